"""Pins the CPU oracle (oracle/pcs_oracle.c) before anything is checked
against it: the reference's own known-answer tests, the golden vectors made by
the real reference (tests/golden/make_golden.py), and -- when oracle/_ref is
built -- live randomized agreement with the reference library."""
import numpy as np
import pytest

from conftest import METHOD_NAMES, load_sampler_goldens, load_sort_goldens
from paper_2208_08795_b200 import synth

LINE = np.array([[float(x), 0.0, 0.0] for x in range(8)])


def test_splitmix_kats(oracle):
    # proj/tests/test_core.cpp:77-90
    assert oracle.splitmix(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert oracle.splitmix(42, 2) == [0xBDD732262FEB6E95, 0x28EFE333B266F103]
    assert list(synth.splitmix_next(0, 3)) == oracle.splitmix(0, 3)
    u = (int(synth.splitmix_next(0, 1)[0]) >> 11) * 2.0**-53
    assert abs(u - 0.8833108082136426) < 1e-15


def test_update_window_kats(oracle):
    # proj/tests/test_sampler.cpp:77-84
    assert oracle.update_window(0, 64, 10, 8) == (6, 14)
    assert oracle.update_window(0, 64, 1, 8) == (0, 5)
    assert oracle.update_window(0, 64, 63, 4) == (61, 64)
    assert oracle.update_window(0, 64, 20, 1) == (20, 21)
    assert oracle.update_window(0, 64, 20, 3) == (19, 22)
    assert oracle.update_window(32, 64, 33, 8) == (32, 37)


def test_line_cloud_traces(oracle):
    # proj/tests/test_sampler.cpp:88-100, 102-113, 277-291
    assert oracle.sample("fps", LINE[:4], 2)[0].tolist() == [0, 3]
    assert oracle.sample("fps", LINE[:4], 3)[0].tolist() == [0, 3, 1]
    assert oracle.sample("fps", LINE[:4], 4)[0].tolist() == [0, 3, 1, 2]
    idx, _, st = oracle.sample("npdu_fps", LINE, 3, k=2)
    assert idx.tolist() == [0, 1, 2] and st.tolist() == [3, 2, 2 * 8, 2]
    assert oracle.sample("npdu_fps", LINE, 3, k=4)[0].tolist() == [0, 2, 4]
    idx, _, st = oracle.sample("fps", synth.random_cloud(100, 17), 1)
    assert idx.tolist() == [0] and st.tolist() == [0, 0, 0, 0]


def test_op_count_pins(oracle):
    # proj/tests/acceptance_main.cpp:224-246, test_sampler.cpp:196-208
    cloud = synth.random_cloud(2048, 777, 10.0)
    assert oracle.sample("fps", cloud, 512, first="random", seed=1)[2][0] == 1046528
    assert oracle.sample("afps", cloud, 512, 32, first="random", seed=1)[2][0] == 30720
    assert oracle.sample("npdu_afps", cloud, 512, 32, 16, first="random", seed=1)[2][0] <= 7680
    assert oracle.sample("afps", synth.random_cloud(10, 3), 4, 3)[2][0] == 4
    assert oracle.sample("npdu_fps", synth.random_cloud(64, 4), 10, k=1, first="random",
                         seed=8)[2][0] == 9


def _naive_fps(pts, c, first):
    # proj/tests/oracle.hpp:12-43: recompute min distance to the whole set.
    n = len(pts)
    chosen = [first]
    taken = np.zeros(n, bool)
    taken[first] = True
    while len(chosen) < c:
        best, best_d = n, -1.0
        for j in range(n):
            if taken[j]:
                continue
            near = -1.0
            for s in chosen:
                dx, dy, dz = pts[j] - pts[s]
                dd = dx * dx + dy * dy + dz * dz
                if near < 0 or dd < near:
                    near = dd
            if near > best_d:
                best, best_d = j, near
        chosen.append(best)
        taken[best] = True
    return chosen


def test_matches_naive_oracle(oracle):
    # proj/tests/acceptance_main.cpp:75-124 (reduced)
    rng = np.random.default_rng(190410)
    for t in range(12):
        n = int(rng.integers(4, 60))
        c = int(rng.integers(1, min(n, 16) + 1))
        pts = synth.random_cloud(n, 500 + t)
        assert oracle.sample("fps", pts, c)[0].tolist() == _naive_fps(pts, c, 0)


@pytest.mark.parametrize("name", sorted(load_sampler_goldens()))
def test_oracle_matches_reference_goldens(oracle, name):
    g = load_sampler_goldens()[name]
    idx, sec, st = oracle.sample(METHOD_NAMES[int(g["method"])], g["points"], int(g["c"]),
                                 int(g["m"]), int(g["k"]),
                                 "random" if int(g["random_first"]) else "fixed", int(g["seed"]))
    np.testing.assert_array_equal(idx, g["indices"])
    np.testing.assert_array_equal(sec, g["sector_of"])
    np.testing.assert_array_equal(st, g["stats"])


def test_oracle_exact_sort_goldens(oracle):
    for name, g in load_sort_goldens().items():
        axis = int(name[-1])
        _, out = oracle.exact_sort(g["points"], axis)
        np.testing.assert_array_equal(out, g["sorted"])


def test_oracle_matches_live_reference(oracle, reference):
    rng = np.random.default_rng(260856)
    for t in range(120):
        n = int(rng.integers(4, 300))
        c = int(rng.integers(1, n + 1))
        m = int(rng.integers(1, c + 1))
        k = int(rng.integers(1, 30))
        pts = synth.random_cloud(n, 9000 + t)
        if t % 4 == 0:
            pts[: n // 2] = 1.0
        for meth in ("fps", "afps", "npdu_fps", "npdu_afps"):
            first = "random" if t % 2 else "fixed"
            a = oracle.sample(meth, pts, c, m, k, first, t)
            b = reference.sample(meth, pts, c, m, k, first, t)
            for x, y in zip(a, b):
                np.testing.assert_array_equal(x, y)


def test_oracle_trace_matches_reference(oracle, reference):
    pts = synth.random_cloud(50, 404)
    for k in (0, 5):
        i1, s1, t1 = oracle.local_fps(pts, 0, 50, 20, k=k, trace=True)
        i2, s2, t2 = reference.local_fps_trace(pts, 0, 50, 20, k=k)
        np.testing.assert_array_equal(i1, i2)
        np.testing.assert_array_equal(s1, s2)
        np.testing.assert_array_equal(t1, t2)


def test_error_messages_match_reference(oracle, reference):
    pts = synth.random_cloud(10, 1)
    bad = [("fps", 0, 1, 0), ("fps", 11, 1, 0), ("afps", 4, 5, 0), ("afps", 11, 2, 0),
           ("afps", 4, 0, 0), ("npdu_afps", 4, 20, 3), ("npdu_fps", 4, 1, 0),
           ("npdu_afps", 4, 2, 0)]
    for meth, c, m, k in bad:
        with pytest.raises(ValueError) as e1:
            oracle.sample(meth, pts, c, m, k)
        with pytest.raises(ValueError) as e2:
            reference.sample(meth, pts, c, m, k)
        assert str(e1.value) == str(e2.value)
