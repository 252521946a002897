"""Benchmark: FPS / AFPS / NPDU-AFPS sampling throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the reference CPU path, same config

Metric (BASELINE.json): sampled points/s (and clouds/s), whole job. A step is
one pass of the hot path over one batch resident in HBM: the per-cloud stable
axis sort (when the config sorts) plus the sampler, both hand-written sm_100a
kernels. Timing: CUDA events on the launching stream around each step, an L2
flush (a 512 MiB write, > 126 MB L2) between steps outside the events,
barrier + synchronize on both sides of the K timed steps, max over ranks.

Multi-GPU (BASELINE cfg4 "batch 128 sharded across 8 GPUs"): the batch is
split by cloud, rank r sampling clouds shard.split(B, N, r) -- strong
scaling, the job's work is fixed; a single large cloud (cfg5-1m) splits by
sector run. The weak-scaling form (every rank its own full batch) is
reported beside it as `weak`.

Also reported: `e2e` (the same metric through the public C-ABI host entry
with host buffers -- pinned H2D of the batch, sort + sample, D2H of indices
+ stats -- timed with the host clock around the synchronous call),
`roofline` (the sampler kernel's FP64 work against the measured FP64 peak),
`cpu_baseline` (the unmodified reference, oracle/_ref, on this host's cores,
bounded sample, best of 3), `parity` (the timed output against the
reference's indices for the cpu_baseline's clouds), `workloads` (every
BASELINE config measured the same way, N=1 only), `clocks` (nvidia-smi
during the timed region).

The reference arm never loads the CUDA library: the generators are loaded
by file path (paper_2208_08795_b200/synth.py is plain numpy), not through
the package, whose import loads libpcs_gpu.so.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Per-GPU workloads (BASELINE.json configs; BASELINE's w -> k = 2w + 1).
WORKLOADS = {
    "cfg1": dict(gen="cube", B=1, N=2048, method="fps", C=512, M=1, K=None, sort="x"),
    "cfg2": dict(gen="prim4", B=16, N=2048, method="afps", C=512, M=8, K=None, sort="x"),
    "cfg3": dict(gen="prim6", B=64, N=8192, method="npdu_afps", C=2048, M=16, K=65, sort="x"),
    "cfg3-afps": dict(gen="prim6", B=64, N=8192, method="afps", C=2048, M=16, K=None, sort="x"),
    "cfg3-fps": dict(gen="prim6", B=64, N=8192, method="fps", C=2048, M=1, K=None, sort="x"),
    "cfg4": dict(gen="lidar", B=128, N=32768, method="npdu_afps", C=8192, M=32, K=129, sort=None),
}
for _n in (2048, 4096, 8192, 16384, 32768):
    WORKLOADS[f"cfg5-fps-{_n}"] = dict(gen="cube", B=256, N=_n, method="fps", C=_n // 4, M=1,
                                       K=None, sort="x")
    for _m in (1, 4, 16, 64, 256):
        WORKLOADS[f"cfg5-afps{_m}-{_n}"] = dict(gen="cube", B=256, N=_n, method="afps",
                                                C=_n // 4, M=_m, K=None, sort="x")
    WORKLOADS[f"cfg5-npdu-{_n}"] = dict(gen="cube", B=256, N=_n, method="npdu_afps", C=_n // 4,
                                        M=16, K=65, sort="x")

# one 1M-point cloud: under torchrun its sectors are split across the ranks
# (strong scaling, BASELINE cfg5), each rank sorting the cloud itself
WORKLOADS["cfg5-1m"] = dict(gen="cube", B=1, N=1 << 20, method="afps", C=(1 << 20) // 4, M=1024,
                            K=None, sort="x")
# the streaming vanilla-FPS engine (north_star item 4): one cloud too large
# for any on-chip engine, d[] in global memory
WORKLOADS["stream-fps-1m"] = dict(gen="cube", B=1, N=1 << 20, method="fps", C=2048, M=1,
                                  K=None, sort="x")

# latency probes: one NPDU sector per warp, 1 warp / 148 warps / 4096 warps
for _b in (1, 148, 4096):
    WORKLOADS[f"lat-npdu-{_b}"] = dict(gen="cube", B=_b, N=1024, method="npdu_fps", C=256, M=1,
                                       K=129, sort=None)

DEFAULT_WORKLOAD = "cfg4"
# --eager: every step launched from Python (default: the step's launches are
# captured once in a CUDA graph and replayed, no host work between them)
EAGER = False
# the `workloads` object of the default run: every BASELINE config
SWEEP = (["cfg1", "cfg2", "cfg3", "cfg3-afps", "cfg3-fps", "cfg4"]
         + [f"cfg5-{v}-{n}" for n in (2048, 4096, 8192, 16384, 32768)
            for v in ("fps", "afps1", "afps4", "afps16", "afps64", "afps256", "npdu")]
         + ["cfg5-1m", "stream-fps-1m"])
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak.json")
HBM_FALLBACK_GBS = 6543.7  # MEASURED_PEAKS.json of this pool (r01/r02)


def _synth():
    """paper_2208_08795_b200/synth.py loaded by path: plain numpy, and the
    package import (which loads the CUDA library) stays out of the
    reference arm."""
    mod = sys.modules.get("pcs_synth_bench")
    if mod is None:
        path = os.path.join(ROOT, "paper_2208_08795_b200", "synth.py")
        spec = importlib.util.spec_from_file_location("pcs_synth_bench", path)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        sys.modules["pcs_synth_bench"] = mod
    return mod


def make_input(w, seed_base=0):
    synth = _synth()
    g = w["gen"]
    if g == "cube":
        return synth.uniform_cube(w["B"], w["N"], seed_base)
    if g.startswith("prim"):
        return synth.primitives(w["B"], w["N"], int(g[4:]), seed=seed_base + 1)
    if g == "lidar":
        return synth.lidar_sweep(w["B"], seed=seed_base + 4)
    raise ValueError(g)


def host_sorted(w, xyz):
    if w["sort"] is None:
        return xyz
    return _synth().stable_sort_np(xyz, "xyz".index(w["sort"]))[0]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 3:
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [r for r in self.rows if not (r[2] & 0x1)] or self.rows
        mask = 0
        for r in loaded:
            mask |= r[2]
        return {"sm_mhz": float(np.median([r[0] for r in loaded])),
                "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": [v for k, v in self.REASONS.items() if mask & k and k != 0x1],
                "samples": len(loaded)}


def _json_file(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def ncu_traffic(workload):
    """DRAM bytes per launch of the sampler kernel (and its issue rate) from
    the committed ncu --set full capture for this workload
    (profiles/ncu_traffic.json, made by tools/ncu_sweep.sh)."""
    d = _json_file("ncu_traffic.json").get(workload)
    if not d:
        return None, "no ncu capture for this workload", None, None
    return float(d["dram_bytes"]), d["source"], d.get("ipc_per_sm"), d.get("fp64_pipe_pct")


def fp64_peak():
    d = _json_file("fp64_peak.json")
    if "fp64_tflops" in d:
        return float(d["fp64_tflops"]), d.get("source", FP64_PEAK_FILE)
    return None, "missing"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK_GBS, "MEASURED_PEAKS.json absent: this pool's r01 measurement"


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(w, xyz_sorted, budget_s=20.0, repeats=3):
    """The unmodified reference (oracle/_ref) on the host: one cloud per
    worker thread, sampler at threads=1 (proj/src/bench.cpp:90-92,104-120),
    timed around the sampler calls only, best of `repeats` runs
    (proj/tests/acceptance_main.cpp:63-71). Bounded: a prefix of the batch
    sized to ~budget_s of single-core work; a single cloud runs the
    reference's own sector threading (threads = cores, sampler.cpp:25-46)
    and, when even that is too long, its first c' picks (FPS is greedy: the
    first c' picks of a run equal a run with c = c').

    Returns the baseline dict plus the reference's indices for the sampled
    clouds (the parity check)."""
    from oracle import Reference

    ref = Reference()
    workers = os.cpu_count() or 1
    B, C = w["B"], w["C"]
    if B == 1:
        pts = xyz_sorted[0].astype(np.float64)
        c = C
        sectored = w["method"] in ("afps", "npdu_afps")
        per_pick = None
        if not sectored:
            # time 64 picks single-threaded, then size the prefix
            t0 = time.perf_counter()
            ref.sample(w["method"], pts, min(64, C), 1, w["K"] or 0)
            per_pick = (time.perf_counter() - t0) / min(64, C)
            c = int(max(64, min(C, budget_s / max(per_pick, 1e-9))))
        best, idx = None, None
        for _ in range(max(1, repeats)):
            t0 = time.perf_counter()  # (ctypes call: no Python objects made inside)
            idx, _, _ = ref.sample(w["method"], pts, c, w["M"], w["K"] or 0,
                                   threads=workers if sectored else 1)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        res = {"value": c / best, "unit": "sampled points/s",
               "cores": workers if sectored else 1, "kind": "reference",
               "clouds_per_s": (c / C) / best,
               "sample": (f"the 1 cloud, reference sector threads = {workers}, best of "
                          f"{max(1, repeats)}" if sectored else
                          f"the 1 cloud's first {c} of {C} picks (greedy prefix), 1 thread, "
                          f"best of {max(1, repeats)}"),
               "cpu_model": _cpu_model()}
        return res, np.asarray(idx)[None, :], np.array([0])
    probe = xyz_sorted[:1]
    _, _, t1 = ref.sample_batch_f32(w["method"], probe, C, w["M"], w["K"] or 0, workers=1)
    per_cloud = max(t1, 1e-6)
    nb = int(max(1, min(B, budget_s / per_cloud)))
    nb = max(min(nb, B), min(B, workers))
    sample = xyz_sorted[:nb]
    best, idx = None, None
    for _ in range(max(1, repeats)):
        idx, _, secs = ref.sample_batch_f32(w["method"], sample, C, w["M"], w["K"] or 0,
                                            workers=workers)
        best = secs if best is None else min(best, secs)
    res = {"value": nb * C / best, "unit": "sampled points/s", "cores": min(workers, nb),
           "kind": "reference", "clouds_per_s": nb / best,
           "sample": f"{nb} of {B} clouds of the same batch (pre-sorted on the host), "
                     f"{min(workers, nb)} worker threads, best of {max(1, repeats)}, "
                     f"single-core probe {per_cloud * 1e3:.2f} ms/cloud",
           "cpu_model": _cpu_model()}
    return res, idx, np.arange(nb)


def parity_of(gpu_idx, ref_idx, clouds):
    """Mismatching clouds between the device output and the reference's
    indices (a prefix of each row when the reference ran fewer picks)."""
    c = ref_idx.shape[1]
    bad = [int(b) for i, b in enumerate(clouds) if not np.array_equal(gpu_idx[b, :c], ref_idx[i])]
    return {"clouds": int(len(clouds)), "picks_per_cloud": int(c), "mismatches": len(bad),
            "mismatched_clouds": bad[:8], "against": "oracle/_ref (the unmodified reference)"}


def launches_per_step(w, n_sort_launches=None):
    """Our kernels per step (csrc/sort_kernels.cu, csrc/sample_dispatch.cu):
    one sampler launch; the axis sort is one launch up to 256K fp32 points,
    otherwise the device-wide radix (histogram, scan, scatter per 8-bit
    pass)."""
    sort = 0
    if w["sort"]:
        sort = 1 if w["N"] <= 16 * 16384 else 3 * 4
    return 1 + sort


def arm_config(workload, w, world, mode):
    """The `config` object both arms print (identical for the same workload)."""
    return {"workload": workload, "clouds": w["B"], "points_per_cloud": w["N"],
            "samples_per_cloud": w["C"], "method": w["method"], "m": w["M"], "k": w["K"],
            "sort": w["sort"], "generator": w["gen"], "coords": "fp32 in, fp64 math",
            "l2": "flushed between steps (512 MiB write)",
            "parallelism": {"batch": f"clouds split over {world} GPU(s)",
                            "sector": f"sector-split x{world}",
                            "replica": f"replicas x{world} (vanilla FPS on one cloud does "
                                       "not shard: one global argmax per iteration)",
                            "weak": f"dp{world}"}[mode]}


def run_mode(w, world):
    """How the job spreads over `world` GPUs: a batch splits by cloud; one
    AFPS / NPDU-AFPS cloud by sector run; one vanilla-FPS cloud (or fewer
    sectors than GPUs) only by replica."""
    if world <= 1 or w["B"] > 1:
        return "batch"
    if w["method"] in ("afps", "npdu_afps") and w["M"] >= world:
        return "sector"
    return "replica"


def _loaded_native():
    """Shared objects of this repo mapped into the process (the reference
    arm must show only oracle/ ones)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")}
    except OSError:
        return None
    return sorted(os.path.relpath(p, ROOT) for p in paths if p.startswith(ROOT))


def run_reference_arm(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    xyz = make_input(w)
    res, _, _ = cpu_reference(w, host_sorted(w, xyz), budget_s=8.0, repeats=args.steps)
    mode = run_mode(w, args.gpus)
    line = {"metric": "sampled points/s", "value": res["value"], "unit": "sampled points/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak" if mode == "replica" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(args.workload, w, args.gpus, mode),
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "clouds_per_s": res["clouds_per_s"], "cpu_model": res["cpu_model"],
            "e2e": {"value": res["value"], "unit": "sampled points/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "native_libraries": _loaded_native()}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- GPU arm
class no_gc:
    """Python's cyclic GC paused inside a timed region (a full collection
    stalled single timed calls by 5-30 ms); collected right before."""

    def __enter__(self):
        import gc

        gc.collect()
        gc.disable()

    def __exit__(self, *a):
        import gc

        gc.enable()


class Runner:
    """One workload on this rank's GPU: the step (sort + sample), the sort
    and the sampler alone, the host-buffer e2e call."""

    def __init__(self, pcs, torch, dev, w, xyz_host, shard_spec=None):
        self.pcs, self.torch, self.dev, self.w = pcs, torch, dev, w
        self.xyz_host = xyz_host
        self.xyz = torch.from_numpy(xyz_host).to(dev)
        self.sh = shard_spec  # sector shard of one large cloud, or None
        self.flush = None
        self.eager = EAGER or shard_spec is not None
        self.graphs, self.graph_errors = [], []

    def sample_sorted(self, xs):
        w, pcs, sh = self.w, self.pcs, self.sh
        if sh is None:
            return pcs.sample(xs, w["C"], method=w["method"], m=w["M"], k=w["K"])
        from paper_2208_08795_b200 import shard

        return shard.sample_sector_shard(xs, sh, w["method"], w["K"])

    def sample_perm(self, x, perm):
        """The step's sampler launch alone: the unsorted clouds and the sort
        permutation (what sample(sort=...) launches after the sort)."""
        w, pcs = self.w, self.pcs
        if perm is None:
            return self.sample_sorted(x)
        from paper_2208_08795_b200 import ops

        return ops.sample_with_perm(x, perm, w["C"], method=w["method"], m=w["M"], k=w["K"])

    def step(self, x):
        w, pcs = self.w, self.pcs
        if self.sh is None:
            return pcs.sample(x, w["C"], method=w["method"], m=w["M"], k=w["K"], sort=w["sort"])
        xs = pcs.sort_axis(x, w["sort"])[0] if w["sort"] else x
        return self.sample_sorted(xs)

    def _flush(self, i):
        if self.flush is None:
            self.flush = self.torch.empty(512 * 1024 * 1024 // 4, dtype=self.torch.float32,
                                          device=self.dev)
        self.flush.fill_(float(i))

    def graphed(self, fn):
        """`fn` captured once in a CUDA graph (the step's launches replayed
        without host work between them) -> (replay, static outputs); falls
        back to (fn, None) when the launches cannot be captured."""
        torch = self.torch
        if self.eager:
            return fn, None
        try:
            s = torch.cuda.Stream(device=self.dev)
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                fn()
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            # thread_local: other threads' CUDA calls (e.g. the NCCL watchdog
            # under torchrun) must not invalidate the capture
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                out = fn()
            torch.cuda.synchronize()
            self.graphs.append(g)

            def replay():
                g.replay()
                return out

            return replay, out
        except Exception as exc:  # e.g. an engine that cannot be captured
            torch.cuda.synchronize()
            self.graph_errors.append(f"{type(exc).__name__}: {exc}")
            return fn, None

    def timed(self, fn, steps, per_step_sync=False):
        """Sum of CUDA-event times of `fn` over `steps` calls, L2 flushed
        before each (outside the events). Returns (ms_total, last output)."""
        torch = self.torch
        fn()  # one untimed call: first-use allocations stay outside the events
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        out = None
        with no_gc():
            for i in range(steps):
                self._flush(i)
                starts[i].record()
                out = fn()
                ends[i].record()
                if per_step_sync:
                    torch.cuda.synchronize()
            torch.cuda.synchronize()
        return sum(s.elapsed_time(e) for s, e in zip(starts, ends)), out

    def e2e(self, steps, warmup, world=1, dist=None):
        """The C-ABI host entry (pcs_sample_host_batch): pinned batch in,
        host arrays out, one synchronous native call per step, timed with
        the host clock after the flush has completed."""
        torch, w, pcs = self.torch, self.w, self.pcs
        pinned = torch.from_numpy(self.xyz_host).pin_memory()
        sh = self.sh

        def call():
            if sh is None:
                return pcs.sample_host_batch(pinned, w["C"], method=w["method"], m=w["M"],
                                             k=w["K"], sort=w["sort"])
            res = self.step(pinned.to(self.dev, non_blocking=True))
            return tuple(t.cpu() for t in res)

        # warm-up: at least W steps and 0.5 s -- the host link ramps up over
        # the first ~15 transfers after idling (tools/e2e_dbg.py)
        # (each call's result is held until the next returns, as in the timed
        # loop: two live result sets, so the pinned host allocator has grown to
        # both before timing -- otherwise the second timed call paid a ~2 ms
        # cudaHostAlloc, tools/e2e_dbg.py)
        t_warm = time.perf_counter()
        r = None
        for i in range(max(warmup, 1000)):
            r = call()
            if i + 1 >= warmup and time.perf_counter() - t_warm > 0.5:
                break
        # and the timed loop's own sequence (flush, synchronize, call) a few
        # times: its first run after a new input was measured at ~30 ms once
        for i in range(3):
            self._flush(i)
            torch.cuda.synchronize()
            r = call()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        total = 0.0
        per_call = []
        with no_gc():
            for i in range(steps):
                self._flush(i)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = call()
                dt = time.perf_counter() - t0
                per_call.append(dt * 1e3)
                total += dt
        e_ms = total * 1e3
        if dist is not None:
            red = torch.device("cpu") if dist.get_backend() == "gloo" else self.dev
            t = torch.tensor([e_ms], dtype=torch.float64, device=red)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e_ms /= steps
        # the PCIe floor on this box: one plain H2D of the same pinned batch
        dst = torch.empty(pinned.shape, dtype=pinned.dtype, device=self.dev)
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h2d = []
        for _ in range(5):
            es.record()
            dst.copy_(pinned, non_blocking=True)
            ee.record()
            torch.cuda.synchronize()
            h2d.append(es.elapsed_time(ee))
        del dst
        nbytes = pinned.numel() * pinned.element_size()
        return {"ms_per_step": e_ms, "min_ms": min(per_call), "max_ms": max(per_call),
                "median_ms": float(np.median(per_call)),
                "h2d_floor_ms": min(h2d),
                "h2d_gbps": nbytes / min(h2d) / 1e6, "h2d_bytes_per_step": int(nbytes),
                "d2h_bytes_per_step": int(sum(t.nbytes if hasattr(t, "nbytes") else
                                              t.numel() * t.element_size() for t in r)),
                "timer": "host perf_counter around the synchronous call, after "
                         "torch.cuda.synchronize() on the L2 flush",
                "path": ("C-ABI pcs_sample_host_batch (pinned host tensor in, host arrays "
                         "out): chunked H2D overlapped with sort+sample, D2H of indices, "
                         "stats (and perm when sorting)") if sh is None else
                        "pinned H2D, sort, sample of this rank's sectors, D2H"}


def sort_bytes(w):
    """Algorithmic HBM bytes of the step's axis sort: read the cloud (12N),
    write the permutation (4N). (The gathered copy is never written: the
    sampler stages through the permutation.)"""
    return 0 if not w["sort"] else w["B"] * w["N"] * 16


def stream_bytes(w):
    """the streaming engine's algorithmic bytes per cloud,
    (C-1)*N*28 (xyz 12 B read, d 8 B read + 8 B written per point and
    iteration) + 12N + 4C."""
    return w["B"] * ((w["C"] - 1) * w["N"] * 28 + 12 * w["N"] + 4 * w["C"])


def measure_workload(pcs, torch, dev, name, w, steps, warmup, xyz_host, cpu_budget_s=2.0):
    """One `workloads` entry (N=1): step / sort / sampler times, kernel,
    roofline fractions, e2e, cpu_baseline and parity."""
    import gc

    gc.collect()  # the previous workload's buffers go now, not inside a timed region
    torch.cuda.synchronize()
    r = Runner(pcs, torch, dev, w, xyz_host)
    for _ in range(warmup):
        out = r.step(r.xyz)
    torch.cuda.synchronize()
    evals = int(out[1][:, 0].sum().item())
    ms, out = r.timed(r.graphed(lambda: r.step(r.xyz))[0], steps)
    ms /= steps
    gpu_idx = out[0].cpu().numpy()
    eager_ms = r.timed(lambda: r.step(r.xyz), steps)[0] / steps
    sort_ms = 0.0
    xs = r.xyz
    perm = None
    if w["sort"]:
        # the step's sort: the permutation only (the sampler stages through it)
        sort_ms = r.timed(r.graphed(lambda: pcs.sort_perm(r.xyz, w["sort"]))[0], steps)[0] / steps
        perm = pcs.sort_perm(r.xyz, w["sort"])
    samp_ms = r.timed(r.graphed(lambda: r.sample_perm(xs, perm))[0], steps)[0] / steps
    peak, _ = fp64_peak()
    hbm, _ = hbm_peak()
    kern = pcs.kernel_family(w["method"], w["N"], w["M"], w["K"], batch=w["B"])
    entry = {"ms_per_step": ms, "sampled_pts_per_s": w["B"] * w["C"] / (ms * 1e-3),
             "clouds_per_s": w["B"] / (ms * 1e-3), "eager_ms_per_step": eager_ms,
             "launch": "cuda graph replay" if r.graphs else "eager",
             "sort_ms": sort_ms, "sampler_ms": samp_ms,
             "kernel": kern, "dist_evals_per_step": evals,
             "fp64_frac_algorithmic": (8.0 * evals / (samp_ms * 1e-3) / 1e12 / peak)
             if peak else None}
    _, _, _, fp64_pct = ncu_traffic(name)
    entry["fp64_pipe_executed_frac"] = (fp64_pct / 100.0) if fp64_pct is not None else None
    if w["sort"]:
        entry["sort_hbm_frac"] = sort_bytes(w) / (sort_ms * 1e-3) / 1e9 / hbm
    if kern.startswith("stream"):
        entry["stream_hbm_frac"] = stream_bytes(w) / (samp_ms * 1e-3) / 1e9 / hbm
        entry["stream_note"] = "d[] and xyz stay L2-resident (20 B/pt x 1M < 126 MB L2)"
    e = r.e2e(max(6, steps), 2)
    e["value"] = w["B"] * w["C"] / (e["ms_per_step"] * 1e-3)
    e["unit"] = "sampled points/s"
    entry["e2e"] = e
    try:
        cpu, ref_idx, clouds = cpu_reference(w, host_sorted(w, xyz_host), budget_s=cpu_budget_s,
                                             repeats=2)
        entry["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        entry["parity"] = parity_of(gpu_idx, ref_idx, clouds)
        entry["e2e_vs_cpu"] = e["value"] / cpu["value"]
    except Exception as exc:  # the checker is optional on the box
        entry["cpu_baseline"] = {"value": None, "sample": f"unavailable: {exc}"}
    return entry


def run_sweep(pcs, torch, dev, names, budget_s, steps=5, warmup=3):
    """The `workloads` object: every BASELINE config under a wall budget."""
    out, cache = {}, {}
    t0 = time.perf_counter()
    for name in names:
        if time.perf_counter() - t0 > budget_s:
            out[name] = {"skipped": f"wall budget of {budget_s:.0f} s spent"}
            continue
        w = WORKLOADS[name]
        key = (w["gen"], w["B"], w["N"])
        if key not in cache:
            cache.clear()
            cache[key] = make_input(w)
        try:
            out[name] = measure_workload(pcs, torch, dev, name, w, steps, warmup, cache[key])
        except Exception as exc:  # keep the sweep going; report the failure
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
    out["_wall_s"] = time.perf_counter() - t0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-workloads", action="store_true")
    ap.add_argument("--eager", action="store_true",
                    help="launch every step from Python instead of replaying a CUDA graph")
    ap.add_argument("--workloads", default=None,
                    help="comma-separated subset of the sweep (default: every BASELINE config)")
    ap.add_argument("--workloads-budget", type=float, default=150.0)
    args = ap.parse_args()
    global EAGER
    EAGER = args.eager
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference_arm(args, w)

    import torch
    import torch.distributed as dist

    import paper_2208_08795_b200 as pcs
    from paper_2208_08795_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PCS_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0 over gloo,
    # to run the torchrun path on a one-GPU box
    share = os.environ.get("PCS_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if share else dev  # gloo reduces host tensors
    args.warmup = max(args.warmup, 3)
    B, N, C = w["B"], w["N"], w["C"]

    # strong scaling: the job is the configured batch. Several clouds split
    # by cloud (BASELINE cfg4: 128 over 8 GPUs = 16 per GPU); one cloud
    # splits by sector run, every rank sorting the cloud itself
    mode = run_mode(w, world)
    xyz_all = make_input(w)
    sh = None
    if mode == "sector":
        sh = shard.sector_shard(N, C, w["M"], world, rank)
        xyz_host, b0 = xyz_all, 0
    elif mode == "replica":
        xyz_host, b0 = xyz_all, 0
    else:
        b0, b1 = shard.split(B, world, rank)
        xyz_host = np.ascontiguousarray(xyz_all[b0:b1])
    r = Runner(pcs, torch, dev, w, xyz_host, sh)

    for _ in range(args.warmup):
        out = r.step(r.xyz)
    torch.cuda.synchronize()
    evals_local = int(out[1][:, 0].sum().item())

    # ---- device-resident throughput (value)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_fn = r.graphed(lambda: r.step(r.xyz))[0]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ms, out = r.timed(step_fn, args.steps)
    if world > 1:
        dist.barrier()
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    gpu_idx = out[0].cpu().numpy()
    # the same step launched eagerly from Python (host work between launches)
    eager_ms = r.timed(lambda: r.step(r.xyz), args.steps)[0]
    t = torch.tensor([eager_ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    eager_ms = float(t.item()) / args.steps
    total_samples = B * C * (world if mode == "replica" else 1)
    pts_per_s = total_samples / (ms_per_step * 1e-3)

    # ---- weak scaling beside it: every rank its own full batch
    weak = None
    if world > 1 and mode == "batch":
        rw = Runner(pcs, torch, dev, w, make_input(w, seed_base=1000 * rank))
        for _ in range(args.warmup):
            rw.step(rw.xyz)
        dist.barrier()
        wfn = rw.graphed(lambda: rw.step(rw.xyz))[0]
        dist.barrier()
        wms = rw.timed(wfn, args.steps)[0]
        t = torch.tensor([wms], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wms = float(t.item()) / args.steps
        weak = {"value": world * B * C / (wms * 1e-3), "unit": "sampled points/s",
                "ms_per_step": wms, "clouds_per_gpu": B,
                "note": "every rank samples its own full batch (seeded by rank)"}
        del rw

    # ---- sampler kernel alone (roofline): sort once, time only the sampler
    if sh is None:
        perm = pcs.sort_perm(r.xyz, w["sort"]) if w["sort"] else None
        kern_ms = r.timed(r.graphed(lambda: r.sample_perm(r.xyz, perm))[0], args.steps,
                          per_step_sync=True)[0] / args.steps
    else:
        xs = pcs.sort_axis(r.xyz, w["sort"])[0] if w["sort"] else r.xyz
        kern_ms = r.timed(lambda: r.sample_sorted(xs), args.steps,
                          per_step_sync=True)[0] / args.steps
    peak, peak_src = fp64_peak()
    flops = 8.0 * evals_local
    achieved = flops / (kern_ms * 1e-3) / 1e12
    traffic, traffic_src, ipc, fp64_pct = ncu_traffic(args.workload)
    kernel = ("none (empty shard)" if sh is not None and sh.empty else
              pcs.kernel_family(w["method"], sh.n if sh else N, sh.m if sh else w["M"], w["K"],
                                batch=xyz_host.shape[0]))
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if peak else None,
                "traffic": traffic if world == 1 and mode == "batch" else None,
                "traffic_source": traffic_src,
                # what actually limits the serial update->argmax->pivot chain:
                # issued instructions per SM-cycle (ncu) against the 4 schedulers
                "issue": ({"ipc_per_sm": ipc, "peak_ipc": 4.0, "frac": ipc / 4.0}
                          if ipc else None),
                "fp64_pipe_executed_frac": (fp64_pct / 100.0) if fp64_pct is not None else None,
                "algorithmic_hbm_bytes": xyz_host.shape[0] * N * 12 + xyz_host.shape[0] * C * 4,
                "kernel": kernel, "kernel_ms": kern_ms, "algorithmic_flops": flops,
                "peak_source": peak_src,
                "note": "FP64 flops = 8 x dist_evals (3 sub, 3 mul, 2 add; no FMA) of this "
                        "rank's launch; the argmax work is not counted; kernel_ms = CUDA "
                        "events on the launching stream, synchronised per launch"}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = r.e2e(args.steps, args.warmup, world, dist if world > 1 else None)
        e2e["value"] = total_samples / (e2e["ms_per_step"] * 1e-3)
        e2e["unit"] = "sampled points/s"

    # ---- reference on the host: baseline (N=1) and parity (rank 0's clouds)
    cpu, parity = None, None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            res, ref_idx, clouds = cpu_reference(
                w, host_sorted(w, xyz_host if mode == "batch" else xyz_all))
            if world == 1:
                cpu = {k: res[k] for k in ("value", "unit", "cores", "kind", "sample",
                                            "cpu_model")}
            if mode == "batch":
                parity = parity_of(gpu_idx, ref_idx, clouds)
            else:  # rank 0's sectors are the first out slots of the cloud
                c0 = min(gpu_idx.shape[1], ref_idx.shape[1])
                parity = parity_of(gpu_idx[:, :c0], ref_idx[:, :c0], clouds)
        except Exception as exc:  # the checker is optional on the box
            cpu = {"value": None, "unit": "sampled points/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    sweep = None
    if world == 1 and not args.no_workloads:
        names = args.workloads.split(",") if args.workloads else SWEEP
        sweep = run_sweep(pcs, torch, dev, names, args.workloads_budget)

    if rank == 0:
        line = {
            "metric": "sampled points/s", "value": pts_per_s, "unit": "sampled points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "launch": ("cuda graph replay of the captured step (sort + sampler launches)"
                       if r.graphs else "eager"), "eager_ms_per_step": eager_ms,
            "scaling": "weak" if mode == "replica" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "clouds_per_s": B * (world if mode == "replica" else 1) / (ms_per_step * 1e-3),
            "config": arm_config(args.workload, w, world, mode),
            "gpu_launches": args.steps * launches_per_step(w),
            "dist_evals_per_step_rank0": evals_local,
            "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
            "weak": weak, "clocks": clocks.summary(), "workloads": sweep,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
