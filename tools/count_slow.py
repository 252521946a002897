"""Debug: how often the TMEM NPDU kernel takes its exact slow path, per
bench workload (needs a -DPCS_COUNT_SLOW build, which adds the count to
stats[2]). usage: python tools/count_slow.py ROOT wl..."""
import sys
root = sys.argv[1]
sys.path.insert(0, root)
import paper_2208_08795_b200 as pcs  # noqa: E402
sys.path.insert(1, ".")
import bench  # noqa: E402
import torch  # noqa: E402

for name in sys.argv[2:]:
    w = bench.WORKLOADS[name]
    x = torch.from_numpy(bench.make_input(w)).cuda()
    idx, st = pcs.sample(x, w["C"], method=w["method"], m=w["M"], k=w["K"], sort=w["sort"])[:2]
    st = st.cpu().numpy()
    it = st[:, 3].sum()
    excess = st[:, 2].sum() - (w["N"] // w["M"]) * it
    print(name, "iterations", int(it), "slow", int(excess), "frac", float(excess) / it)
