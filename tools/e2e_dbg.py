import sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2208_08795_b200 as pcs
w = bench.WORKLOADS[sys.argv[1]]
xh = bench.make_input(w)
pinned = torch.from_numpy(xh).pin_memory()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
call = lambda: pcs.sample_host_batch(pinned, w["C"], method=w["method"], m=w["M"], k=w["K"], sort=w["sort"])
for i in range(30): call()
for mode in ("flush", "noflush", "flush_sleep"):
    ts = []
    for i in range(30):
        if mode != "noflush":
            flush.fill_(i % 255)
        torch.cuda.synchronize()
        if mode == "flush_sleep": time.sleep(0.002)
        t0 = time.perf_counter(); r = call(); ts.append((time.perf_counter() - t0) * 1e3)
    print(mode, "mean %.3f median %.3f" % (np.mean(ts), np.median(ts)), [round(t, 2) for t in ts])
