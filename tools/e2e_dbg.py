import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2208_08795_b200 as pcs
from paper_2208_08795_b200 import synth
x = torch.from_numpy(synth.lidar_sweep(128, seed=4)).pin_memory()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
def step():
    return pcs.sample(x, 8192, method="npdu_afps", m=32, k=129)
for _ in range(3): step()
torch.cuda.synchronize()
for mode in ("flush", "noflush", "flush", "noflush"):
    ts=[]; ws=[]
    for i in range(20):
        if mode == "flush": flush.fill_(float(i))
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0=time.perf_counter()
        es.record(); step(); ee.record(); torch.cuda.synchronize()
        ws.append((time.perf_counter()-t0)*1e3)
        ts.append(es.elapsed_time(ee))
    print(mode, "ev", np.round(ts,2).tolist())
    print(mode, "wall", np.round(ws,2).tolist())
