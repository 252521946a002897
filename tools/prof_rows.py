import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs
from paper_2208_08795_b200 import synth
lib = ctypes.CDLL(pcs.LIB_PATH)
for N in (2048, 8192, 32768):
    x = torch.from_numpy(synth.stable_sort_np(synth.uniform_cube(1, N, 1), 0)[0]).cuda()
    import os; os.environ["PCS_SAMPLER"] = "rows"
    pcs.sample(x, N // 4, method="fps"); torch.cuda.synchronize()
    out = np.zeros(8, np.uint64); lib.pcs_debug_rprof(out.ctypes.data_as(ctypes.c_void_p))
    pcs.sample(x, N // 4, method="fps"); torch.cuda.synchronize()
    out = np.zeros(8, np.uint64); lib.pcs_debug_rprof(out.ctypes.data_as(ctypes.c_void_p))
    it = N // 4 - 1
    W = {2048: 8, 8192: 16, 32768: 16}[N]
    names = ["test", "test+process", "warp_argmax", "cta_exchange", "cluster+pivot", "tail"]
    print(N, {n: round(int(v) / it / W, 1) for n, v in zip(names, out[:6])},
          "cand rows/iter/CTA", round(int(out[6]) / it, 1), "pairs/iter/warp", round(int(out[7]) / it / W, 2))
