import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs
from paper_2208_08795_b200 import synth
lib = ctypes.CDLL(pcs.LIB_PATH)
for B in (1, 4096):
    x = torch.from_numpy(synth.uniform_cube(B, 1024, 1)).cuda()
    for _ in range(2): pcs.sample(x, 256, method="npdu_fps", k=129)
    torch.cuda.synchronize()
    out = np.zeros(8, np.uint64)
    lib.pcs_debug_prof(out.ctypes.data_as(ctypes.c_void_p))
    names = ["pivot", "window", "tmem_ld", "compute", "tmem_st", "row_red", "argmax", "tail"]
    print(B, {n: round(int(v) / 255, 1) for n, v in zip(names, out)}, "total", round(int(out.sum()) / 255, 1))
