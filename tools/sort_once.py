"""One warm sort_axis call on a (B, N, 3) cube batch (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

B, N = int(sys.argv[1]), int(sys.argv[2])
x = torch.from_numpy(synth.uniform_cube(B, N, 1)).cuda()
for _ in range(3):
    pcs.sort_perm(x, "x")
torch.cuda.synchronize()
print("ok")
