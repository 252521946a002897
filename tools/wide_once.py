"""One warm NPDU-AFPS call on 4 cfg4 LiDAR clouds (128 sectors: the W-warp
npdu_wide_kernel) -- an ncu target: the last launch is the measured one."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
x = torch.from_numpy(synth.lidar_sweep(B, seed=1)).cuda()
for _ in range(3):
    pcs.sample(x, 8192, method="npdu_afps", m=32, k=129)
torch.cuda.synchronize()
print(pcs.kernel_family("npdu_afps", 32768, 32, 129, batch=B))
