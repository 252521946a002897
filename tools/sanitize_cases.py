"""Small invocations of every kernel family (for compute-sanitizer)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

x = torch.from_numpy(synth.uniform_cube(3, 4099, 1)).cuda()
pcs.sample(x, 300, method="fps")                              # Morton TMEM
pcs.sample(x, 300, method="afps", m=4)                        # full kernel
pcs.sample(x, 300, method="npdu_afps", m=4, k=129)            # NPDU wide (<= 148 sectors)
xb = torch.from_numpy(synth.uniform_cube(40, 4099, 4)).cuda()
pcs.sample(xb, 300, method="npdu_afps", m=4, k=129)           # NPDU TMEM (160 sectors)
pcs.sample(xb[:, :1000], 300, method="npdu_afps", m=1, k=65)  # NPDU wide, P=4
pcs.sample(x, 300, method="npdu_fps", k=65)                   # TMEM rows, window mode
pcs.sample(x.double(), 300, method="fps")                     # Morton smem (fp64)
pcs.sample(x.double(), 300, method="npdu_afps", m=2, k=33)    # NPDU warp kernel
pcs.sort_axis(x, "y")                                         # register bitonic
pcs.sort_axis(torch.from_numpy(synth.uniform_cube(1, 70000, 2)).cuda(), "x")      # cluster
pcs.sort_axis(torch.from_numpy(synth.uniform_cube(1, 300000, 2)).cuda(), "x")     # device radix
big = torch.from_numpy(synth.uniform_cube(1, 20000, 5)).cuda()
pcs.sample(big, 50, method="fps")                             # Morton TMEM cluster
xs = torch.from_numpy(synth.uniform_cube(40, 8192, 6)).cuda()
xs[1, :5000, 0] = 0.5                                         # a huge bucket: flagged
pcs.sort_perm(xs, "x")                                        # bucket sort + flagged radix
xm = torch.from_numpy(synth.uniform_cube(700, 4096, 7)).cuda()
pcs.sample(xm, 1024, method="npdu_afps", m=4, k=129)          # NPDU TMEM, high-word keys
pcs.sample(torch.from_numpy(synth.uniform_cube(1, 2048, 8)).cuda(), 300, method="fps")  # cluster
import os
os.environ["PCS_SAMPLER"] = "stream"
pcs.reload_knobs()
pcs.sample(x, 100, method="fps")                              # streaming engine
os.environ["PCS_SAMPLER"] = "rows"
os.environ["PCS_MORTON"] = "0"
pcs.reload_knobs()
pcs.sample(x, 100, method="npdu_fps", k=65)                   # slab rows
del os.environ["PCS_SAMPLER"], os.environ["PCS_MORTON"]
pcs.reload_knobs()
pts = synth.random_cloud(500, 3)
pcs.fps(pts, 50)
pcs.npdu_afps(pts, 50, 5, 9)
pcs.local_fps(pts, 10, 400, 30, k=7, trace=True)              # wide kernel, fp64 + trace
pcs.sample_host_batch(synth.uniform_cube(4, 1000, 3), 100, method="npdu_afps", m=2, k=33, sort="x")
idx = pcs.sample(x, 100, method="afps", m=2)[0]
pcs.quality(x, idx)
torch.cuda.synchronize()
print("ok")
