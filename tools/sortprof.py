import torch, sys
sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs
from paper_2208_08795_b200 import synth
x = torch.from_numpy(synth.uniform_cube(256, 8192, 1)).cuda()
for _ in range(3): pcs.sort_axis(x, "x")
torch.cuda.synchronize()
