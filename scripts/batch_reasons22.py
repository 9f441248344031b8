import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rgg

g = gen_rgg(1 << 22, 0.55, 1)
dg = D.DeviceGraph.from_host(g)
D.integrated_map_device(dg, (4, 8, 6), (1, 10, 100), 0.03, 0)
torch.cuda.synchronize()
