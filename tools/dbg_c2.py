import dilu_inputs as di
from paper_2503_05130_b200 import DiluSim
import torch
wl = di.c2(seed=0)
s = DiluSim.from_workload(wl)
for n in [1, 59, 540, 3000]:
    s.scale_step(n)
torch.cuda.synchronize()
print(s.metrics()[1].tolist()[14])
