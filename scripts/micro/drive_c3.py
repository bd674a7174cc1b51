import torch
from paper_2512_05906_b200.engine import poisson_drive_device
for _ in range(2):
    m = poisson_drive_device(100000, 16, 1000, 1e-3, 16e-3, 12e-3, 1)
torch.cuda.synchronize()
