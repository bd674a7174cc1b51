"""Device PoissonDrive at C3 x 16 trials (for an ncu capture of k_poisson_drive)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

from paper_2512_05906_b200.engine import poisson_drive_device  # noqa: E402

for _ in range(2):
    m = poisson_drive_device(100000, 16, 1000, 1e-3, 16e-3, 12e-3, 1)
torch.cuda.synchronize()
print("ok", m.shape)
