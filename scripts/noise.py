"""Run-to-run variance of the fwd/bwd launches: several engines (fresh
allocations) x several passes each, C3 x 16 trials."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_05906_b200.engine import Engine  # noqa: E402

net, mask, amp, T = bench.make_inputs("C3", 16, 0)
md = torch.from_numpy(mask.view(np.int32)).cuda()
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    eng = Engine(net.n, 16, T)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(md, torch.from_numpy(amp).cuda().float())
    fw, bw = [], []
    for it in range(int(os.environ.get("NOISE_ITERS", "6"))):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        out = eng.forward()
        b.record()
        eng.backward((2 * (out["v"] - 0.25)), want_amp=False)
        c.record()
        torch.cuda.synchronize()
        fw.append(a.elapsed_time(b))
        bw.append(b.elapsed_time(c))
    print(f"engine {rep}: fwd " + " ".join(f"{x:.1f}" for x in fw) + " | bwd " + " ".join(f"{x:.1f}" for x in bw),
          flush=True)
    del eng
    torch.cuda.empty_cache()
