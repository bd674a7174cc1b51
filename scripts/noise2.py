import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2512_05906_b200.engine import Engine
net, mask, amp, T = bench.make_inputs("C3", 16, 0)
md = torch.from_numpy(mask.view(np.int32)).cuda()
eng = Engine(net.n, 16, T)
eng.set_network(net.rowptr, net.col, net.weight, net.delay)
eng.set_drive(md, torch.from_numpy(amp).cuda().float())
mode = sys.argv[1]
def it():
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record(); out = eng.forward(); b.record()
    vbar = (2.0 * (out["v"] - 0.25)).to(eng.dtype)
    gw, gd, _ = eng.backward(vbar, want_amp=False); c.record()
    return (a, b, c)
evs = []
for i in range(3): it()
torch.cuda.synchronize()
if mode == "counters": eng.counters()
if mode == "sleep": time.sleep(0.5)
torch.cuda.synchronize()
for i in range(8): evs.append(it())
torch.cuda.synchronize()
print(mode, "bwd", " ".join("%.1f" % b.elapsed_time(c) for a, b, c in evs))
