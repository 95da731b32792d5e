"""GPU timeline of one config-2 step (torch.profiler / CUPTI): kernels in
order with start offsets and the idle gaps between them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2510_04094_b200 import batch as BT, workloads as W
from paper_2510_04094_b200.problems import ivp

cfg = W.CONFIGS[2]
B = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.batch
bt = W.linear_batch(cfg, 0, B)
cond = ivp(bt.instances[0].conditions())
pipe = BT.SharedGridPipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond, B)
coef = torch.as_tensor(bt.coef, device="cuda")
forc = torch.as_tensor(bt.forcing, device="cuda")
vals = torch.as_tensor(bt.cond_values, device="cuda")
for _ in range(3):
    pipe.run_device(coef, forc, vals)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    pipe.run_device(coef, forc, vals)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
tot_gap = 0.0
for e in ev:
    gap = e.time_range.start - prev_end
    tot_gap += max(gap, 0)
    print(f"{(e.time_range.start - t0):9.1f} us  +gap {gap:7.1f}  dur {e.time_range.elapsed_us():8.1f}  {e.name[:70]}")
    prev_end = max(prev_end, e.time_range.end)
print(f"span {prev_end - t0:.1f} us, gaps {tot_gap:.1f} us")
