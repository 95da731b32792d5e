"""GPU timeline of steady-state SingleSolvePipeline calls (config argv[1],
default 1; argv[2] calls, default 6): kernels with start and duration.
WORLD=N: config 4's row-sharded pipeline over rank 0's slab of N."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2510_04094_b200 import linear as L, workloads as W
from paper_2510_04094_b200.problems import ivp

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ncall = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = W.CONFIGS[cid]
bt = W.linear_batch(cfg, 0, 1)
cond = ivp(bt.instances[0].conditions())
world = int(os.environ.get("WORLD", "1"))
rows = None
if world > 1:
    from paper_2510_04094_b200 import dist as DI
    rows = DI.row_ranges(bt.pts.size, world)[0]
    # the K all-reduce stood in for by a copy of the full K (tools/c4_rank_model.py)
    _f = L.SingleSolvePipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond)
    _e = torch.cuda.Event()
    _e.record()
    _f.run_device(torch.as_tensor(bt.pts, device="cuda"),
                  torch.as_tensor(bt.coef[0], device="cuda"),
                  torch.as_tensor(bt.forcing[0], device="cuda"), input_event=_e)
    torch.cuda.synchronize()
    _K = _f._kcur.clone()
    del _f
    DI.allreduce_sum = lambda t, group=None: t.copy_(_K)
pipe = L.SingleSolvePipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond,
                             rows=rows)
pts = torch.as_tensor(bt.pts, device="cuda")
coef = torch.as_tensor(bt.coef[0], device="cuda")
forc = torch.as_tensor(bt.forcing[0], device="cuda")
ev_in = torch.cuda.Event()
ev_in.record()
for _ in range(12):
    pipe.run_device(pts, coef, forc, input_event=ev_in)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(ncall):
        pipe.run_device(pts, coef, forc, input_event=ev_in)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{(e.time_range.start - t0):9.1f} us  dur {e.time_range.elapsed_us():8.1f}  "
          f"{e.name[:60]}")
print(f"span {ev[-1].time_range.end - t0:.1f} us for {ncall} calls")
