"""GPU timeline of one single-instance solve (config argv[1], default 0):
kernels with start offsets and the idle gaps between them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2510_04094_b200 import linear as L, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = W.CONFIGS[cid]
bt = W.linear_batch(cfg, 0, 1)
cond = ivp(bt.instances[0].conditions())
pts = torch.as_tensor(bt.pts, device="cuda")
coef = torch.as_tensor(bt.coef[0], device="cuda")
forc = torch.as_tensor(bt.forcing[0], device="cuda")


def solve():
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), bt.landmarks)
    E = L.gram_ext_device(fm, cfg.order, pts, coef, forc)
    Ac, beta, vals = L.condition_rows(cond, fm)
    sy = L.AssembledSystem(bt.pts, cfg.gamma, None, None, None,
                           Ac.reshape(len(cond.entries), -1), beta, vals, fm, cfg.order, E)
    return L._kkt_solve(sy)


if len(sys.argv) > 2:
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    solve = __import__(sys.argv[2]).make(cfg, bt, cond, pts, coef, forc)
for _ in range(5):
    solve()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    solve()
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
ev0 = torch.cuda.Event(enable_timing=True)
ev1 = torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(20):
    solve()
ev1.record()
torch.cuda.synchronize()
print(f"plain: {ev0.elapsed_time(ev1) / 20 * 1e3:.1f} us per solve")
