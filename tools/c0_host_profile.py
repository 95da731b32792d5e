"""Host cost of steady-state SingleSolvePipeline calls (config argv[1], default
0): wall time per call with the GPU far ahead, and a cProfile of 2000 calls."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2510_04094_b200 import linear as L, workloads as W
from paper_2510_04094_b200.problems import ivp

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = W.CONFIGS[cid]
bt = W.linear_batch(cfg, 0, 1)
cond = ivp(bt.instances[0].conditions())
pipe = L.SingleSolvePipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond)
pts = torch.as_tensor(bt.pts, device="cuda")
coef = torch.as_tensor(bt.coef[0], device="cuda")
forc = torch.as_tensor(bt.forcing[0], device="cuda")
ev = torch.cuda.Event()
ev.record()
for _ in range(30):
    pipe.run_device(pts, coef, forc, input_event=ev)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    pipe.run_device(pts, coef, forc, input_event=ev)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host {1e6 * (t1 - t0) / n:.1f} us/call, wall {1e6 * (t2 - t0) / n:.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    pipe.run_device(pts, coef, forc, input_event=ev)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
