"""Timeline of pipelined config-3 batches (NP streams): ladder-kernel start/end
per stream and the host time per step (GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp

cfg = W.CONFIGS[3]
B = 256
g = W.grid(cfg)
lm = W.equidistant_landmarks(g, cfg.m)
insts = [W.instance(3, 0, i) for i in range(B)]
pts = g[1:]
fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                         np.array([i.quad_coeff for i in insts]),
                         np.array([i.sin_coeff for i in insts]))
vals = np.array([[i.conditions()[0][2]] for i in insts])
cond = ivp([(0.0, 0, 0.0)])
NP = int(sys.argv[1]) if len(sys.argv) > 1 else 3
streams = [torch.cuda.Stream() for _ in range(NP)]
slots = [None] * NP
tol_t = 1e-10 * (1.0 + cfg.gamma)
host = []


def step(k):
    s = k % NP
    t0 = time.perf_counter()
    if slots[s] is not None:
        eng, norms, ist = slots[s]
        eng.ladder_collect(norms, ist)
    t1 = time.perf_counter()
    with torch.cuda.stream(streams[s]):
        fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
        eng = NW.NewtonBatch(fm, g, cond, vals, cfg.gamma, family=fam)
        starts = eng.ladder_starts()
        t2 = time.perf_counter()
        norms, ist = eng.ladder_launch(*starts, cfg.newton_max_iters, tol_t)
        slots[s] = (eng, norms, ist)
    host.append((t1 - t0, t2 - t1, time.perf_counter() - t2))


for k in range(4):
    step(k)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(4, 10):
        step(k)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
      and "ladder" in e.name]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"ladder start {(e.time_range.start - t0) / 1e3:8.2f} ms  end "
          f"{(e.time_range.end - t0) / 1e3:8.2f} ms")
print("host per step (collect, setup, launch) ms:",
      [tuple(round(x * 1e3, 2) for x in h) for h in host[4:]])
