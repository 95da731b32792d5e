"""Where does a config-3 step spend its time?  Counts and times NewtonBatch
methods (host wall clock, each call synchronising as it already does)."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp

cfg = W.CONFIGS[3]
B = cfg.batch
g = W.grid(cfg)
lm = W.equidistant_landmarks(g, cfg.m)
insts = [W.instance(3, 0, i) for i in range(B)]
pts = g[1:]
fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                         np.array([i.quad_coeff for i in insts]),
                         np.array([i.sin_coeff for i in insts]))
vals = np.array([[i.conditions()[0][2]] for i in insts])
cond = ivp([(0.0, 0, 0.0)])
stats = collections.defaultdict(lambda: [0, 0.0, 0])


def wrap(name):
    f = getattr(NW.NewtonBatch, name)

    def g(self, *a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(self, *a, **k)
        torch.cuda.synchronize()
        s = stats[name]
        s[0] += 1
        s[1] += time.perf_counter() - t
        ids = a[0] if a else None
        s[2] += len(ids) if isinstance(ids, (list, tuple)) else 0
        return r
    setattr(NW.NewtonBatch, name, g)


for nm in ("residual", "direction", "candidate", "solve_once", "const_state", "_line_search",
           "linearized_state", "model_state"):
    wrap(nm)
for rep in range(2):
    stats.clear()
    torch.cuda.synchronize()
    t = time.perf_counter()
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
    eng = NW.NewtonBatch(fm, g, cond, vals, cfg.gamma, family=fam)
    st, X, tr, rung = eng.solve(max_iters=cfg.newton_max_iters)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t
print(f"total {tot*1e3:.1f} ms  status {np.bincount(st, minlength=4)}  rungs {np.bincount(rung)}")
for k, (n, s, ni) in sorted(stats.items(), key=lambda x: -x[1][1]):
    print(f"{k:18s} calls {n:6d}  {s*1e3:8.1f} ms  {s/n*1e6 if n else 0:8.1f} us/call  ids/call {ni/max(n,1):.1f}")
