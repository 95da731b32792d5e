import sys, os, numpy as np
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
sys.path.insert(0, os.getcwd())
import torch
from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp
cfg = W.CONFIGS[3]; B = 256
g = W.grid(cfg); lm = W.equidistant_landmarks(g, cfg.m)
insts = [W.instance(3, 0, i) for i in range(B)]
pts = g[1:]
fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]), np.array([i.quad_coeff for i in insts]), np.array([i.sin_coeff for i in insts]))
vals = np.array([[i.conditions()[0][2]] for i in insts])
cond = ivp([(0.0, 0, 0.0)])
fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
eng = NW.NewtonBatch(fm, g, cond, vals, cfg.gamma, family=fam)
st, X, tr, rung = eng.solve(max_iters=cfg.newton_max_iters)
t = eng.total_iterations
print("iterations: mean %.1f median %d p90 %d p99 %d max %d sum %d" % (t.mean(), np.median(t), np.percentile(t,90), np.percentile(t,99), t.max(), t.sum()))
print("rungs", np.bincount(rung))
print("top 10", sorted(t)[-10:])
print("regs/occupancy: B", B)
