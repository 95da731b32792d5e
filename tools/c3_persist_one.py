"""One damped persistent Newton rung on the config-3 batch (profiling driver)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp

B = 256
cfg = W.CONFIGS[3]
g = W.grid(cfg); lm = W.equidistant_landmarks(g, cfg.m); pts = g[1:]
insts = [W.instance(3, 0, i) for i in range(B)]
fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                         np.array([i.quad_coeff for i in insts]), np.array([i.sin_coeff for i in insts]))
vals = np.array([[i.conditions()[0][2]] for i in insts])
fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
eng = NW.NewtonBatch(fm, g, ivp([(0.0, 0, 0.0)]), vals, cfg.gamma, family=fam)
ids = list(range(B))
x0 = eng.linearized_state(ids)[0]
st, Xn, tr = eng.solve_once(ids, x0, cfg.gamma, 1e-10 * (1 + cfg.gamma), True, cfg.newton_max_iters)
torch.cuda.synchronize()
print("status", np.bincount(st, minlength=4).tolist())
