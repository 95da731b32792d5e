"""cProfile of one config-3 step (host-side view: which calls block or cost)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp

cfg = W.CONFIGS[3]
g = W.grid(cfg)
lm = W.equidistant_landmarks(g, cfg.m)
insts = [W.instance(3, 0, i) for i in range(cfg.batch)]
pts = g[1:]
fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                         np.array([i.quad_coeff for i in insts]),
                         np.array([i.sin_coeff for i in insts]))
vals = np.array([[i.conditions()[0][2]] for i in insts])
cond = ivp([(0.0, 0, 0.0)])


def step():
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
    eng = NW.NewtonBatch(fm, g, cond, vals, cfg.gamma, family=fam)
    eng.solve(max_iters=cfg.newton_max_iters)


for _ in range(2):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
