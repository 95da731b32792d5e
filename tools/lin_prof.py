import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W, batch as BT
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp
cfg = W.CONFIGS[3]; B = cfg.batch; g = W.grid(cfg); lm = W.equidistant_landmarks(g, cfg.m)
insts = [W.instance(3, 0, i) for i in range(B)]; pts = g[1:]
fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]), np.array([i.quad_coeff for i in insts]), np.array([i.sin_coeff for i in insts]))
vals = np.array([[i.conditions()[0][2]] for i in insts]); cond = ivp([(0.0, 0, 0.0)])
fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
eng = NW.NewtonBatch(fm, g, cond, vals, cfg.gamma, family=fam)
ids = list(range(176))
T = {}
orig_solve = BT.LinearBatchSolver.solve
def timed(name, f):
    def w(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter(); r = f(*a, **k); torch.cuda.synchronize()
        T[name] = T.get(name, 0) + time.perf_counter() - t; return r
    return w
BT.LinearBatchSolver.solve = timed("solver.solve", BT.LinearBatchSolver.solve)
BT.LinearBatchSolver.__init__ = timed("solver.init", BT.LinearBatchSolver.__init__)
eng.model_state = timed("model_state", eng.model_state)
eng.const_state = timed("const_state", eng.const_state)
for rep in range(3):
    T.clear()
    torch.cuda.synchronize(); t = time.perf_counter()
    eng.linearized_state(ids)
    torch.cuda.synchronize(); T["total"] = time.perf_counter() - t
    print({k: round(v * 1e3, 2) for k, v in T.items()})
