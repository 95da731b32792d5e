"""Time every BASELINE config through the public API on one GPU (diagnostic)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_04094_b200 import _lib, linear as L, newton as NW, nystrom as N, workloads as W  # noqa
from paper_2510_04094_b200.kernel import RbfKernel  # noqa
from paper_2510_04094_b200.problems import ivp  # noqa


def single(cid, reps=5, n=None):
    cfg = W.CONFIGS[cid] if n is None else W.scaled(W.CONFIGS[cid], n=n)
    bt = W.linear_batch(cfg, 0, 1)
    cond = ivp(bt.instances[0].conditions())
    pts = torch.as_tensor(bt.pts, device="cuda")
    coef = torch.as_tensor(bt.coef[0], device="cuda")
    forc = torch.as_tensor(bt.forcing[0], device="cuda")

    def run():
        fm = N.build_feature_map(RbfKernel(cfg.sigma2), bt.landmarks)
        E = L.gram_ext_device(fm, cfg.order, pts, coef, forc)
        Ac, beta, vals = L.condition_rows(cond, fm)
        sy = L.AssembledSystem(bt.pts, cfg.gamma, -bt.coef[0, -1], bt.forcing[0], bt.coef[0],
                               Ac.reshape(len(cond.entries), -1), beta, vals, fm, cfg.order, E)
        return fm, L.solve(sy, fm)
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fm, mdl = run()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    y = mdl.predict(0, bt.grid[:: max(1, bt.grid.size // 4096)])
    return min(ts), fm.m_eff


def newton(B=256):
    cfg = W.CONFIGS[3]
    g = W.grid(cfg)
    lm = W.equidistant_landmarks(g, cfg.m)
    insts = [W.instance(3, 0, i) for i in range(B)]
    pts = g[1:]
    fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                             np.array([i.quad_coeff for i in insts]),
                             np.array([i.sin_coeff for i in insts]))
    vals = np.array([[i.conditions()[0][2]] for i in insts])
    cond = ivp([(0.0, 0, 0.0)])
    t0 = time.perf_counter()
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
    eng = NW.NewtonBatch(fm, g, cond, vals, cfg.gamma, family=fam)
    st, X, tr, rung = eng.solve(max_iters=cfg.newton_max_iters)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    its = sum(len(t) - 1 for t in tr)
    return dt, np.bincount(st, minlength=4), np.bincount(rung, minlength=6), its


if __name__ == "__main__":
    for cid in (0, 1):
        dt, me = single(cid)
        print(f"c{cid}: {dt*1e3:.3f} ms/solve (m_eff {me})", flush=True)
    for n in (1 << 18, 1 << 22):
        dt, me = single(4, reps=3, n=n)
        print(f"c4 n={n}: {dt*1e3:.2f} ms/solve (m_eff {me})", flush=True)
    for B in (16, 256):
        dt, st, rg, its = newton(B)
        print(f"c3 B={B}: {dt:.3f} s, status {st.tolist()}, rungs {rg.tolist()}, newton its {its}",
              flush=True)
