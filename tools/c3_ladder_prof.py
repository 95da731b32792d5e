"""Ladder kernel profile on the config-3 batch: per-instance chain clocks by phase,
wave structure, and the host-side parts of one step."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W, _lib
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp

B = 256
cfg = W.CONFIGS[3]
g = W.grid(cfg); lm = W.equidistant_landmarks(g, cfg.m); pts = g[1:]
insts = [W.instance(3, 0, i) for i in range(B)]
fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                         np.array([i.quad_coeff for i in insts]), np.array([i.sin_coeff for i in insts]))
vals = np.array([[i.conditions()[0][2]] for i in insts])
lib = _lib.load()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    eng = NW.NewtonBatch(fm, g, ivp([(0.0, 0, 0.0)]), vals, cfg.gamma, family=fam)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    ids = list(range(B))
    x0c = eng.const_state(ids); xl, _ = eng.linearized_state(ids)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    st, X, tr, rung = eng.solve(max_iters=cfg.newton_max_iters)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"fmap {1e3*(t1-t0):.2f} ms, engine {1e3*(t2-t1):.2f} ms, starts {1e3*(t3-t2):.2f} ms, solve {1e3*(t4-t3):.2f} ms")
prof = torch.zeros((B, 8), dtype=torch.int64, device="cuda")
lib.nys_newton_persist_profile(prof.data_ptr())
st, X, tr, rung = eng.solve(max_iters=cfg.newton_max_iters)
torch.cuda.synchronize()
lib.nys_newton_persist_profile(None)
p = prof.cpu().numpy().astype(float)
tot = p[:, :4].sum(1)
o = np.argsort(-tot)
print("phase totals over instances (Gclk): resid/ls %.2f reduce %.2f LU %.2f step %.2f trials %d" % (
    p[:, 0].sum() / 1e9, p[:, 1].sum() / 1e9, p[:, 2].sum() / 1e9, p[:, 3].sum() / 1e9, p[:, 5].sum()))
for j in o[:8]:
    print(f"inst {j}: rung {rung[j]} status {st[j]} chain {tot[j]/1.9e6:.2f} ms  resid/ls {p[j,0]/1e6:.1f}M reduce {p[j,1]/1e6:.1f}M LU {p[j,2]/1e6:.1f}M step {p[j,3]/1e6:.1f}M trials {int(p[j,5])}")
print("chain ms quantiles", np.percentile(tot / 1.9e6, [50, 90, 99, 100]).round(2))
print("first-wave (0..147) max", (tot[:148] / 1.9e6).max().round(2), "second wave max", (tot[148:] / 1.9e6).max().round(2))
