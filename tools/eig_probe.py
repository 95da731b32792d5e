"""Eigensolver probe: sweeps, time and parity of y_hat vs golden for several
stopping thresholds (NYS_EIG_TOLSCALE).  Run on the GPU box."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, "%s"); sys.path.insert(0, "%s/tests")
from paper_2510_04094_b200 import nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from conftest import load_golden
from gpu_util import fmap_from_golden, solve_golden_instance, rel_l2
out = []
for cid in (0, 1, 2, 4):
    c = W.CONFIGS[cid]; g = W.grid(W.scaled(c, n=min(c.n, 1 << 16))); lm = W.equidistant_landmarks(g, c.m)
    fm = N.build_feature_map(RbfKernel(c.sigma2), lm); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3): fm = N.build_feature_map(RbfKernel(c.sigma2), lm)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
    out.append(f"c{cid}: m_eff={fm.m_eff} sweeps={fm._host['sweeps']} {dt*1e3:.2f}ms")
for name in ("cat_p2", "cat_p12", "cat_p16", "c1_seed0", "c2_seed0_i0-7"):
    gd = load_golden(name); fm = fmap_from_golden(gd); sy, mdl = solve_golden_instance(gd, fm, 0)
    out.append(f"{name}: m_eff={fm.m_eff}/{int(gd['m_eff'])} dyhat={rel_l2(mdl.predict(0, gd['grid']), gd['yhat'][0]):.2e}")
print(" | ".join(out))
''' % (ROOT, ROOT)
for ts in sys.argv[1:] or ["1"]:
    env = dict(os.environ, NYS_EIG_TOLSCALE=ts)
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print("tolscale", ts, "->", r.stdout.strip() or r.stderr[-2000:])
