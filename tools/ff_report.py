"""Full-feature comparator: device vs reference goldens (error, yardstick, time)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "tests")
from conftest import load_golden  # noqa: E402
from test_gpu_full_feature import _problem, _rel  # noqa: E402

from paper_2510_04094_b200 import baselines as BL  # noqa: E402

g = load_golden("full_feature")
for pid in g["pids"]:
    key = f"p{int(pid)}"
    prob = _problem(g, key)
    n = int(g[f"{key}_n"])
    args = (prob, float(g[f"{key}_gamma"]), float(g[f"{key}_sigma2"]), n)
    BL.full_feature_baseline(*args)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        model, secs = BL.full_feature_baseline(*args)
        ts.append(secs)
    y = model.predict(0, BL.grid_for(prob, n))
    print(f"P{int(pid)} n={n} m_eff dev {model.feature_map.m_eff} ref {int(g[key + '_m_eff'])}"
          f"  |y-ref| {_rel(y, g[key + '_yhat']):.2e}  yardstick {_rel(g[key + '_yhat_dsyev'], g[key + '_yhat']):.2e}"
          f"  train dev {np.median(ts) * 1e3:.1f} ms  ref {float(g[key + '_seconds']) * 1e3:.0f} ms")
# n = 5000 (the cap), P7 shape
key = "p7"
prob = _problem(g, key)
for n in (2000, 5000):
    grid = BL.grid_for(prob, n)
    from paper_2510_04094_b200 import nystrom as N, linear as L
    from paper_2510_04094_b200.kernel import RbfKernel
    t0 = time.perf_counter()
    fm = N.build_feature_map(RbfKernel(float(g[key + "_sigma2"])), grid)
    torch.cuda.synchronize()
    print(f"n={n}: compressed eig {1e3 * (time.perf_counter() - t0):.1f} ms, m_eff {fm.m_eff}, rank {fm._host['compressed']}")
