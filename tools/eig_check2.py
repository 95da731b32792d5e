import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_04094_b200 import nystrom as N, workloads as W  # noqa
from paper_2510_04094_b200.kernel import RbfKernel  # noqa
for cid in (2, 2, 2, 4, 4):
    c = W.CONFIGS[cid]
    g = W.grid(W.scaled(c, n=min(c.n, 1 << 16)))
    lm = W.equidistant_landmarks(g, c.m)
    A = np.exp(-(lm[:, None] - lm[None, :]) ** 2 / c.sigma2)
    for rep in range(3):
        fm = N.build_feature_map(RbfKernel(c.sigma2), lm)
        lam = fm.d_eigvals.cpu().numpy(); V = fm.d_eigvecs.cpu().numpy()
        print(cid, rep, fm.m_eff, f"resid={np.abs(A @ V - V * lam).max():.2e}", lam[-3:])
