"""Cluster eigensolver (64 < m <= 256) against numpy and the one-CTA kernel:
eigenvalues, residual, orthogonality, time per call (diagnostic, GPU box)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_04094_b200 import nystrom as N  # noqa: E402
from paper_2510_04094_b200.kernel import RbfKernel  # noqa: E402

algo = os.environ.get("NYS_EIG_ALGO", "cluster")
for m, T, s2 in ((256, 100.0, 0.25), (256, 2.0, 0.01), (200, 5.0, 0.04), (129, 3.0, 0.05),
                 (100, 1.0, 0.01), (67, 1.0, 0.02), (80, 1.0, 0.3)):
    lm = np.linspace(0.0, T, m)
    A = np.exp(-(lm[:, None] - lm[None, :]) ** 2 / s2)
    fm = N.build_feature_map(RbfKernel(s2), lm)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fm = N.build_feature_map(RbfKernel(s2), lm)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    lam = fm.d_eigvals.cpu().numpy()
    V = fm.d_eigvecs.cpu().numpy()
    ref = np.sort(np.linalg.eigvalsh(A))[::-1]
    err = np.abs(lam - ref).max() / ref[0]
    res = np.abs(A @ V - V * lam).max()
    orth = np.abs(V.T @ V - np.eye(m)).max()
    ok = err < 1e-13 and res < 1e-12 and orth < 1e-12
    print(f"[{algo}] m={m} T={T} s2={s2} m_eff={fm.m_eff} eigerr/s0={err:.2e} resid={res:.2e} "
          f"orth={orth:.2e} {dt * 1e3:.3f} ms/call {'OK' if ok else 'BAD'}")
