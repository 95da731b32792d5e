"""Compare the device eigendecomposition against numpy (diagnostic)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_04094_b200 import nystrom as N, workloads as W  # noqa: E402
from paper_2510_04094_b200.kernel import RbfKernel  # noqa: E402

for cid in (0, 2, 4):
    c = W.CONFIGS[cid]
    g = W.grid(W.scaled(c, n=min(c.n, 1 << 16)))
    lm = W.equidistant_landmarks(g, c.m)
    A = np.exp(-(lm[:, None] - lm[None, :]) ** 2 / c.sigma2)
    fm = N.build_feature_map(RbfKernel(c.sigma2), lm)
    lam = fm.d_eigvals.cpu().numpy()
    V = fm.d_eigvecs.cpu().numpy()
    ref = np.sort(np.linalg.eigvalsh(A))[::-1]
    err = np.abs(lam - ref)
    print(f"c{cid} m={c.m} maxerr={err.max():.3e} at {err.argmax()} resid={np.abs(A @ V - V * lam).max():.3e} "
          f"orth={np.abs(V.T @ V - np.eye(c.m)).max():.3e}")
    bad = np.where(err > 1e-12 * ref[0])[0]
    print("  bad idx", bad[:20], lam[bad[:5]], ref[bad[:5]])
