"""Golden vectors for ridge leverage-score landmark selection: the LIVE
reference's ``nystrom.ridge_leverage_scores`` and ``select_landmarks(LeverageScore)``
(nystrom.py:58-103) on a few grids.

Build container only:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_leverage.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from nysode import nystrom  # noqa: E402
from nysode.kernel import RbfKernel  # noqa: E402

# (name, grid, sigma2 or None for the default score kernel, ridge, m, seeds)
CASES = [
    ("u50", np.linspace(0.0, 1.0, 50), None, 1e-6, 10, (3, 4, 5)),
    ("u300", np.linspace(-1.0, 2.0, 300), 0.01, 1e-6, 40, (0, 1)),
    ("u1000", np.linspace(0.0, 1.0, 1000), 0.01, 1e-6, 50, (0, 7)),
    ("u1000r4", np.linspace(0.0, 10.0, 1000), None, 1e-4, 64, (2,)),
    ("u4000", np.linspace(0.0, 1.0, 4000), None, 1e-6, 100, (0,)),
]


def main():
    out = {}
    for name, grid, s2, ridge, m, seeds in CASES:
        kern = RbfKernel(sigma2=s2) if s2 is not None else None
        score_k = kern or RbfKernel(sigma2=max(float(grid[-1] - grid[0]) / 10.0, 1e-6) ** 2)
        scores = nystrom.ridge_leverage_scores(score_k, grid, ridge)
        out[f"{name}_grid"] = grid
        out[f"{name}_sigma2"] = np.array(score_k.sigma2)
        out[f"{name}_ridge"] = np.array(ridge)
        out[f"{name}_scores"] = scores
        out[f"{name}_m"] = np.array(m)
        out[f"{name}_seeds"] = np.array(seeds)
        out[f"{name}_explicit_kernel"] = np.array(kern is not None)
        for sd in seeds:
            lm = nystrom.select_landmarks(nystrom.LeverageScore(seed=sd, ridge=ridge, kernel=kern),
                                          grid, m)
            out[f"{name}_lm{sd}"] = lm
    out["cases"] = np.array([c[0] for c in CASES])
    np.savez_compressed(os.path.join(HERE, "leverage.npz"), **out)
    print("wrote leverage.npz", {c[0]: len(c[5]) for c in CASES})


SKETCH_CASES = [
    ("s4001", np.linspace(0.0, 1.0, 4001), None, 1e-6, 30, (0,)),
    ("s6000", np.linspace(-2.0, 3.0, 6000), None, 1e-6, 50, (1, 2)),
    ("s10000", np.linspace(0.0, 1.0, 10000), 0.01, 1e-6, 80, (0,)),
    ("s8192r", np.linspace(0.0, 4.0, 8192), 0.09, 1e-5, 64, (3,)),
]


def main_sketch():
    out = {}
    for name, grid, s2, ridge, m, seeds in SKETCH_CASES:
        kern = RbfKernel(sigma2=s2) if s2 is not None else None
        score_k = kern or RbfKernel(sigma2=max(float(grid[-1] - grid[0]) / 10.0, 1e-6) ** 2)
        scores = nystrom.ridge_leverage_scores(score_k, grid, ridge)
        # the same sketch with the LAPACK dsyev driver instead of dsyevd: the
        # reference's own sensitivity to its eigensolver (the parity yardstick)
        idx = np.linspace(0, grid.size - 1, 2000).round().astype(int)
        from nysode import kernel as kmod
        C = kmod.kernel_matrix(score_k, 0, grid, grid[idx])
        W = C[idx, :]
        import scipy.linalg as sl
        vals, vecs = sl.eigh((W + W.T) / 2.0, driver="ev")
        keep = vals > vals.max() * 1e-12
        A = C @ (vecs[:, keep] / np.sqrt(vals[keep]))
        inner = np.linalg.solve(A.T @ A + grid.size * ridge * np.eye(A.shape[1]), A.T)
        alt = np.clip(np.einsum("ij,ji->i", A, inner), 1e-300, None)
        out[f"{name}_n"] = np.array(grid.size)
        out[f"{name}_lo"] = np.array(grid[0])
        out[f"{name}_hi"] = np.array(grid[-1])
        out[f"{name}_sigma2"] = np.array(score_k.sigma2)
        out[f"{name}_ridge"] = np.array(ridge)
        out[f"{name}_scores"] = scores
        out[f"{name}_scores_dsyev"] = alt
        out[f"{name}_keep"] = np.array(int(keep.sum()))
        out[f"{name}_m"] = np.array(m)
        out[f"{name}_seeds"] = np.array(seeds)
        out[f"{name}_explicit_kernel"] = np.array(kern is not None)
        for sd in seeds:
            lm = nystrom.select_landmarks(nystrom.LeverageScore(seed=sd, ridge=ridge, kernel=kern),
                                          grid, m)
            out[f"{name}_lm{sd}"] = lm
        print(name, "keep", int(keep.sum()), "self-sens", float(np.max(np.abs(alt / scores - 1))))
    out["cases"] = np.array([c[0] for c in SKETCH_CASES])
    np.savez_compressed(os.path.join(HERE, "leverage_sketch.npz"), **out)


if __name__ == "__main__":
    main()
    main_sketch()
