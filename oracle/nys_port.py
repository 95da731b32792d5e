"""CPU oracle: NumPy restatement of the reference's linear hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` legs may import this module,
and only as the checker or the timed CPU baseline -- never as the product.

Restated from the reference package ``nysode`` (``/root/reference/pkg/src/nysode``),
array-in / array-out, following the same NumPy/BLAS operation order so that it
reproduces the reference to round-off (pinned against ``tests/golden/*.npz``,
which ``tests/golden/make_golden.py`` generates by importing the live
reference in the build container).  Each function cites the lines it follows.
"""
from __future__ import annotations

from typing import Callable, Sequence, Union

import numpy as np

DROP_TOL = 1e-16            # nystrom.py:21
KKT_TOL = 1e-8              # linear.py:33

ArrayOrFn = Union[np.ndarray, Callable]


class OracleError(RuntimeError):
    pass


# ---------------------------------------------------------------- kernel.py


def hermite_coeffs(sigma2: float, order: int) -> np.ndarray:
    """Low-degree-first coefficients of P_order (kernel.py:26-37).

    P_0 = 1, P_{a+1}(d) = (2 d / sigma2) P_a(d) - P_a'(d).
    """
    c = np.array([1.0])
    for _ in range(order):
        up = np.concatenate(([0.0], c)) * (2.0 / sigma2)
        dc = c[1:] * np.arange(1, c.size)
        up[: dc.size] -= dc
        c = up
    return c


def rbf_block(sigma2: float, order: int, rows, cols) -> np.ndarray:
    """d^a K(rows_i, cols_j)/d cols_j^a, d = rows_i - cols_j (kernel.py:75-92)."""
    d = np.asarray(rows, dtype=float)[:, None] - np.asarray(cols, dtype=float)[None, :]
    e = np.exp(-(d * d) / sigma2)
    if order == 0:
        return e
    acc = np.zeros_like(d)
    for c in hermite_coeffs(sigma2, order)[::-1]:        # _horner, kernel.py:62-66
        acc = acc * d + c
    return acc * e


# ---------------------------------------------------------------- nystrom.py


def equidistant(grid: np.ndarray, m: int) -> np.ndarray:
    """nystrom.py:84-91 (Equidistant)."""
    n = grid.size
    if m < 2 or m > n:
        raise OracleError(f"landmark count {m} outside 2..{n}")
    return grid[np.round(np.arange(m) * (n - 1) / (m - 1)).astype(int)]


LEVERAGE_EXACT_LIMIT = 4000  # nystrom.py:25


def leverage_scores(sigma2: float, grid, ridge: float) -> np.ndarray:
    """Ridge leverage scores (nystrom.py:58-81).

    n <= 4000: diag of solve(Omega + n ridge I, Omega); otherwise the uniform
    column sketch of :71-80.  Clipped below at 1e-300 (:81).
    """
    grid = np.asarray(grid, dtype=float)
    n = grid.size
    if n <= LEVERAGE_EXACT_LIMIT:
        omega = rbf_block(sigma2, 0, grid, grid)
        res = np.linalg.solve(omega + n * ridge * np.eye(n), omega)
        return np.clip(np.diagonal(res).copy(), 1e-300, None)
    # uniform column sketch (nystrom.py:71-80)
    c = LEVERAGE_EXACT_LIMIT // 2
    idx = np.linspace(0, n - 1, c).round().astype(int)
    C = rbf_block(sigma2, 0, grid, grid[idx])
    W = C[idx, :]
    vals, vecs = np.linalg.eigh((W + W.T) / 2.0)
    keep = vals > vals.max() * 1e-12
    A = C @ (vecs[:, keep] / np.sqrt(vals[keep]))
    inner = np.linalg.solve(A.T @ A + n * ridge * np.eye(A.shape[1]), A.T)
    return np.clip(np.einsum("ij,ji->i", A, inner), 1e-300, None)


def leverage_landmarks(scores: np.ndarray, seed: int, m: int) -> np.ndarray:
    """Landmark indices drawn from the scores (nystrom.py:95-103)."""
    rng = np.random.default_rng(seed)
    p = scores / scores.sum()
    return np.sort(rng.choice(scores.size, size=m, replace=False, p=p))


def leverage_default_sigma2(grid) -> float:
    """Neutral score kernel: length scale span / 10 (nystrom.py:97-100)."""
    span = float(grid[-1] - grid[0])
    return max(span / 10.0, 1e-6) ** 2


def eig_landmarks(sigma2: float, landmarks, drop_tol: float = DROP_TOL):
    """Kept eigenpairs of Omega_mm, descending (nystrom.py:136-160).

    Returns (s, V): s (m_eff,), V (m, m_eff).
    """
    lm = np.asarray(landmarks, dtype=float)
    if lm.size >= 2 and np.min(np.diff(np.sort(lm))) <= 1e-12:
        raise OracleError("degenerate landmarks")
    om = rbf_block(sigma2, 0, lm, lm)
    s, v = np.linalg.eigh((om + om.T) / 2.0)
    idx = np.argsort(s)[::-1]
    s, v = s[idx], v[:, idx]
    keep = s > max(drop_tol * s[0], 0.0)
    return s[keep], v[:, keep]


def scaled_basis(s: np.ndarray, v: np.ndarray) -> np.ndarray:
    """W = V / sqrt(s) (nystrom.py:120-121)."""
    return v / np.sqrt(s)


def features(sigma2, landmarks, W, order: int, pts) -> np.ndarray:
    """Psi_order(pts) = K_order(L, pts)^T W, shape (|pts|, m_eff) (nystrom.py:123-127)."""
    pts = np.atleast_1d(np.asarray(pts, dtype=float))
    return rbf_block(sigma2, order, landmarks, pts).T @ W


# ---------------------------------------------------------------- linear.py


def _values(x: ArrayOrFn, pts: np.ndarray) -> np.ndarray:
    return np.asarray(x(pts) if callable(x) else x, dtype=float)


def assemble(order: int, coeffs: Sequence[ArrayOrFn], forcing: ArrayOrFn,
             cond: Sequence[tuple[float, int, float]], grid, gamma: float,
             sigma2: float, landmarks, W, kind: str = "ivp"):
    """Primal KKT matrix and rhs (linear.py:90-137).

    ``coeffs`` / ``forcing`` are either callables of t (the reference's spec) or
    arrays already sampled on the constraint points.  Returns a dict with
    M, rhs, D, g, r, Ac, beta, values, pts.
    """
    grid = np.asarray(grid, dtype=float)
    if gamma <= 0:
        raise ValueError("gamma must be positive")
    pts = grid[1:] if kind == "ivp" else grid[1:-1]              # linear.py:66-68
    D = features(sigma2, landmarks, W, order, pts)
    fvals = []
    for k, fk in enumerate(coeffs, start=1):                      # linear.py:104-112
        fv = _values(fk, pts)
        if not np.all(np.isfinite(fv)):
            raise FloatingPointError(f"coefficient f_{k} non-finite")
        fvals.append(fv)
        D = D - fv[:, None] * features(sigma2, landmarks, W, order - k, pts)
    g = -fvals[-1]
    r = _values(forcing, pts)
    if not np.all(np.isfinite(r)):
        raise FloatingPointError("forcing non-finite")
    Ac = np.array([features(sigma2, landmarks, W, o, [t])[0] for (t, o, _) in cond])
    beta = np.array([1.0 if o == 0 else 0.0 for (_, o, _) in cond])
    vals = np.array([v for (_, _, v) in cond])
    me = W.shape[1]
    side = me + 1 + len(cond)
    M = np.zeros((side, side))                                    # linear.py:123-131
    M[:me, :me] = np.eye(me) / gamma + D.T @ D
    M[:me, me] = D.T @ g
    M[me, :me] = M[:me, me]
    M[me, me] = g @ g
    M[:me, me + 1:] = Ac.T
    M[me + 1:, :me] = Ac
    M[me, me + 1:] = beta
    M[me + 1:, me] = beta
    rhs = np.concatenate([D.T @ r, [g @ r], vals])               # linear.py:133
    return dict(M=M, rhs=rhs, D=D, g=g, r=r, Ac=Ac, beta=beta, values=vals, pts=pts)


def solve_kkt(M: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """LU solve + one refinement step (linear.py:140-158)."""
    try:
        x = np.linalg.solve(M, rhs)
        x = x + np.linalg.solve(M, rhs - M @ x)
    except np.linalg.LinAlgError as exc:
        raise OracleError(f"singular KKT system: {exc}") from exc
    if not np.all(np.isfinite(x)):
        raise OracleError("non-finite KKT solution")
    return x


def predict(sigma2, landmarks, W, omega, bias, order: int, pts) -> np.ndarray:
    """y_hat^(order) = Psi_order omega (+ b at order 0) (linear.py:47-53)."""
    out = features(sigma2, landmarks, W, order, pts) @ omega
    return out + bias if order == 0 else out


def kkt_report(sys_: dict, x: np.ndarray) -> dict:
    """check_kkt (linear.py:161-189)."""
    me = sys_["D"].shape[1]
    om, b, lam = x[:me], x[me], x[me + 1:]
    lin = float(np.max(np.abs(sys_["M"] @ x - sys_["rhs"])))
    cres = np.abs(sys_["Ac"] @ om + sys_["beta"] * b - sys_["values"])
    e = sys_["D"] @ om + sys_["g"] * b - sys_["r"]
    scale = float(np.max(np.abs(sys_["rhs"])))
    passed = lin <= KKT_TOL * max(scale, 1.0) and bool(np.all(cres <= KKT_TOL))
    return dict(linear_residual=lin, rhs_scale=scale, condition_residuals=cres,
                ode_residuals=e, passed=passed)


def solve_linear_instance(order, coeffs, forcing, cond, grid, gamma, sigma2,
                          m: int, drop_tol: float = DROP_TOL):
    """The harness train scope for one linear ODE (harness.py:152-163):
    landmarks -> eigendecomposition -> assemble -> solve.  Returns a dict."""
    grid = np.asarray(grid, dtype=float)
    lm = equidistant(grid, m)
    s, v = eig_landmarks(sigma2, lm, drop_tol)
    W = scaled_basis(s, v)
    sy = assemble(order, coeffs, forcing, cond, grid, gamma, sigma2, lm, W)
    x = solve_kkt(sy["M"], sy["rhs"])
    me = W.shape[1]
    return dict(landmarks=lm, s=s, V=v, W=W, x=x, omega=x[:me], bias=float(x[me]),
                lam=x[me + 1:], system=sy, m_eff=me)


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
