"""CPU oracle: NumPy restatement of the reference's Newton-KKT path.

TEST INFRASTRUCTURE ONLY (see oracle/nys_port.py for the import rule).

Follows ``/root/reference/pkg/src/nysode/newton.py``: unknowns
x = (omega, b, lambda, y_aux); residual = gradient of the Lagrangian
(newton.py:128-147); analytic Hessian (newton.py:160-211); Newton loop with
optional backtracking (newton.py:279-349); gamma continuation
(newton.py:352-373); the five-rung retry ladder (newton.py:376-412).
The dense (m_eff + 1 + p + n_c)-side LU of the reference is kept here on
purpose: the oracle must take the reference's path, not the device's Schur
shortcut.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import nys_port as lin


class Divergence(RuntimeError):
    pass


class SingularJac(RuntimeError):
    pass


class MaxIters(RuntimeError):
    def __init__(self, msg, x, trace):
        super().__init__(msg)
        self.x = x
        self.trace = trace


@dataclass
class NlSpec:
    """rhs(t, y, y', ..), partials[j] = df/dy^(j), second[(j,k)] (problems.py:44-52)."""
    order: int
    rhs: Callable
    partials: Sequence[Callable]
    second: dict


@dataclass
class Trace:
    norms: list = field(default_factory=list)
    converged: bool = False
    floor: float = 0.0
    x: Optional[np.ndarray] = None
    rung: int = 0
    solves: int = 0        # _solve_once invocations that produced iterations


class Work:
    """newton.py:92-125."""

    def __init__(self, spec: NlSpec, cond, grid, gamma, sigma2, landmarks, W):
        self.spec, self.cond = spec, list(cond)
        self.grid = np.asarray(grid, dtype=float)
        self.gamma = float(gamma)
        self.sigma2, self.lm, self.W = sigma2, landmarks, W
        self.pts = self.grid[1:]
        p = spec.order
        self.S = [lin.features(sigma2, landmarks, W, j, self.pts) for j in range(p + 1)]
        self.Ac = np.array([lin.features(sigma2, landmarks, W, o, [t])[0]
                            for (t, o, _) in self.cond])
        self.beta = np.array([1.0 if o == 0 else 0.0 for (_, o, _) in self.cond])
        self.values = np.array([v for (_, _, v) in self.cond])
        self.m = W.shape[1]
        self.nc = self.pts.size
        self.ncond = len(self.cond)
        self.side = self.m + 1 + self.ncond + self.nc

    def split(self, x):
        m, k = self.m, self.ncond
        return x[:m], float(x[m]), x[m + 1:m + 1 + k], x[m + 1 + k:]

    def args(self, om, y):
        out = [self.pts, y]
        for j in range(1, self.spec.order):
            out.append(self.S[j] @ om)
        return out


def residual(w: Work, x) -> np.ndarray:
    """newton.py:128-147."""
    sp, gm, p = w.spec, w.gamma, w.spec.order
    om, b, lam, y = w.split(x)
    a = w.args(om, y)
    f = np.asarray(sp.rhs(*a), dtype=float)
    e1 = w.S[p] @ om - f
    e2 = y - w.S[0] @ om - b
    if not (np.all(np.isfinite(e1)) and np.all(np.isfinite(f))):
        raise Divergence("non-finite rhs")
    Fo = om + gm * (w.S[p].T @ e1) - gm * (w.S[0].T @ e2) + w.Ac.T @ lam
    for j in range(1, p):
        Fo -= gm * (w.S[j].T @ (np.asarray(sp.partials[j](*a), dtype=float) * e1))
    Fb = -gm * np.sum(e2) + w.beta @ lam
    Fl = w.Ac @ om + w.beta * b - w.values
    Fy = -gm * np.asarray(sp.partials[0](*a), dtype=float) * e1 + gm * e2
    return np.concatenate([Fo, [Fb], Fl, Fy])


def _sec(sp: NlSpec, j, k, a):
    key = (j, k) if (j, k) in sp.second else (k, j)
    return np.asarray(sp.second[key](*a), dtype=float)


def jacobian(w: Work, x) -> np.ndarray:
    """Analytic Hessian (newton.py:160-211)."""
    sp, gm, p, m, nc, nk = w.spec, w.gamma, w.spec.order, w.m, w.nc, w.ncond
    om, b, lam, y = w.split(x)
    a = w.args(om, y)
    f = np.asarray(sp.rhs(*a), dtype=float)
    e1 = w.S[p] @ om - f
    fp = [np.asarray(sp.partials[j](*a), dtype=float) for j in range(p)]
    G = w.S[p].copy()
    for j in range(1, p):
        G -= fp[j][:, None] * w.S[j]
    J = np.zeros((w.side, w.side))
    o, bi, li, yi = slice(0, m), m, slice(m + 1, m + 1 + nk), slice(m + 1 + nk, w.side)
    Joo = np.eye(m) + gm * (G.T @ G) + gm * (w.S[0].T @ w.S[0])
    for j in range(1, p):
        for k in range(1, p):
            Joo -= gm * (w.S[j].T @ ((_sec(sp, j, k, a) * e1)[:, None] * w.S[k]))
    J[o, o] = Joo
    J[o, bi] = gm * np.sum(w.S[0], axis=0)
    J[bi, o] = J[o, bi]
    J[bi, bi] = gm * nc
    J[o, li] = w.Ac.T
    J[li, o] = w.Ac
    J[bi, li] = w.beta
    J[li, bi] = w.beta
    Joy = -gm * (G.T * fp[0][None, :]) - gm * w.S[0].T
    for j in range(1, p):
        Joy -= gm * (w.S[j].T * (_sec(sp, j, 0, a) * e1)[None, :])
    J[o, yi] = Joy
    J[yi, o] = Joy.T
    J[bi, yi] = -gm * np.ones(nc)
    J[yi, bi] = -gm * np.ones(nc)
    J[yi, yi] = np.diag(gm * (1.0 + fp[0] ** 2 - _sec(sp, 0, 0, a) * e1))
    return J


def const_state(w: Work) -> np.ndarray:
    """newton.py:226-237 (IVP: b = first order-0 condition value)."""
    b = [v for (_, o, v) in w.cond if o == 0][0]
    return np.concatenate([np.zeros(w.m), [b], np.zeros(w.ncond), np.full(w.nc, b)])


def linearized_state(w: Work) -> np.ndarray:
    """newton.py:240-276: linear ODE about (y = b0, derivatives 0)."""
    sp, p = w.spec, w.spec.order
    b0 = const_state(w)[w.m]

    def _a(t):
        t = np.asarray(t, dtype=float)
        return [t, np.full_like(t, b0)] + [np.zeros_like(t)] * (p - 1)

    coeffs = [(lambda t, k=k: np.asarray(sp.partials[p - k](*_a(t)), dtype=float))
              for k in range(1, p + 1)]

    def forcing(t):
        a = _a(t)
        return (np.asarray(sp.rhs(*a), dtype=float)
                - np.asarray(sp.partials[0](*a), dtype=float) * b0)

    sy = lin.assemble(p, coeffs, forcing, w.cond, w.grid, w.gamma, w.sigma2, w.lm, w.W)
    xl = lin.solve_kkt(sy["M"], sy["rhs"])
    om, b = xl[:w.m], float(xl[w.m])
    yv = lin.predict(w.sigma2, w.lm, w.W, om, b, 0, w.pts)
    return np.concatenate([om, [b], np.zeros(w.ncond), yv])


def solve_once(w: Work, x, max_iters: int, tol: float, damping) -> tuple[np.ndarray, Trace]:
    """newton.py:279-349."""
    tr = Trace()
    F = residual(w, x)
    nrm = float(np.max(np.abs(F)))
    tr.norms.append(nrm)
    jn = 0.0
    for _ in range(max_iters):
        if nrm <= tol:
            tr.converged = True
            break
        if nrm > 1e12:
            raise Divergence(f"residual {nrm:.3e} > 1e12")
        J = jacobian(w, x)
        jn = float(np.max(np.sum(np.abs(J), axis=1)))
        try:
            dx = np.linalg.solve(J, -F)
        except np.linalg.LinAlgError as exc:
            raise SingularJac(str(exc)) from exc
        if not np.all(np.isfinite(dx)):
            raise SingularJac("non-finite step")
        if damping is not None:
            shrink, halvings = damping
            al = 1.0
            for _h in range(halvings):
                try:
                    if float(np.max(np.abs(residual(w, x + al * dx)))) <= nrm:
                        break
                except Divergence:
                    pass
                al *= shrink
            x = x + al * dx
        else:
            x = x + dx
        F = residual(w, x)
        nrm = float(np.max(np.abs(F)))
        tr.norms.append(nrm)
    else:
        if nrm <= tol:
            tr.converged = True
    tr.floor = np.finfo(float).eps * jn
    tr.x = x
    if not tr.converged and nrm > tol:
        raise MaxIters(f"no convergence in {max_iters}", x, tr)
    return x, tr


CONT_GAMMAS = (1e0, 1e2, 1e4)      # newton.py:349


def continuation(w: Work, max_iters: int, tol: float):
    """newton.py:352-373."""
    x = None
    for g in [g for g in CONT_GAMMAS if g < w.gamma]:
        wg = Work(w.spec, w.cond, w.grid, g, w.sigma2, w.lm, w.W)
        try:
            xg, _ = solve_once(wg, x if x is not None else const_state(wg),
                               max_iters, 1e-8 * (1.0 + g), (0.5, 30))
        except MaxIters as exc:
            xg = exc.x
        om, b = xg[:wg.m], float(xg[wg.m])
        yv = lin.predict(w.sigma2, w.lm, w.W, om, b, 0, wg.pts)
        x = np.concatenate([om, [b], np.zeros(wg.ncond), yv])
    return solve_once(w, x if x is not None else const_state(w), max_iters, tol, (0.5, 30))


def solve_nonlinear(spec: NlSpec, cond, grid, gamma, sigma2, landmarks, W,
                    max_iters: int = 100, tol: Optional[float] = None):
    """Retry ladder (newton.py:376-412).  Returns (x, trace); on total failure
    re-raises the last exception like the reference."""
    w = Work(spec, cond, grid, gamma, sigma2, landmarks, W)
    tol = 1e-10 * (1.0 + gamma) if tol is None else tol           # newton.py:60-61
    rungs = (
        lambda: solve_once(w, const_state(w), max_iters, tol, None),
        lambda: solve_once(w, const_state(w), max_iters, tol, (0.5, 30)),
        lambda: solve_once(w, linearized_state(w), max_iters, tol, None),
        lambda: solve_once(w, linearized_state(w), max_iters, tol, (0.5, 30)),
        lambda: continuation(w, max_iters, tol),
    )
    last = None
    for i, rung in enumerate(rungs, start=1):
        try:
            x, tr = rung()
            tr.rung = i
            return x, tr
        except (Divergence, SingularJac, MaxIters) as exc:
            last = exc
    raise last
