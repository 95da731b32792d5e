"""Newton-iterated primal KKT solve for nonlinear first-order ODEs, on the B200.

Mirror of ``pkg/src/nysode/newton.py`` (names, options, exceptions, the
five-rung retry ladder and its semantics), with the numerics on the device
(C ABI ``nys_newton_*``):

* residual / gradient of the Lagrangian -- ``nys_newton_residual_f64``
  (newton.py:128-147);
* Newton direction -- the Jacobian's y-block is diagonal (newton.py:210), so
  J delta = -F is solved by a Schur complement onto (omega, b, lambda):
  DMMA-accumulated reduced system (``nys_newton_reduced_f64``) + batched LU
  (``nys_lu_solve_f64``) + diagonal back-substitution (``nys_newton_step_f64``)
  instead of the reference's dense (m_eff+2+n_c)-side LU (newton.py:307);
* damping, continuation and the ladder (newton.py:279-412) stay on the host,
  batched: every instance of a rung advances in the same kernel launches and
  drops out when it converges, diverges, hits a singular step or exhausts the
  iteration budget.

Two ways to give the nonlinearity f(t, y):
* :class:`SeparableFamily` -- f = g(t) + alpha y^2 + beta sin(y), evaluated on
  the device (config 3: y' = -k y^2 + g and y' = sin y + g);
* a reference ``NonlinearOdeSpec`` (callables) -- evaluated on the host at the
  current y every residual call (the generic drop-in path; slower).

First- and second-order problems run on the device (p = 2: newton2.cu, the
SURVEY.md §8f next-row 2 families P14 / P15, with host-sampled callables);
higher orders raise ``NotImplementedError``.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._refcompat import ref_base
from . import _lib
from .linear import PrimalModel, condition_rows, constraint_points, predict_batch
from .nystrom import NystromFeatureMap


class PartialsMissingError(*ref_base("newton", "PartialsMissingError", ValueError)):
    pass


class SingularJacobianError(*ref_base("newton", "SingularJacobianError",
                                     np.linalg.LinAlgError)):
    pass


class DivergenceError(*ref_base("newton", "DivergenceError", RuntimeError)):
    pass


class MaxItersExceeded(*ref_base("newton", "MaxItersExceeded", RuntimeError)):
    def __init__(self, message: str, model: PrimalModel, trace: "NewtonTrace"):
        # the reference's __init__ (newton.py:42-45) only stores the same two
        # attributes; RuntimeError's works for both bases
        RuntimeError.__init__(self, message)
        self.model = model
        self.trace = trace


@dataclass(frozen=True)
class NewtonOptions:
    """newton.py:52-61."""

    max_iters: int = 100
    tol: Optional[float] = None
    damping: Optional[tuple] = None
    jacobian: str = "analytic"
    fd_step: float = 1e-6

    def resolved_tol(self, gamma: float) -> float:
        return self.tol if self.tol is not None else 1e-10 * (1.0 + gamma)


@dataclass
class NewtonTrace:
    residual_norms: list = field(default_factory=list)
    converged: bool = False
    floor_estimate: float = 0.0
    final_state: Optional["NewtonState"] = None
    rung: int = 0

    @property
    def iterations(self) -> int:
        return max(len(self.residual_norms) - 1, 0)


@dataclass(frozen=True)
class NewtonState:
    omega: np.ndarray
    bias: float
    multipliers: np.ndarray
    y_aux: np.ndarray
    iteration: int = 0
    residual_norm: float = np.inf

    def pack(self) -> np.ndarray:
        return np.concatenate([self.omega, [self.bias], self.multipliers, self.y_aux])


@dataclass
class SeparableFamily:
    """f(t, y) = g(t) + alpha y^2 + beta sin(y), sampled g on the constraint points."""

    g: np.ndarray         # (B, n_c)
    alpha: np.ndarray     # (B,)
    beta: np.ndarray      # (B,)


# outcome codes of a batched solve_once
OK, MAXITERS, DIVERGED, SINGULAR = 0, 1, 2, 3
_CONTINUATION_GAMMAS = (1e0, 1e2, 1e4)     # newton.py:349


class NewtonBatch:
    """Batched Newton-KKT engine for B first-order ODEs sharing grid and fmap."""

    def __init__(self, fmap: NystromFeatureMap, grid, cond, values, gamma: float,
                 family: Optional[SeparableFamily] = None, specs: Optional[Sequence] = None):
        lib, torch = _lib.require_device()
        self.lib, self.torch = lib, torch
        self.fmap = fmap
        dev = self.dev = fmap.device
        self.grid = np.asarray(grid, dtype=float)
        self.cond = cond
        self.pts_host = constraint_points(cond, self.grid)
        self.n_c = self.pts_host.size
        self.values = np.asarray(values, dtype=float).reshape(-1, len(cond.entries))
        self.B = self.values.shape[0]
        self.nk = len(cond.entries)
        self.me = fmap.m_eff
        self.nz = self.me + 1 + self.nk
        self.ldx = self.nz + self.n_c
        self.gamma_target = float(gamma)
        if (family is None) == (specs is None):
            raise ValueError("give exactly one of family / specs")
        self.family, self.specs = family, specs
        orders = {1} if specs is None else {int(sp.order) for sp in specs}
        if len(orders) != 1 or not orders <= {1, 2}:
            raise NotImplementedError("device Newton: one common order p in {1, 2} per batch")
        self.p = orders.pop()
        f64 = dict(dtype=torch.float64, device=dev)
        self.pts = _lib.as_f64(self.pts_host, dev)
        st = _lib.stream_ptr()
        # shared feature rows S0, S1 (dense + transposed) and the DMMA-packed copy
        self.S0 = fmap.feature_matrix_device(0, self.pts).contiguous()
        self.S1 = fmap.feature_matrix_device(1, self.pts).contiguous()
        self.S0T = torch.empty((self.me, self.n_c), **f64)
        self.S1T = torch.empty((self.me, self.n_c), **f64)
        _lib.call("nys_transpose_f64", _lib.ptr(self.S0), self.n_c, self.me, _lib.ptr(self.S0T), st)
        _lib.call("nys_transpose_f64", _lib.ptr(self.S1), self.n_c, self.me, _lib.ptr(self.S1T), st)
        pack = "nys_newton_pack" if self.p == 1 else "nys_newton2_pack"
        self.packed = torch.zeros(getattr(lib, pack + "_doubles")(self.me, self.n_c), **f64)
        _lib.call(pack + "_f64", _lib.ptr(fmap.d_landmarks), fmap.m, _lib.ptr(fmap.d_W),
                  fmap.ldw, self.me, float(fmap.kernel.sigma2), _lib.ptr(self.pts), self.n_c,
                  _lib.ptr(self.packed), st)
        if self.p == 2:   # Psi_2 rows (transposed) for e1 = S2 omega - f and the step
            S2 = fmap.feature_matrix_device(2, self.pts).contiguous()
            self.S2T = torch.empty((self.me, self.n_c), **f64)
            _lib.call("nys_transpose_f64", _lib.ptr(S2), self.n_c, self.me, _lib.ptr(self.S2T),
                      st)
        Ac, beta, _ = condition_rows(cond, fmap)
        self.Ac = _lib.as_f64(Ac.reshape(self.nk, self.me), dev)
        self.betac = _lib.as_f64(beta, dev)
        self.vals = _lib.as_f64(self.values, dev)
        B, ldx = self.B, self.ldx
        self.X = torch.zeros((B, ldx), **f64)
        self.Xc = torch.zeros((B, ldx), **f64)
        self.F = torch.zeros((B, ldx), **f64)
        self.D = torch.zeros((B, ldx), **f64)
        self.norm = torch.zeros(B, **f64)
        self.aux = torch.zeros((B, 3 if self.p == 1 else 6, self.n_c), **f64)
        self.work = torch.zeros((B, 2, self.n_c), **f64)
        self.gam = torch.full((B,), self.gamma_target, **f64)
        self.alpha = torch.ones(B, **f64)
        self.K = torch.zeros((B, self.nz, self.nz), **f64)
        self.rz = torch.zeros((B, self.nz), **f64)
        self.dz = torch.zeros((B, self.nz), **f64)
        self.info = torch.zeros(B, dtype=torch.int32, device=dev)
        if family is not None:
            self.g = _lib.as_f64(family.g, dev)
            self.fal = _lib.as_f64(family.alpha, dev)
            self.fbe = _lib.as_f64(family.beta, dev)
            self.fy = self.fyy = None
        else:
            self.g = torch.zeros((B, self.n_c), **f64)
            self.fy = torch.zeros((B, self.n_c), **f64)
            self.fyy = torch.zeros((B, self.n_c), **f64)
            self.fal = self.fbe = None
            need = [(0, 0)] if self.p == 1 else [(0, 0), (0, 1), (1, 1)]
            for sp in specs:
                tab = sp.rhs_second_partials
                if tab is None or any(k not in tab and k[::-1] not in tab for k in need):
                    raise PartialsMissingError(
                        "rhs_second_partials required for analytic Jacobian")
            if self.p == 2:   # f, f_y, f_y', f_yy, f_yy', f_y'y' at (t, y, y')
                self.samples = torch.zeros((6, B, self.n_c), **f64)
        self.launches = 0

    # -------------------------------------------------------------- kernels
    def _idx(self, ids):
        """Device index tensor for an id list; the active sets of consecutive
        iterations repeat, so they are cached (one small H2D copy per new set)."""
        key = tuple(ids)
        cache = self.__dict__.setdefault("_idx_cache", {})
        t = cache.get(key)
        if t is None:
            if len(cache) > 256:
                cache.clear()
            t = self.torch.as_tensor(np.asarray(ids, dtype=np.int32), device=self.dev)
            cache[key] = t
        return t

    def _sample_host(self, X, ids):
        """Sampled mode: evaluate the spec callables at the current y (host);
        p = 2 also at y' = S1 omega (newton.py:120-125: derivatives from the model)."""
        if self.p == 2:
            return self._sample_host2(X, ids)
        Y = X[:, self.nz:].cpu().numpy()
        t = self.pts_host
        for b in ids:
            sp = self.specs[b]
            y = Y[b]
            self.g[b] = _lib.as_f64(np.asarray(sp.rhs(t, y), dtype=float), self.dev)
            self.fy[b] = _lib.as_f64(np.asarray(sp.rhs_partials[0](t, y), dtype=float), self.dev)
            self.fyy[b] = _lib.as_f64(np.asarray(sp.rhs_second_partials[(0, 0)](t, y),
                                                 dtype=float), self.dev)

    def _sample_host2(self, X, ids):
        idx_t = self._idx(ids)
        Y = X[idx_t, self.nz:].cpu().numpy()
        YP = predict_batch(self.fmap, X[idx_t, :self.me + 1], 1, self.pts).cpu().numpy()
        t = self.pts_host
        host = np.empty((6, len(ids), self.n_c))
        for r, b in enumerate(ids):
            sp = self.specs[b]
            a = (t, Y[r], YP[r])
            tab = sp.rhs_second_partials
            sec = lambda j, k: tab[(j, k)] if (j, k) in tab else tab[(k, j)]  # noqa: E731
            host[0, r] = np.asarray(sp.rhs(*a), dtype=float)
            host[1, r] = np.asarray(sp.rhs_partials[0](*a), dtype=float)
            host[2, r] = np.asarray(sp.rhs_partials[1](*a), dtype=float)
            host[3, r] = np.asarray(sec(0, 0)(*a), dtype=float)
            host[4, r] = np.asarray(sec(0, 1)(*a), dtype=float)
            host[5, r] = np.asarray(sec(1, 1)(*a), dtype=float)
        self.samples[:, idx_t] = self.torch.as_tensor(host, device=self.dev)

    def residual(self, X, ids, idx_t=None, read: bool = True):
        """F(X[b]) for b in ids; returns max|F| per id (NaN = non-finite rhs),
        or None without the read-back (read=False: F / aux for the next
        direction only)."""
        if self.specs is not None:
            self._sample_host(X, ids)
        idx_t = self._idx(ids) if idx_t is None else idx_t
        self._residual_launch(X, idx_t, len(ids))
        return self.norm[idx_t].cpu().numpy() if read else None

    def _ws2(self, nb):
        wsb = self.lib.nys_newton2_workspace_bytes(self.me, self.n_c, nb)
        return _lib.WORKSPACE.get(wsb, self.dev), wsb

    def _residual_launch(self, X, idx_t, nb):
        if self.p == 2:
            ws, wsb = self._ws2(nb)
            _lib.call("nys_newton2_residual_f64", _lib.ptr(self.S0T), _lib.ptr(self.S1T),
                      _lib.ptr(self.S2T), self.me, self.n_c, _lib.ptr(self.samples), self.B,
                      _lib.ptr(self.Ac), _lib.ptr(self.betac), _lib.ptr(self.vals), self.nk,
                      _lib.ptr(self.gam), _lib.ptr(X), self.ldx, _lib.ptr(idx_t), nb,
                      _lib.ptr(self.F), _lib.ptr(self.norm), _lib.ptr(self.aux), _lib.ptr(ws), wsb,
                      _lib.stream_ptr())
            return
        _lib.call("nys_newton_residual_f64", _lib.ptr(self.S0), _lib.ptr(self.S1),
                  _lib.ptr(self.S0T), _lib.ptr(self.S1T), self.me, self.n_c, _lib.ptr(self.g),
                  _lib.ptr(self.fy), _lib.ptr(self.fyy), _lib.ptr(self.fal), _lib.ptr(self.fbe),
                  _lib.ptr(self.Ac), _lib.ptr(self.betac), _lib.ptr(self.vals), self.nk,
                  _lib.ptr(self.gam), _lib.ptr(X), self.ldx, _lib.ptr(idx_t), nb,
                  _lib.ptr(self.F), _lib.ptr(self.norm), _lib.ptr(self.aux), _lib.ptr(self.work),
                  _lib.stream_ptr())

    def direction(self, ids, sync: bool = True):
        """Newton direction D[b] at X[b] (aux/F from the last residual at X);
        returns LU info per id (sync=False: the device tensor, read later
        together with the line search's first trial norms)."""
        idx_t = self._idx(ids)
        nb, st = len(ids), _lib.stream_ptr()
        if self.p == 2:
            return self._direction2(idx_t, nb, st)
        wsb = self.lib.nys_newton_reduced_workspace_bytes(self.me, self.n_c, nb)
        ws = _lib.WORKSPACE.get(wsb, self.dev) if wsb else None
        _lib.call("nys_newton_reduced_ws_f64", _lib.ptr(self.packed), self.me, self.n_c,
                  _lib.ptr(self.aux), _lib.ptr(self.F), self.ldx, _lib.ptr(self.gam),
                  _lib.ptr(self.Ac), _lib.ptr(self.betac), self.nk, _lib.ptr(idx_t), nb,
                  _lib.ptr(self.K), _lib.ptr(self.rz), _lib.ptr(ws), wsb, st)
        _lib.call("nys_lu_solve_f64", _lib.ptr(self.K), _lib.ptr(self.rz), self.nz, nb,
                  _lib.ptr(self.dz), _lib.ptr(self.info), st)
        _lib.call("nys_newton_step_f64", _lib.ptr(self.S0), _lib.ptr(self.S1), self.me, self.n_c,
                  self.nk, _lib.ptr(self.aux), _lib.ptr(self.F), _lib.ptr(self.dz),
                  _lib.ptr(self.gam), _lib.ptr(self.X), _lib.ptr(self.D), _lib.ptr(self.Xc),
                  _lib.ptr(self.alpha), self.ldx, _lib.ptr(idx_t), nb, 1, st)
        # LU info and the finiteness of D in one read-back
        bad = ~self.torch.isfinite(self.D[idx_t]).all(dim=1)
        both = self.torch.where(bad, self.torch.full_like(self.info[:nb], _lib.INFO_NONFINITE),
                                self.info[:nb])
        return both.cpu().numpy() if sync else both

    def _direction2(self, idx_t, nb, st):
        ws, wsb = self._ws2(nb)
        _lib.call("nys_newton2_reduced_f64", _lib.ptr(self.packed), self.me, self.n_c,
                  _lib.ptr(self.aux), _lib.ptr(self.F), self.ldx, _lib.ptr(self.gam),
                  _lib.ptr(self.Ac), _lib.ptr(self.betac), self.nk, _lib.ptr(idx_t), nb,
                  _lib.ptr(self.K), _lib.ptr(self.rz), _lib.ptr(ws), wsb, st)
        _lib.call("nys_lu_solve_f64", _lib.ptr(self.K), _lib.ptr(self.rz), self.nz, nb,
                  _lib.ptr(self.dz), _lib.ptr(self.info), st)
        _lib.call("nys_newton2_step_f64", _lib.ptr(self.S0T), _lib.ptr(self.S1T),
                  _lib.ptr(self.S2T), self.me, self.n_c, self.nk, _lib.ptr(self.aux),
                  _lib.ptr(self.F), _lib.ptr(self.dz), _lib.ptr(self.gam), _lib.ptr(self.X),
                  _lib.ptr(self.D), _lib.ptr(self.Xc), _lib.ptr(self.alpha), self.ldx,
                  _lib.ptr(idx_t), nb, st)
        bad = ~self.torch.isfinite(self.D[idx_t]).all(dim=1)
        both = self.torch.where(bad, self.torch.full_like(self.info[:nb], _lib.INFO_NONFINITE),
                                self.info[:nb])
        return both.cpu().numpy()

    def candidate(self, ids, alphas):
        """Xc[b] = X[b] + alpha_b D[b]."""
        idx_t = self._idx(ids)
        pin = self.__dict__.get("_alpha_pin")
        if pin is None:   # pinned staging: the upload is asynchronous (no host sync)
            pin = self._alpha_pin = self.torch.empty(self.B, dtype=self.torch.float64).pin_memory()
        n = len(ids)
        pin.numpy()[:n] = np.asarray(alphas, dtype=float)
        self.alpha[idx_t] = pin[:n].to(self.dev, non_blocking=True)
        _lib.call("nys_newton_step_f64", _lib.ptr(self.S0), _lib.ptr(self.S1), self.me, self.n_c,
                  self.nk, _lib.ptr(self.aux), _lib.ptr(self.F), _lib.ptr(self.dz),
                  _lib.ptr(self.gam), _lib.ptr(self.X), _lib.ptr(self.D), _lib.ptr(self.Xc),
                  _lib.ptr(self.alpha), self.ldx, _lib.ptr(idx_t), len(ids), 0,
                  _lib.stream_ptr())

    def _line_search(self, ids, ref, shrink, halvings, chunks=(1, 3), with_norms=False,
                     info_d=None):
        """Step halving of newton.py:305-318 with the trial steps evaluated in
        batches: alpha_k = shrink^k for a chunk of k at once (one host sync per
        chunk instead of per halving), then the first accepted k per instance --
        the same alpha the sequential loop stops at, because every trial's
        residual depends only on its own instance and alpha.  Never-accepted
        instances get shrink^halvings, as the sequential loop leaves them."""
        torch = self.torch
        alphas = [1.0]
        for _ in range(halvings):
            alphas.append(alphas[-1] * shrink)   # the loop's repeated products
        out = {b: alphas[halvings] for b in ids}
        tn = {}   # accepted trial norms: bit-identical to the residual at the candidate
        info = np.full(len(ids), _lib.INFO_OK, dtype=np.int64)
        left = list(range(len(ids)))
        key = (shrink, halvings)
        cache = self.__dict__.setdefault("_alpha_cache", {})
        al_all = cache.get(key)
        if al_all is None:   # the ladder on the device once (no H2D per chunk)
            al_all = cache[key] = torch.tensor(alphas, dtype=torch.float64, device=self.dev)
        k0, c = 0, 0
        while left and k0 < halvings:
            # growing chunks: most steps are accepted at alpha = 1 or after a few
            # halvings; the rest of the ladder goes in one batch
            kk = min(chunks[c] if c < len(chunks) else halvings - k0, halvings - k0)
            c += 1
            sub = [ids[r] for r in left]
            idx_t = self._idx(sub)
            nb = len(sub)
            norms = torch.empty((kk, nb), dtype=torch.float64, device=self.dev)
            al_t = al_all[k0:k0 + kk]
            sb = self.lib.nys_newton_trial_scratch_bytes(self.me, self.n_c, nb, kk)
            scratch = _lib.WORKSPACE.get(sb, self.dev) if sb else None
            _lib.call("nys_newton_trial_norms_f64", _lib.ptr(self.S0T), _lib.ptr(self.S1T),
                      self.me, self.n_c, _lib.ptr(self.g), _lib.ptr(self.fy), _lib.ptr(self.fyy),
                      _lib.ptr(self.fal), _lib.ptr(self.fbe), _lib.ptr(self.Ac),
                      _lib.ptr(self.betac), _lib.ptr(self.vals), self.nk, _lib.ptr(self.gam),
                      _lib.ptr(self.X), _lib.ptr(self.D), self.ldx, _lib.ptr(idx_t), nb,
                      _lib.ptr(al_t), kk, _lib.ptr(norms), _lib.ptr(scratch) if sb else None, sb,
                      _lib.stream_ptr())
            if info_d is not None:
                # the direction's LU info rides on the first read-back; instances
                # it flags leave the search (newton.py:307-310: no step for them)
                both = self.torch.cat([norms.reshape(-1), info_d.to(norms.dtype)]).cpu().numpy()
                nh = both[:kk * nb].reshape(kk, nb)
                info = both[kk * nb:].astype(np.int64)
                info_d = None
                keep = np.flatnonzero(info[left] == _lib.INFO_OK)
                nh = nh[:, keep]
                left = [left[c] for c in keep]
            else:
                nh = norms.cpu().numpy()
            # first accepted trial per instance (vectorised over the instances)
            ok = np.isfinite(nh) & (nh <= np.asarray([ref[r] for r in left])[None, :])
            hit = ok.any(axis=0)
            first = ok.argmax(axis=0)
            for c in np.flatnonzero(hit):
                out[ids[left[c]]] = alphas[k0 + int(first[c])]
                tn[ids[left[c]]] = float(nh[first[c], c])
            left = [left[c] for c in np.flatnonzero(~hit)]
            k0 += kk
        if info_d is not None:   # no trial chunk ran (halvings == 0)
            info = info_d.cpu().numpy().astype(np.int64)
        if with_norms:
            return out, tn, info
        return out

    # -------------------------------------------------------------- states
    def const_state(self, ids):
        """omega = 0, b = first order-0 IVP value, y = b (newton.py:226-237)."""
        j0 = [j for j, bc in enumerate(self.cond.entries) if bc.order == 0]
        if self.cond.kind == "ivp":
            b0 = self.values[ids, j0[0]]
        else:
            b0 = self.values[ids][:, j0].mean(axis=1)
        x = np.zeros((len(ids), self.ldx))
        x[:, self.me] = b0
        x[:, self.nz:] = b0[:, None]
        return x

    def model_state(self, ids, x):
        """(omega, b, 0, S0 omega + b) -- continuation hand-off (newton.py:369-372)."""
        torch = self.torch
        xd = _lib.as_f64(x[:, :self.me + 1], self.dev)
        y = predict_batch(self.fmap, xd, 0, self.pts).cpu().numpy()
        out = np.zeros((len(ids), self.ldx))
        out[:, :self.me + 1] = x[:, :self.me + 1]
        out[:, self.nz:] = y
        return out

    def linearized_state(self, ids):
        """Warm start from the ODE linearised about (y = b0) (newton.py:240-276):
        y' = f(t, b0) + f_y(t, b0) (y - b0), solved by the batched linear path."""
        from .batch import LinearBatchSolver

        x0 = self.const_state(ids)
        b0 = x0[:, self.me]
        t = self.pts_host
        p = self.p
        if self.family is not None:   # vectorised over the instances, on the device
            # y = b0 is constant along t, so the y-dependent terms are one scalar
            # per instance; forcing = (g + c) - d elementwise, the same two
            # roundings the host form makes
            fam = self.family
            torch = self.torch
            ida = np.asarray(ids)
            a, be = fam.alpha[ida], fam.beta[ida]
            c = a * b0 * b0 + be * np.sin(b0)
            fy = 2.0 * a * b0 + be * np.cos(b0)
            sc = torch.as_tensor(np.stack([c, fy, fy * b0]), device=self.dev)
            idx_t = self._idx(ids)
            coef = sc[1][:, None, None].expand(len(ids), 1, self.n_c).contiguous()
            forcing = (self.g.index_select(0, idx_t.long()) + sc[0][:, None]) - sc[2][:, None]
        else:
            coef = np.empty((len(ids), p, self.n_c))
            forcing = np.empty((len(ids), self.n_c))
        for r, b in enumerate(ids if self.family is None else ()):
            yb = np.full_like(t, b0[r])
            if p == 2:   # args (t, b0, 0); f_k = df/dy^(p-k) (newton.py:256-266)
                sp = self.specs[b]
                a = (t, yb, np.zeros_like(t))
                for k in (1, 2):
                    coef[r, k - 1] = np.asarray(sp.rhs_partials[p - k](*a), dtype=float)
                forcing[r] = (np.asarray(sp.rhs(*a), dtype=float)
                              - np.asarray(sp.rhs_partials[0](*a), dtype=float) * b0[r])
                continue
            sp = self.specs[b]
            f0 = np.asarray(sp.rhs(t, yb), dtype=float)
            fy = np.asarray(sp.rhs_partials[0](t, yb), dtype=float)
            coef[r, 0] = fy
            forcing[r] = f0 - fy * b0[r]
        solver = self.__dict__.get("_lin_solver")
        if solver is None:   # one batched linear solver (max batch B) for every rung
            solver = LinearBatchSolver(self.fmap, self.grid, self.gamma_target, p, self.cond,
                                       self.B)
            self._lin_solver = solver
        xl, info = solver.solve(coef, forcing, self.values[ids])
        xl = xl.cpu().numpy()
        info = info.cpu().numpy()
        out = self.model_state(ids, xl)
        return out, info

    # -------------------------------------------------------------- solve_once
    def persistent(self) -> bool:
        """The device-resident loop (nys_newton_solve_once_f64) serves the
        separable family at p = 1; NYS_NEWTON_PERSIST=0 selects the
        host-orchestrated multi-kernel loop (same arithmetic)."""
        import os

        return (self.family is not None and self.p == 1
                and os.environ.get("NYS_NEWTON_PERSIST", "1") != "0")

    def _solve_once_device(self, ids, x0, gamma, tol, damping, max_iters, shrink, halvings):
        """newton._solve_once for every instance in ids at once, entirely on
        the device: one CTA per instance loops until converged / max iterations
        / diverged / singular.  One read-back (status, iterations, trace)."""
        torch = self.torch
        nid = len(ids)
        idx_all = self._idx(ids)
        self.X[idx_all] = _lib.as_f64(x0, self.dev)
        self.gam[idx_all] = _lib.as_f64(np.broadcast_to(np.asarray(gamma, dtype=float), (nid,)),
                                        self.dev)
        tolv = self.__dict__.get("_tolv")
        if tolv is None:
            tolv = self._tolv = torch.zeros(self.B, dtype=torch.float64, device=self.dev)
        tolv[idx_all] = _lib.as_f64(np.broadcast_to(np.asarray(tol, dtype=float), (nid,)),
                                    self.dev)
        wd = int(self.lib.nys_newton_solve_once_work_doubles(self.me, self.n_c, self.nk))
        work = self.__dict__.get("_pwork")
        if work is None or work.numel() < nid * wd:
            work = self._pwork = torch.empty(self.B * wd, dtype=torch.float64, device=self.dev)
        outs = self.__dict__.get("_pouts")
        if outs is None or outs[0].shape[1] < max_iters + 1:
            outs = self._pouts = (torch.empty((self.B, max_iters + 1), dtype=torch.float64,
                                              device=self.dev),
                                  torch.empty(2 * self.B, dtype=torch.int32, device=self.dev))
        norms, ist = outs[0][:nid, :max_iters + 1].contiguous(), outs[1]
        _lib.call("nys_newton_solve_once_f64", _lib.ptr(self.S0), _lib.ptr(self.S1),
                  _lib.ptr(self.S0T), _lib.ptr(self.S1T), _lib.ptr(self.packed), self.me,
                  self.n_c, _lib.ptr(self.g), _lib.ptr(self.fal), _lib.ptr(self.fbe),
                  _lib.ptr(self.Ac), _lib.ptr(self.betac), _lib.ptr(self.vals), self.nk,
                  _lib.ptr(self.gam), _lib.ptr(tolv), _lib.ptr(self.X), self.ldx,
                  _lib.ptr(idx_all), nid, 1 if damping else 0, float(shrink), int(halvings),
                  int(max_iters), _lib.ptr(work), work.numel() * 8, _lib.ptr(norms),
                  _lib.ptr(ist), _lib.ptr(ist[self.B:]), _lib.stream_ptr())
        self.launches += 1
        nr = norms.cpu().numpy()
        st_its = ist.cpu().numpy()
        its, status = st_its[:nid], st_its[self.B:self.B + nid].astype(int)
        traces = [[float(v) for v in nr[r, :its[r] + 1]] for r in range(nid)]
        Xn = self.X[idx_all].cpu().numpy()
        return status, Xn, traces

    def solve_once(self, ids, x0, gamma, tol, damping, max_iters, shrink=0.5, halvings=30):
        """Batched newton._solve_once (newton.py:279-349).

        Returns (status[len(ids)], X rows (np), traces)."""
        if self.persistent():
            return self._solve_once_device(list(ids), x0, gamma, tol, damping, max_iters,
                                           shrink, halvings)
        torch = self.torch
        ids = list(ids)
        nid = len(ids)
        idx_all = self._idx(ids)
        self.X[idx_all] = _lib.as_f64(x0, self.dev)
        g = np.broadcast_to(np.asarray(gamma, dtype=float), (nid,))
        self.gam[idx_all] = _lib.as_f64(g, self.dev)
        tol = np.broadcast_to(np.asarray(tol, dtype=float), (nid,))
        pos = {b: r for r, b in enumerate(ids)}
        status = np.full(nid, -1)
        norm = self.residual(self.X, ids, idx_all)
        traces = [[float(v)] for v in norm]
        its = np.zeros(nid, dtype=int)
        bad0 = ~np.isfinite(norm)
        status[bad0] = DIVERGED           # _residual raised at the initial state
        ids_a = np.asarray(ids)
        act = np.flatnonzero(status < 0)          # positions r of the active instances
        while act.size:
            # the per-iteration checks of newton.py:296-303, vectorised over r
            nr = norm[act]
            ok = nr <= tol[act]
            mx = ~ok & (its[act] >= max_iters)
            dv = ~ok & ~mx & (nr > 1e12)
            status[act[ok]] = OK
            status[act[mx]] = MAXITERS
            status[act[dv]] = DIVERGED
            act = act[~(ok | mx | dv)]
            if not act.size:
                break
            known = None
            if damping and self.specs is None:
                # direction, then the batched line search; the LU info is read back
                # with the first trial norms (one host sync instead of two)
                active = ids_a[act].tolist()
                info_d = self.direction(active, sync=False)
                alpha, known, info = self._line_search(active, norm[act].tolist(), shrink,
                                                       halvings, with_norms=True, info_d=info_d)
                sing = info != _lib.INFO_OK
                status[act[sing]] = SINGULAR
                act = act[~sing]
                if not act.size:
                    break
                active = ids_a[act].tolist()
                self.candidate(active, [alpha[b] for b in active])
            else:
                info = np.asarray(self.direction(ids_a[act].tolist()))
                sing = info != _lib.INFO_OK
                status[act[sing]] = SINGULAR
                act = act[~sing]
                if not act.size:
                    break
                active = ids_a[act].tolist()
                if damping:   # sampled specs: halving through the host-sampled residual
                    alpha = {b: 1.0 for b in active}
                    searching = list(active)
                    for _ in range(halvings):
                        if not searching:
                            break
                        self.candidate(searching, [alpha[b] for b in searching])
                        cn = self.residual(self.Xc, searching)
                        nxt = []
                        for b, v in zip(searching, cn):
                            if np.isfinite(v) and v <= norm[pos[b]]:
                                continue            # accepted
                            alpha[b] *= shrink
                            nxt.append(b)
                        searching = nxt
                    self.candidate(active, [alpha[b] for b in active])
                else:
                    self.candidate(active, [1.0] * len(active))
            act_t = self._idx(active)
            self.X[act_t] = self.Xc[act_t]
            if known is not None and len(known) == len(active):
                # every step was accepted by a trial whose norm is bit-identical
                # to the residual at the new point: no read-back needed
                self.residual(self.X, active, act_t, read=False)
                newn = np.array([known[b] for b in active])
            else:
                newn = np.asarray(self.residual(self.X, active, act_t))
            its[act] += 1
            norm[act] = newn
            for r, v in zip(act.tolist(), newn.tolist()):
                traces[r].append(float(v))
            fin = np.isfinite(newn)
            status[act[~fin]] = DIVERGED        # _residual raised after the update
            act = act[fin]
        # loop ended: converged check after exhausting iterations (newton.py:331-333)
        for r in range(nid):
            if status[r] == MAXITERS and norm[r] <= tol[r]:
                status[r] = OK
        Xn = self.X[idx_all].cpu().numpy()
        return status, Xn, traces

    # -------------------------------------------------------------- ladder
    def ladder_starts(self):
        """Constant and linearised starts of every instance, formed on the
        device without a host round trip (the latter by one batched linear
        solve and the model hand-off y = Psi_0 omega + b; the same roundings
        as const_state / linearized_state)."""
        torch = self.torch
        ids = list(range(self.B))
        if self.family is None:
            x0c = _lib.as_f64(self.const_state(ids), self.dev)
            xl, _ = self.linearized_state(ids)
            return x0c, _lib.as_f64(xl, self.dev)
        from .batch import LinearBatchSolver

        B, me, nz = self.B, self.me, self.nz
        j0 = [j for j, bc in enumerate(self.cond.entries) if bc.order == 0]
        b0 = (self.values[:, j0[0]] if self.cond.kind == "ivp"
              else self.values[:, j0].mean(axis=1))
        fam = self.family
        a, be = fam.alpha, fam.beta
        c = a * b0 * b0 + be * np.sin(b0)
        fy = 2.0 * a * b0 + be * np.cos(b0)
        sc = torch.as_tensor(np.stack([b0, c, fy, fy * b0]), device=self.dev)
        x0c = torch.zeros((B, self.ldx), dtype=torch.float64, device=self.dev)
        x0c[:, me] = sc[0]
        x0c[:, nz:] = sc[0][:, None]
        coef = sc[2][:, None, None].expand(B, 1, self.n_c).contiguous()
        forcing = (self.g + sc[1][:, None]) - sc[3][:, None]
        solver = self.__dict__.get("_lin_solver")
        if solver is None:
            solver = LinearBatchSolver(self.fmap, self.grid, self.gamma_target, self.p, self.cond,
                                       self.B)
            self._lin_solver = solver
        xl, _ = solver.solve_device(coef, forcing, self.vals)
        x0l = torch.zeros((B, self.ldx), dtype=torch.float64, device=self.dev)
        x0l[:, :me + 1] = xl[:, :me + 1]
        x0l[:, nz:] = predict_batch(self.fmap, xl[:, :me + 1].contiguous(), 0, self.pts)
        return x0c, x0l

    def ladder_launch(self, x0c, x0l, max_iters, tol_t):
        """One nys_newton_ladder_f64 launch over all B instances; device
        outputs (norms[B, max_iters + 1], ints[4 B]: iterations, status, rung,
        iterations over all rungs), X updated in place.  No host sync."""
        torch = self.torch
        B = self.B
        idx_all = self._idx(list(range(B)))
        self.gam.fill_(self.gamma_target)
        tolv = self.__dict__.get("_tolv")
        if tolv is None:
            tolv = self._tolv = torch.zeros(B, dtype=torch.float64, device=self.dev)
        tolv.fill_(float(tol_t))
        wd = int(self.lib.nys_newton_solve_once_work_doubles(self.me, self.n_c, self.nk))
        work = self.__dict__.get("_pwork")
        if work is None or work.numel() < B * wd:
            work = self._pwork = torch.empty(B * wd, dtype=torch.float64, device=self.dev)
        outs = self.__dict__.get("_louts")
        if outs is None or outs[0].shape[1] != max_iters + 1:
            outs = self._louts = (torch.empty((B, max_iters + 1), dtype=torch.float64,
                                              device=self.dev),
                                  torch.empty(4 * B, dtype=torch.int32, device=self.dev))
        norms, ist = outs
        _lib.call("nys_newton_ladder_f64", _lib.ptr(self.S0), _lib.ptr(self.S1),
                  _lib.ptr(self.S0T), _lib.ptr(self.S1T), _lib.ptr(self.packed), self.me,
                  self.n_c, _lib.ptr(self.g), _lib.ptr(self.fal), _lib.ptr(self.fbe),
                  _lib.ptr(self.Ac), _lib.ptr(self.betac), _lib.ptr(self.vals), self.nk,
                  _lib.ptr(self.gam), _lib.ptr(tolv), _lib.ptr(x0c), _lib.ptr(x0l),
                  _lib.ptr(self.X), self.ldx, _lib.ptr(idx_all), B, 0.5, 30, int(max_iters),
                  _lib.ptr(work), work.numel() * 8, _lib.ptr(norms), _lib.ptr(ist),
                  _lib.ptr(ist[B:]), _lib.ptr(ist[2 * B:]), _lib.stream_ptr())
        self.launches += 1
        return norms, ist

    def _solve_ladder_device(self, max_iters, tol_t):
        """The whole ladder in one launch (nys_newton_ladder_f64): both starts
        are formed up front for every instance, then each instance climbs the
        rungs on its own CTA without waiting for the others."""
        norms, ist = self.ladder_launch(*self.ladder_starts(), max_iters, tol_t)
        return self.ladder_collect(norms, ist)

    def ladder_collect(self, norms, ist):
        """Read back one ladder launch's outcomes (status, X, traces, rung;
        total_iterations kept on the engine) -- the host half of
        _solve_ladder_device, so a caller may keep several launches in flight
        (one engine per launch) and collect each later."""
        B = self.B
        nr = norms.cpu().numpy()
        v = ist.cpu().numpy()
        its, status, rung = v[:B], v[B:2 * B].astype(int), v[2 * B:3 * B].astype(int)
        self.total_iterations = v[3 * B:4 * B].astype(int)
        traces = [[float(x) for x in nr[r, :its[r] + 1]] for r in range(B)]
        return status, self.X.cpu().numpy(), traces, rung

    def solve(self, max_iters: int = 100, tol: Optional[float] = None):
        """Retry ladder (newton.py:376-412) for all B instances.

        Returns (status[B], X[B, ldx] np, traces list, rung[B]); status is the
        outcome of the rung that finished the instance (OK) or of the last rung."""
        gam = self.gamma_target
        if self.persistent():
            return self._solve_ladder_device(max_iters,
                                             1e-10 * (1.0 + gam) if tol is None else tol)
        tol_t = 1e-10 * (1.0 + gam) if tol is None else tol
        B = self.B
        status = np.full(B, -1)
        X = np.zeros((B, self.ldx))
        traces = [None] * B
        rung = np.zeros(B, dtype=int)

        def record(ids, st, Xn, tr, r):
            for k, b in enumerate(ids):
                status[b] = st[k]
                X[b] = Xn[k]
                traces[b] = tr[k]
                rung[b] = r

        todo = list(range(B))
        plans = [(1, "const", None), (2, "const", (0.5, 30)), (3, "lin", None),
                 (4, "lin", (0.5, 30))]
        for r, init, damp in plans:
            if not todo:
                break
            if init == "const":
                x0 = self.const_state(todo)
            else:
                x0, _ = self.linearized_state(todo)
            st, Xn, tr = self.solve_once(todo, x0, gam, tol_t, damp is not None, max_iters)
            record(todo, st, Xn, tr, r)
            todo = [b for b in todo if status[b] != OK]
        if todo:
            # rung 5: gamma continuation (newton.py:352-373)
            stages = [g for g in _CONTINUATION_GAMMAS if g < gam]
            x_cur = self.const_state(todo)
            alive = list(todo)
            failed = {}
            for g in stages:
                if not alive:
                    break
                x0 = np.stack([x_cur[todo.index(b)] for b in alive])
                st, Xn, tr = self.solve_once(alive, x0, g, 1e-8 * (1.0 + g), True, max_iters)
                nxt = []
                for k, b in enumerate(alive):
                    if st[k] in (OK, MAXITERS):            # MaxIters tolerated
                        nxt.append(b)
                    else:
                        failed[b] = (st[k], Xn[k], tr[k])  # Divergence / Singular escape
                if nxt:
                    sel = [alive.index(b) for b in nxt]
                    xs = self.model_state(nxt, Xn[sel])
                    for k, b in enumerate(nxt):
                        x_cur[todo.index(b)] = xs[k]
                alive = nxt
            if alive:
                x0 = np.stack([x_cur[todo.index(b)] for b in alive])
                st, Xn, tr = self.solve_once(alive, x0, gam, tol_t, True, max_iters)
                record(alive, st, Xn, tr, 5)
            for b, (s, xb, tb) in failed.items():
                status[b], X[b], traces[b], rung[b] = s, xb, tb, 5
        return status, X, traces, rung

    def model(self, xrow) -> PrimalModel:
        me = self.me
        return PrimalModel(omega=xrow[:me].copy(), bias=float(xrow[me]),
                           multipliers=xrow[me + 1:self.nz].copy(), feature_map=self.fmap)


def _raise_for(status, msg, model, trace):
    if status == DIVERGED:
        raise DivergenceError(msg)
    if status == SINGULAR:
        raise SingularJacobianError(msg)
    if status == MAXITERS:
        raise MaxItersExceeded(msg, model, trace)


def solve_nonlinear(spec, cond, fmap: NystromFeatureMap, grid, gamma: float,
                    opts: NewtonOptions = NewtonOptions(), x0: Optional[NewtonState] = None):
    """newton.solve_nonlinear (newton.py:376-412) for one first- or second-order spec."""
    if spec.order not in (1, 2):
        raise NotImplementedError("device Newton supports orders p = 1 and p = 2")
    if opts.jacobian != "analytic":
        raise NotImplementedError("finite-difference Jacobians are not on the device path")
    values = np.array([[bc.value for bc in cond.entries]])
    eng = NewtonBatch(fmap, grid, cond, values, gamma, specs=[spec])
    tol = opts.resolved_tol(float(gamma))
    if x0 is not None or opts.damping is not None:
        xs = x0.pack()[None] if x0 is not None else eng.const_state([0])
        st, Xn, tr = eng.solve_once([0], xs, gamma, tol, opts.damping is not None, opts.max_iters,
                                    *(opts.damping or (0.5, 30)))
        status, xrow, trace_l, rung = st[0], Xn[0], tr[0], 0
    else:
        status_a, X, traces, rungs = eng.solve(opts.max_iters, opts.tol)
        status, xrow, trace_l, rung = status_a[0], X[0], traces[0], rungs[0]
    model = eng.model(xrow)
    trace = NewtonTrace(residual_norms=list(trace_l), converged=status == OK, rung=int(rung))
    trace.final_state = NewtonState(xrow[:eng.me], float(xrow[eng.me]), xrow[eng.me + 1:eng.nz],
                                    xrow[eng.nz:], iteration=trace.iterations,
                                    residual_norm=trace_l[-1])
    if status != OK:
        _raise_for(status, f"Newton failed (status {status}, residual {trace_l[-1]:.3e})",
                   model, trace)
    return model, trace
