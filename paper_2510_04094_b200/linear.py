"""Primal KKT assembly and direct solve for linear ODEs, on the B200.

Mirror of ``pkg/src/nysode/linear.py`` (same names, arguments, exceptions).
What moved to the GPU:

* :func:`assemble` samples the spec callables on the constraint points on the
  host (exactly like linear.py:103-116, so the values are the reference's),
  then calls the fused feature+Gram kernel (``nys_fused_gram_f64``): the
  n x m feature matrices are never formed.  The system keeps the extended Gram
  E = [D g r]^T [D g r] on the device; ``matrix`` / ``rhs`` are built on demand.
* :func:`solve` is the batched device LU + one refinement step
  (``nys_kkt_solve_f64``, linear.py:140-158).
* :meth:`PrimalModel.predict` and :func:`check_kkt` run on the device
  (``nys_predict_f64``, ``nys_ode_residual_f64``).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Optional

import os

import numpy as np

from ._refcompat import ref_base
from . import _lib
from .nystrom import NystromFeatureMap

KKT_RESIDUAL_TOL = 1e-8          # linear.py:33
# kernel-space Gram for m_eff + 2 > 72 is only parity-safe on well-conditioned
# landmark matrices (1.3e-13 at cond 28, 2.6e-5 when m_eff < m)
KSPACE_MAX_COND = 1e6
SMALL_NB_MAX = 9                 # register-resident fused kernel: m_eff + 2 <= 72


class SingularSystemError(*ref_base("linear", "SingularSystemError", np.linalg.LinAlgError)):
    """Direct solve failed or produced non-finite entries (linear.py:36-37)."""


class IllConditionedLargeMapError(RuntimeError):
    """m_eff + 2 > 72 with an ill-conditioned landmark matrix: the large-m
    device path (kernel-space Gram) would not be parity-safe."""


@dataclass(frozen=True)
class PrimalModel:
    omega: np.ndarray
    bias: float
    multipliers: np.ndarray
    feature_map: NystromFeatureMap

    def x_device(self):
        _, torch = _lib.require_device()
        x = np.concatenate([self.omega, [self.bias]])
        return _lib.as_f64(x, self.feature_map.device)

    def predict_device(self, ell: int, points):
        """y_hat^(ell)(points) as a device tensor (linear.py:47-53)."""
        return predict_batch(self.feature_map, self.x_device().reshape(1, -1), ell, points)[0]

    def predict(self, ell: int, points) -> np.ndarray:
        return self.predict_device(ell, points).cpu().numpy()


def predict_batch(fmap: NystromFeatureMap, x, ell: int, points):
    """Rows x[b] = (omega_b, b_b, ...) sharing fmap -> (B, |points|) device tensor."""
    lib, torch = _lib.require_device()
    pts = _lib.as_f64(np.atleast_1d(points) if not hasattr(points, "device") else points,
                      fmap.device).reshape(-1)
    x = _lib.as_f64(x, fmap.device)
    B, ldx = x.shape
    out = torch.empty((B, pts.numel()), dtype=torch.float64, device=fmap.device)
    _lib.call("nys_predict_f64", _lib.ptr(fmap.d_landmarks), fmap.m, _lib.ptr(fmap.d_W), fmap.ldw,
              fmap.m_eff, float(fmap.kernel.sigma2), int(ell), _lib.ptr(pts), pts.numel(),
              _lib.ptr(x), ldx, B, _lib.ptr(out), pts.numel(), _lib.stream_ptr())
    return out


def condition_rows(cond, fmap: NystromFeatureMap):
    """(A_c, beta, values) -- linear.py:56-63; feature rows from the device."""
    rows, bias_coeffs, values = [], [], []
    for bc in cond.entries:
        rows.append(fmap.feature_deriv(bc.order, bc.point))
        bias_coeffs.append(1.0 if bc.order == 0 else 0.0)
        values.append(bc.value)
    return np.array(rows), np.array(bias_coeffs), np.array(values)


def constraint_points(cond, grid: np.ndarray) -> np.ndarray:
    """t_2..t_n for IVPs, t_2..t_{n-1} for BVPs (linear.py:66-68)."""
    return grid[1:] if cond.kind == "ivp" else grid[1:-1]


def gram_ext_device(fmap: NystromFeatureMap, order: int, pts, coef, forcing,
                    row_begin: int = 0, row_end: Optional[int] = None):
    """E = [D g r]^T [D g r] over rows [row_begin, row_end) of the sampled
    constraint system (device tensors in, (m_eff+2)^2 device tensor out)."""
    lib, torch = _lib.require_device()
    dev = fmap.device
    pts = _lib.as_f64(pts, dev).reshape(-1)
    coef = _lib.as_f64(coef, dev).reshape(order, -1)
    forcing = _lib.as_f64(forcing, dev).reshape(-1)
    n_c = pts.numel()
    row_end = n_c if row_end is None else row_end
    me = fmap.m_eff
    if "compressed" in fmap._host:
        return _gram_ext_explicit(fmap, order, pts, coef, forcing, row_begin, row_end)
    if (me + 2 + 7) // 8 > SMALL_NB_MAX and fmap.condition > KSPACE_MAX_COND:
        raise IllConditionedLargeMapError(
            f"m_eff={me} with cond(Omega)={fmap.condition:.2e} > {KSPACE_MAX_COND:.0e}")
    E = torch.empty((me + 2, me + 2), dtype=torch.float64, device=dev)
    wsb = lib.nys_fused_gram_workspace_bytes(row_end - row_begin, fmap.m, me, order)
    ws = _lib.WORKSPACE.get(wsb, dev)
    _lib.call("nys_fused_gram_f64", _lib.ptr(fmap.d_landmarks), fmap.m, _lib.ptr(fmap.d_W),
              fmap.ldw, me, float(fmap.kernel.sigma2), int(order), _lib.ptr(pts), _lib.ptr(coef),
              _lib.ptr(forcing), n_c, int(row_begin), int(row_end), _lib.ptr(E), _lib.ptr(ws),
              wsb, _lib.stream_ptr())
    return E


def _gram_ext_explicit(fmap, order, pts, coef, forcing, row_begin, row_end):
    """Large landmark sets: Psi_0..Psi_p as explicit device matrices (the
    reference's own per-order feature matrices, linear.py:103-112), then
    E = [D g r]^T [D g r] (nys_explicit_gram_f64)."""
    lib, torch = _lib.require_device()
    dev = fmap.device
    me = fmap.m_eff
    n = row_end - row_begin
    psi = torch.empty((order + 1, max(n, 1), me), dtype=torch.float64, device=dev)
    st = _lib.stream_ptr()
    for ell in range(order + 1):
        _lib.call("nys_feature_matrix_f64", _lib.ptr(fmap.d_landmarks), fmap.m,
                  _lib.ptr(fmap.d_W), fmap.ldw, me, float(fmap.kernel.sigma2), ell,
                  _lib.ptr(pts) + 8 * row_begin, n, _lib.ptr(psi[ell]), me, st)
    c = coef[:, row_begin:row_end].contiguous()
    f = forcing[row_begin:row_end].contiguous()
    E = torch.empty((me + 2, me + 2), dtype=torch.float64, device=dev)
    wsb = lib.nys_explicit_gram_workspace_bytes(n, me)
    ws = _lib.WORKSPACE.get(wsb, dev)
    _lib.call("nys_explicit_gram_f64", _lib.ptr(psi), n, me, int(order), _lib.ptr(c), _lib.ptr(f),
              _lib.ptr(E), _lib.ptr(ws), wsb, st)
    return E


@dataclass(eq=False)
class AssembledSystem:
    """linear.py:71-87; D is not materialised."""

    constraint_points: np.ndarray
    gamma: float
    g: np.ndarray
    r: np.ndarray
    coeff_values: np.ndarray         # (p, n_c) f_k on the constraint points
    cond_rows: np.ndarray
    cond_bias: np.ndarray
    cond_values: np.ndarray
    fmap: NystromFeatureMap
    order: int
    d_gram: Any                      # (m_eff+2)^2 device tensor
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def side(self) -> int:
        return self.fmap.m_eff + 1 + self.cond_values.size

    def _kkt(self):
        if "x" not in self._cache:
            self._cache.update(_kkt_solve(self, want_matrix=True))
        return self._cache

    @property
    def matrix(self) -> np.ndarray:
        return self._kkt()["M"].cpu().numpy()[0]

    @property
    def rhs(self) -> np.ndarray:
        return self._kkt()["rhs"].cpu().numpy()[0]

    @property
    def D(self) -> np.ndarray:
        """Materialises D on request only (linear.py:103-112 order)."""
        fm = self.fmap
        D = fm.feature_matrix_device(self.order, self.constraint_points)
        for k in range(1, self.order + 1):
            fk = _lib.as_f64(self.coeff_values[k - 1], fm.device)
            D = D - fk[:, None] * fm.feature_matrix_device(self.order - k, self.constraint_points)
        return D.cpu().numpy()


def assemble(spec, cond, fmap: NystromFeatureMap, grid, gamma: float) -> AssembledSystem:
    """linear.py:90-137 -- callables sampled on host, Gram on the GPU."""
    grid = np.asarray(grid, dtype=float)
    if gamma <= 0:
        raise ValueError(f"gamma must be positive, got {gamma}")
    p = spec.order
    pts = constraint_points(cond, grid)
    coeff_vals = []
    for k, fk in enumerate(spec.coeffs, start=1):
        fkv = np.asarray(fk(pts), dtype=float)
        if not np.all(np.isfinite(fkv)):
            raise FloatingPointError(f"coefficient f_{k} non-finite on constraint points")
        coeff_vals.append(np.broadcast_to(fkv, pts.shape))
    r = np.asarray(spec.forcing(pts), dtype=float)
    if not np.all(np.isfinite(r)):
        raise FloatingPointError("forcing non-finite on constraint points")
    r = np.broadcast_to(r, pts.shape)
    coef = np.stack(coeff_vals)
    Ac, beta, values = condition_rows(cond, fmap)
    E = gram_ext_device(fmap, p, pts, coef, r)
    return AssembledSystem(constraint_points=pts, gamma=float(gamma), g=-coef[-1], r=r,
                           coeff_values=coef, cond_rows=Ac.reshape(len(cond.entries), -1),
                           cond_bias=beta, cond_values=values, fmap=fmap, order=p, d_gram=E)


def _kkt_solve(system: AssembledSystem, want_matrix: bool = False):
    lib, torch = _lib.require_device()
    fm = system.fmap
    dev = fm.device
    me, nk = fm.m_eff, system.cond_values.size
    side = me + 1 + nk
    Ac = _lib.as_f64(system.cond_rows.reshape(nk, me) if nk else np.zeros((0, me)), dev)
    beta = _lib.as_f64(system.cond_bias, dev)
    vals = _lib.as_f64(system.cond_values.reshape(1, nk), dev)
    x = torch.empty((1, side), dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    M = torch.empty((1, side, side), dtype=torch.float64, device=dev) if want_matrix else None
    rhs = torch.empty((1, side), dtype=torch.float64, device=dev) if want_matrix else None
    wsb = lib.nys_kkt_workspace_bytes(me, nk, 1)
    ws = _lib.WORKSPACE.get(wsb, dev) if wsb else None
    _lib.call("nys_kkt_solve_f64", _lib.ptr(system.d_gram), me, nk, _lib.ptr(Ac), _lib.ptr(beta),
              _lib.ptr(vals), float(system.gamma), 1, _lib.ptr(x), _lib.ptr(info), _lib.ptr(M),
              _lib.ptr(rhs), _lib.ptr(ws), wsb, _lib.stream_ptr())
    return dict(x=x, info=info, M=M, rhs=rhs)


def raise_for_info(code: int):
    if code == _lib.INFO_SINGULAR:
        raise SingularSystemError("Singular matrix")
    if code == _lib.INFO_NONFINITE:
        raise SingularSystemError("solution contains non-finite entries")


def solve(system: AssembledSystem, fmap: NystromFeatureMap) -> PrimalModel:
    """Dense partial-pivoting solve + one refinement step (linear.py:140-158)."""
    res = system._cache if "x" in system._cache else _kkt_solve(system)
    raise_for_info(int(res["info"][0]))
    x = res["x"][0].cpu().numpy()
    me = fmap.m_eff
    return PrimalModel(omega=x[:me], bias=float(x[me]), multipliers=x[me + 1:], feature_map=fmap)


@dataclass(frozen=True)
class KktReport:
    linear_residual: float
    rhs_scale: float
    condition_residuals: np.ndarray
    ode_residuals: np.ndarray

    @property
    def passed(self) -> bool:
        bound = KKT_RESIDUAL_TOL * max(self.rhs_scale, 1.0)
        return bool(self.linear_residual <= bound
                    and np.all(self.condition_residuals <= KKT_RESIDUAL_TOL))


def check_kkt(model: PrimalModel, system: AssembledSystem) -> KktReport:
    """linear.py:161-189; e = D omega + g b - r from a device kernel (no D)."""
    lib, torch = _lib.require_device()
    x = np.concatenate([model.omega, [model.bias], model.multipliers])
    M, rhs = system.matrix, system.rhs
    lin = float(np.max(np.abs(M @ x - rhs)))
    cond_res = np.abs(system.cond_rows @ model.omega + system.cond_bias * model.bias
                      - system.cond_values)
    fm = system.fmap
    dev = fm.device
    pts = _lib.as_f64(system.constraint_points, dev)
    coef = _lib.as_f64(system.coeff_values, dev)
    r = _lib.as_f64(system.r, dev)
    xd = _lib.as_f64(x, dev)
    e = torch.empty(pts.numel(), dtype=torch.float64, device=dev)
    _lib.call("nys_ode_residual_f64", _lib.ptr(fm.d_landmarks), fm.m, _lib.ptr(fm.d_W), fm.ldw,
              fm.m_eff, float(fm.kernel.sigma2), system.order, _lib.ptr(pts), _lib.ptr(coef),
              _lib.ptr(r), pts.numel(), _lib.ptr(xd), _lib.ptr(e), _lib.stream_ptr())
    return KktReport(linear_residual=lin, rhs_scale=float(np.max(np.abs(rhs))),
                     condition_residuals=cond_res, ode_residuals=e.cpu().numpy())


def predict(model: PrimalModel, ell: int, points) -> np.ndarray:
    return model.predict(ell, points)


def _cluster_eig(m: int) -> bool:
    """Landmark counts whose eigendecomposition runs on an 8-CTA cluster
    (csrc/eig_cluster.cu: 68 < m <= 256, the sizes whose one-CTA buffers spill
    out of shared memory)."""
    return 68 < m <= 256 and os.environ.get("NYS_EIG_ALGO", "") != "dc1"


class SingleSolvePipeline:
    """One linear ODE per call on a fixed grid / landmark set (configs 0, 1, 4):
    the reference's assemble + solve (linear.py:90-158) as a device pipeline.

    Per call: the landmark eigendecomposition (its m_eff read-back is the one
    host sync), then -- replayed from a CUDA graph captured on the first call
    with the same buffers -- the condition rows A_c (feature rows at the
    condition points, nys_feature_matrix_f64), the fused feature+Gram kernel and
    the KKT LU + refinement.  Inputs are device tensors; x / info come back in
    buffers owned by the pipeline (overwritten by the next call).  The
    eigendecomposition runs on 2-3 (NYS_EIG_STREAMS) side streams in
    rotation with one buffer set per call in flight, so consecutive calls'
    eigensolvers run concurrently and overlap the previous calls' Gram and KKT
    (NYS_EIG_OVERLAP=0 turns this off); with m_eff + 2 > 72 the kernel-space
    Gram also runs concurrently with it on another side stream.
    NYS_GRAPHS=0 runs everything eagerly.
    """

    # concurrent eigendecompositions: enough that the one-CTA eigensolver
    # (B200, D&C: 0.14 ms at m = 20, 0.30 ms at m = 50, 3.7 ms at m = 256) keeps
    # up with the rest of a call (measured ~0.06, ~0.07 and 2.4 ms): 3 up to
    # m = 32, 5 up to 128, else 2 (each one holds an SM); NYS_EIG_STREAMS overrides
    EIG_STREAMS = int(os.environ.get("NYS_EIG_STREAMS", "0"))

    def _n_eig_streams(self) -> int:
        if self.EIG_STREAMS > 0:
            return self.EIG_STREAMS
        m = self.landmarks.size
        if _cluster_eig(m):
            # one 8-SM cluster eigensolver (1.3 ms at m = 256) per call: one in
            # flight keeps up with a 2.4 ms call; with row shards the Gram is
            # short and more run concurrently (each takes 8 of the Gram's SMs):
            # two for half the rows, three for a quarter, four below
            # (tools/c4_rank_model.py)
            rows = getattr(self, "_rows", None)
            if rows is None:
                return 1
            frac = (rows[1] - rows[0]) / max(1, getattr(self, "_n_grid", rows[1]))
            return 2 if frac > 0.3 else (3 if frac > 0.15 else 4)
        if getattr(self, "_rows", None) is not None:
            return 4   # row shards make the Gram short: more eigensolvers in flight
        if self.WHOLE and (m + 2 + 7) // 8 <= SMALL_NB_MAX:
            # whole-call graphs: every set's call runs concurrently, so the set
            # count is the number of solves in flight: a call's chain (c0 ~0.2 ms,
            # c1 ~0.4 ms) over ~22 us of host time per call
            return int(os.environ.get("NYS_INFLIGHT", "12" if m <= 32 else "16")) - 1
        return 3 if m <= 32 else (5 if m <= 128 else 2)

    def _eig_sms(self) -> int:
        """SMs one in-flight eigendecomposition holds."""
        return 8 if _cluster_eig(self.landmarks.size) else 1

    def __init__(self, landmarks, sigma2: float, grid, gamma: float, order: int, cond,
                 drop_tol: float = 1e-16, device=None, rows=None, group=None):
        """rows=(lo, hi): row-sharded mode (config 4 on several GPUs, dist.py):
        this rank's kernel-space Gram covers collocation rows [lo, hi) and one
        all-reduce(SUM) of K (before the projection; (m+2)^2 doubles) over
        ``group`` (default: the world) completes it; every rank then runs the
        identical projection and KKT.  Requires the kernel-space path."""
        from .kernel import RbfKernel
        from .nystrom import EigBuffers

        lib, torch = _lib.require_device()
        self.lib, self.torch = lib, torch
        if gamma <= 0:
            raise ValueError(f"gamma must be positive, got {gamma}")
        self.kernel = RbfKernel(float(sigma2))
        self._rows, self._group = (None if rows is None else tuple(int(v) for v in rows)), group
        self._n_grid = int(np.asarray(grid).size)
        self.landmarks = np.asarray(landmarks, dtype=float).reshape(-1)
        self.gamma, self.order, self.cond, self.drop_tol = float(gamma), int(order), cond, drop_tol
        self.eig = EigBuffers(self.landmarks, device)
        self.device = self.eig.device
        self.nk = len(cond.entries)
        self.cond_pts = _lib.as_f64([bc.point for bc in cond.entries], self.device)
        self.beta = _lib.as_f64([1.0 if bc.order == 0 else 0.0 for bc in cond.entries],
                                self.device)
        self.vals = _lib.as_f64([bc.value for bc in cond.entries], self.device).reshape(1, -1)
        self._shape = None
        self._graph = None
        self._eigbufs = None
        self._pending = []
        self._me_known = None
        self._cond_known = None
        # kernel-space Gram (m_eff + 2 > 72) needs no eigenvectors: when the
        # landmark count allows that path it is launched speculatively on a side
        # stream with one SM left free, concurrent with the eigendecomposition
        m = self.landmarks.size
        self._kspace = ((m + 2 + 7) // 8 > SMALL_NB_MAX and (m + 2 + 7) // 8 <= 64
                        and os.environ.get("NYS_KSPACE_OVERLAP", "1") != "0")
        if self._kspace:
            self._side = torch.cuda.Stream(device=self.device)
            self._kev = torch.cuda.Event()
            # one SM per concurrent eigensolver and one for the previous call's
            # KKT, which may overlap this call's Gram (input_event)
            self._kctas = (torch.cuda.get_device_properties(self.device).multi_processor_count
                           - self._eig_sms() * self._n_eig_streams() - 1)
            self._kn_c = None
        if rows is not None and not self._kspace:
            raise NotImplementedError("row-sharded SingleSolvePipeline needs the kernel-space "
                                      "Gram (m + 2 > 72 landmarks)")

    def _verify_pending(self, keep: int = 0):
        """Check steady-state eigendecompositions (m_eff, info) once their
        events have completed, leaving the newest ``keep`` unchecked (so the
        host never waits for the eigensolver that is still running)."""
        while len(self._pending) > keep:
            self._check(*self._pending.pop(0))

    def _check(self, ev, buf, me):
        ev.synchronize()
        m_eff, info = int(buf.meta_np[0]), int(buf.meta_np[1])
        if (info & 0xFF) == _lib.INFO_DEGENERATE:
            from .nystrom import DegenerateLandmarksError
            raise DegenerateLandmarksError("two landmarks coincide within 1e-12")
        if m_eff != me:
            raise RuntimeError(f"landmark eigendecomposition changed m_eff {me} -> {m_eff} "
                               "between calls on the same landmarks")

    def _calls_next(self) -> int:
        """Buffer set the next overlapped call will use."""
        n = self._n_eig_streams() + 1
        return self.__dict__.get("_calls", 0) % n

    def _k_for(self, par):
        """Kernel-space Gram buffer of buffer set par (one per set, so the next
        call's Gram never overwrites a K the previous projection still reads)."""
        ks = self.__dict__.setdefault("_K_sets", {})
        k = ks.get(par)
        if k is None:
            m = self.landmarks.size
            k = ks[par] = self.torch.empty((m + 2, m + 2), dtype=self.torch.float64,
                                           device=self.device)
        return k

    def _kspace_launch(self, pts, coef, forcing, kpar=0, input_event=None):
        torch, lib = self.torch, self.lib
        n_c = int(pts.numel())
        m = self.landmarks.size
        if self._kn_c != n_c:
            self.kgws_b = lib.nys_kspace_gram_workspace_bytes(n_c, m, self._kctas)
            self.kgws = torch.empty(self.kgws_b, dtype=torch.uint8, device=self.device)
            self.kpws_b = lib.nys_kspace_project_workspace_bytes(m, m)
            self.kpws = torch.empty(self.kpws_b, dtype=torch.uint8, device=self.device)
            self._kn_c = n_c
        if input_event is not None:
            # the caller's event marks its inputs final: the Gram need not wait
            # for the caller's earlier work (the previous call's KKT)
            self._side.wait_event(input_event)
        else:
            self._side.wait_stream(torch.cuda.current_stream(self.device))
        done = self.__dict__.get("_eig_done")
        if done is not None and done[kpar] is not None:
            self._side.wait_event(done[kpar])   # the last projection that read K_kpar
        K = self._kcur = self._k_for(kpar)
        _lib.call("nys_kspace_gram_f64", _lib.ptr(self.eig.d_lm), m, float(self.kernel.sigma2),
                  self.order, _lib.ptr(pts), _lib.ptr(coef), _lib.ptr(forcing), n_c,
                  *((0, n_c) if self._rows is None else self._rows),
                  self._kctas, _lib.ptr(K), _lib.ptr(self.kgws), self.kgws_b,
                  self._side.cuda_stream)
        self._kev.record(self._side)

    def _buffers(self, me: int, n_c: int):
        torch, lib = self.torch, self.lib
        if self._shape == (me, n_c):
            return
        f64 = dict(dtype=torch.float64, device=self.device)
        m = self.landmarks.size
        self.Ac = torch.zeros((max(self.nk, 1), me), **f64)
        self.E = torch.empty((me + 2, me + 2), **f64)
        self.gws_b = lib.nys_fused_gram_workspace_bytes(n_c, m, me, self.order)
        self.gws = torch.empty(self.gws_b, dtype=torch.uint8, device=self.device)
        self.kws_b = lib.nys_kkt_workspace_bytes(me, self.nk, 1)
        self.kws = (torch.empty(self.kws_b, dtype=torch.uint8, device=self.device)
                    if self.kws_b else None)
        self.x = torch.empty((1, me + 1 + self.nk), **f64)
        self.info = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._shape = (me, n_c)
        self._graph = None

    def _rows_args(self, fm, Ac):
        """Argument tuples of the condition-row launches (linear.py:56-63) into Ac."""
        me = fm.m_eff
        return [(_lib.ptr(fm.d_landmarks), fm.m, _lib.ptr(fm.d_W), fm.ldw, me,
                 float(fm.kernel.sigma2), int(bc.order), _lib.ptr(self.cond_pts) + 8 * mu, 1,
                 _lib.ptr(Ac) + 8 * mu * me, me) for mu, bc in enumerate(self.cond.entries)]

    def _ac_for(self, par, me):
        """Condition rows of buffer set par: they depend on W only, so the
        overlapped path computes them on the eigensolver's stream."""
        sets = self.__dict__.setdefault("_Ac_sets", {})
        a = sets.get(par)
        if a is None or a.shape[1] != me:
            a = sets[par] = self.torch.zeros((max(self.nk, 1), me), dtype=self.torch.float64,
                                             device=self.device)
        return a

    def _post(self, fm, pts, coef, forcing, use_k=False, Ac=None, K=None, E=None, part="all",
              gws=None, xi=None, kws=None, kpws=None):
        me, m, st = fm.m_eff, fm.m, _lib.stream_ptr()
        E = self.E if E is None else E
        gws = self.gws if gws is None else gws
        kws = self.kws if kws is None else kws
        kpws = self.__dict__.get("kpws") if kpws is None else kpws
        x, info = (self.x, self.info) if xi is None else xi
        if part != "kkt":
            if Ac is None:   # rows here (otherwise already computed on the eig stream)
                Ac = self.Ac
                for args in self._rows_args(fm, Ac):
                    _lib.call("nys_feature_matrix_f64", *args, st)
            n_c = pts.numel()
            if use_k:
                _lib.call("nys_kspace_project_f64", _lib.ptr(self._kcur if K is None else K), m,
                          _lib.ptr(fm.d_W), fm.ldw, me,
                          _lib.ptr(E), _lib.ptr(kpws), self.kpws_b, st)
            else:
                _lib.call("nys_fused_gram_f64", _lib.ptr(fm.d_landmarks), m, _lib.ptr(fm.d_W),
                          fm.ldw, me, float(fm.kernel.sigma2), self.order, _lib.ptr(pts),
                          _lib.ptr(coef), _lib.ptr(forcing), n_c, 0, n_c, _lib.ptr(E),
                          _lib.ptr(gws), self.gws_b, st)
        if part != "gram":
            _lib.call("nys_kkt_solve_f64", _lib.ptr(E), me, self.nk, _lib.ptr(Ac),
                      _lib.ptr(self.beta), _lib.ptr(self.vals), self.gamma, 1, _lib.ptr(x),
                      _lib.ptr(info), None, None, _lib.ptr(kws), self.kws_b, st)

    # kernel-space path (config 4): each buffer set's projection + KKT (one CTA,
    # ~0.45 ms at side 259) runs on the set's own stream with the set's own E,
    # workspaces and outputs, so consecutive calls' KKTs overlap each other (with
    # row shards the Gram is short and one KKT per call in series would bound the
    # step); NYS_KSPACE_SETS=0 keeps them on the caller's stream
    KSETS = os.environ.get("NYS_KSPACE_SETS", "1") != "0"

    def _set_res(self, q, me):
        """Per-set E, (x, info), KKT and projection workspaces (kernel-space sets)."""
        rs = self.__dict__.setdefault("_set_res_d", {})
        r = rs.get(q)
        if r is None or r[0] != me:
            torch = self.torch
            xs = (torch.empty_like(self.x), torch.zeros_like(self.info))
            kws = (torch.empty(self.kws_b, dtype=torch.uint8, device=self.device)
                   if self.kws_b else None)
            kpws = torch.empty(self.kpws_b, dtype=torch.uint8, device=self.device)
            r = rs[q] = (me, dict(E=self._e_for(q, me), xi=xs, kws=kws, kpws=kpws))
        return r[1]

    def _set_stream(self, q):
        ss = self.__dict__.setdefault("_set_streams", {})
        st = ss.get(q)
        if st is None:
            st = ss[q] = self.torch.cuda.Stream(device=self.device)
        return st

    def _e_for(self, par, me):
        es = self.__dict__.setdefault("_E_sets", {})
        e = es.get(par)
        if e is None or e.shape[0] != me + 2:
            e = es[par] = self.torch.empty((me + 2, me + 2), dtype=self.torch.float64,
                                           device=self.device)
        return e

    def _split_capture(self, fm, pts, coef, forcing, Ac, E):
        """Two graphs for the fused-Gram path: the Gram (replayed on a side
        stream that waits only for the inputs and W) and the KKT (on the
        caller's stream), so call k+1's Gram overlaps call k's KKT."""
        torch = self.torch
        out = []
        for part in ("gram", "kkt"):
            n0 = self.lib.nys_launch_count()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                self._post(fm, pts, coef, forcing, False, Ac, None, E, part)
            out += [g, self.lib.nys_launch_count() - n0]
        return tuple(out)

    # configs 0/1 steady state: each buffer set's WHOLE call (eigendecomposition,
    # condition rows, fused Gram, KKT) is one CUDA graph replayed on the set's own
    # stream with the set's own workspace and outputs, so consecutive calls
    # (independent solves) run concurrently on different SMs and the host pays one
    # replay per call; NYS_WHOLE_GRAPH=0 keeps the per-stage replays
    WHOLE = os.environ.get("NYS_WHOLE_GRAPH", "1") != "0"

    def _capture_whole(self, q, fm, pts, coef, forcing):
        torch, lib = self.torch, self.lib
        me = fm.m_eff
        gw = self.__dict__.setdefault("_gws_sets", {})
        if q not in gw:
            gw[q] = torch.empty(self.gws_b, dtype=torch.uint8, device=self.device)
        xs = self.__dict__.setdefault("_X_sets", {})
        if q not in xs:
            xs[q] = (torch.empty_like(self.x), torch.zeros_like(self.info))
        Ac, E = self._ac_for(q, me), self._e_for(q, me)
        # two graphs on the set's stream: the eigendecomposition and condition rows
        # need no inputs (they start as soon as the set is free), the Gram and KKT
        # wait for the inputs
        n0 = lib.nys_launch_count()
        ge = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ge, capture_error_mode="thread_local"):
            st = _lib.stream_ptr()
            rc = lib.nys_landmark_eig_f64(*self._eig_args[q], st)
            if rc:
                _lib.check(rc, "nys_landmark_eig_f64")
            for args in self._rows_args(fm, Ac):
                _lib.call("nys_feature_matrix_f64", *args, st)
        gp = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gp, capture_error_mode="thread_local"):
            self._post(fm, pts, coef, forcing, False, Ac, None, E, "all", gw[q], xs[q])
        return (ge, gp, lib.nys_launch_count() - n0, ge.raw_cuda_graph_exec(),
                gp.raw_cuda_graph_exec())

    def _run_whole(self, plan, input_event):
        torch = self.torch
        n = len(self._eigbufs)
        par = self._calls % n
        self._calls += 1
        # the set's previous call (n calls ago) is checked now; newer ones later,
        # so the host never waits for work still in flight
        self._verify_pending(keep=n - 1)
        ws = self.__dict__.setdefault("_wstreams", {})
        sd = ws.get(par)
        if sd is None:
            st = torch.cuda.Stream(device=self.device)
            evs = (torch.cuda.Event(), torch.cuda.Event())
            for e in evs:   # create the CUDA events now (lazy in torch)
                e.record(st)
            sd = ws[par] = (st, evs[0], evs[1], st.cuda_stream, evs[0].cuda_event,
                            evs[1].cuda_event)
        ge, gp, nl = plan[par][:3]
        di = self.__dict__.get("_dev_index")
        if di is None:
            di = self._dev_index = torch.device(self.device).index or 0
        # the caller's current stream by its raw handle (torch.cuda.current_stream()
        # resolves the device on every call: ~half the host cost of a call)
        caller = torch._C._cuda_getCurrentRawStream(di)
        rc = self.lib.nys_replay_pair(
            sd[3], plan[par][3], None if input_event is None else input_event.cuda_event,
            plan[par][4], sd[4], caller, sd[5])
        if rc:
            _lib.check(rc, "nys_replay_pair")
        _lib.note_graph_launches(nl)
        self._pending.append((sd[1], self._eigbufs[par], self._me_known))
        self.eig = self._eigbufs[par]
        self.x, self.info = self._X_sets[par]
        return self.x, self.info

    def _gram_side(self):
        side = self.__dict__.get("_gside")
        if side is None:
            side = self._gside = self.torch.cuda.Stream(device=self.device)
            self._gram_ev = [self.torch.cuda.Event() for _ in self._eigbufs]
        return side

    def _replay_split(self, plan_par, par, input_event, cur):
        """Gram graph on the side stream (inputs + W + this set's E free), KKT
        graph on the caller's stream after it."""
        torch = self.torch
        gg, nlg, gk, nlk = plan_par
        side = self._gram_side()
        if input_event is not None:
            side.wait_event(input_event)
        else:
            side.wait_stream(cur)
        side.wait_event(self._eig_ev[par])
        if self._eig_done[par] is not None:
            side.wait_event(self._eig_done[par])   # E of this set: its last KKT is done
        with torch.cuda.stream(side):
            gg.replay()
        gev = self._gram_ev[par]
        gev.record(side)
        cur.wait_event(gev)
        gk.replay()
        _lib.note_graph_launches(nlg + nlk)

    def _run_fast(self, plan, input_event=None):
        """Steady-state call for inputs whose graphs exist for every buffer set
        (configs 0/1): rotate the set and the eigensolver stream, launch the
        eigendecomposition with pre-bound arguments, replay the set's graph --
        the same work as the general path with a fraction of its host cost."""
        n = len(self._eigbufs)
        par = self._calls % n
        es = self._eig_streams[self._calls % len(self._eig_streams)]
        self._calls += 1
        es.wait_event(self._post_ev[par])   # the set's last reader has finished
        self._verify_pending(keep=len(self._eig_streams))
        buf = self._eigbufs[par]
        sh = es.cuda_stream
        rc = self.lib.nys_landmark_eig_f64(*self._eig_args[par], sh)
        if rc:
            _lib.check(rc, "nys_landmark_eig_f64")
        for args in self._rows_bound[par]:   # condition rows need W only: same stream
            rc = self.lib.nys_feature_matrix_f64(*args, sh)
            if rc:
                _lib.check(rc, "nys_feature_matrix_f64")
        ev = self._eig_ev[par]
        ev.record(es)
        self._pending.append((ev, buf, self._me_known))
        cur = self.torch.cuda.current_stream()
        p = plan[par]
        if len(p) == 4:
            self._replay_split(p, par, input_event, cur)
        else:
            cur.wait_event(ev)
            p[0].replay()
            _lib.note_graph_launches(p[1])
        post = self._post_ev[par]
        post.record(cur)
        self._eig_done[par] = post
        self.eig = buf
        return self.x, self.info

    def _capture(self, fm, pts, coef, forcing, use_k, Ac=None, K=None, res=None):
        torch = self.torch
        n0 = self.lib.nys_launch_count()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            self._post(fm, pts, coef, forcing, use_k, Ac, K, **(res or {}))
        return g, self.lib.nys_launch_count() - n0

    def run_device(self, pts, coef, forcing, input_event=None):
        """pts (n_c,), coef (p, n_c), forcing (n_c,) device float64 -> (x (1, side), info).

        input_event: optional CUDA event after which the inputs are final (e.g.
        the caller's H2D, or recorded once for static inputs); the kernel-space
        Gram then waits on it instead of on all earlier work of the current
        stream, so it can overlap the previous call's KKT."""
        import os

        from .nystrom import build_feature_map, launch_eig_pinned

        torch = self.torch
        whole = self.__dict__.get("_whole")
        if whole:
            plan = whole.get((pts.data_ptr(), coef.data_ptr(), forcing.data_ptr()))
            if plan is not None:
                return self._run_whole(plan, input_event)
            # new input buffers: let the whole-call graphs in flight on the sets'
            # own streams finish before the staged path reuses the sets
            torch.cuda.synchronize(self.device)
        fast = self.__dict__.get("_fast")
        if fast:
            plan = fast.get((pts.data_ptr(), coef.data_ptr(), forcing.data_ptr()))
            if plan is not None:
                return self._run_fast(plan, input_event)
        cur = torch.cuda.current_stream()
        graphs = os.environ.get("NYS_GRAPHS", "1") != "0"
        overlap = graphs and os.environ.get("NYS_EIG_OVERLAP", "1") != "0"
        kpar = self._calls_next() if overlap else 0
        if self._kspace and input_event is None:
            # the caller's work so far (its inputs), before this call's
            # eigendecomposition is joined into the stream: the Gram waits only
            # for that
            pre = self.__dict__.get("_pre_ev")
            if pre is None:
                pre = self._pre_ev = torch.cuda.Event()
            pre.record(cur)
            input_event = pre
        par = None
        kset = self._kspace and overlap and self.KSETS
        post_st = cur
        if overlap:
            # the eigendecomposition (one CTA, FP64-latency bound) runs on
            # EIG_STREAMS side streams in rotation, each call with its own buffer
            # set (EIG_STREAMS + 1 sets), so consecutive calls' eigensolvers run
            # concurrently on different SMs and overlap the Gram/KKT of earlier
            # calls; a set is rewritten only after the main-stream work that last
            # read it (event)
            if self._eigbufs is None:
                from .nystrom import EigBuffers
                ns = self._n_eig_streams()
                self._eigbufs = [self.eig] + [EigBuffers(self.landmarks, self.device)
                                              for _ in range(ns)]
                self._eig_done = [None] * (ns + 1)
                self._eig_ev = [torch.cuda.Event() for _ in range(ns + 1)]
                self._post_ev = [torch.cuda.Event() for _ in range(ns + 1)]
                self._fm_cache = {}
                self._eig_streams = [torch.cuda.Stream(device=self.device) for _ in range(ns)]
                self._calls = 0
            par = self._calls % len(self._eigbufs)
            es = self._eig_streams[self._calls % len(self._eig_streams)]
            self._calls += 1
            if kset:
                post_st = self._set_stream(par)
            if self._eig_done[par] is not None:
                es.wait_event(self._eig_done[par])
            self._verify_pending(keep=len(self._eig_streams))
            buf = self._eigbufs[par]
            if self._me_known is None:
                # first call: synchronous build (m_eff, degenerate check, cond gate)
                with torch.cuda.stream(es):
                    fm = build_feature_map(self.kernel, self.landmarks, self.drop_tol,
                                           buffers=buf)
                self._me_known = fm.m_eff
                self._cond_known = fm.condition
                for args in self._rows_args(fm, self._ac_for(par, fm.m_eff)):
                    _lib.call("nys_feature_matrix_f64", *args, es.cuda_stream)
                cur.wait_stream(es)
                if post_st is not cur:
                    post_st.wait_stream(cur)
            else:
                # steady state: the same landmarks give the same m_eff (deterministic
                # kernels), so the host does not wait for the eigensolver; this
                # call's m_eff / info are checked at the start of the next call
                fm = self._fm_cache.get(par)
                if fm is None:
                    fm = self._fm_cache[par] = NystromFeatureMap(
                        kernel=self.kernel, landmarks=self.landmarks, m_eff=self._me_known,
                        device=self.device, d_landmarks=buf.d_lm, d_W=buf.W, d_eigvals=buf.s,
                        d_eigvecs=buf.V)
                launch_eig_pinned(self.kernel, buf, self.drop_tol, es, self._eig_ev[par])
                for args in self._rows_args(fm, self._ac_for(par, self._me_known)):
                    _lib.call("nys_feature_matrix_f64", *args, es.cuda_stream)
                ev = self._eig_ev[par]
                ev.record(es)
                self._pending.append((ev, buf, self._me_known))
                post_st.wait_event(ev)
            self.eig = buf
        else:
            fm = build_feature_map(self.kernel, self.landmarks, self.drop_tol, buffers=self.eig)
        if self._kspace:
            # launched after the eigendecomposition: an 8-SM cluster eigensolver
            # (68 < m <= 256) must find its SMs in one GPC before the Gram's CTAs
            # spread over the rest, else it waits for the whole Gram
            self._kspace_launch(pts, coef, forcing, kpar, input_event)
        me = fm.m_eff
        big = (me + 2 + 7) // 8 > SMALL_NB_MAX
        if self._kspace:   # inputs and K are shared with the side stream
            post_st.wait_event(self._kev)
            if post_st is not cur:   # the fused-Gram fallback (small m_eff) reads the inputs
                post_st.wait_event(input_event)
            if self._rows is not None:   # partial K of this rank's rows -> full K
                from .dist import allreduce_sum
                with torch.cuda.stream(post_st):
                    allreduce_sum(self._kcur, self._group)
        cond_omega = self._cond_known if par is not None else fm.condition
        if big and cond_omega > KSPACE_MAX_COND:
            raise IllConditionedLargeMapError(
                f"m_eff={me} with cond(Omega)={fm.condition:.2e} > {KSPACE_MAX_COND:.0e}")
        use_k = self._kspace and big
        n_c = int(pts.numel())
        self._buffers(me, n_c)
        if not graphs:
            self._post(fm, pts, coef, forcing, use_k)
            return self.x, self.info
        with torch.cuda.stream(post_st):
            self._post_graphs(fm, pts, coef, forcing, me, n_c, use_k, par, kset, input_event,
                              post_st)
        if par is not None:
            ev = self._post_ev[par]
            ev.record(post_st)
            self._eig_done[par] = ev
            if post_st is not cur:
                cur.wait_event(ev)
                self.x, self.info = self._set_res(par, me)["xi"]
        return self.x, self.info

    def _post_graphs(self, fm, pts, coef, forcing, me, n_c, use_k, par, kset, input_event, cur):
        """Replay (or run eagerly and capture) the post-eigendecomposition graphs
        of buffer set par on the current stream (``cur``)."""
        torch = self.torch
        key = (me, pts.data_ptr(), coef.data_ptr(), forcing.data_ptr(), n_c, use_k,
               fm.d_W.data_ptr())
        if self._graph is None:
            self._graph = {}
        # split Gram / KKT graphs (call k+1's Gram overlaps call k's KKT) pay off
        # once the KKT is long; for tiny systems the extra stream hops cost more
        split = (not use_k) and par is not None and me >= 32 and not kset
        if split:
            key = key + ("split",)
        hit = self._graph.get(key)
        if hit is not None:
            if split:
                self._replay_split(hit, par, input_event, cur)
            else:
                hit[0].replay()
                _lib.note_graph_launches(hit[1])
        else:
            Ac = None if par is None else self._ac_for(par, me)
            Kp = (self._k_for(par) if par is not None else self._kcur) if use_k else None
            Ep = self._e_for(par, me) if split else None
            # eager: this call's result + the kernels' one-time attribute setup
            if kset:
                self._post(fm, pts, coef, forcing, use_k, Ac, Kp, **self._set_res(par, me))
            else:
                self._post(fm, pts, coef, forcing, use_k, Ac, Kp, Ep)
            if split:
                self._graph[key] = self._split_capture(fm, pts, coef, forcing, Ac, Ep)
                # the eager Gram ran on this stream: later side-stream Grams (shared
                # workspace) must follow it
                self._gram_side().wait_stream(cur)
            else:
                self._graph[key] = self._capture(fm, pts, coef, forcing, use_k, Ac, Kp,
                                                 self._set_res(par, me) if kset else None)
            if par is not None:
                # the other eigendecomposition buffer sets will come round with
                # the same inputs: capture theirs now (capture does not execute),
                # so steady-state calls only replay
                self._fm_cache.setdefault(par, fm)
                for q, b2 in enumerate(self._eigbufs):
                    f2 = self._fm_cache.get(q)
                    if f2 is None:
                        f2 = self._fm_cache[q] = NystromFeatureMap(
                            kernel=self.kernel, landmarks=self.landmarks, m_eff=me,
                            device=self.device, d_landmarks=b2.d_lm, d_W=b2.W, d_eigvals=b2.s,
                            d_eigvecs=b2.V)
                    k2 = key[:6] + (f2.d_W.data_ptr(),) + key[7:]
                    if k2 in self._graph:
                        continue
                    if split:
                        self._graph[k2] = self._split_capture(f2, pts, coef, forcing,
                                                              self._ac_for(q, me),
                                                              self._e_for(q, me))
                    else:
                        self._graph[k2] = self._capture(f2, pts, coef, forcing, use_k,
                                                        self._ac_for(q, me),
                                                        self._k_for(q) if use_k else None,
                                                        self._set_res(q, me) if kset else None)
                if not self._kspace:   # steady state for these inputs: _run_fast
                    plan = [self._graph[key[:6] + (b2.W.data_ptr(),) + key[7:]]
                            for b2 in self._eigbufs]
                    self.__dict__.setdefault("_fast", {})[key[1:4]] = plan
                    self._eig_args = [
                        (_lib.ptr(b2.d_lm), self.landmarks.size, float(self.kernel.sigma2),
                         float(self.drop_tol), _lib.ptr(b2.s), _lib.ptr(b2.V), _lib.ptr(b2.W),
                         _lib.ptr(b2.meta_h), _lib.ptr(b2.meta_h) + 4, _lib.ptr(b2.ws), b2.wsb)
                        for b2 in self._eigbufs]
                    self._rows_bound = [self._rows_args(self._fm_cache[q], self._ac_for(q, me))
                                        for q in range(len(self._eigbufs))]
                    if self.WHOLE and self._rows is None:
                        # every set's previous work has finished before its
                        # whole-call graph is first replayed on its own stream
                        torch.cuda.synchronize(self.device)
                        self.__dict__.setdefault("_whole", {})[key[1:4]] = [
                            self._capture_whole(q, self._fm_cache[q], pts, coef, forcing)
                            for q in range(len(self._eigbufs))]

    def host_block(self, pts, coef, forcing):
        """The samples of one call as ONE pinned host block [pts | coef (p x n_c) |
        forcing] (one H2D per call) -- what run_host takes.  The reference's
        callers hold these as NumPy arrays (linear.py:103-116 samples the spec
        on the host)."""
        blk = np.concatenate([np.asarray(pts, dtype=np.float64).reshape(-1),
                              np.asarray(coef, dtype=np.float64).reshape(-1),
                              np.asarray(forcing, dtype=np.float64).reshape(-1)])
        n_c = int(np.asarray(pts).size)
        if blk.size != n_c * (2 + self.order):
            raise ValueError(f"expected pts (n_c,), coef ({self.order}, n_c), forcing (n_c,)")
        return self.torch.from_numpy(blk).pin_memory()

    def run_host(self, block_h, x_h, stages: int = 0):
        """One call from pinned host memory to pinned host memory: ``block_h`` (see
        host_block) is uploaded on a copy stream into one of ``stages`` device
        sets used in rotation (default 3 on the kernel-space path, else 4), the
        solve runs as in run_device with the upload's event as its input event,
        and x lands in ``x_h`` (pinned, (1, side)) behind it on the current
        stream.  Nothing blocks the host: call k + 1's upload overlaps call k's
        solve, and a set is refilled only after the solve that last read it.
        Returns (x_h, info) with info the device int32[1] of this call's buffer
        set (0 ok; read it after synchronising).  Two C calls + run_device per
        solve."""
        torch = self.torch
        hs = self.__dict__.get("_hstage")
        n = int(block_h.numel())
        ns = int(stages) if stages else (3 if self._kspace else 4)
        if hs is None or hs["n"] != n or len(hs["dev"]) != ns:
            p = self.order
            if n % (p + 2):
                raise ValueError(f"block of {n} doubles is not (p + 2) * n_c with p = {p}")
            n_c = n // (p + 2)
            if hs is not None:   # in-flight calls still read the old sets
                torch.cuda.synchronize(self.device)
            dev = [torch.empty(n, dtype=torch.float64, device=self.device) for _ in range(ns)]
            evs = [(torch.cuda.Event(), torch.cuda.Event()) for _ in range(ns)]
            copy = torch.cuda.Stream(device=self.device)
            for r, f in evs:   # torch creates the CUDA events lazily
                r.record(copy)
                f.record(copy)
            hs = self._hstage = dict(
                n=n, dev=dev, copy=copy, evs=evs, calls=0, used=[False] * ns,
                views=[(d[:n_c], d[n_c:n_c * (p + 1)].view(p, n_c), d[n_c * (p + 1):])
                       for d in dev],
                raw=[(d.data_ptr(), r.cuda_event, f.cuda_event) for d, (r, f) in zip(dev, evs)],
                di=torch.device(self.device).index or 0)
        if not (block_h.is_pinned() and x_h.is_pinned()):
            raise ValueError("run_host needs pinned host tensors (host_block / pin_memory())")
        k = hs["calls"] % ns
        hs["calls"] += 1
        dptr, ready, free = hs["raw"][k]
        caller = torch._C._cuda_getCurrentRawStream(hs["di"])
        rc = self.lib.nys_stage_upload(dptr, block_h.data_ptr(), n * 8, hs["copy"].cuda_stream,
                                       free if hs["used"][k] else None, ready, caller)
        if rc:
            _lib.check(rc, "nys_stage_upload")
        hs["used"][k] = True
        x, info = self.run_device(*hs["views"][k], input_event=hs["evs"][k][0])
        rc = self.lib.nys_stage_download(x_h.data_ptr(), x.data_ptr(), x.numel() * 8, caller, free)
        if rc:
            _lib.check(rc, "nys_stage_download")
        return x_h, info

    def model(self):
        """PrimalModel of the last call (raises the reference's errors from info)."""
        self._verify_pending()
        raise_for_info(int(self.info[0]))
        x = self.x[0].cpu().numpy()
        me = self._shape[0]
        fm = NystromFeatureMap(kernel=self.kernel, landmarks=self.landmarks, m_eff=me,
                               device=self.device, d_landmarks=self.eig.d_lm, d_W=self.eig.W,
                               d_eigvals=self.eig.s, d_eigvecs=self.eig.V)
        return PrimalModel(omega=x[:me], bias=float(x[me]), multipliers=x[me + 1:],
                           feature_map=fm)
