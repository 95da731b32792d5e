"""Landmark selection and the explicit Nystrom feature map, on the B200.

Mirror of ``pkg/src/nysode/nystrom.py`` (same names, arguments, errors):

* :func:`select_landmarks` -- host index logic, identical to nystrom.py:84-106;
  for ``LeverageScore`` the scores come from the device
  (:func:`ridge_leverage_scores`, C-ABI ``nys_leverage_scores_f64``) and the
  draw uses the reference's own numpy Generator stream on the host.
* :func:`build_feature_map` -- device Jacobi eigendecomposition of Omega_mm
  (C-ABI ``nys_landmark_eig_f64``), replacing nystrom.py:136-160.
* :class:`NystromFeatureMap` -- holds the device copies (landmarks, W);
  ``eigenvalues`` / ``eigenvectors`` are fetched to the host lazily so the
  reference's attributes keep working.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Optional

import os

import numpy as np

from ._refcompat import ref_base
from . import _lib
from .kernel import RbfKernel, check_order

DEFAULT_DROP_TOL = 1e-16     # nystrom.py:21
_LEVERAGE_EXACT_LIMIT = 4000  # nystrom.py:25


class DegenerateLandmarksError(*ref_base("nystrom", "DegenerateLandmarksError", ValueError)):
    """Two landmarks coincide within 1e-12 (nystrom.py:29-30)."""


class InvalidCountError(*ref_base("nystrom", "InvalidCountError", ValueError)):
    """Landmark count outside 2..n (nystrom.py:33-34)."""


@dataclass(frozen=True)
class Equidistant:
    pass


@dataclass(frozen=True)
class Random:
    seed: int = 0


@dataclass(frozen=True)
class LeverageScore:
    seed: int = 0
    ridge: float = 1e-6
    kernel: Optional[RbfKernel] = None


def select_landmarks(strategy, grid, m: int) -> np.ndarray:
    """Pick m distinct grid points (nystrom.py:84-106)."""
    grid = np.asarray(grid, dtype=float)
    n = grid.size
    if m < 2 or m > n:
        raise InvalidCountError(f"landmark count m={m} must satisfy 2 <= m <= n={n}")
    name = type(strategy).__name__
    if name == "Equidistant":
        idx = np.round(np.arange(m) * (n - 1) / (m - 1)).astype(int)
    elif name == "Random":
        rng = np.random.default_rng(strategy.seed)
        idx = np.sort(rng.choice(n, size=m, replace=False))
    elif name == "LeverageScore":
        # nystrom.py:95-103: default score kernel is an RBF of length span / 10
        rng = np.random.default_rng(strategy.seed)
        score_kernel = strategy.kernel
        if score_kernel is None:
            span = float(grid[-1] - grid[0])
            score_kernel = RbfKernel(sigma2=max(span / 10.0, 1e-6) ** 2)
        scores = ridge_leverage_scores(score_kernel, grid, strategy.ridge)
        p = scores / scores.sum()
        idx = np.sort(rng.choice(n, size=m, replace=False, p=p))
    else:
        raise TypeError(f"unknown sampling strategy {strategy!r}")
    return grid[idx]


_SKETCH_PCHOL_TOL = 1e-15    # stop of the sketch compression (diag of W is 1)
DENSE_EIG_MAX_M = 512        # nys_landmark_eig_f64 (D&C <= 256, QL <= 512)
# compression stop for large landmark sets (diag of Omega is 1): 1e-18, below
# the drop rule's 1e-16 s_0, so the compressed spectrum reaches the same tail a
# dense dsyevd keeps (catalog P1/P7/P8/P12/P16 at m = n = 1000: y_hat within
# 1.9e-7 .. 6.0e-7 of the reference; with 1e-16, P16 drifts to 1.9e-6)
_LARGE_PCHOL_TOL = float(os.environ.get("NYS_PCHOL_TOL", "1e-18"))
_LARGE_MAX_RANK = 256
_SKETCH_MAX_RANK = 256       # r x r eigensolver limit (divide and conquer)


def ridge_leverage_scores(k: RbfKernel, grid, ridge: float, device=None) -> np.ndarray:
    """diag(Omega (Omega + n ridge I)^-1) over the grid (nystrom.py:58-81).

    Exact branch (n <= 4000): 1 - n ridge diag(A^-1) from one tiled DMMA
    Cholesky + inverse sweep on the device (``nys_leverage_scores_f64``).
    Sketch branch (n > 4000, nystrom.py:71-80): the same column sketch
    (c = 2000 points idx = linspace(0, n-1, c).round(), chosen on the host as
    the reference does); the sketch matrix is compressed on the device by a
    pivoted Cholesky and its kept spectrum (vals > 1e-12 vals.max()) taken from
    the small G^T G eigenproblem (``nys_pchol_rbf_f64`` +
    ``nys_leverage_sketch_f64``).  A sketch whose numerical rank exceeds 256
    raises ``NotImplementedError`` instead of falling back to the host.
    """
    grid = np.asarray(grid, dtype=float).reshape(-1)
    n = grid.size
    lib, torch = _lib.require_device()
    device = torch.device(device or "cuda")
    d_grid = _lib.as_f64(grid, device)
    scores = torch.empty(n, dtype=torch.float64, device=device)
    info = torch.zeros(1, dtype=torch.int32, device=device)
    st = _lib.stream_ptr()
    if n <= _LEVERAGE_EXACT_LIMIT:
        wsb = lib.nys_leverage_workspace_bytes(n)
        ws = _lib.WORKSPACE.get(wsb, device)
        _lib.call("nys_leverage_scores_f64", _lib.ptr(d_grid), n, float(k.sigma2), float(ridge),
                  _lib.ptr(scores), _lib.ptr(info), _lib.ptr(ws), wsb, st)
    else:
        c = _LEVERAGE_EXACT_LIMIT // 2
        idx = np.linspace(0, n - 1, c).round().astype(int)      # nystrom.py:72
        d_x = _lib.as_f64(grid[idx], device)
        cap = _SKETCH_MAX_RANK
        G = torch.empty(cap * c, dtype=torch.float64, device=device)
        out = torch.zeros(2, dtype=torch.int32, device=device)
        _lib.call("nys_pchol_rbf_f64", _lib.ptr(d_x), c, float(k.sigma2), _SKETCH_PCHOL_TOL,
                  cap, _lib.ptr(G), _lib.ptr(out), st)
        r, converged = (int(v) for v in out.cpu())
        if not converged:
            raise NotImplementedError(
                f"sketch kernel matrix has numerical rank > {cap}; the device eigensolver "
                "for the sketch branch stops there")
        wsb = lib.nys_leverage_sketch_workspace_bytes(n, c, r)
        ws = _lib.WORKSPACE.get(wsb, device)
        _lib.call("nys_leverage_sketch_f64", _lib.ptr(d_grid), n, _lib.ptr(d_x), c,
                  float(k.sigma2), float(ridge), _lib.ptr(G), r, _lib.ptr(scores),
                  _lib.ptr(info), _lib.ptr(ws), wsb, st)
    if int(info.item()) != _lib.INFO_OK:
        raise np.linalg.LinAlgError("leverage system is not numerically positive definite")
    return scores.cpu().numpy()


@dataclass(eq=False)
class NystromFeatureMap:
    """Feature map phi(t) = Lambda^{-1/2} V^T k(t, L) with device-resident W."""

    kernel: RbfKernel
    landmarks: np.ndarray
    m_eff: int
    device: Any
    d_landmarks: Any                 # (m,) float64 tensor
    d_W: Any                         # (m, m) float64 tensor; columns >= m_eff are 0
    d_eigvals: Any                   # (m,) descending
    d_eigvecs: Any                   # (m, m)
    _host: dict = field(default_factory=dict, repr=False)

    @property
    def m(self) -> int:
        return int(self.landmarks.size)

    @property
    def ldw(self) -> int:
        """Row stride of d_W (m for the dense eigensolvers, the rank cap for
        the compressed large-m path)."""
        return int(self.d_W.shape[1])

    @property
    def eigenvalues(self) -> np.ndarray:
        if "s" not in self._host:
            self._host["s"] = self.d_eigvals[: self.m_eff].cpu().numpy()
        return self._host["s"]

    @property
    def eigenvectors(self) -> np.ndarray:
        if "v" not in self._host:
            self._host["v"] = self.d_eigvecs[:, : self.m_eff].cpu().numpy()
        return self._host["v"]

    @property
    def condition(self) -> float:
        """s_max / s_min over the retained eigenvalues."""
        s = self.eigenvalues
        return float(s[0] / s[-1])

    def feature_matrix_device(self, ell: int, points):
        """Psi_ell(points) as a (|points|, m_eff) device tensor (nystrom.py:123-127)."""
        check_order(ell)
        lib, torch = _lib.require_device()
        pts = _lib.as_f64(np.atleast_1d(points) if not hasattr(points, "device") else points,
                          self.device).reshape(-1)
        out = torch.empty((pts.numel(), self.m_eff), dtype=torch.float64, device=self.device)
        _lib.call("nys_feature_matrix_f64", _lib.ptr(self.d_landmarks), self.m, _lib.ptr(self.d_W),
                  self.ldw, self.m_eff, float(self.kernel.sigma2), int(ell), _lib.ptr(pts),
                  pts.numel(), _lib.ptr(out), self.m_eff, _lib.stream_ptr())
        return out

    def feature_matrix(self, ell: int, points) -> np.ndarray:
        return self.feature_matrix_device(ell, points).cpu().numpy()

    def feature(self, t: float) -> np.ndarray:
        return self.feature_matrix(0, [t])[0]

    def feature_deriv(self, ell: int, t: float) -> np.ndarray:
        return self.feature_matrix(ell, [t])[0]


class EigBuffers:
    """Device buffers of one landmark set's eigendecomposition, reused across
    repeated builds (SharedGridPipeline): the landmarks are copied once and the
    m_eff read-back goes through pinned memory -- no per-step allocations or
    pageable copies on the critical path.  A feature map built into these
    buffers is overwritten by the next build."""

    def __init__(self, landmarks, device=None):
        lib, torch = _lib.require_device()
        self.landmarks = np.asarray(landmarks, dtype=float).reshape(-1).copy()
        self.device = torch.device(device or "cuda")
        m = self.landmarks.size
        f64 = dict(dtype=torch.float64, device=self.device)
        self.d_lm = _lib.as_f64(self.landmarks, self.device)
        self.s = torch.empty(m, **f64)
        self.V = torch.empty((m, m), **f64)
        self.W = torch.empty((m, m), **f64)
        self.meta = torch.zeros(2, dtype=torch.int32, device=self.device)   # m_eff, info
        self.meta_h = torch.zeros(2, dtype=torch.int32).pin_memory()
        self.meta_np = self.meta_h.numpy()   # host view (no tensor iteration on checks)
        self.s_h = torch.zeros(m, dtype=torch.float64).pin_memory()   # eigenvalues, same sync
        self.wsb = lib.nys_landmark_eig_workspace_bytes(m)
        self.ws = torch.empty(self.wsb, dtype=torch.uint8, device=self.device) if self.wsb else None


def launch_eig_async(k: RbfKernel, buffers: EigBuffers, drop_tol: float, stream):
    """Enqueue the eigendecomposition into ``buffers`` on ``stream`` without
    waiting for it: m_eff / info land in ``buffers.meta_h`` (pinned) when the
    returned event completes.  For pipelines that already know m_eff from an
    earlier build of the same landmarks and verify it one call later."""
    lib, torch = _lib.require_device()
    m = buffers.landmarks.size
    with torch.cuda.stream(stream):
        _lib.call("nys_landmark_eig_f64", _lib.ptr(buffers.d_lm), m, float(k.sigma2),
                  float(drop_tol), _lib.ptr(buffers.s), _lib.ptr(buffers.V), _lib.ptr(buffers.W),
                  _lib.ptr(buffers.meta), _lib.ptr(buffers.meta) + 4, _lib.ptr(buffers.ws),
                  buffers.wsb, stream.cuda_stream)
        buffers.meta_h.copy_(buffers.meta, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
    return ev


def launch_eig_pinned(k: RbfKernel, buffers: EigBuffers, drop_tol: float, stream, event):
    """Steady-state form of launch_eig_async for pipelines: the eigensolver
    writes m_eff / info straight into the pinned host words (device-visible
    under unified addressing: no D2H copy op), on ``stream`` by handle (no
    stream context switch), and ``event`` (reused) is recorded after it."""
    m = buffers.landmarks.size
    _lib.call("nys_landmark_eig_f64", _lib.ptr(buffers.d_lm), m, float(k.sigma2),
              float(drop_tol), _lib.ptr(buffers.s), _lib.ptr(buffers.V), _lib.ptr(buffers.W),
              _lib.ptr(buffers.meta_h), _lib.ptr(buffers.meta_h) + 4, _lib.ptr(buffers.ws),
              buffers.wsb, stream.cuda_stream)
    event.record(stream)
    return event


def build_feature_map(k: RbfKernel, landmarks, drop_tol: float = DEFAULT_DROP_TOL,
                      device=None, buffers: Optional[EigBuffers] = None) -> NystromFeatureMap:
    """Eigendecompose Omega_mm on the GPU and keep s > max(drop_tol s_0, 0)."""
    landmarks = np.asarray(landmarks, dtype=float).reshape(-1)
    if not 0 <= drop_tol < 1:
        raise ValueError(f"drop_tol must lie in [0, 1), got {drop_tol}")
    lib, torch = _lib.require_device()
    m = landmarks.size
    if m > DENSE_EIG_MAX_M:
        return _build_compressed(k, landmarks, drop_tol, device)
    if buffers is not None:
        if not np.array_equal(buffers.landmarks, landmarks):
            raise ValueError("EigBuffers hold a different landmark set")
        device = buffers.device
        d_lm, s, V, W, meta, ws, wsb = (buffers.d_lm, buffers.s, buffers.V, buffers.W,
                                        buffers.meta, buffers.ws, buffers.wsb)
    else:
        device = torch.device(device or "cuda")
        d_lm = _lib.as_f64(landmarks, device)
        s = torch.empty(m, dtype=torch.float64, device=device)
        V = torch.empty((m, m), dtype=torch.float64, device=device)
        W = torch.empty((m, m), dtype=torch.float64, device=device)
        meta = torch.zeros(2, dtype=torch.int32, device=device)   # m_eff, info
        wsb = lib.nys_landmark_eig_workspace_bytes(m)
        ws = _lib.WORKSPACE.get(wsb, device) if wsb else None
    _lib.call("nys_landmark_eig_f64", _lib.ptr(d_lm), m, float(k.sigma2), float(drop_tol),
              _lib.ptr(s), _lib.ptr(V), _lib.ptr(W), _lib.ptr(meta), _lib.ptr(meta) + 4,
              _lib.ptr(ws), wsb, _lib.stream_ptr())
    if buffers is not None:
        buffers.meta_h.copy_(meta, non_blocking=True)
        buffers.s_h.copy_(s, non_blocking=True)
        torch.cuda.current_stream(device).synchronize()
        m_eff, info = (int(v) for v in buffers.meta_h)
    else:
        m_eff, info = (int(v) for v in meta.cpu())
    sweeps, info = info >> 8, info & 0xFF      # bits 8+: Jacobi sweeps (diagnostic)
    if info == _lib.INFO_DEGENERATE:
        raise DegenerateLandmarksError("two landmarks coincide within 1e-12")
    fm = NystromFeatureMap(kernel=k, landmarks=landmarks, m_eff=m_eff, device=device,
                           d_landmarks=d_lm, d_W=W, d_eigvals=s, d_eigvecs=V)
    fm._host["sweeps"] = sweeps
    if buffers is not None:
        fm._host["s"] = buffers.s_h[:m_eff].numpy().copy()
    return fm


def _build_compressed(k: RbfKernel, landmarks: np.ndarray, drop_tol: float, device=None):
    """Feature map of a large landmark set (m > 512, e.g. the m = n comparator
    of baselines.py:170-194).

    Omega = K(L, L) is compressed on the device by a pivoted Cholesky
    (Omega ~ G G^T, stopped when the largest remaining diagonal is below 1e-16),
    and the eigenpairs of G G^T come from the r x r problem G^T G with the
    reference's drop rule s > max(drop_tol s_0, 0) (nystrom.py:150-154).  The
    kept spectrum is the numerical range of Omega; eigenpairs at the rounding
    floor (s ~ 1e-16 s_0) are noise in the reference's dense dsyevd as well.
    """
    if landmarks.size >= 2 and np.min(np.diff(np.sort(landmarks))) <= 1e-12:
        raise DegenerateLandmarksError("two landmarks coincide within 1e-12")   # nystrom.py:145
    lib, torch = _lib.require_device()
    device = torch.device(device or "cuda")
    m = landmarks.size
    d_lm = _lib.as_f64(landmarks, device)
    cap = _LARGE_MAX_RANK
    G = torch.empty(cap * m, dtype=torch.float64, device=device)
    out = torch.zeros(2, dtype=torch.int32, device=device)
    st = _lib.stream_ptr()
    _lib.call("nys_pchol_rbf_f64", _lib.ptr(d_lm), m, float(k.sigma2), _LARGE_PCHOL_TOL, cap,
              _lib.ptr(G), _lib.ptr(out), st)
    r, converged = (int(v) for v in out.cpu())
    if not converged:
        raise NotImplementedError(
            f"landmark kernel matrix (m={m}) has numerical rank > {cap}: beyond the device "
            "eigensolver of the compressed path")
    s = torch.empty(r, dtype=torch.float64, device=device)
    V = torch.zeros((m, r), dtype=torch.float64, device=device)
    W = torch.zeros((m, r), dtype=torch.float64, device=device)
    meta = torch.zeros(2, dtype=torch.int32, device=device)
    wsb = lib.nys_landmark_eig_compressed_workspace_bytes(r)
    ws = _lib.WORKSPACE.get(wsb, device)
    _lib.call("nys_landmark_eig_compressed_f64", _lib.ptr(G), m, r, float(drop_tol), _lib.ptr(s),
              _lib.ptr(V), _lib.ptr(W), r, _lib.ptr(meta), _lib.ptr(meta) + 4, _lib.ptr(ws), wsb,
              st)
    m_eff = int(meta[0].item())
    fm = NystromFeatureMap(kernel=k, landmarks=landmarks, m_eff=m_eff, device=device,
                           d_landmarks=d_lm, d_W=W, d_eigvals=s, d_eigvecs=V)
    fm._host["compressed"] = r
    return fm
