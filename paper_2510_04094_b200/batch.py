"""Batched linear solves for B ODEs sharing grid, landmarks and sigma (config 2).

The reference solves one spec per call (``linear.assemble`` + ``linear.solve``,
linear.py:90-158), recomputing the feature matrices every time.  A batch that
shares the feature map lets the GPU form Psi_0..Psi_p once and spend the rest
on per-instance row combines + Gram (``nys_batch_gram_f64``) and B small KKT
solves (``nys_batch_kkt_solve_f64``) -- one stream, no host round trip.

Entry points:
* :class:`LinearBatchSolver` -- array API: sampled coefficient rows
  ``coef[B, p, n_c]``, ``forcing[B, n_c]``, condition values ``values[B, p]``
  (host or device); returns device ``x[B, side]`` and ``info[B]``.
* :func:`solve_many` -- reference-style API over lists of ``LinearOdeSpec`` /
  ``Conditions`` (samples the callables on the host exactly like
  linear.py:103-116) returning ``PrimalModel`` objects.
"""
from __future__ import annotations

import os
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .linear import PrimalModel, condition_rows, constraint_points, raise_for_info
from .nystrom import NystromFeatureMap


class LinearBatchSolver:
    def __init__(self, fmap: NystromFeatureMap, grid, gamma: float, order: int, cond,
                 max_batch: int):
        if gamma <= 0:
            raise ValueError(f"gamma must be positive, got {gamma}")
        lib, torch = _lib.require_device()
        self.lib, self.torch = lib, torch
        self.fmap = fmap
        self.gamma = float(gamma)
        self.order = int(order)
        self.cond = cond
        grid = np.asarray(grid, dtype=float)
        self.pts_host = constraint_points(cond, grid)
        self.n_c = self.pts_host.size
        dev = fmap.device
        self.pts = _lib.as_f64(self.pts_host, dev)
        Ac, beta, _ = condition_rows(cond, fmap)
        self.n_cond = len(cond.entries)
        self.Ac = _lib.as_f64(Ac.reshape(self.n_cond, fmap.m_eff), dev)
        self.beta = _lib.as_f64(beta, dev)
        self.side = fmap.m_eff + 1 + self.n_cond
        self.max_batch = int(max_batch)
        self.ws_bytes = lib.nys_batch_gram_workspace_bytes(self.n_c, fmap.m_eff, self.order,
                                                          self.max_batch)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.cond_pts = _lib.as_f64([bc.point for bc in cond.entries], dev)

    def refresh_condition_rows(self):
        """A_c[mu] = phi^(order_mu)(point_mu) written straight into the device
        buffer (linear.py:56-63), no host round trip; beta depends only on the
        orders and is unchanged."""
        fm = self.fmap
        st = _lib.stream_ptr()
        for mu, bc in enumerate(self.cond.entries):
            _lib.call("nys_feature_matrix_f64", _lib.ptr(fm.d_landmarks), fm.m, _lib.ptr(fm.d_W),
                      fm.ldw, fm.m_eff, float(fm.kernel.sigma2), int(bc.order),
                      _lib.ptr(self.cond_pts) + 8 * mu, 1, _lib.ptr(self.Ac) + 8 * mu * fm.m_eff,
                      fm.m_eff, st)

    def solve_device(self, coef, forcing, values, out_x=None, out_info=None):
        """coef (B, p, n_c), forcing (B, n_c), values (B, n_cond) device float64
        tensors -> (x (B, side), info (B,)).  Fully stream-ordered, no sync."""
        torch = self.torch
        fm = self.fmap
        B = int(coef.shape[0])
        if B > self.max_batch:
            raise ValueError(f"batch {B} exceeds max_batch {self.max_batch}")
        ws_bytes = self.lib.nys_batch_gram_workspace_bytes(self.n_c, fm.m_eff, self.order, B)
        x = out_x if out_x is not None else torch.empty((B, self.side), dtype=torch.float64,
                                                         device=fm.device)
        info = out_info if out_info is not None else torch.empty(B, dtype=torch.int32,
                                                                 device=fm.device)
        st = _lib.stream_ptr()
        _lib.call("nys_batch_gram_f64", _lib.ptr(fm.d_landmarks), fm.m, _lib.ptr(fm.d_W), fm.ldw,
                  fm.m_eff, float(fm.kernel.sigma2), self.order, _lib.ptr(self.pts), self.n_c,
                  _lib.ptr(coef), _lib.ptr(forcing), B, None, _lib.ptr(self.ws), ws_bytes, st)
        _lib.call("nys_batch_kkt_solve_f64", _lib.ptr(self.ws), self.n_c, fm.m_eff, self.order,
                  self.n_cond, _lib.ptr(self.Ac), _lib.ptr(self.beta), _lib.ptr(values),
                  self.gamma, B, _lib.ptr(x), _lib.ptr(info), st)
        return x, info

    def gram_ext(self, coef, forcing):
        """Dense extended Grams (B, m_eff+2, m_eff+2) -- for tests / inspection."""
        torch = self.torch
        fm = self.fmap
        B = int(coef.shape[0])
        ws_bytes = self.lib.nys_batch_gram_workspace_bytes(self.n_c, fm.m_eff, self.order, B)
        E = torch.empty((B, fm.m_eff + 2, fm.m_eff + 2), dtype=torch.float64, device=fm.device)
        _lib.call("nys_batch_gram_f64", _lib.ptr(fm.d_landmarks), fm.m, _lib.ptr(fm.d_W), fm.ldw,
                  fm.m_eff, float(fm.kernel.sigma2), self.order, _lib.ptr(self.pts), self.n_c,
                  _lib.ptr(coef), _lib.ptr(forcing), B, _lib.ptr(E), _lib.ptr(self.ws), ws_bytes,
                  _lib.stream_ptr())
        return E

    def solve(self, coef, forcing, values):
        dev = self.fmap.device
        coef = _lib.as_f64(coef, dev)
        forcing = _lib.as_f64(forcing, dev)
        values = _lib.as_f64(values, dev).reshape(coef.shape[0], self.n_cond)
        return self.solve_device(coef, forcing, values)


def _sample_specs(specs, pts, p, coef, forcing, lo, hi):
    """Spec callables on the constraint points for specs[lo:hi] (linear.py:104-116:
    the same non-finite checks, in the same order per spec)."""
    for b in range(lo, hi):
        sp = specs[b]
        if sp.order != p:
            raise ValueError("solve_many needs a common ODE order")
        for k, fk in enumerate(sp.coeffs, start=1):
            v = np.asarray(fk(pts), dtype=float)
            if not np.all(np.isfinite(v)):
                raise FloatingPointError(f"coefficient f_{k} non-finite on constraint points")
            coef[b, k - 1] = v
        r = np.asarray(sp.forcing(pts), dtype=float)
        if not np.all(np.isfinite(r)):
            raise FloatingPointError("forcing non-finite on constraint points")
        forcing[b] = r


# host threads sampling the spec callables (NumPy ufuncs release the GIL inside
# their loops); NYS_SAMPLE_THREADS=1 samples on the calling thread
_SAMPLE_THREADS = int(os.environ.get("NYS_SAMPLE_THREADS", "0")) or min(16, os.cpu_count() or 1)
_POOL = None


def solve_many(specs: Sequence, conds: Sequence, fmap: NystromFeatureMap, grid,
               gamma: float) -> list[PrimalModel]:
    """Reference-style batch: one PrimalModel per (spec, cond), same grid/fmap.

    Condition points and orders must be shared (values may differ).  The spec
    callables are sampled on a host thread pool in contiguous chunks (each spec's
    checks and errors as in linear.py:104-116; the first failing chunk's error is
    raised)."""
    if len(specs) != len(conds) or not specs:
        raise ValueError("need matching, non-empty spec and condition lists")
    grid = np.asarray(grid, dtype=float)
    c0 = conds[0]
    key = [(bc.point, bc.order) for bc in c0.entries]
    for c in conds:
        if c.kind != c0.kind or [(bc.point, bc.order) for bc in c.entries] != key:
            raise ValueError("solve_many needs shared condition points/orders")
    p = specs[0].order
    pts = constraint_points(c0, grid)
    coef = np.empty((len(specs), p, pts.size))
    forcing = np.empty((len(specs), pts.size))
    nb = len(specs)
    nt = min(_SAMPLE_THREADS, max(1, nb // 64))
    if nt <= 1:
        _sample_specs(specs, pts, p, coef, forcing, 0, nb)
    else:
        global _POOL
        if _POOL is None:
            from concurrent.futures import ThreadPoolExecutor
            _POOL = ThreadPoolExecutor(max_workers=_SAMPLE_THREADS)
        bounds = [nb * i // nt for i in range(nt + 1)]
        futs = [_POOL.submit(_sample_specs, specs, pts, p, coef, forcing, bounds[i], bounds[i + 1])
                for i in range(nt)]
        for f in futs:   # in chunk order: the lowest failing chunk's error wins
            f.result()
    values = np.array([[bc.value for bc in c.entries] for c in conds])
    solver = LinearBatchSolver(fmap, grid, gamma, p, c0, len(specs))
    x, info = solver.solve(coef, forcing, values)
    x = x.cpu().numpy()
    info = info.cpu().numpy()
    me = fmap.m_eff
    out = []
    for b in range(len(specs)):
        raise_for_info(int(info[b]))
        out.append(PrimalModel(omega=x[b, :me], bias=float(x[b, me]), multipliers=x[b, me + 1:],
                               feature_map=fmap))
    return out


class SharedGridPipeline:
    """One config-2 step from scratch: landmark eigendecomposition (once per
    shared landmark set), shared features, per-instance Gram, KKT solves.

    ``run_device`` takes device-resident samples; ``run_host`` takes pinned
    host arrays, streams them in ``chunks`` on a copy stream overlapped with
    the compute stream, and returns the solutions in pinned host memory --
    the end-to-end path a caller with host data uses.
    """

    def __init__(self, landmarks, sigma2: float, grid, gamma: float, order: int, cond,
                 max_batch: int, drop_tol: float = 1e-16, device=None):
        from .kernel import RbfKernel
        from .nystrom import build_feature_map

        self.landmarks = np.asarray(landmarks, dtype=float)
        self.kernel = RbfKernel(float(sigma2))
        self.grid = np.asarray(grid, dtype=float)
        self.gamma, self.order, self.cond = float(gamma), int(order), cond
        self.max_batch, self.drop_tol = int(max_batch), drop_tol
        self._build = build_feature_map
        self.device = device
        self.solver = None

    def _prepare_fmap(self, eigbuf=None, stream=None):
        """Eigendecomposition + solver object; True when the solver is new."""
        from .nystrom import EigBuffers
        if eigbuf is None:
            if getattr(self, "_eigbuf", None) is None:
                self._eigbuf = EigBuffers(self.landmarks, self.device)
            eigbuf = self._eigbuf
        if stream is None:
            fm = self._build(self.kernel, self.landmarks, self.drop_tol, buffers=eigbuf)
        else:
            torch = _lib.require_device()[1]
            with torch.cuda.stream(stream):
                fm = self._build(self.kernel, self.landmarks, self.drop_tol, buffers=eigbuf)
            torch.cuda.current_stream().wait_stream(stream)
        if self.solver is None or self.solver.fmap.m_eff != fm.m_eff:
            self.solver = LinearBatchSolver(fm, self.grid, self.gamma, self.order, self.cond,
                                            self.max_batch)
            self._graphs = None
            return self.solver, True
        self.solver.fmap = fm
        return self.solver, False

    def prepare(self):
        """Eigendecomposition + solver state (the per-landmark-set work)."""
        solver, fresh = self._prepare_fmap()
        if not fresh:   # same shapes: keep the workspace, refresh the condition rows on device
            solver.refresh_condition_rows()
        return solver

    def run_device(self, coef, forcing, values, out_x=None, out_info=None):
        """One step on device-resident samples.  After the eigendecomposition
        (whose m_eff read-back is the step's one host sync) the condition-row
        refresh, Psi pack, Gram and KKT launches are replayed from a CUDA graph
        captured on the first call with the same buffers (NYS_GRAPHS=0 turns
        this off).  The eigendecomposition itself runs on a side stream with two
        alternating buffer sets, so consecutive calls overlap it with the
        previous call's Gram (NYS_EIG_OVERLAP=0 turns this off).  Without
        out_x/out_info the results land in buffers owned by the pipeline and are
        overwritten by the next call."""
        import os

        from .nystrom import EigBuffers

        torch = _lib.require_device()[1]
        graphs = os.environ.get("NYS_GRAPHS", "1") != "0"
        if graphs and os.environ.get("NYS_EIG_OVERLAP", "1") != "0":
            # Two eigen-buffer sets used alternately, the eigendecomposition on its
            # own stream: this call's (one-SM) eigensolver runs while the previous
            # call's Gram is still executing.  A set is overwritten only after the
            # main-stream work of the call that last read it (event).
            if getattr(self, "_eigbufs", None) is None:
                self._eigbufs = [EigBuffers(self.landmarks, self.device) for _ in range(2)]
                self._eig_done = [None, None]
                self._eig_stream = torch.cuda.Stream(device=self._eigbufs[0].device)
                self._parity = 0
            k = self._parity
            self._parity ^= 1
            if self._eig_done[k] is not None:
                self._eig_stream.wait_event(self._eig_done[k])
            solver, fresh = self._prepare_fmap(self._eigbufs[k], self._eig_stream)
        else:
            k = None
            solver, fresh = self._prepare_fmap()
        B = int(coef.shape[0])
        if out_x is None or out_info is None:
            if getattr(self, "_outs", None) is None or self._outs[0].shape != (B, solver.side):
                self._outs = (torch.empty((B, solver.side), dtype=torch.float64,
                                          device=solver.fmap.device),
                              torch.empty(B, dtype=torch.int32, device=solver.fmap.device))
            out_x = self._outs[0] if out_x is None else out_x
            out_info = self._outs[1] if out_info is None else out_info

        def post():
            solver.refresh_condition_rows()
            solver.solve_device(coef, forcing, values, out_x, out_info)

        if not graphs:
            post()
            return out_x, out_info
        key = (id(solver), solver.fmap.m_eff, solver.fmap.d_W.data_ptr(), B, coef.data_ptr(),
               forcing.data_ptr(), values.data_ptr(), out_x.data_ptr(), out_info.data_ptr())
        if fresh or getattr(self, "_graphs", None) is None:
            self._graphs = {}
        hit = self._graphs.get(key)
        if hit is not None:
            hit[0].replay()
            _lib.note_graph_launches(hit[1])
        else:
            post()   # eager: this call's result, and the kernels' one-time attribute setup
            lib = _lib.load()
            n0 = lib.nys_launch_count()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                post()
            self._graphs[key] = (g, lib.nys_launch_count() - n0)
        if k is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self._eig_done[k] = ev
        return out_x, out_info

    def run_host(self, coef_h, forcing_h, values_h, x_h, info_h, chunks: int = 4,
                 dev_bufs=None):
        """Pinned host in -> pinned host out.  dev_bufs: optional preallocated
        device staging (coef, forcing, values, x, info) for the full batch, or a
        list of such sets used in rotation: the copy stream then refills a set as
        soon as the solve that last read it has finished, so this call's H2D
        overlaps the previous call's solve (otherwise it waits for all earlier
        work on the current stream)."""
        torch = _lib.require_device()[1]
        dev = torch.device(self.device or "cuda")
        B = coef_h.shape[0]
        free_ev = None
        if isinstance(dev_bufs, list):
            k = getattr(self, "_host_calls", 0)
            self._host_calls = k + 1
            if not hasattr(self, "_host_free") or len(self._host_free) != len(dev_bufs):
                self._host_free = [None] * len(dev_bufs)
            slot = k % len(dev_bufs)
            free_ev = self._host_free[slot]
            dev_bufs = dev_bufs[slot]
        else:
            slot = None
        if dev_bufs is None:
            dev_bufs = (torch.empty(coef_h.shape, dtype=torch.float64, device=dev),
                        torch.empty(forcing_h.shape, dtype=torch.float64, device=dev),
                        torch.empty(values_h.shape, dtype=torch.float64, device=dev),
                        None, None)
        dc, df, dv, dx, di = dev_bufs
        comp = torch.cuda.current_stream()
        copy = getattr(self, "_copy_stream", None)
        if copy is None:
            copy = self._copy_stream = torch.cuda.Stream(device=dev)
        if slot is None:
            copy.wait_stream(comp)
        elif free_ev is not None:
            copy.wait_event(free_ev)
        bounds = np.linspace(0, B, chunks + 1).astype(int)
        ready = []
        with torch.cuda.stream(copy):
            for c in range(chunks):
                a, b = bounds[c], bounds[c + 1]
                dc[a:b].copy_(coef_h[a:b], non_blocking=True)
                df[a:b].copy_(forcing_h[a:b], non_blocking=True)
                dv[a:b].copy_(values_h[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
                ready.append(ev)
        # eigendecomposition of the shared landmark set runs while the samples
        # are still crossing PCIe on the copy stream
        solver = self.prepare()
        if dx is None:
            dx = torch.empty((B, solver.side), dtype=torch.float64, device=dev)
            di = torch.empty(B, dtype=torch.int32, device=dev)
        if tuple(dx.shape) != (B, solver.side) or tuple(x_h.shape) != (B, solver.side):
            raise ValueError(f"solution buffers must be ({B}, {solver.side})")
        for c in range(chunks):
            a, b = bounds[c], bounds[c + 1]
            comp.wait_event(ready[c])
            solver.solve_device(dc[a:b], df[a:b], dv[a:b], dx[a:b], di[a:b])
        if slot is not None:
            ev = torch.cuda.Event()
            ev.record(comp)
            self._host_free[slot] = ev
        x_h.copy_(dx, non_blocking=True)
        info_h.copy_(di, non_blocking=True)
        return x_h, info_h
