"""Race and bounds evidence for the lock-free / shared-memory-heavy kernels.

compute-sanitizer is closed on this GPU pool (runs under it have left GPUs
needing a reset; tools/sanitize.sh is kept for pools that allow it), so these
tests look for the two classes of defect it would report by their effects:

* races -- every call is repeated many times while a side stream keeps other
  kernels resident, so CTA placement, warp drift and the TMA / mbarrier
  hand-over timing change from call to call; a race on a shared-memory stage
  (gram_batch.cu's lock-free stage release), on the replica slab sums
  (gram_large.cu) or on the DSMEM exchanges (eig_cluster.cu) shows up as a
  result that is not bit-identical to the first call.  Every reduction in
  these kernels is fixed-order, so bit-identity is the contract.
* out-of-bounds writes -- outputs and workspaces are carved out of larger
  buffers whose guard regions hold a sentinel; any byte written outside the
  documented extent changes a guard.

Shapes are the bench's own (c2: n = 4096, m = 64; c4: m = 256 on n = 2^20 of
the c4 grid; c3's Newton ladder on 64 instances).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 4096            # doubles of guard on each side
SENTINEL = -7.25e301    # any write of a real result changes it
REPEATS = 12


def _guarded(torch, n_doubles, dev):
    buf = torch.full((n_doubles + 2 * GUARD,), SENTINEL, dtype=torch.float64, device=dev)
    return buf, buf[GUARD:GUARD + n_doubles]


def _guards_intact(buf):
    return bool((buf[:GUARD] == SENTINEL).all()) and bool((buf[-GUARD:] == SENTINEL).all())


class _Contention:
    """Keeps a side stream busy with GEMMs while the tested calls run."""

    def __init__(self, torch, dev):
        self.torch = torch
        self.side = torch.cuda.Stream(device=dev)
        self.a = torch.randn(2048, 2048, device=dev)

    def kick(self, i):
        torch = self.torch
        with torch.cuda.stream(self.side):
            for _ in range(1 + i % 3):
                self.a = torch.tanh(self.a @ self.a * 1e-3)


def test_batch_gram_and_kkt_race_and_bounds():
    """c2 shape: the batched Gram (TMA ring released by the last warp, no CTA
    barrier) and the batched KKT reading its partials -- bit-identical over
    repeats under contention, nothing written outside E / x / info / ws."""
    import torch

    from paper_2510_04094_b200 import _lib
    from paper_2510_04094_b200 import batch as BT
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200 import workloads as W
    from paper_2510_04094_b200.kernel import RbfKernel
    from paper_2510_04094_b200.problems import BoundaryCondition, Conditions

    lib, _ = _lib.require_device()
    cfg = W.scaled(W.CONFIGS[2], batch=1000)     # 125 CTAs: a partial wave, ragged tail
    bt = W.linear_batch(cfg, seed=3)
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), bt.landmarks)
    dev = fm.device
    cond = Conditions("ivp", tuple(BoundaryCondition(*c) for c in bt.instances[0].conditions()))
    solver = BT.LinearBatchSolver(fm, bt.grid, cfg.gamma, cfg.order, cond, cfg.batch)
    B, n_c, me, p = cfg.batch, solver.n_c, fm.m_eff, cfg.order
    coef = torch.as_tensor(bt.coef, device=dev).contiguous()
    forc = torch.as_tensor(bt.forcing, device=dev).contiguous()
    vals = torch.as_tensor(bt.cond_values, device=dev).reshape(B, -1).contiguous()
    wsb = lib.nys_batch_gram_workspace_bytes(n_c, me, p, B)
    wsbuf, ws = _guarded(torch, (wsb + 7) // 8, dev)
    ebuf, E = _guarded(torch, B * (me + 2) ** 2, dev)
    xbuf, x = _guarded(torch, B * solver.side, dev)
    ibuf = torch.full((B + 2 * GUARD,), -12345, dtype=torch.int32, device=dev)
    info = ibuf[GUARD:GUARD + B]
    load = _Contention(torch, dev)
    st = _lib.stream_ptr()
    first = None
    for i in range(REPEATS):
        load.kick(i)
        _lib.call("nys_batch_gram_f64", _lib.ptr(fm.d_landmarks), fm.m, _lib.ptr(fm.d_W),
                  fm.ldw, me, float(fm.kernel.sigma2), p, _lib.ptr(solver.pts), n_c,
                  _lib.ptr(coef), _lib.ptr(forc), B, _lib.ptr(E), _lib.ptr(ws), wsb, st)
        _lib.call("nys_batch_kkt_solve_f64", _lib.ptr(ws), n_c, me, p, solver.n_cond,
                  _lib.ptr(solver.Ac), _lib.ptr(solver.beta), _lib.ptr(vals), float(cfg.gamma),
                  B, _lib.ptr(x), _lib.ptr(info), st)
        got = (E.clone(), x.clone(), info.clone())
        if first is None:
            first = got
            assert bool((info == 0).all())
        else:
            assert torch.equal(got[0], first[0]), f"gram differs on repeat {i}"
            assert torch.equal(got[1], first[1]), f"solution differs on repeat {i}"
            assert torch.equal(got[2], first[2])
    torch.cuda.synchronize()
    assert _guards_intact(wsbuf) and _guards_intact(ebuf) and _guards_intact(xbuf)
    assert bool((ibuf[:GUARD] == -12345).all()) and bool((ibuf[-GUARD:] == -12345).all())
    # and the guarded run equals the product entry
    xs, _ = solver.solve(coef, forc, vals)
    assert torch.equal(xs.reshape(-1), first[1])


def test_kspace_gram_race_and_bounds():
    """c4 shape on 2^20 rows: kernel-space Gram (per-CTA windows, replica slabs
    added in fixed order, slab reduce) + projection -- bit-identical over
    repeats under contention and at a CTA cap, guards intact."""
    import torch

    from paper_2510_04094_b200 import _lib
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200 import workloads as W
    from paper_2510_04094_b200.kernel import RbfKernel

    lib, _ = _lib.require_device()
    cfg = W.CONFIGS[4]
    bt = W.linear_batch(cfg, 0, 1)
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), bt.landmarks)
    dev = fm.device
    lo, hi = 1_000_000, 1_000_000 + (1 << 20) + 17          # ragged range mid-grid
    pts = torch.as_tensor(bt.pts, device=dev)
    coef = torch.as_tensor(bt.coef[0], device=dev).contiguous()
    forc = torch.as_tensor(bt.forcing[0], device=dev).contiguous()
    n_c, m, me, p = pts.numel(), fm.m, fm.m_eff, cfg.order
    load = _Contention(torch, dev)
    st = _lib.stream_ptr()
    results = {}
    for cap in (0, 100):
        wsb = lib.nys_kspace_gram_workspace_bytes(n_c, m, cap)
        wsbuf, ws = _guarded(torch, (wsb + 7) // 8, dev)
        kbuf, K = _guarded(torch, (m + 2) ** 2, dev)
        pwsb = lib.nys_kspace_project_workspace_bytes(m, me)
        pbuf, pws = _guarded(torch, (pwsb + 7) // 8, dev)
        ebuf, E = _guarded(torch, (me + 2) ** 2, dev)
        first = None
        for i in range(REPEATS // 2):
            load.kick(i)
            _lib.call("nys_kspace_gram_f64", _lib.ptr(fm.d_landmarks), m, float(fm.kernel.sigma2),
                      p, _lib.ptr(pts), _lib.ptr(coef), _lib.ptr(forc), n_c, lo, hi, cap,
                      _lib.ptr(K), _lib.ptr(ws), wsb, st)
            _lib.call("nys_kspace_project_f64", _lib.ptr(K), m, _lib.ptr(fm.d_W), fm.ldw, me,
                      _lib.ptr(E), _lib.ptr(pws), pwsb, st)
            got = (K.clone(), E.clone())
            if first is None:
                first = got
            else:
                assert torch.equal(got[0], first[0]), f"K differs on repeat {i} (cap {cap})"
                assert torch.equal(got[1], first[1])
        torch.cuda.synchronize()
        for b in (wsbuf, kbuf, pbuf, ebuf):
            assert _guards_intact(b), f"write outside its extent (cap {cap})"
        results[cap] = first[0]
    # a different CTA count changes the row ranges, hence the summation order:
    # equal to rounding only
    d = float((results[0] - results[100]).abs().max() / results[0].abs().max())
    assert d <= 1e-13, d


@pytest.mark.parametrize("m", [64, 256])
def test_landmark_eig_race_and_bounds(m):
    """One-CTA (m = 64) and 8-CTA cluster (m = 256, DSMEM st.async exchanges
    counted by mbarrier transaction bytes) eigensolvers: bit-identical over
    repeats under contention, guards intact."""
    import torch

    from paper_2510_04094_b200 import _lib
    from paper_2510_04094_b200 import workloads as W

    lib, _ = _lib.require_device()
    cfg = W.CONFIGS[4] if m == 256 else W.CONFIGS[2]
    bt = W.linear_batch(cfg, 0, 1)
    dev = torch.device("cuda")
    lm = torch.as_tensor(bt.landmarks, device=dev)
    assert lm.numel() == m
    wsb = lib.nys_landmark_eig_workspace_bytes(m)
    wsbuf, ws = _guarded(torch, (wsb + 7) // 8, dev)
    sbuf, s = _guarded(torch, m, dev)
    vbuf, V = _guarded(torch, m * m, dev)
    wbuf, Wm = _guarded(torch, m * m, dev)
    ibuf = torch.full((2 + 2 * GUARD,), -777, dtype=torch.int32, device=dev)
    me, info = ibuf[GUARD:GUARD + 1], ibuf[GUARD + 1:GUARD + 2]
    load = _Contention(torch, dev)
    st = _lib.stream_ptr()
    first = None
    for i in range(REPEATS):
        load.kick(i)
        _lib.call("nys_landmark_eig_f64", _lib.ptr(lm), m, float(cfg.sigma2), 1e-12,
                  _lib.ptr(s), _lib.ptr(V), _lib.ptr(Wm), _lib.ptr(me), _lib.ptr(info),
                  _lib.ptr(ws), wsb, st)
        got = (s.clone(), V.clone(), Wm.clone(), me.clone())
        if first is None:
            first = got
            assert int(info) == 0
        else:
            for a, b in zip(got, first):
                assert torch.equal(a, b), f"eigensolver output differs on repeat {i}"
    torch.cuda.synchronize()
    for b in (wsbuf, sbuf, vbuf, wbuf):
        assert _guards_intact(b)
    assert bool((ibuf[:GUARD] == -777).all()) and bool((ibuf[-GUARD:] == -777).all())
    # and the spectrum is right
    ev = np.sort(first[0].cpu().numpy())[::-1]
    K = np.exp(-np.subtract.outer(bt.landmarks, bt.landmarks) ** 2 / cfg.sigma2)
    ref = np.sort(np.linalg.eigvalsh(K))[::-1]
    assert np.max(np.abs(ev - ref)) <= 1e-12 * ref[0]


def test_newton_ladder_repeatable_under_contention():
    """c3 (64 instances): the whole retry ladder in one kernel (one CTA per
    instance, 8 warps sharing the reduction trees and the LU rows) gives
    bit-identical iterates, statuses and rungs over repeats under contention."""
    import torch

    from paper_2510_04094_b200 import newton as NW
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200 import workloads as W
    from paper_2510_04094_b200.kernel import RbfKernel
    from paper_2510_04094_b200.problems import ivp

    cfg = W.CONFIGS[3]
    g = W.grid(cfg)
    lm = W.equidistant_landmarks(g, cfg.m)
    insts = [W.instance(3, 0, i) for i in range(64)]
    pts = g[1:]
    fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                             np.array([i.quad_coeff for i in insts]),
                             np.array([i.sin_coeff for i in insts]))
    vals = np.array([[i.conditions()[0][2]] for i in insts])
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
    eng = NW.NewtonBatch(fm, g, ivp([(0.0, 0, 0.0)]), vals, cfg.gamma, family=fam)
    load = _Contention(torch, fm.device)
    first = None
    for i in range(4):
        load.kick(i)
        status, X, traces, rung = eng.solve(max_iters=cfg.newton_max_iters)
        got = (np.asarray(status).copy(), np.asarray(X).copy(), np.asarray(rung).copy(),
               [np.asarray(t).copy() for t in traces])
        if first is None:
            first = got
            assert int((got[0] == NW.OK).sum()) >= 56
        else:
            assert np.array_equal(got[0], first[0]) and np.array_equal(got[2], first[2])
            assert np.array_equal(got[1], first[1]), f"iterates differ on repeat {i}"
            for a, b in zip(got[3], first[3]):
                assert np.array_equal(a, b)
