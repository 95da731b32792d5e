"""GPU tests of the device pipelines and the reference's error behaviour
(golden fixtures only; the GPU box has no /root/reference)."""
import os

import numpy as np
import pytest

from conftest import load_golden
from gpu_util import conditions, fmap_from_golden, rel_l2

pytestmark = pytest.mark.gpu


def _predict(fm, x, grid):
    from paper_2510_04094_b200 import linear as L
    return L.predict_batch(fm, x, 0, grid).cpu().numpy()


@pytest.mark.parametrize("name", ["c0_seed0", "c1_seed0", "c4_n16384"])
def test_single_pipeline_matches_reference_and_replays(name):
    """SingleSolvePipeline (eig + graph-replayed condition rows / Gram / KKT):
    y_hat within 1e-6 of the reference, and the replayed call reproduces the
    first (eager) call bit for bit."""
    import torch

    from paper_2510_04094_b200 import linear as L
    g = load_golden(name)
    cond = conditions(g, 0)
    pipe = L.SingleSolvePipeline(g["landmarks"], float(g["sigma2"]), g["grid"],
                                 float(g["gamma"]), int(g["order"]), cond)
    pts = torch.as_tensor(g["pts"], device="cuda")
    coef = torch.as_tensor(g["coef"][0], device="cuda")
    forc = torch.as_tensor(g["forcing"][0], device="cuda")
    x1 = pipe.run_device(pts, coef, forc)[0].clone()
    x2 = pipe.run_device(pts, coef, forc)[0].clone()   # captured graph now exists
    x3 = pipe.run_device(pts, coef, forc)[0].clone()   # replay
    assert torch.equal(x1, x2) and torch.equal(x2, x3)
    mdl = pipe.model()
    y = mdl.predict(0, g["grid"])
    assert rel_l2(y, g["yhat"][0]) <= 1e-6
    if name.startswith("c4"):
        # m = 256: the kernel-space Gram ran on the side stream, concurrent with
        # the eigendecomposition; the serial path gives the same model
        assert pipe._kspace
        import os
        os.environ["NYS_KSPACE_OVERLAP"] = "0"
        try:
            serial = L.SingleSolvePipeline(g["landmarks"], float(g["sigma2"]), g["grid"],
                                           float(g["gamma"]), int(g["order"]), cond)
        finally:
            del os.environ["NYS_KSPACE_OVERLAP"]
        assert not serial._kspace
        xs = serial.run_device(pts, coef, forc)[0]
        ys = serial.model().predict(0, g["grid"])
        assert rel_l2(y, ys) <= 1e-12
        assert float(torch.max(torch.abs(xs - x1))) <= 1e-9 * float(torch.max(torch.abs(xs)))


@pytest.mark.parametrize("name", ["c1_seed0", "c4_n16384"])
def test_single_pipeline_rotating_buffers(name):
    """Eigendecompositions on rotating side streams with one buffer set per call
    in flight, inputs alternating between two staging sets (the e2e path):
    every call reproduces the first bit for bit."""
    import torch

    from paper_2510_04094_b200 import linear as L
    g = load_golden(name)
    pipe = L.SingleSolvePipeline(g["landmarks"], float(g["sigma2"]), g["grid"],
                                 float(g["gamma"]), int(g["order"]), conditions(g, 0))
    ins = [tuple(torch.as_tensor(a, device="cuda").clone() for a in
                 (g["pts"], g["coef"][0], g["forcing"][0])) for _ in range(2)]
    xs = [pipe.run_device(*ins[k % 2])[0].clone() for k in range(9)]
    assert len(pipe._eigbufs) == pipe._n_eig_streams() + 1
    assert all(torch.equal(xs[0], x) for x in xs[1:])
    # inputs marked final by an event: the kernel-space Gram (c4) may overlap
    # the previous call's KKT; same results
    ready = torch.cuda.Event()
    ready.record()
    xe = [pipe.run_device(*ins[k % 2], input_event=ready)[0].clone() for k in range(21)]
    assert all(torch.equal(xs[0], x) for x in xe)
    if name.startswith("c4"):   # each set's projection + KKT on the set's own stream
        assert len(pipe._set_streams) == len(pipe._eigbufs)
    if name.startswith("c1"):   # configs 0/1: whole-call graphs, all sets in flight
        assert len(pipe._whole) == 2 and all(len(p) == len(pipe._eigbufs)
                                             for p in pipe._whole.values())


@pytest.mark.parametrize("name", ["c0_seed0", "c1_seed0", "c4_n16384"])
def test_single_pipeline_run_host_matches_run_device(name):
    """run_host (pinned host block in, pinned x out, staging sets in rotation):
    calls alternating between two different right-hand sides, issued back to back
    without synchronising, each return the device path's solution for ITS
    inputs -- a stale or overwritten staging set would give the other one's."""
    import torch

    from paper_2510_04094_b200 import linear as L
    g = load_golden(name)
    pipe = L.SingleSolvePipeline(g["landmarks"], float(g["sigma2"]), g["grid"],
                                 float(g["gamma"]), int(g["order"]), conditions(g, 0))
    forc = [g["forcing"][0], 0.5 * g["forcing"][0] + 1.0]
    want = []
    for f in forc:
        ins = tuple(torch.as_tensor(a, device="cuda") for a in (g["pts"], g["coef"][0], f))
        want.append(pipe.run_device(*ins)[0].cpu().clone())
    assert not torch.equal(want[0], want[1])
    blocks = [pipe.host_block(g["pts"], g["coef"][0], f) for f in forc]
    outs = [torch.empty(want[0].shape, dtype=torch.float64).pin_memory() for _ in range(14)]
    infos = [pipe.run_host(blocks[k % 2], outs[k])[1] for k in range(14)]
    torch.cuda.synchronize()
    assert all(int(i[0]) == 0 for i in infos)
    for k, x in enumerate(outs):
        assert torch.equal(x, want[k % 2]), k
    with pytest.raises(ValueError):
        pipe.run_host(torch.zeros(blocks[0].numel(), dtype=torch.float64), outs[0])


def test_single_pipeline_row_shards_sum_to_full():
    """Row-sharded SingleSolvePipeline (config 4 on N GPUs): the kernel-space
    Grams of two row slabs add up to the single-GPU one (the all-reduce is the
    identity at world size 1, so the slabs are summed here)."""
    import torch

    from paper_2510_04094_b200 import dist as D
    from paper_2510_04094_b200 import linear as L
    g = load_golden("c4_n16384")
    args = (g["landmarks"], float(g["sigma2"]), g["grid"], float(g["gamma"]), int(g["order"]),
            conditions(g, 0))
    ins = tuple(torch.as_tensor(a, device="cuda") for a in (g["pts"], g["coef"][0], g["forcing"][0]))
    full = L.SingleSolvePipeline(*args)
    full.run_device(*ins)
    Ks = []
    for lo, hi in D.row_ranges(g["pts"].size, 2):
        p = L.SingleSolvePipeline(*args, rows=(lo, hi))
        assert p._n_eig_streams() == 2   # two 8-SM cluster eigensolvers in flight
        p._kspace_launch(*ins)
        torch.cuda.synchronize()
        Ks.append(p._kcur.clone())
    torch.cuda.synchronize()
    Kf = full._kcur
    scale = float(torch.max(torch.abs(Kf)))
    assert float(torch.max(torch.abs(Ks[0] + Ks[1] - Kf))) <= 1e-12 * scale


def test_shared_pipeline_host_staging_rotation():
    """SharedGridPipeline.run_host with two device staging sets in rotation
    (this call's H2D overlaps the previous call's solve) == run_device."""
    import torch

    from paper_2510_04094_b200 import batch as BT
    g = load_golden("c2_seed0_i0-7")
    cond = conditions(g, 0)
    pipe = BT.SharedGridPipeline(g["landmarks"], float(g["sigma2"]), g["grid"],
                                 float(g["gamma"]), 2, cond, 8)
    coef = torch.as_tensor(g["coef"], device="cuda")
    forc = torch.as_tensor(g["forcing"], device="cuda")
    vals = torch.as_tensor(g["cond_values"], device="cuda")
    xd = pipe.run_device(coef, forc, vals)[0].cpu()
    side = xd.shape[1]
    hs = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
          for a in (g["coef"], g["forcing"], g["cond_values"])]
    bufs = [(torch.empty_like(coef), torch.empty_like(forc), torch.empty_like(vals),
             torch.empty((8, side), dtype=torch.float64, device="cuda"),
             torch.empty(8, dtype=torch.int32, device="cuda")) for _ in range(2)]
    for _ in range(3):
        x_h = torch.empty((8, side), dtype=torch.float64).pin_memory()
        i_h = torch.empty(8, dtype=torch.int32).pin_memory()
        pipe.run_host(*hs, x_h, i_h, chunks=2, dev_bufs=bufs)
        torch.cuda.synchronize()
        assert (i_h.numpy() == 0).all()
        assert torch.equal(x_h, xd)


def test_shared_pipeline_graph_equals_eager():
    import torch

    from paper_2510_04094_b200 import batch as BT
    g = load_golden("c2_seed0_i0-7")
    cond = conditions(g, 0)
    coef = torch.as_tensor(g["coef"], device="cuda")
    forc = torch.as_tensor(g["forcing"], device="cuda")
    vals = torch.as_tensor(g["cond_values"], device="cuda")
    pipe = BT.SharedGridPipeline(g["landmarks"], float(g["sigma2"]), g["grid"],
                                 float(g["gamma"]), 2, cond, 8)
    xs = [pipe.run_device(coef, forc, vals)[0].clone() for _ in range(3)]
    os.environ["NYS_GRAPHS"] = "0"
    try:
        xe = pipe.run_device(coef, forc, vals)[0].clone()
    finally:
        del os.environ["NYS_GRAPHS"]
    assert all(torch.equal(xs[0], x) for x in xs[1:] + [xe])
    fm = pipe.solver.fmap
    Y = _predict(fm, xs[0], g["grid"])
    for b in range(8):
        assert rel_l2(Y[b], g["yhat"][b]) <= 1e-6


def test_blocked_kkt_matches_scalar_cholesky():
    """kkt_block.cu (DMMA-blocked omega Cholesky + Schur) against the scalar
    whole-H Cholesky on the same Grams: the same solutions to 1e-9 in y_hat."""
    import torch

    from paper_2510_04094_b200 import batch as BT
    g = load_golden("c2_seed0_i0-7")
    fm = fmap_from_golden(g)
    solver = BT.LinearBatchSolver(fm, g["grid"], float(g["gamma"]), 2, conditions(g, 0), 8)
    xb, ib = solver.solve(g["coef"], g["forcing"], g["cond_values"])
    xb = xb.clone()
    os.environ["NYS_KKT_SCALAR"] = "1"
    try:
        xs, is_ = solver.solve(g["coef"], g["forcing"], g["cond_values"])
    finally:
        del os.environ["NYS_KKT_SCALAR"]
    assert (ib.cpu().numpy() == 0).all() and (is_.cpu().numpy() == 0).all()
    Yb = _predict(fm, xb, g["grid"])
    Ys = _predict(fm, xs, g["grid"])
    for b in range(8):
        assert rel_l2(Yb[b], Ys[b]) <= 1e-9


def test_large_kkt_cholesky_matches_lu():
    """kkt_big.cu (c4-shaped side 259) against the reference's LU (kkt.cu)."""
    from gpu_util import solve_golden_instance

    g = load_golden("c4_n16384")
    fm = fmap_from_golden(g)
    _, m_chol = solve_golden_instance(g, fm, 0)
    os.environ["NYS_KKT_LU"] = "1"
    try:
        _, m_lu = solve_golden_instance(g, fm, 0)
    finally:
        del os.environ["NYS_KKT_LU"]
    y1 = m_chol.predict(0, g["grid"])
    y2 = m_lu.predict(0, g["grid"])
    assert rel_l2(y1, y2) <= 1e-10
    assert rel_l2(y1, g["yhat"][0]) <= 1e-6


@pytest.mark.parametrize("name", ["c0_seed0", "c1_seed0", "cat_p12", "cat_p16"])
def test_small_kkt_cholesky_matches_lu(name):
    """Single small systems (one CTA: Cholesky + Schur, kkt_chol.cu) against
    the reference's LU on the same assembled system; P12 / P16 are a BVP and a
    fourth-order problem (more conditions, other side lengths)."""
    from gpu_util import solve_golden_instance

    g = load_golden(name)
    fm = fmap_from_golden(g)
    _, m_chol = solve_golden_instance(g, fm, 0)
    os.environ["NYS_KKT_LU"] = "1"
    try:
        _, m_lu = solve_golden_instance(g, fm, 0)
    finally:
        del os.environ["NYS_KKT_LU"]
    y1 = m_chol.predict(0, g["grid"])
    y2 = m_lu.predict(0, g["grid"])
    assert rel_l2(y1, y2) <= 1e-9
    assert rel_l2(y1, g["yhat"][0]) <= 1e-6


def test_singular_system_raises():
    """Two identical conditions make M singular: linear.solve raises
    SingularSystemError like linear.py:148-151 (and so does the batch path)."""
    from gpu_util import ArraySpec

    from paper_2510_04094_b200 import batch as BT
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200.problems import BoundaryCondition, Conditions
    g = load_golden("c0_seed0")
    fm = fmap_from_golden(g)
    bc = BoundaryCondition(float(g["cond_points"][0]), int(g["cond_orders"][0]),
                           float(g["cond_values"][0][0]))
    cond = Conditions("ivp", (bc, bc))
    spec = ArraySpec(int(g["order"]), g["coef"][0], g["forcing"][0], g["pts"])
    sy = L.assemble(spec, cond, fm, g["grid"], float(g["gamma"]))
    with pytest.raises(L.SingularSystemError):
        L.solve(sy, fm)
    solver = BT.LinearBatchSolver(fm, g["grid"], float(g["gamma"]), int(g["order"]), cond, 2)
    vals = np.array([[bc.value, bc.value]] * 2)
    _, info = solver.solve(np.stack([g["coef"][0]] * 2), np.stack([g["forcing"][0]] * 2), vals)
    info = info.cpu().numpy()
    assert (info != 0).all()
    with pytest.raises(L.SingularSystemError):
        L.raise_for_info(int(info[0]))


def test_degenerate_landmarks_and_bad_arguments_raise():
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200.kernel import RbfKernel
    with pytest.raises(N.DegenerateLandmarksError):
        N.build_feature_map(RbfKernel(0.01), np.array([0.0, 0.5, 0.5, 1.0]))
    with pytest.raises(ValueError):
        N.build_feature_map(RbfKernel(0.01), np.linspace(0, 1, 5), drop_tol=1.5)
    g = load_golden("c0_seed0")
    fm = fmap_from_golden(g)
    from gpu_util import ArraySpec
    spec = ArraySpec(int(g["order"]), g["coef"][0], g["forcing"][0], g["pts"])
    with pytest.raises(ValueError):
        L.assemble(spec, conditions(g, 0), fm, g["grid"], 0.0)
    bad = g["forcing"][0].copy()
    bad[3] = np.nan
    spec_bad = ArraySpec(int(g["order"]), g["coef"][0], bad, g["pts"])
    with pytest.raises(FloatingPointError):
        L.assemble(spec_bad, conditions(g, 0), fm, g["grid"], float(g["gamma"]))
