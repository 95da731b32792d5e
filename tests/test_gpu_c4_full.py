"""Config 4 at its FULL size (n = 2^22, m = 256) against the live reference.

Golden: tests/golden/make_c4_full.py -- the unmodified reference's
feature_matrix / condition_rows / solve / predict, row-chunked (SURVEY.md
§8(d)), y_hat stored on every 64th grid point.  Inputs are regenerated from the
seed by workloads.linear_batch.  These cases exercise what only exists at
scale: the exp recurrence on the uniform grid, exact-underflow block skipping,
the 145-CTA slab reduce and the kernel-space reassociation, plus the row-shard
split used on N GPUs (slab Grams summed in rank order).
Bar (north star): y_hat within 1e-6 relative L2 of the reference; error vs
y* within 1 % of the reference's.
"""
import numpy as np
import pytest

from conftest import load_golden
from gpu_util import rel_l2

pytestmark = pytest.mark.gpu

YHAT_TOL = 1e-6
ERR_TOL = 0.01


@pytest.fixture(scope="module")
def c4():
    from paper_2510_04094_b200 import workloads as W

    g = load_golden("c4_full")
    cfg = W.CONFIGS[4]
    bt = W.linear_batch(cfg, 0, 1)
    assert int(g["n"]) == cfg.n and float(g["sigma2"]) == cfg.sigma2
    return g, cfg, bt


def _check_yhat(g, cfg, bt, y_dev):
    stride = int(g["stride"])
    y = y_dev.cpu().numpy()
    sub = y[::stride]
    rel = rel_l2(sub, g["yhat_sub"])
    err = rel_l2(y, bt.instances[0].sol(bt.grid))
    ref_err = float(g["err_vs_exact"])
    print(f"c4 full: y_hat rel L2 {rel:.3e} on {sub.size} points; err vs y* {err:.6e} "
          f"(reference {ref_err:.6e})")
    assert rel <= YHAT_TOL, rel
    assert abs(err - ref_err) <= ERR_TOL * ref_err, (err, ref_err)
    # every grid point, not only the stored ones: per-chunk sums of y_hat
    chunk = int(g["chunk"])
    csum = np.add.reduceat(y, np.arange(0, y.size, chunk))
    # Cauchy-Schwarz: |sum_chunk (y - y_ref)| <= sqrt(chunk) ||y - y_ref||_2
    scale = np.sqrt(chunk * g["chunk_sumsq"].sum())
    assert np.all(np.abs(csum - g["chunk_sum"]) <= YHAT_TOL * scale)


def test_c4_full_api_matches_reference(c4):
    """linear.assemble + solve + predict (the drop-in API) at n = 2^22."""
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200.kernel import RbfKernel
    from paper_2510_04094_b200.problems import ivp

    g, cfg, bt = c4
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), bt.landmarks)
    assert fm.m_eff == int(g["m_eff"])
    inst = bt.instances[0]

    class Spec:
        order = cfg.order
        coeffs = inst.coeff_fns()
        forcing = staticmethod(inst.forcing_fn)

    sy = L.assemble(Spec, ivp(inst.conditions()), fm, bt.grid, cfg.gamma)
    mdl = L.solve(sy, fm)
    M = sy.matrix
    Mg = g["M"]
    me = fm.m_eff
    # D^T D block: same basis up to eigenvector signs -> compare the basis-free
    # scalars and the spectrum-invariant norm
    assert abs(M[me, me] - Mg[me, me]) <= 1e-12 * abs(Mg[me, me])         # g^T g
    np.testing.assert_allclose(np.linalg.norm(M[:me, :me]), np.linalg.norm(Mg[:me, :me]),
                               rtol=1e-10)
    rep = L.check_kkt(mdl, sy)
    assert rep.passed, (rep.linear_residual, rep.rhs_scale)
    _check_yhat(g, cfg, bt, mdl.predict_device(0, bt.grid))


def test_c4_full_row_shards_match_reference(c4):
    """The N-GPU split: slab Grams over dist.row_ranges(n_c, 8) summed in rank
    order (what the all-reduce computes), then the KKT solve -- same y_hat."""
    import torch

    from paper_2510_04094_b200 import dist as DI
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200.kernel import RbfKernel
    from paper_2510_04094_b200.problems import ivp

    g, cfg, bt = c4
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), bt.landmarks)
    dev = fm.device
    pts = torch.as_tensor(bt.pts, device=dev)
    coef = torch.as_tensor(bt.coef[0], device=dev)
    forc = torch.as_tensor(bt.forcing[0], device=dev)
    full = L.gram_ext_device(fm, cfg.order, pts, coef, forc)
    for world in (2, 8):
        E = None
        for lo, hi in DI.row_ranges(bt.pts.size, world):
            Er = L.gram_ext_device(fm, cfg.order, pts, coef, forc, lo, hi).clone()
            E = Er if E is None else E + Er
        d = float((E - full).abs().max() / full.abs().max())
        assert d <= 1e-13, (world, d)
    cond = ivp(bt.instances[0].conditions())
    Ac, beta, vals = L.condition_rows(cond, fm)
    sy = L.AssembledSystem(constraint_points=bt.pts, gamma=cfg.gamma, g=None, r=None,
                           coeff_values=None, cond_rows=Ac.reshape(len(cond.entries), -1),
                           cond_bias=beta, cond_values=vals, fmap=fm, order=cfg.order,
                           d_gram=E)
    mdl = L.solve(sy, fm)
    _check_yhat(g, cfg, bt, mdl.predict_device(0, bt.grid))


def test_c4_full_pipeline_matches_reference(c4):
    """SingleSolvePipeline (the bench's c4 path: overlapped eigensolver streams,
    CUDA-graph replay) at n = 2^22, three consecutive calls."""
    import torch

    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200.problems import ivp

    g, cfg, bt = c4
    dev = torch.device("cuda", 0)
    pipe = L.SingleSolvePipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order,
                                 ivp(bt.instances[0].conditions()), device=dev)
    pts = torch.as_tensor(bt.pts, device=dev)
    coef = torch.as_tensor(bt.coef[0], device=dev)
    forc = torch.as_tensor(bt.forcing[0], device=dev)
    xs = []
    for _ in range(3):
        x, info = pipe.run_device(pts, coef, forc)
        xs.append(x.clone())
    torch.cuda.synchronize()
    assert int(info[0]) == 0
    assert all(torch.equal(xs[0], x) for x in xs[1:])
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200.kernel import RbfKernel

    fm = N.NystromFeatureMap(kernel=RbfKernel(cfg.sigma2), landmarks=pipe.landmarks,
                             m_eff=pipe._shape[0], device=dev, d_landmarks=pipe.eig.d_lm,
                             d_W=pipe.eig.W, d_eigvals=pipe.eig.s, d_eigvecs=pipe.eig.V)
    me = fm.m_eff
    y = L.predict_batch(fm, xs[0][:, :me + 1], 0, bt.grid)[0]
    _check_yhat(g, cfg, bt, y)
