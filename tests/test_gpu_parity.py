"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the oracle.  Bar: y_hat within 1e-6 relative L2 of the reference
(north star), error vs the manufactured solution within 1 % of the reference's."""
import numpy as np
import pytest

from conftest import load_golden
from gpu_util import conditions, fmap_from_golden, rel_l2, solve_golden_instance
from oracle import nys_port as O

pytestmark = pytest.mark.gpu

YHAT_TOL = 1e-6          # north star: relative L2 of y_hat vs the reference
ERR_TOL = 0.01           # north star: error vs y* within 1 % of the reference's


@pytest.mark.parametrize("name", ["c0_seed0", "c1_seed0", "c2_seed0_i0-7", "cat_p2", "cat_p12",
                                  "cat_p16", "c4_n16384"])
def test_eigendecomposition_matches_reference(name):
    g = load_golden(name)
    fm = fmap_from_golden(g)
    ref = g["eigvals"]
    if not name.startswith("cat"):
        assert fm.m_eff == int(g["m_eff"])
    else:   # catalog spectra run into the 1e-16 noise floor: m_eff may shift a little
        assert abs(fm.m_eff - int(g["m_eff"])) <= 5, (fm.m_eff, int(g["m_eff"]))
    assert fm._host["sweeps"] < 30 * fm.m, fm._host["sweeps"]   # QL iterations
    k = min(fm.m_eff, ref.size)
    np.testing.assert_allclose(fm.eigenvalues[:k], ref[:k], rtol=0, atol=1e-13 * ref[0])
    V = fm.eigenvectors
    np.testing.assert_allclose(V.T @ V, np.eye(fm.m_eff), atol=1e-12)


@pytest.mark.parametrize("name", ["c0_seed0", "c1_seed0", "cat_p2", "cat_p12", "cat_p16",
                                  "c4_n16384"])
def test_linear_solve_matches_reference(name):
    g = load_golden(name)
    fm = fmap_from_golden(g)
    sy, model = solve_golden_instance(g, fm, 0)
    y = model.predict(0, g["grid"])
    assert rel_l2(y, g["yhat"][0]) <= YHAT_TOL
    if "err_vs_exact" in g:
        from paper_2510_04094_b200 import workloads as W
        cid = int(name[1])
        cfg = W.CONFIGS[cid] if cid != 4 else W.scaled(W.CONFIGS[4], n=g["grid"].size)
        ys = W.instance(cid, 0, 0, cfg).sol(g["grid"])
        err = rel_l2(y, ys)
        assert abs(err - g["err_vs_exact"][0]) <= ERR_TOL * g["err_vs_exact"][0]


@pytest.mark.parametrize("name", ["c0_seed0", "c1_seed0", "cat_p16"])
def test_fused_gram_matches_oracle_same_basis(name):
    """With the device's own W, E from the fused kernel equals the oracle's
    [D g r]^T [D g r] built with the reference's operation order."""
    g = load_golden(name)
    fm = fmap_from_golden(g)
    Wd = fm.d_W[:, :fm.m_eff].cpu().numpy()
    sy, _ = solve_golden_instance(g, fm, 0)
    E = sy.d_gram.cpu().numpy()
    osy = O.assemble(int(g["order"]), list(g["coef"][0]), g["forcing"][0],
                     [(float(t), int(o), float(v)) for t, o, v in
                      zip(g["cond_points"], g["cond_orders"], g["cond_values"][0])],
                     g["grid"], float(g["gamma"]), float(g["sigma2"]), g["landmarks"], Wd,
                     kind=str(g["kind"]))
    Dx = np.column_stack([osy["D"], osy["g"], osy["r"]])
    Eo = Dx.T @ Dx
    scale = np.abs(Dx).max(axis=0)
    den = np.outer(scale, scale) * Dx.shape[0]
    err = np.abs(E - Eo)
    assert np.all(err[den == 0] == 0)
    rel = err[den > 0] / den[den > 0]
    assert rel.max() <= 1e-8   # 4th-order (P16) polynomials cancel more
    # the assembled KKT matrix (linear.py:123-133 layout) equals the oracle's
    M = sy.matrix
    np.testing.assert_allclose(M, osy["M"], rtol=0, atol=1e-9 * np.abs(osy["M"]).max())


@pytest.mark.parametrize("name", ["c0_seed0", "c1_seed0", "cat_p12", "c4_n16384"])
def test_kkt_solve_matches_lapack(name):
    """Device LU + refinement vs LAPACK dgesv on the SAME assembled M: the
    reference's backward-stability bound (reference tests/test_linear.py:79-86)
    and identical predictions.  (x itself may differ in its ill-conditioned
    directions -- cond(M) reaches 1e15 -- without moving y_hat.)"""
    from paper_2510_04094_b200 import linear as L
    g = load_golden(name)
    fm = fmap_from_golden(g)
    sy, model = solve_golden_instance(g, fm, 0)
    M, rhs = sy.matrix, sy.rhs
    x_ref = np.linalg.solve(M, rhs)
    x_ref = x_ref + np.linalg.solve(M, rhs - M @ x_ref)
    x = np.concatenate([model.omega, [model.bias], model.multipliers])
    assert np.max(np.abs(M @ x - rhs)) <= 1e-8 * max(np.abs(rhs).max(), 1.0)
    me = fm.m_eff
    ref_model = L.PrimalModel(x_ref[:me], float(x_ref[me]), x_ref[me + 1:], fm)
    assert rel_l2(model.predict(0, g["grid"]), ref_model.predict(0, g["grid"])) <= 1e-8


def test_check_kkt_certificate():
    from paper_2510_04094_b200 import linear as L
    g = load_golden("cat_p2")
    fm = fmap_from_golden(g)
    sy, model = solve_golden_instance(g, fm, 0)
    rep = L.check_kkt(model, sy)
    assert rep.passed
    # the certificate's e = D w + g b - r (linear.py:175-189) against D assembled
    # by the oracle restatement (linear.py:90-137) in the device's own basis W
    # (so the comparison isolates the fused residual kernel, not the basis)
    W = fm.d_W.cpu().numpy()[:, :fm.m_eff]
    cond = [(float(t), int(o), float(v)) for t, o, v in
            zip(g["cond_points"], g["cond_orders"], g["cond_values"][0])]
    orc = O.assemble(int(g["order"]), list(g["coef"][0]), g["forcing"][0], cond, g["grid"],
                     float(g["gamma"]), float(g["sigma2"]), g["landmarks"], W, str(g["kind"]))
    e_ref = orc["D"] @ model.omega + orc["g"] * model.bias - orc["r"]
    np.testing.assert_allclose(rep.ode_residuals, e_ref,
                               atol=1e-9 * max(1.0, np.abs(orc["r"]).max()))


def test_batch_config2_matches_reference():
    from paper_2510_04094_b200 import batch as BT
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import workloads as W
    g = load_golden("c2_seed0_i0-7")
    fm = fmap_from_golden(g)
    solver = BT.LinearBatchSolver(fm, g["grid"], float(g["gamma"]), 2, conditions(g, 0), 8)
    x, info = solver.solve(g["coef"], g["forcing"], g["cond_values"])
    assert (info.cpu().numpy() == 0).all()
    Y = L.predict_batch(fm, x, 0, g["grid"]).cpu().numpy()
    cfg = W.CONFIGS[2]
    for b in range(8):
        assert rel_l2(Y[b], g["yhat"][b]) <= YHAT_TOL
        ys = W.instance(2, 0, b, cfg).sol(g["grid"])
        err = rel_l2(Y[b], ys)
        assert abs(err - g["err_vs_exact"][b]) <= ERR_TOL * g["err_vs_exact"][b]
    # batch Gram == single-instance fused Gram for the same instance
    E = solver.gram_ext(L._lib.as_f64(g["coef"], fm.device), L._lib.as_f64(g["forcing"], fm.device))
    sy, _ = solve_golden_instance(g, fm, 3)
    E1 = sy.d_gram.cpu().numpy()
    scale = np.abs(E1).max()
    np.testing.assert_allclose(E[3].cpu().numpy(), E1, rtol=0, atol=1e-9 * scale)


@pytest.mark.parametrize("name", ["c1_seed0", "c4_n16384"])
def test_row_range_partials_sum_to_full_gram(name):
    """Row sharding contract of nys_fused_gram_f64 (dist.py): partial extended
    Grams over disjoint row slabs add up to the full one."""
    from paper_2510_04094_b200 import dist as D
    from paper_2510_04094_b200 import linear as L
    g = load_golden(name)
    fm = fmap_from_golden(g)
    dev = fm.device
    pts = L._lib.as_f64(g["pts"], dev)
    coef = L._lib.as_f64(g["coef"][0], dev)
    forc = L._lib.as_f64(g["forcing"][0], dev)
    full = L.gram_ext_device(fm, int(g["order"]), pts, coef, forc).cpu().numpy()
    parts = sum(L.gram_ext_device(fm, int(g["order"]), pts, coef, forc, lo, hi).cpu().numpy()
                for lo, hi in D.row_ranges(g["pts"].size, 3))
    np.testing.assert_allclose(parts, full, rtol=0, atol=1e-11 * np.abs(full).max())


@pytest.mark.parametrize("uniform", [False, True])
@pytest.mark.parametrize("m", [80, 94, 134, 150, 256])
def test_large_m_kspace_gram_matches_oracle(m, uniform):
    """Large-m kernel (gram_large.cu) for every super-block shape: NB % 4 in
    {3, 0, 1 (stub + corner), 3, 1} -- E = W_ext^T [G g r]^T [G g r] W_ext
    with G built by the oracle's rbf_block (kernel.py:75-92).  Random points
    take the per-entry exp() path, a linspace grid the exp recurrence."""
    import torch

    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200.kernel import RbfKernel

    sigma2, p, n = 0.25, 2, 3001
    rng = np.random.default_rng(m)
    lm = np.linspace(0.0, 0.39 * (m - 1), m)
    pts = np.sort(rng.uniform(lm[0], lm[-1], n))
    if uniform:
        pts = np.linspace(lm[0] - 0.3, lm[-1] + 0.2, n)
    coef = rng.normal(size=(p, n))
    forcing = rng.normal(size=n)
    fm = N.build_feature_map(RbfKernel(sigma2), lm)
    assert fm.m_eff == m and fm.condition < L.KSPACE_MAX_COND
    E = L.gram_ext_device(fm, p, torch.as_tensor(pts, device="cuda"),
                          torch.as_tensor(coef, device="cuda"),
                          torch.as_tensor(forcing, device="cuda")).cpu().numpy()
    G = O.rbf_block(sigma2, p, lm, pts).T.copy()
    for k in range(1, p + 1):
        G -= coef[k - 1][:, None] * O.rbf_block(sigma2, p - k, lm, pts).T
    X = np.column_stack([G, -coef[p - 1], forcing])
    K = X.T @ X
    Wd = fm.d_W[:, :m].cpu().numpy()
    Wx = np.zeros((m + 2, m + 2))
    Wx[:m, :m] = Wd
    Wx[m, m] = Wx[m + 1, m + 1] = 1.0
    Eo = Wx.T @ K @ Wx
    assert np.allclose(E, E.T, rtol=0, atol=0)
    np.testing.assert_allclose(E, Eo, rtol=0, atol=1e-11 * np.abs(Eo).max())


@pytest.mark.parametrize("sigma", [0.25, 0.3, 0.35, 0.4, 0.45, 0.5, 0.55, 0.6])
def test_kspace_gram_every_window_width(sigma):
    """Kernel-space Gram at m = 256 with the live window swept through every
    width (sigma 0.25 .. 0.6 on landmarks 0.39 apart: ~6 .. 13 live blocks per
    CTA), so each ragged super-tile pattern of large_kspace_kernel (4 x n and
    n x n edge tiles, n = 1..3, each with its own unpredicated DMMA loop) is the
    one that runs somewhere; uniform grid (exp recurrence), three row tiles per
    CTA.  Checked against G built by the oracle's rbf_block (kernel.py:75-92)."""
    import torch

    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200.kernel import RbfKernel

    m, p, n = 256, 2, 148 * 32 * 3 + 5
    sigma2 = sigma * sigma
    rng = np.random.default_rng(int(sigma * 100))
    lm = np.linspace(0.0, 0.39 * (m - 1), m)
    pts = np.linspace(lm[0] - 0.1, lm[-1] + 0.1, n)
    coef = rng.normal(size=(p, n))
    forcing = rng.normal(size=n)
    fm = N.build_feature_map(RbfKernel(sigma2), lm)
    assert fm.m_eff == m and fm.condition < L.KSPACE_MAX_COND
    E = L.gram_ext_device(fm, p, torch.as_tensor(pts, device="cuda"),
                          torch.as_tensor(coef, device="cuda"),
                          torch.as_tensor(forcing, device="cuda")).cpu().numpy()
    G = O.rbf_block(sigma2, p, lm, pts).T.copy()
    for k in range(1, p + 1):
        G -= coef[k - 1][:, None] * O.rbf_block(sigma2, p - k, lm, pts).T
    X = np.column_stack([G, -coef[p - 1], forcing])
    K = X.T @ X
    Wx = np.zeros((m + 2, m + 2))
    Wx[:m, :m] = fm.d_W[:, :m].cpu().numpy()
    Wx[m, m] = Wx[m + 1, m + 1] = 1.0
    Eo = Wx.T @ K @ Wx
    assert np.allclose(E, E.T, rtol=0, atol=0)
    np.testing.assert_allclose(E, Eo, rtol=0, atol=1e-11 * np.abs(Eo).max())


@pytest.mark.parametrize("case", ["n300", "n500", "sparse"])
def test_kspace_gram_coarse_uniform_grids(case):
    """Uniform grids that are coarse against sigma: the exp recurrence of
    large_kspace_kernel (e_j = e_A rho_A^j Q^{j(j-1)/2}) would overflow rho_A^j
    within one anchor period (h / sigma = 0.67 at n = 300 gave NaN), so those
    row ranges must take the exp()-per-entry path (rec_span_ok).  "sparse": a
    long domain with landmarks 23 sigma apart and five row tiles per CTA."""
    import torch

    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200.kernel import RbfKernel

    sigma2, p = 0.25, 2
    if case == "sparse":
        m, n = 80, 148 * 32 * 5
        lm = np.linspace(0.0, 924.0, m)
    else:
        m, n = 256, int(case[1:])
        lm = np.linspace(0.0, 0.39 * (m - 1), m)
    rng = np.random.default_rng(n)
    pts = np.linspace(lm[0] - 0.1, lm[-1] + 0.1, n)
    coef = rng.normal(size=(p, n))
    forcing = rng.normal(size=n)
    fm = N.build_feature_map(RbfKernel(sigma2), lm)
    assert fm.m_eff == m and fm.condition < L.KSPACE_MAX_COND
    E = L.gram_ext_device(fm, p, torch.as_tensor(pts, device="cuda"),
                          torch.as_tensor(coef, device="cuda"),
                          torch.as_tensor(forcing, device="cuda")).cpu().numpy()
    G = O.rbf_block(sigma2, p, lm, pts).T.copy()
    for k in range(1, p + 1):
        G -= coef[k - 1][:, None] * O.rbf_block(sigma2, p - k, lm, pts).T
    X = np.column_stack([G, -coef[p - 1], forcing])
    K = X.T @ X
    Wx = np.zeros((m + 2, m + 2))
    Wx[:m, :m] = fm.d_W[:, :m].cpu().numpy()
    Wx[m, m] = Wx[m + 1, m + 1] = 1.0
    Eo = Wx.T @ K @ Wx
    assert np.isfinite(E).all()
    np.testing.assert_allclose(E, Eo, rtol=0, atol=1e-11 * np.abs(Eo).max())


def test_kspace_gram_random_shapes():
    """Kernel-space Gram against the oracle on 40 seeded random shapes: m in
    71..256 (equidistant or jittered landmarks), p in {1, 2}, sigma 0.2..3
    landmark spacings, n from 97 to 60000 rows, uniform grids (exp recurrence
    where its range check allows it: h / sigma runs from 8e-4 to 4.7) and random
    points (exp per entry).  Shapes outside the kernel-space gate (m_eff < m or
    cond(Omega) > 1e6) are skipped; at least 30 must remain."""
    import torch

    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200.kernel import RbfKernel

    rng = np.random.default_rng(12345)
    checked = 0
    for case in range(40):
        m, p = int(rng.integers(71, 257)), int(rng.integers(1, 3))
        spacing = float(rng.uniform(0.05, 3.0))
        sigma = float(rng.uniform(0.6, 3.0)) * spacing * rng.choice([1.0, 0.3])
        n = int(rng.choice([97, 300, 1000, 5000, 20000, 60000]))
        uniform = bool(rng.integers(0, 2))
        lm = np.linspace(0.0, spacing * (m - 1), m)
        if rng.integers(0, 2):
            lm = np.sort(lm + rng.uniform(-0.2, 0.2, m) * spacing)
        pts = (np.linspace(lm[0] - 0.3 * spacing, lm[-1] + 0.2 * spacing, n) if uniform
               else np.sort(rng.uniform(lm[0], lm[-1], n)))
        coef, forcing = rng.normal(size=(p, n)), rng.normal(size=n)
        sigma2 = sigma * sigma
        fm = N.build_feature_map(RbfKernel(sigma2), lm)
        if fm.m_eff != m or fm.condition >= L.KSPACE_MAX_COND:
            continue
        E = L.gram_ext_device(fm, p, torch.as_tensor(pts, device="cuda"),
                              torch.as_tensor(coef, device="cuda"),
                              torch.as_tensor(forcing, device="cuda")).cpu().numpy()
        G = O.rbf_block(sigma2, p, lm, pts).T.copy()
        for k in range(1, p + 1):
            G -= coef[k - 1][:, None] * O.rbf_block(sigma2, p - k, lm, pts).T
        X = np.column_stack([G, -coef[p - 1], forcing])
        K = X.T @ X
        Wx = np.zeros((m + 2, m + 2))
        Wx[:m, :m] = fm.d_W[:, :m].cpu().numpy()
        Wx[m, m] = Wx[m + 1, m + 1] = 1.0
        Eo = Wx.T @ K @ Wx
        assert np.isfinite(E).all(), (case, m, p, n, uniform)
        np.testing.assert_allclose(E, Eo, rtol=0, atol=1e-11 * np.abs(Eo).max(),
                                   err_msg=f"case {case}: m={m} p={p} n={n} uniform={uniform}")
        checked += 1
    assert checked >= 30


def test_fused_gram_random_shapes():
    """Fused feature + Gram kernel (m_eff + 2 <= 72, configs 0/1) against the
    oracle on 48 seeded random shapes: m 2..70, order 1..3, n from 3 to 20000
    rows (uniform or random points, some outside the landmark span),
    cond(Omega) up to ~1e6.  E = [D g r]^T [D g r] with D from the oracle's
    rbf_block (kernel.py:75-92, linear.py:103-114) in the device's basis W."""
    import torch

    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200.kernel import RbfKernel

    rng = np.random.default_rng(777)
    checked = 0
    for case in range(48):
        m, p = int(rng.integers(2, 71)), int(rng.integers(1, 4))
        spacing = float(rng.uniform(0.02, 1.0))
        sigma = float(rng.uniform(0.4, 2.5)) * spacing
        n = int(rng.choice([3, 9, 33, 100, 999, 4097, 20000]))
        lm = np.linspace(0.0, spacing * (m - 1), m)
        pts = (np.sort(rng.uniform(lm[0] - spacing, lm[-1] + spacing, n)) if rng.integers(0, 2)
               else np.linspace(lm[0], lm[-1] + spacing, n))
        coef, forcing = rng.normal(size=(p, n)), rng.normal(size=n)
        sigma2 = sigma * sigma
        fm = N.build_feature_map(RbfKernel(sigma2), lm)
        me = fm.m_eff
        if me + 2 > 72:
            continue
        E = L.gram_ext_device(fm, p, torch.as_tensor(pts, device="cuda"),
                              torch.as_tensor(coef, device="cuda"),
                              torch.as_tensor(forcing, device="cuda")).cpu().numpy()
        W = fm.d_W[:, :me].cpu().numpy()
        Psi = [O.rbf_block(sigma2, ell, lm, pts).T @ W for ell in range(p + 1)]
        D = Psi[p].copy()
        for k in range(1, p + 1):
            D -= coef[k - 1][:, None] * Psi[p - k]
        X = np.column_stack([D, -coef[p - 1], forcing])
        Eo = X.T @ X
        assert np.isfinite(E).all(), (case, m, p, n)
        np.testing.assert_allclose(E, Eo, rtol=0, atol=1e-10 * np.abs(Eo).max(),
                                   err_msg=f"case {case}: m={m} m_eff={me} p={p} n={n}")
        checked += 1
    assert checked >= 40


def test_batch_solver_random_shapes():
    """LinearBatchSolver (batched Gram + KKT, config 2's path) on 16 seeded random
    shapes -- m 8..70 (every m_eff class: the DMMA-blocked KKT for multiples of
    8, the packed Cholesky otherwise, a dropped eigenpair), n 65..4096, B 1..150,
    sigma 0.05..0.3, gamma 1e6..1e9: y_hat of the first, middle and last instance
    within 1e-6 of the oracle restatement (observed <= 4e-10), same m_eff, info 0."""
    from paper_2510_04094_b200 import batch as BT
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200 import workloads as W
    from paper_2510_04094_b200.kernel import RbfKernel
    from paper_2510_04094_b200.problems import ivp

    rng = np.random.default_rng(2024)
    for case in range(16):
        m = int(rng.integers(8, 71))
        n = int(rng.choice([65, 257, 1000, 2049, 4096]))
        B = int(rng.choice([1, 3, 8, 17, 64, 150]))
        sigma = float(rng.choice([0.05, 0.1, 0.15, 0.2, 0.3]))
        gamma = float(rng.choice([1e6, 1e8, 1e9]))
        cfg = W.scaled(W.CONFIGS[2], n=n, m=m, batch=B, sigma=sigma, gamma=gamma)
        bt = W.linear_batch(cfg, seed=case)
        fm = N.build_feature_map(RbfKernel(cfg.sigma2), bt.landmarks)
        cond = ivp([(t, int(o), 0.0) for t, o in zip(bt.cond_points, bt.cond_orders)])
        solver = BT.LinearBatchSolver(fm, bt.grid, cfg.gamma, cfg.order, cond, cfg.batch)
        x, info = solver.solve(bt.coef, bt.forcing, bt.cond_values)
        Y = L.predict_batch(fm, x, 0, bt.grid).cpu().numpy()
        assert (info.cpu().numpy() == 0).all(), case
        for b in sorted({0, B // 2, B - 1}):
            ref = O.solve_linear_instance(cfg.order, list(bt.coef[b]), bt.forcing[b],
                                          bt.instances[b].conditions(), bt.grid, cfg.gamma,
                                          cfg.sigma2, cfg.m)
            assert ref["m_eff"] == fm.m_eff, (case, ref["m_eff"], fm.m_eff)
            yref = O.predict(cfg.sigma2, ref["landmarks"], ref["W"], ref["omega"], ref["bias"],
                             0, bt.grid)
            err = O.rel_l2(Y[b], yref)
            assert err <= 1e-6, f"case {case} (m={m} n={n} B={B} sigma={sigma}): {err:.2e}"


def test_solve_many_callables_match_array_batch():
    """Reference-style callables through solve_many (host sampling on the thread
    pool) give the same solutions as the array batch entry."""
    from paper_2510_04094_b200 import batch as BT
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200 import workloads as W
    from paper_2510_04094_b200.kernel import RbfKernel
    from paper_2510_04094_b200.problems import BoundaryCondition, Conditions, LinearOdeSpec

    cfg = W.scaled(W.CONFIGS[2], n=1025, batch=200)
    bt = W.linear_batch(cfg, seed=0)
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), bt.landmarks)
    specs = [LinearOdeSpec(2, inst.coeff_fns(), inst.forcing_fn, inst.domain)
             for inst in bt.instances]
    conds = [Conditions("ivp", tuple(BoundaryCondition(*c) for c in inst.conditions()))
             for inst in bt.instances]
    models = BT.solve_many(specs, conds, fm, bt.grid, cfg.gamma)
    solver = BT.LinearBatchSolver(fm, bt.grid, cfg.gamma, cfg.order, conds[0], cfg.batch)
    x, info = solver.solve(bt.coef, bt.forcing, bt.cond_values)
    x = x.cpu().numpy()
    assert (info.cpu().numpy() == 0).all()
    for b in (0, 77, 199):
        np.testing.assert_array_equal(models[b].omega, x[b, :fm.m_eff])
