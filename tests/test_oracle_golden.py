"""Pin the CPU oracle (oracle/) against golden vectors produced by the live
reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import newton_port as NP
from oracle import nys_port as O
from paper_2510_04094_b200 import workloads as W
from conftest import load_golden

LINEAR = ["c0_seed0", "c1_seed0", "c2_seed0_i0-7", "c4_n16384", "cat_p2", "cat_p12", "cat_p16"]


def _cond(g, b):
    return [(float(t), int(o), float(v)) for t, o, v in
            zip(g["cond_points"], g["cond_orders"], g["cond_values"][b])]


@pytest.mark.parametrize("name", LINEAR)
def test_oracle_reproduces_reference(name):
    g = load_golden(name)
    s, v = O.eig_landmarks(float(g["sigma2"]), g["landmarks"])
    assert s.size == int(g["m_eff"])
    np.testing.assert_allclose(s, g["eigvals"], rtol=0, atol=1e-13 * g["eigvals"][0])
    Wb = O.scaled_basis(s, v)
    grid = g["grid"]
    kind = str(g["kind"])
    nb = g["coef"].shape[0]
    for b in range(min(nb, 3)):
        coef = list(g["coef"][b])
        sy = O.assemble(int(g["order"]), coef, g["forcing"][b], _cond(g, b), grid,
                        float(g["gamma"]), float(g["sigma2"]), g["landmarks"], Wb, kind=kind)
        np.testing.assert_allclose(sy["M"], g["M"][b], rtol=1e-12, atol=1e-12 * np.abs(g["M"][b]).max())
        x = O.solve_kkt(sy["M"], sy["rhs"])
        me = Wb.shape[1]
        y = O.predict(float(g["sigma2"]), g["landmarks"], Wb, x[:me], x[me], 0, grid)
        assert O.rel_l2(y, g["yhat"][b]) <= 1e-12


def test_oracle_newton_reproduces_reference():
    g = load_golden("c3_seed0_i0-3")
    cfg = W.CONFIGS[3]
    s, v = O.eig_landmarks(float(g["sigma2"]), g["landmarks"])
    Wb = O.scaled_basis(s, v)
    for j, idx in enumerate(g["indices"][:2]):
        inst = W.instance(3, 0, int(idx))
        spec = NP.NlSpec(1, inst.rhs, (inst.rhs_y,), {(0, 0): inst.rhs_yy})
        try:
            x, tr = NP.solve_nonlinear(spec, inst.conditions(), g["grid"], cfg.gamma, cfg.sigma2,
                                       g["landmarks"], Wb, max_iters=cfg.newton_max_iters)
        except NP.MaxIters as exc:
            x, tr = exc.x, exc.trace
        me = Wb.shape[1]
        y = O.predict(cfg.sigma2, g["landmarks"], Wb, x[:me], x[me], 0, g["grid"])
        assert O.rel_l2(y, g["yhat"][j]) <= 1e-9
        np.testing.assert_allclose(tr.norms, g[f"norms_{j}"], rtol=1e-6)


def test_kernel_known_answers():
    # kernel.py closed forms (tests/test_kernel.py:11-56 of the reference)
    assert O.rbf_block(1.0, 0, [0.0], [0.0])[0, 0] == 1.0
    assert abs(O.rbf_block(1.0, 0, [1.0], [0.0])[0, 0] - np.exp(-1.0)) <= 1e-15
    assert abs(O.rbf_block(10.0, 0, [2.0], [-1.0])[0, 0] - np.exp(-0.9)) <= 1e-15
    assert O.rbf_block(1.0, 1, [0.3], [0.3])[0, 0] == 0.0
    assert abs(O.rbf_block(1.0, 2, [0.0], [0.0])[0, 0] + 2.0) <= 1e-15
    assert abs(O.rbf_block(1.0, 4, [1.0], [0.0])[0, 0] - (16 - 48 + 12) * np.exp(-1.0)) <= 1e-13
    np.testing.assert_allclose(O.hermite_coeffs(2.0, 2), [-1.0, 0.0, 1.0])


def test_two_landmark_eigenvalues():
    s, _ = O.eig_landmarks(1.0, [0.0, 1.0])
    c = np.exp(-1.0)
    np.testing.assert_allclose(s, [1 + c, 1 - c], rtol=1e-12)


def test_oracle_newton2_reproduces_reference():
    """Second-order Newton (p = 2): the oracle port against the live reference's
    golden (tests/golden/make_newton2.py) -- pins the oracle for newton2.cu."""
    g = load_golden("n2_seed0_i0-5")
    s, v = O.eig_landmarks(float(g["sigma2"]), g["landmarks"])
    Wb = O.scaled_basis(s, v)
    for j, idx in enumerate(g["indices"][:2]):
        inst = W.nonlinear2_instance(0, int(idx))
        spec = NP.NlSpec(2, inst.rhs, (inst.rhs_y, inst.rhs_yp), inst.second_partials())
        x, tr = NP.solve_nonlinear(spec, inst.conditions(), g["grid"], float(g["gamma"]),
                                   float(g["sigma2"]), g["landmarks"], Wb,
                                   max_iters=W.NONLINEAR2["newton_max_iters"])
        me = Wb.shape[1]
        y = O.predict(float(g["sigma2"]), g["landmarks"], Wb, x[:me], x[me], 0, g["grid"])
        assert O.rel_l2(y, g["yhat"][j]) <= 1e-9
        np.testing.assert_allclose(tr.norms, g[f"norms_{j}"], rtol=1e-6)


def _lev_cases():
    g = load_golden("leverage")
    return g, [str(c) for c in g["cases"]]


def test_oracle_leverage_reproduces_reference():
    """Exact leverage scores and the seeded draw (nystrom.py:58-103)."""
    g, cases = _lev_cases()
    for c in cases:
        grid = g[f"{c}_grid"]
        if grid.size > 1000:          # the 4000-point solve is checked on the GPU side
            continue
        s2 = float(g[f"{c}_sigma2"])
        if not bool(g[f"{c}_explicit_kernel"]):
            assert s2 == O.leverage_default_sigma2(grid)
        sc = O.leverage_scores(s2, grid, float(g[f"{c}_ridge"]))
        np.testing.assert_allclose(sc, g[f"{c}_scores"], rtol=1e-12, atol=0)
        for sd in g[f"{c}_seeds"]:
            idx = O.leverage_landmarks(sc, int(sd), int(g[f"{c}_m"]))
            np.testing.assert_array_equal(grid[idx], g[f"{c}_lm{int(sd)}"])


def test_oracle_leverage_sketch_reproduces_reference():
    """Sketch branch (nystrom.py:71-80) on the smallest golden grid."""
    g = load_golden("leverage_sketch")
    c = "s4001"
    grid = np.linspace(float(g[f"{c}_lo"]), float(g[f"{c}_hi"]), int(g[f"{c}_n"]))
    sc = O.leverage_scores(float(g[f"{c}_sigma2"]), grid, float(g[f"{c}_ridge"]))
    np.testing.assert_allclose(sc, g[f"{c}_scores"], rtol=1e-12, atol=0)
    idx = O.leverage_landmarks(sc, 0, int(g[f"{c}_m"]))
    np.testing.assert_array_equal(grid[idx], g[f"{c}_lm0"])
