"""GPU parity for the nonlinear (Newton-KKT) path, config 3, against the
reference's golden vectors (tests/golden/c3_seed0_i0-3.npz)."""
import numpy as np
import pytest

from conftest import load_golden
from gpu_util import rel_l2

pytestmark = pytest.mark.gpu

YHAT_TOL = 1e-6


def _engine(g, specs=False):
    from paper_2510_04094_b200 import newton as NW
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200 import workloads as W
    from paper_2510_04094_b200.kernel import RbfKernel
    from paper_2510_04094_b200.problems import ivp

    fm = N.build_feature_map(RbfKernel(float(g["sigma2"])), g["landmarks"])
    cond = ivp([(0.0, 0, 0.0)])
    vals = g["y0"].reshape(-1, 1)
    if specs:
        from paper_2510_04094_b200.problems import NonlinearOdeSpec
        sp = []
        for i in g["indices"]:
            inst = W.instance(3, 0, int(i))
            sp.append(NonlinearOdeSpec(1, inst.rhs, (inst.rhs_y,), (0.0, 1.0),
                                       {(0, 0): inst.rhs_yy}))
        return NW.NewtonBatch(fm, g["grid"], cond, vals, float(g["gamma"]), specs=sp), fm
    kinds = [str(k) for k in g["kinds"]]
    alpha = np.array([-k if kd == "quad" else 0.0 for k, kd in zip(g["k"], kinds)])
    beta = np.array([1.0 if kd == "sin" else 0.0 for kd in kinds])
    fam = NW.SeparableFamily(g["g"], alpha, beta)
    return NW.NewtonBatch(fm, g["grid"], cond, vals, float(g["gamma"]), family=fam), fm


@pytest.mark.parametrize("specs", [False, True])
def test_newton_ladder_matches_reference(specs):
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import newton as NW
    g = load_golden("c3_seed0_i0-3")
    eng, fm = _engine(g, specs)
    status, X, traces, rung = eng.solve(max_iters=20)
    Y = L.predict_batch(fm, X[:, :eng.me + 1], 0, g["grid"]).cpu().numpy()
    for j in range(len(g["indices"])):
        ref_status = str(g["status"][j])
        ours = "converged" if status[j] == NW.OK else ("max_iters" if status[j] == NW.MAXITERS
                                                       else f"failed{status[j]}")
        # instances the reference converges must converge here with the same y_hat;
        # a reference MaxIters outcome is the last iterate of a non-converging
        # sequence (harness.py:173-175) and is rounding-chaotic: status only logged
        if ref_status == "converged":
            assert ours == ref_status, (j, ours, ref_status, rung[j], traces[j][-3:])
        print(j, ours, "rung", rung[j], "its", len(traces[j]) - 1, "ref its", len(g[f"norms_{j}"]) - 1,
              "dyhat", rel_l2(Y[j], g["yhat"][j]), traces[j][:4], list(g[f"norms_{j}"][:4]))
        if ref_status == "converged":
            assert rel_l2(Y[j], g["yhat"][j]) <= YHAT_TOL, (j, rel_l2(Y[j], g["yhat"][j]))


def test_newton_residual_matches_oracle():
    """Device residual F(x) equals the oracle's newton_port.residual at a random x."""
    from oracle import newton_port as NP
    from paper_2510_04094_b200 import workloads as W
    g = load_golden("c3_seed0_i0-3")
    eng, fm = _engine(g)
    rng = np.random.default_rng(0)
    x = np.zeros((eng.B, eng.ldx))
    x[:, :eng.me] = rng.normal(scale=0.1, size=(eng.B, eng.me))
    x[:, eng.me] = 0.5
    x[:, eng.nz:] = 1.0 + 0.1 * rng.normal(size=(eng.B, eng.n_c))
    eng.X[:] = eng.torch.as_tensor(x, device=eng.dev)
    ids = list(range(eng.B))
    eng.residual(eng.X, ids)
    F = eng.F.cpu().numpy()
    Wd = fm.d_W[:, :fm.m_eff].cpu().numpy()
    for j, i in enumerate(g["indices"]):
        inst = W.instance(3, 0, int(i))
        spec = NP.NlSpec(1, inst.rhs, (inst.rhs_y,), {(0, 0): inst.rhs_yy})
        w = NP.Work(spec, inst.conditions(), g["grid"], float(g["gamma"]), float(g["sigma2"]),
                    g["landmarks"], Wd)
        Fo = NP.residual(w, x[j])
        scale = np.abs(Fo).max()
        np.testing.assert_allclose(F[j], Fo, rtol=0, atol=1e-9 * scale)


def test_batched_step_halving_is_bit_identical():
    """nys_newton_trial_norms_f64 (the batched line search) returns exactly the
    norms of materialising each candidate and running the residual."""
    import torch

    from paper_2510_04094_b200 import _lib
    g = load_golden("c3_seed0_i0-3")
    eng, fm = _engine(g)
    ids = list(range(eng.B))
    eng.X[:] = torch.as_tensor(eng.const_state(ids), device=eng.dev)
    eng.residual(eng.X, ids)
    info = eng.direction(ids)
    assert (info == 0).all()
    alphas = [1.0, 0.5, 0.25, 0.125]
    seq = []
    for a in alphas:
        eng.candidate(ids, [a] * len(ids))
        seq.append(eng.residual(eng.Xc, ids))
    seq = np.array(seq)
    idx_t = eng._idx(ids)
    norms = torch.empty((len(alphas), len(ids)), dtype=torch.float64, device=eng.dev)
    al_t = torch.tensor(alphas, dtype=torch.float64, device=eng.dev)
    sb = eng.lib.nys_newton_trial_scratch_bytes(eng.me, eng.n_c, len(ids), len(alphas))
    scratch = torch.empty(max(sb, 8), dtype=torch.uint8, device=eng.dev)
    _lib.call("nys_newton_trial_norms_f64", _lib.ptr(eng.S0T), _lib.ptr(eng.S1T), eng.me,
              eng.n_c, _lib.ptr(eng.g), None, None, _lib.ptr(eng.fal), _lib.ptr(eng.fbe),
              _lib.ptr(eng.Ac), _lib.ptr(eng.betac), _lib.ptr(eng.vals), eng.nk,
              _lib.ptr(eng.gam), _lib.ptr(eng.X), _lib.ptr(eng.D), eng.ldx, _lib.ptr(idx_t),
              len(ids), _lib.ptr(al_t), len(alphas), _lib.ptr(norms), _lib.ptr(scratch), sb,
              _lib.stream_ptr())
    got = norms.cpu().numpy()
    assert np.array_equal(got, seq, equal_nan=True), (got, seq)


def test_config3_census_matches_reference():
    """All 256 config-3 bench instances against the live reference's outcomes
    (tests/golden/c3_census_seed0.npz, make_c3_census.py): instances the
    reference converges converge here with y_hat within the north-star 1e-6;
    outcome disagreements are confined to the reference's non-converging,
    rounding-chaotic instances."""
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import newton as NW
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200 import workloads as W
    from paper_2510_04094_b200.kernel import RbfKernel
    from paper_2510_04094_b200.problems import ivp

    ref = load_golden("c3_census_seed0")
    cfg = W.CONFIGS[3]
    g = W.grid(cfg)
    lm = W.equidistant_landmarks(g, cfg.m)
    B = ref["status"].size
    insts = [W.instance(3, 0, i) for i in range(B)]
    pts = g[1:]
    fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                             np.array([i.quad_coeff for i in insts]),
                             np.array([i.sin_coeff for i in insts]))
    vals = np.array([[i.conditions()[0][2]] for i in insts])
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
    eng = NW.NewtonBatch(fm, g, ivp([(0.0, 0, 0.0)]), vals, cfg.gamma, family=fam)
    status, X, traces, rung = eng.solve(max_iters=cfg.newton_max_iters)
    me = eng.me
    Y = L.predict_batch(fm, X[:, :me + 1], 0, g).cpu().numpy()
    conv = np.flatnonzero(ref["status"] == 0)
    from oracle import nys_port as O
    Wr = O.scaled_basis(ref["eigvals"], ref["eigvecs"])     # the reference's own basis
    Phi = O.features(cfg.sigma2, lm, Wr, 0, g)
    Yr = ref["x"][conv, :Wr.shape[1]] @ Phi.T + ref["x"][conv, Wr.shape[1]][:, None]
    bad, lost = [], []
    for j, i in enumerate(conv):
        if status[i] != NW.OK:
            lost.append(int(i))
            continue
        d = rel_l2(Y[i], Yr[j])
        if d > YHAT_TOL:
            bad.append((int(i), d))
    both = [int(i) for i in conv if status[i] == NW.OK]
    its = np.array([len(traces[i]) - 1 for i in both])
    same_its = int((its == ref["iterations"][both]).sum())
    agree = int((status == ref["status"]).sum())
    print("status agreement", agree, "/", B, "ours", np.bincount(status, minlength=4),
          "ref", np.bincount(ref["status"], minlength=4), "| ref-converged lost", lost,
          "rungs", [int(rung[i]) for i in lost], "| same iteration count", same_its, "/",
          len(both), "| y_hat mismatches", bad)
    assert not bad, bad
    # Outcome flips sit on knife-edge trajectories.  Yardstick: the reference
    # against itself (make_c3_census.py) -- with only LAPACK's eigensolver
    # driver swapped (status_dsyev) it loses 6 of its converged instances and
    # agrees on 240 of 256 outcomes; with its landmark matrix moved by at most
    # one ulp per entry (status_perturbed, 3 seeds) it agrees on 237-243 and
    # loses 4-9.  The device must do at least as well as the driver swap.
    self_lost = int(((ref["status"] == 0) & (ref["status_dsyev"] != 0)).sum())
    self_agree = int((ref["status"] == ref["status_dsyev"]).sum())
    pert = [(int((ref["status"] == p).sum()), int(((ref["status"] == 0) & (p != 0)).sum()))
            for p in ref["status_perturbed"]]
    print("reference self-sensitivity: dsyev agreement", self_agree, "lost", self_lost,
          "| 1-ulp perturbations (agreement, lost)", pert)
    assert len(lost) <= self_lost, lost
    assert agree >= self_agree, (agree, self_agree)


# ---------------------------------------------------------------- p = 2
def _engine2(g):
    from paper_2510_04094_b200 import newton as NW
    from paper_2510_04094_b200 import nystrom as N
    from paper_2510_04094_b200 import workloads as W
    from paper_2510_04094_b200.kernel import RbfKernel
    from paper_2510_04094_b200.problems import Conditions, BoundaryCondition, NonlinearOdeSpec

    fm = N.build_feature_map(RbfKernel(float(g["sigma2"])), g["landmarks"])
    insts = [W.nonlinear2_instance(0, int(i)) for i in g["indices"]]
    specs = [NonlinearOdeSpec(2, it.rhs, (it.rhs_y, it.rhs_yp), it.domain, it.second_partials())
             for it in insts]
    cond = Conditions("ivp", tuple(BoundaryCondition(*c) for c in insts[0].conditions()))
    vals = np.array([[c[2] for c in it.conditions()] for it in insts])
    eng = NW.NewtonBatch(fm, g["grid"], cond, vals, float(g["gamma"]), specs=specs)
    return eng, fm, insts


def test_newton2_residual_and_direction_match_oracle():
    """p = 2 (newton2.cu): the device residual equals the oracle's, and the
    Schur-reduced Newton direction solves the oracle's dense analytic system
    J d = -F (newton.py:160-211) to a backward error of 1e-12."""
    from oracle import newton_port as NP
    g = load_golden("n2_seed0_i0-5")
    eng, fm, insts = _engine2(g)
    rng = np.random.default_rng(1)
    x = np.zeros((eng.B, eng.ldx))
    x[:, :eng.me] = rng.normal(scale=0.05, size=(eng.B, eng.me))
    x[:, eng.me] = 0.7
    x[:, eng.nz:] = 0.7 + 0.05 * rng.normal(size=(eng.B, eng.n_c))
    eng.X[:] = eng.torch.as_tensor(x, device=eng.dev)
    ids = list(range(eng.B))
    eng.residual(eng.X, ids)
    info = eng.direction(ids)
    assert (info == 0).all()
    F = eng.F.cpu().numpy()
    Dd = eng.D.cpu().numpy()
    Wd = fm.d_W[:, :fm.m_eff].cpu().numpy()
    S0 = fm.feature_matrix(0, eng.pts_host)
    for j, it in enumerate(insts):
        spec = NP.NlSpec(2, it.rhs, (it.rhs_y, it.rhs_yp), it.second_partials())
        w = NP.Work(spec, it.conditions(), g["grid"], float(g["gamma"]), float(g["sigma2"]),
                    g["landmarks"], Wd)
        Fo = NP.residual(w, x[j])
        np.testing.assert_allclose(F[j], Fo, rtol=0, atol=1e-9 * np.abs(Fo).max())
        J = NP.jacobian(w, x[j])
        d = Dd[j]
        # backward error of the device direction in the oracle's dense system
        # (J reaches cond ~1e16 at gamma = 1e8, so forward differences say little)
        berr = np.abs(J @ d + Fo).max() / (np.abs(J).sum(axis=1).max() * np.abs(d).max()
                                           + np.abs(Fo).max())
        assert berr <= 1e-12, (j, berr)
        do = np.linalg.solve(J, -Fo)
        me = eng.me
        yo = S0 @ do[:me] + do[me]
        yd = S0 @ d[:me] + d[me]
        assert rel_l2(yd, yo) <= 1e-3, (j, rel_l2(yd, yo))


def test_newton2_ladder_matches_reference():
    """solve_nonlinear with p = 2 specs against the live reference's outcomes
    (tests/golden/make_newton2.py): same status, y_hat within 1e-6."""
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200 import newton as NW
    g = load_golden("n2_seed0_i0-5")
    eng, fm, insts = _engine2(g)
    status, X, traces, rung = eng.solve(max_iters=30)
    Y = L.predict_batch(fm, X[:, :eng.me + 1], 0, g["grid"]).cpu().numpy()
    for j in range(len(insts)):
        ours = "converged" if status[j] == NW.OK else f"status{status[j]}"
        assert ours == str(g["status"][j]), (j, ours, traces[j][-3:])
        assert rel_l2(Y[j], g["yhat"][j]) <= YHAT_TOL, (j, rel_l2(Y[j], g["yhat"][j]))
        print(j, "its", len(traces[j]) - 1, "ref", int(g["iterations"][j]), "rung", rung[j])
