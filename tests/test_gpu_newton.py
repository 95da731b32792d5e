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
