"""Generate golden vectors by running the LIVE reference (``nysode``).

Run in the build container only (``/root/reference`` does not exist on the GPU
box):  ``PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py``

Each case stores the sampled inputs that cross our C-ABI (grid, landmarks,
coefficient rows, forcing, conditions) together with the reference's outputs
(eigenvalues, m_eff, KKT matrix/rhs, solution x, y_hat on the grid, Newton
traces).  The tests compare (a) the oracle restatement against these vectors
(pinning the oracle) and (b) the CUDA path against them (parity).
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from nysode import linear, newton, nystrom  # noqa: E402
from nysode.kernel import RbfKernel  # noqa: E402
from nysode.problems import (BoundaryCondition, Conditions, LinearOdeSpec,  # noqa: E402
                             NonlinearOdeSpec, get_problem, grid_for)

from paper_2510_04094_b200 import workloads as W  # noqa: E402


def _cond_arrays(entries):
    return (np.array([c[0] for c in entries]), np.array([c[1] for c in entries], np.int32),
            np.array([c[2] for c in entries]))


def linear_case(name, cfg, seed, indices, kind="ivp"):
    g = W.grid(cfg)
    lm = W.equidistant_landmarks(g, cfg.m)
    fmap = nystrom.build_feature_map(RbfKernel(cfg.sigma2), lm)
    pts = g[1:]
    coef, forcing, vals, xs, yh, Ms, rhss, errs = [], [], [], [], [], [], [], []
    for i in indices:
        inst = W.instance(cfg.cid, seed, i, cfg)
        spec = LinearOdeSpec(cfg.order, inst.coeff_fns(), inst.forcing_fn, cfg.domain)
        cond = Conditions("ivp", tuple(BoundaryCondition(*c) for c in inst.conditions()))
        t0 = time.perf_counter()
        sy = linear.assemble(spec, cond, fmap, g, cfg.gamma)
        mdl = linear.solve(sy, fmap)
        dt = time.perf_counter() - t0
        c, r = inst.sample(pts)
        coef.append(c)
        forcing.append(r)
        vals.append([e[2] for e in inst.conditions()])
        xs.append(np.concatenate([mdl.omega, [mdl.bias], mdl.multipliers]))
        y = mdl.predict(0, g)
        yh.append(y)
        ys = inst.sol(g)
        errs.append(np.linalg.norm(y - ys) / np.linalg.norm(ys))
        Ms.append(sy.matrix)
        rhss.append(sy.rhs)
    cp, co, _ = _cond_arrays(inst.conditions())
    out = dict(kind=kind, order=cfg.order, gamma=cfg.gamma, sigma2=cfg.sigma2, m=cfg.m,
               grid=g, landmarks=lm, pts=pts, coef=np.array(coef), forcing=np.array(forcing),
               cond_points=cp, cond_orders=co, cond_values=np.array(vals),
               eigvals=fmap.eigenvalues, eigvecs=fmap.eigenvectors, m_eff=fmap.m_eff,
               x=np.array(xs), yhat=np.array(yh), err_vs_exact=np.array(errs),
               M=np.array(Ms), rhs=np.array(rhss), indices=np.array(indices),
               seconds_per_solve=dt)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: m_eff={fmap.m_eff} side={Ms[0].shape[0]} err={np.median(errs):.3e}")


def catalog_case(name, pid, n=None, m=None):
    """A reference catalog problem, sampled (no reference code is stored)."""
    p = get_problem(pid)
    d = p.defaults
    g = grid_for(p, n or d.n)
    lm = nystrom.select_landmarks(nystrom.Equidistant(), g, m or d.m)
    fmap = nystrom.build_feature_map(RbfKernel(d.sigma2), lm)
    sy = linear.assemble(p.spec, p.conditions, fmap, g, d.gamma)
    mdl = linear.solve(sy, fmap)
    pts = sy.constraint_points
    coef = np.stack([np.asarray(f(pts), dtype=float) for f in p.spec.coeffs])
    forcing = np.asarray(p.spec.forcing(pts), dtype=float)
    ents = [(bc.point, bc.order, bc.value) for bc in p.conditions.entries]
    cp, co, cv = _cond_arrays(ents)
    rep = linear.check_kkt(mdl, sy)
    out = dict(kind=p.conditions.kind, order=p.spec.order, gamma=d.gamma, sigma2=d.sigma2,
               m=lm.size, grid=g, landmarks=lm, pts=pts, coef=coef[None], forcing=forcing[None],
               cond_points=cp, cond_orders=co, cond_values=cv[None],
               eigvals=fmap.eigenvalues, eigvecs=fmap.eigenvectors, m_eff=fmap.m_eff,
               x=np.concatenate([mdl.omega, [mdl.bias], mdl.multipliers])[None],
               yhat=mdl.predict(0, g)[None], M=sy.matrix[None], rhs=sy.rhs[None],
               kkt_linear_residual=rep.linear_residual, problem_id=pid)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: P{pid} order={p.spec.order} kind={p.conditions.kind} m_eff={fmap.m_eff}")


def newton_case(name, cfg, seed, indices):
    g = W.grid(cfg)
    lm = W.equidistant_landmarks(g, cfg.m)
    fmap = nystrom.build_feature_map(RbfKernel(cfg.sigma2), lm)
    rows = []
    for i in indices:
        inst = W.instance(cfg.cid, seed, i, cfg)
        spec = NonlinearOdeSpec(1, inst.rhs, (inst.rhs_y,), cfg.domain,
                                {(0, 0): inst.rhs_yy})
        cond = Conditions("ivp", tuple(BoundaryCondition(*c) for c in inst.conditions()))
        opts = newton.NewtonOptions(max_iters=cfg.newton_max_iters)
        t0 = time.perf_counter()
        try:
            mdl, tr = newton.solve_nonlinear(spec, cond, fmap, g, cfg.gamma, opts)
            status = "converged"
        except newton.MaxItersExceeded as exc:      # harness.py:173-175
            mdl, tr = exc.model, exc.trace
            status = "max_iters"
        dt = time.perf_counter() - t0
        y = mdl.predict(0, g)
        ys = inst.sol(g)
        rows.append(dict(x=np.concatenate([mdl.omega, [mdl.bias], mdl.multipliers]),
                         yhat=y, err=np.linalg.norm(y - ys) / np.linalg.norm(ys),
                         norms=np.array(tr.residual_norms), status=status, seconds=dt,
                         kind=inst.kind, k=inst.k, y0=inst.conditions()[0][2]))
        print(f"  {name}[{i}] {inst.kind} {status} its={tr.iterations} "
              f"err={rows[-1]['err']:.3e} {dt:.2f}s")
    t = g[1:]
    gvals = np.array([W.instance(cfg.cid, seed, i, cfg).g_fn(t) for i in indices])
    out = dict(order=1, gamma=cfg.gamma, sigma2=cfg.sigma2, m=cfg.m, grid=g, landmarks=lm,
               pts=t, g=gvals, kinds=np.array([r["kind"] for r in rows]),
               k=np.array([r["k"] for r in rows]), y0=np.array([r["y0"] for r in rows]),
               eigvals=fmap.eigenvalues, m_eff=fmap.m_eff,
               x=np.array([r["x"] for r in rows]), yhat=np.array([r["yhat"] for r in rows]),
               err_vs_exact=np.array([r["err"] for r in rows]),
               status=np.array([r["status"] for r in rows]),
               seconds=np.array([r["seconds"] for r in rows]),
               indices=np.array(indices))
    for j, r in enumerate(rows):
        out[f"norms_{j}"] = r["norms"]
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def main():
    C = W.CONFIGS
    linear_case("c0_seed0", C[0], 0, [0])
    linear_case("c1_seed0", C[1], 0, [0])
    linear_case("c2_seed0_i0-7", C[2], 0, list(range(8)))
    linear_case("c4_n16384", W.scaled(C[4], n=1 << 14), 0, [0])
    catalog_case("cat_p2", 2, n=2000)
    catalog_case("cat_p12", 12)
    catalog_case("cat_p16", 16)
    newton_case("c3_seed0_i0-3", C[3], 0, [0, 1, 2, 3])
    meta = dict(numpy=np.__version__, python=platform.python_version(),
                blas=str(np.show_config(mode="dicts").get("Build Dependencies", {})
                         .get("blas", {}).get("version")),
                generated=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()))
    with open(os.path.join(HERE, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(meta)


if __name__ == "__main__":
    main()
