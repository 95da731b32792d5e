"""sigma selection for the "tuned" configs (c1, c2, c4) -- oracle side only.

    python oracle/tune_sigma.py [--configs 1 2 4] [--c4-n 262144]

BASELINE.json: c1 "RBF sigma tuned per seed from [0.05, 0.5]", c4 "of config-1
form", c2 one shared sigma (shared landmarks).  SURVEY.md §8(d) ambiguity 2
turns "tuned" into an oracle-side grid search over
``workloads.SIGMA_CANDIDATES`` minimising the relative L2 error of y_hat vs the
manufactured y* on the grid (seed 0, instance 0 -- c2: the mean over instances
0..3).  The rule this repository adds: only sigmas whose error
is REPRODUCIBLE are eligible -- re-running the same restatement with LAPACK's
dsyev driver for the landmark eigenproblem (instead of numpy's dsyevd) must
move the error vs y* by < 1e-3 of itself.  Otherwise the north star's "error
within 1 % of the reference's" gate is unattainable for the reference against
itself (c2 at sigma = 0.3 moves 300 %).

The frozen outcome lives in ``workloads.CONFIGS`` (c1 0.4, c2 0.1, c4 0.5);
this script re-derives it.  c4 is evaluated on a 2^18-point grid of the same
domain by default (--c4-n; the full n = 2^22 takes ~2 min per sigma and
driver): its error vs y* is set by the 256 landmarks on [0, 100], not by n.

TEST / BASELINE INFRASTRUCTURE: the restatement is oracle/nys_port.py
(linear.py:90-158, nystrom.py:136-160); nothing here is product code.
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import nys_port as O  # noqa: E402
from paper_2510_04094_b200 import workloads as W  # noqa: E402

REPRO_TOL = 1e-3


@contextlib.contextmanager
def dsyev_driver():
    import scipy.linalg as sl

    orig = np.linalg.eigh
    np.linalg.eigh = lambda A: sl.eigh(A, driver="ev")
    try:
        yield
    finally:
        np.linalg.eigh = orig


def error_vs_exact(cfg, sigma, indices):
    c = W.scaled(cfg, sigma=sigma)
    g = W.grid(c)
    errs, meff = [], None
    for i in indices:
        inst = W.instance(c.cid, 0, i, c)
        r = O.solve_linear_instance(c.order, inst.coeff_fns(), inst.forcing_fn,
                                    inst.conditions(), g, c.gamma, c.sigma2, c.m)
        y = O.predict(c.sigma2, r["landmarks"], r["W"], r["omega"], r["bias"], 0, g)
        ys = inst.sol(g)
        errs.append(float(np.linalg.norm(y - ys) / np.linalg.norm(ys)))
        meff = r["m_eff"]
    return float(np.mean(errs)), meff


def tune(cid, c4_n):
    cfg = W.CONFIGS[cid]
    if cid == 4:
        cfg = W.scaled(cfg, n=c4_n)
    indices = range(4) if cid == 2 else [0]
    rows = []
    for s in W.SIGMA_CANDIDATES:
        try:
            e, me = error_vs_exact(cfg, s, indices)
            with dsyev_driver():
                e2, _ = error_vs_exact(cfg, s, indices)
        except (O.OracleError, np.linalg.LinAlgError, FloatingPointError) as exc:
            rows.append(dict(sigma=s, error=None, note=str(exc)))
            continue
        swing = abs(e2 - e) / e
        rows.append(dict(sigma=s, m_eff=me, error=e, error_dsyev=e2, swing=swing,
                         eligible=bool(swing < REPRO_TOL)))
    ok = [r for r in rows if r.get("eligible")]
    best = min(ok, key=lambda r: r["error"]) if ok else None
    return dict(config=cid, chosen=best["sigma"] if best else None,
                frozen=W.CONFIGS[cid].sigma, rows=rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--c4-n", type=int, default=1 << 18)
    args = ap.parse_args()
    for cid in args.configs:
        print(json.dumps(tune(cid, args.c4_n)), flush=True)


if __name__ == "__main__":
    main()
