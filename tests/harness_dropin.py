"""Run the UNMODIFIED reference harness with and without the device drop-in.

    python tests/harness_dropin.py            (prints one JSON object)

Needs ``nysode`` importable (``baseline/_ref`` -- the reference installed by
pip, git-ignored -- or ``/root/reference/pkg/src``) and, for the patched leg, a
GPU.  For every case it runs ``nysode.harness.run(config)`` once as shipped and
once after ``paper_2510_04094_b200.dropin.patch_nysode()``,
and reports the harness's own outputs: error metrics, m_eff, Newton status and
trace length, and the relative L2 distance of the two predicted y_hat.
Test helper only (tests/test_gpu_dropin.py); not product code.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "nysode")):
        sys.path.insert(0, p)
        break
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
from nysode import harness  # noqa: E402
from nysode.problems import get_problem, grid_for  # noqa: E402

# (problem id, overrides): P3 linear 1st order, P12 linear BVP, P4 nonlinear
# (Newton ladder), P4 with a 1-iteration budget (ends MaxItersExceeded, which
# harness.py:173 must catch)
CASES = [
    ("P3", 3, {}),
    ("P12", 12, {}),
    ("P4", 4, dict(n=400)),
    ("P4_maxiters", 4, dict(n=400, max_iters=1)),
]


def _one(pid, over):
    cfg = harness.config_from_defaults(pid, **over)
    res = harness.run(cfg)
    grid = grid_for(get_problem(pid), cfg.n)
    y = np.asarray(res.model.predict(0, grid), dtype=float)
    return res, y


def main():
    from paper_2510_04094_b200 import dropin
    from paper_2510_04094_b200 import newton as W1

    import nysode.newton as W0

    out = {"maxiters_is_subclass": issubclass(W1.MaxItersExceeded, W0.MaxItersExceeded)}
    ref = {name: _one(pid, over) for name, pid, over in CASES}
    undo = dropin.patch_nysode()
    try:
        dev = {name: _one(pid, over) for name, pid, over in CASES}
    finally:
        undo()
    for name, _, _ in CASES:
        (r0, y0), (r1, y1) = ref[name], dev[name]
        out[name] = dict(
            ref_mae=r0.metrics.mae, dev_mae=r1.metrics.mae,
            ref_m_eff=r0.m_eff, dev_m_eff=r1.m_eff,
            ref_converged=r0.newton_converged, dev_converged=r1.newton_converged,
            ref_trace_len=len(r0.newton_trace) if r0.newton_trace else None,
            dev_trace_len=len(r1.newton_trace) if r1.newton_trace else None,
            ref_kkt_residual=r0.kkt_residual, dev_kkt_residual=r1.kkt_residual,
            dev_model_type=type(r1.model).__module__,
            yhat_rel_l2=float(np.linalg.norm(y1 - y0) / np.linalg.norm(y0)),
            ref_train_s=r0.timings.train_seconds, dev_train_s=r1.timings.train_seconds)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
