"""Measurements for the SURVEY 8f next rows (leverage scores, full-feature
comparator): device time by CUDA events after warm-up vs the CPU reference
algorithm (oracle restatement, numpy/OpenBLAS on the host cores).  One JSON
line per workload; run on the GPU box: python tools/next_rows_bench.py"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "tests")
from paper_2510_04094_b200 import _lib  # noqa: E402
from paper_2510_04094_b200 import nystrom as N  # noqa: E402
from paper_2510_04094_b200.kernel import RbfKernel  # noqa: E402
from oracle import nys_port as O  # noqa: E402

DMMA_PEAK = 37.15   # TFLOP/s, profiles/fp64_peak.json


def dev_time(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def cpu_time(fn, reps=2):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


def leverage_exact(n):
    grid = np.linspace(0.0, 1.0, n)
    lib, _ = _lib.require_device()
    dev = torch.device("cuda")
    d_grid = _lib.as_f64(grid, dev)
    sc = torch.empty(n, dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    wsb = lib.nys_leverage_workspace_bytes(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    s2 = O.leverage_default_sigma2(grid)
    ms = dev_time(lambda: _lib.call("nys_leverage_scores_f64", d_grid.data_ptr(), n, s2, 1e-6,
                                    sc.data_ptr(), info.data_ptr(), ws.data_ptr(), wsb, st))
    cpu = cpu_time(lambda: O.leverage_scores(s2, grid, 1e-6), reps=1)
    ref = O.leverage_scores(s2, grid, 1e-6)
    nt = (n + 63) // 64
    flops = 2 * (nt * 64) ** 3 / 3          # Cholesky n^3/3 + inverse n^3/3, 2 flop/FMA
    tfs = flops / ms / 1e9
    return dict(workload=f"leverage_exact_n{n}", ms=round(ms, 4), cpu_ms=round(cpu, 1),
                speedup=round(cpu / ms, 1), tflops=round(tfs, 2),
                roofline={"bound": "tensor", "achieved": round(tfs, 2), "peak": DMMA_PEAK,
                          "unit": "TFLOP/s", "frac": round(tfs / DMMA_PEAK, 3)},
                max_rel_vs_cpu=float(np.max(np.abs(sc.cpu().numpy() / ref - 1))))


def leverage_sketch(n):
    grid = np.linspace(0.0, 1.0, n)
    k = RbfKernel(O.leverage_default_sigma2(grid))
    t = []
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sc = N.ridge_leverage_scores(k, grid, 1e-6)
        t.append(time.perf_counter() - t0)
    ms = float(np.median(t[1:]) * 1e3)
    cpu = cpu_time(lambda: O.leverage_scores(k.sigma2, grid, 1e-6), reps=1)
    ref = O.leverage_scores(k.sigma2, grid, 1e-6)
    return dict(workload=f"leverage_sketch_n{n}", ms_host_wall=round(ms, 3), cpu_ms=round(cpu, 1),
                speedup=round(cpu / ms, 1), max_rel_vs_cpu=float(np.max(np.abs(sc / ref - 1))))


def full_feature(n, sigma2=1.0, lo=0.0, hi=20.0):
    """P7 shape (damped oscillator defaults): landmark eig + assemble + KKT."""
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200.problems import BoundaryCondition, Conditions, LinearOdeSpec
    grid = np.linspace(lo, hi, n)
    spec = LinearOdeSpec(2, (lambda t: -0.4 + 0 * t, lambda t: -1.0 + 0 * t),
                         lambda t: np.sin(t), (lo, hi))
    cond = Conditions("ivp", (BoundaryCondition(lo, 0, 1.0), BoundaryCondition(lo, 1, 0.0)))

    def dev():
        fm = N.build_feature_map(RbfKernel(sigma2), grid)
        sy = L.assemble(spec, cond, fm, grid, 1e7)
        return L.solve(sy, fm)
    t = []
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        model = dev()
        t.append(time.perf_counter() - t0)
    ms = float(np.median(t[1:]) * 1e3)
    pts = grid[1:]
    ents = [(lo, 0, 1.0), (lo, 1, 0.0)]

    def cpu():
        s, v = O.eig_landmarks(sigma2, grid)
        W = O.scaled_basis(s, v)
        sy = O.assemble(2, [lambda t: -0.4 + 0 * t, lambda t: -1.0 + 0 * t], np.sin, ents, grid,
                        1e7, sigma2, grid, W)
        return O.solve_kkt(sy["M"], sy["rhs"]), W
    c = cpu_time(cpu, reps=1)
    x, W = cpu()
    me = W.shape[1]
    y_ref = O.predict(sigma2, grid, W, x[:me], x[me], 0, grid)
    y = model.predict(0, grid)
    return dict(workload=f"full_feature_p7shape_n{n}", ms_host_wall=round(ms, 2), cpu_ms=round(c, 1),
                speedup=round(c / ms, 1), m_eff=model.feature_map.m_eff, m_eff_cpu=me,
                rel_l2_vs_cpu=float(np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)))


if __name__ == "__main__":
    cores = len(os.sched_getaffinity(0))
    for row in (leverage_exact(1000), leverage_exact(4000), leverage_sketch(10000),
                leverage_sketch(100000) if False else None, full_feature(1000), full_feature(5000)):
        if row is None:
            continue
        row.update(cpu_cores=cores, cpu_kind="port (oracle restatement, numpy/OpenBLAS)")
        print(json.dumps(row), flush=True)
