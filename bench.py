"""Benchmark: ODE solves/s on BASELINE.json config 2 (B = 4096 linear 2nd-order
IVPs per GPU, n = 4096, m = 64 shared landmarks, FP64).

One step = one batch solved from scratch through the device pipeline:
landmark eigendecomposition (once per shared landmark set) -> shared features
Psi_0..Psi_2 -> per-instance fused row-combine + Gram (DMMA) -> per-instance
KKT LU + refinement.  This is the reference harness' "train" scope
(harness.py:152-163) for a shared-grid batch.

  value  : device-timed, samples already resident in HBM (402 MB > 126 MB L2,
           so no L2 flush is needed between steps)
  e2e    : same step through the public API with pinned HOST buffers: H2D of
           the samples (chunked, overlapped with compute) + D2H of the solutions
  roofline: the batched Gram launch (batch_gram_kernel + its 3 tiny feature
           launches) vs the measured FP64 DMMA peak (profiles/fp64_peak.json)
  cpu_baseline: the oracle restatement of the reference path on this host's
           cores (process pool, 1 BLAS thread per worker), bounded sample

Multi-GPU (torchrun): instances are independent, so each rank solves its own
4096 instances (global instance ids rank*4096 + i) with no collective;
"scaling": "weak"; value = all ranks' solves / max-over-ranks time.

--impl reference: the reference's CPU path (oracle port, all host cores) on the
same config/metric; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CID = 2
FP64_PEAK_FALLBACK_TFLOPS = 37.15   # profiles/fp64_peak.json (DMMA m8n8k4, this pool)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nysb200", choices=["nysb200", "reference"])
    ap.add_argument("--batch", type=int, default=None, help="instances per GPU (default 4096)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--e2e-chunks", type=int, default=4)
    return ap.parse_args()


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _traffic_from_profiles():
    path = os.path.join(ROOT, "profiles", "ncu_batch_gram.json")
    try:
        with open(path) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def _fp64_peak():
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
            return float(json.load(fh)["dmma_m8n8k4_w8_tflops"]), "measured (profiles/fp64_peak.json)"
    except (OSError, ValueError, KeyError):
        return FP64_PEAK_FALLBACK_TFLOPS, "measured earlier (tools/fp64_peak.cu)"


def run_reference(args, world, rank):
    """Reference arm: the oracle port of the reference path on all host cores."""
    if rank != 0:
        return
    from oracle import cpu_baseline as CB

    cores = os.cpu_count() or 1
    per_step_s = 2.0
    for _ in range(args.warmup):
        CB.batch_solves_per_second(CID, cores, per_worker=4)
    vals, solved = [], 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, n, _, _ = CB.batch_solves_per_second(CID, cores, per_worker=10_000, budget_s=per_step_s)
        vals.append(v)
        solved += n
    wall = time.perf_counter() - t0
    value = solved / wall
    line = {
        "impl": "reference", "metric": "ode_solves_per_s", "value": value, "unit": "solves/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (workloads.py, seed 0)",
        "config": {"workload": "c2: B=4096 linear 2nd-order IVPs, n=4096, m=64, sigma=0.1, "
                               "gamma=1e9 (BASELINE.json configs[2])"},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": "port",
                         "sample": f"{solved} instances over {args.steps} steps of "
                                   f"~{per_step_s:.0f} s on a {cores}-process pool "
                                   "(1 BLAS thread each; shared feature map per worker)"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = _args()
    world, rank, local = _dist()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch

    from paper_2510_04094_b200 import _lib
    from paper_2510_04094_b200 import batch as BT
    from paper_2510_04094_b200 import workloads as W
    from paper_2510_04094_b200.problems import ivp

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist

    cfg = W.CONFIGS[CID]
    B = args.batch or cfg.batch
    cfg = W.scaled(cfg, batch=B)
    bt = W.linear_batch(cfg, seed=0, count=B, first=rank * B)
    cond = ivp([(t, int(o), 0.0) for t, o in zip(bt.cond_points, bt.cond_orders)])
    pipe = BT.SharedGridPipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond,
                                 max_batch=B, device=dev)
    coef_d = torch.as_tensor(bt.coef, device=dev)
    forc_d = torch.as_tensor(bt.forcing, device=dev)
    vals_d = torch.as_tensor(bt.cond_values, device=dev)
    side = None
    lib = _lib.load()

    def step():
        return pipe.run_device(coef_d, forc_d, vals_d)

    def barrier():
        torch.cuda.synchronize()
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()

    # ---- warm-up + correctness spot check
    for _ in range(max(args.warmup, 1)):
        x, info = step()
    torch.cuda.synchronize()
    side = x.shape[1]
    bad = int((info != 0).sum())
    if bad:
        raise SystemExit(f"{bad} instances reported singular/non-finite KKT systems")

    # ---- timed device-resident steps
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = lib.nys_launch_count()
    barrier()
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(st)
        for k in range(args.steps):
            ev[k][0].record(st)
            step()
            ev[k][1].record(st)
        t_end.record(st)
        barrier()
    launches = (lib.nys_launch_count() - launches0) / args.steps
    total_ms = t_start.elapsed_time(t_end)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    if pg is not None:
        t = torch.tensor([total_ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total_ms = float(t)
    ms_per_step = total_ms / args.steps
    value = world * B / (ms_per_step / 1e3)

    # ---- roofline: the batched Gram launch alone
    fm = pipe.solver.fmap
    me, n_c, p, m = fm.m_eff, pipe.solver.n_c, cfg.order, cfg.m
    solver = pipe.solver
    ws_bytes = lib.nys_batch_gram_workspace_bytes(n_c, me, p, B)
    g_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    for k in range(args.steps):
        g_ev[k][0].record(st)
        _lib.call("nys_batch_gram_f64", _lib.ptr(fm.d_landmarks), fm.m, _lib.ptr(fm.d_W), fm.m,
                  me, float(cfg.sigma2), p, _lib.ptr(solver.pts), n_c, _lib.ptr(coef_d),
                  _lib.ptr(forc_d), B, None, _lib.ptr(solver.ws), ws_bytes, _lib.stream_ptr())
        g_ev[k][1].record(st)
    torch.cuda.synchronize()
    gram_ms = statistics.median(a.elapsed_time(b) for a, b in g_ev)
    # per instance 2 n_c m_eff^2 + 8 n_c m_eff + 4 n_c (Gram + combine + rhs)
    flops_gram = B * (2.0 * n_c * me * me + 8.0 * n_c * me + 4.0 * n_c)
    flops_shared = 2.0 * (p + 1) * n_c * m * me
    peak, peak_src = _fp64_peak()
    achieved = flops_gram / (gram_ms / 1e3) / 1e12
    nb = (me + 2 + 7) // 8
    executed = B * (4 * ((n_c + 3) // 4)) * (nb * (nb + 1) // 2) * 64 * 2.0
    step_flops = flops_gram + flops_shared

    # ---- e2e through the public API with pinned host buffers
    coef_h = torch.from_numpy(bt.coef).pin_memory()
    forc_h = torch.from_numpy(bt.forcing).pin_memory()
    vals_h = torch.from_numpy(bt.cond_values).pin_memory()
    x_h = torch.empty((B, side), dtype=torch.float64).pin_memory()
    info_h = torch.empty(B, dtype=torch.int32).pin_memory()
    bufs = (torch.empty_like(coef_d), torch.empty_like(forc_d), torch.empty_like(vals_d),
            torch.empty((B, side), dtype=torch.float64, device=dev),
            torch.empty(B, dtype=torch.int32, device=dev))
    for _ in range(2):
        pipe.run_host(coef_h, forc_h, vals_h, x_h, info_h, chunks=args.e2e_chunks, dev_bufs=bufs)
    barrier()
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    e_start.record(st)
    for _ in range(args.steps):
        pipe.run_host(coef_h, forc_h, vals_h, x_h, info_h, chunks=args.e2e_chunks, dev_bufs=bufs)
    e_end.record(st)
    barrier()
    e2e_ms = e_start.elapsed_time(e_end) / args.steps
    if pg is not None:
        t = torch.tensor([e2e_ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_ms = float(t)
    if int((info_h != 0).sum()):
        raise SystemExit("e2e path reported failed instances")
    h2d = coef_h.numel() * 8 + forc_h.numel() * 8 + vals_h.numel() * 8
    d2h = x_h.numel() * 8 + info_h.numel() * 4

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import cpu_baseline as CB

        cores = os.cpu_count() or 1
        v, n, workers, wall = CB.batch_solves_per_second(CID, cores, per_worker=10_000,
                                                        budget_s=args.cpu_seconds)
        cpu = {"value": v, "unit": "solves/s", "cores": workers, "kind": "port",
               "sample": f"{n} config-2 instances in {wall:.1f} s on a {workers}-process pool "
                         "(oracle port of linear.assemble+solve, 1 BLAS thread per worker, "
                         "shared feature map per worker)"}

    if rank == 0:
        line = {
            "metric": "ode_solves_per_s", "value": value, "unit": "solves/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, paper_2510_04094_b200/workloads.py)",
            "config": {"workload": "c2: B=4096 linear 2nd-order IVPs per GPU, n=4096 shared "
                                   "grid on [0,2], m=64 shared landmarks, sigma=0.1 "
                                   "(m_eff=%d), gamma=1e9 (BASELINE.json configs[2])" % me,
                       "global_batch": world * B, "n": cfg.n, "m": cfg.m, "m_eff": me,
                       "parallelism": f"instance-sharded x{world}, no collective",
                       "l2": "samples 402 MB/GPU > 126 MB L2; no flush needed",
                       "step": "eig + shared features + batched Gram + batched KKT"},
            "step_ms_min": min(step_ms), "step_ms_median": statistics.median(step_ms),
            "gpu_launches": launches,
            "e2e": {"value": world * B / (e2e_ms / 1e3), "unit": "solves/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms, "chunks": args.e2e_chunks},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": _traffic_from_profiles(),
                         "kernel": "batch_gram_kernel (+3 psi-pack launches)",
                         "kernel_ms": gram_ms, "algorithmic_flops": flops_gram,
                         "executed_dmma_flops": executed,
                         "executed_frac": executed / (gram_ms / 1e3) / 1e12 / peak,
                         "peak_source": peak_src + "; MEASURED_PEAKS.json has no FP64 entry",
                         "note": "algorithmic F (SURVEY.md 8d) counts the full m_eff^2 Gram; "
                                 "the kernel computes the upper block triangle only"},
            "step_tflops": step_flops / (ms_per_step / 1e3) / 1e12 / world,
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
