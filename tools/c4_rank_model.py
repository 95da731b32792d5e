"""Modelled per-rank c4 step at N ranks on ONE GPU: the product pipeline
(SingleSolvePipeline(rows=...)) over rank 0's row slab of N, i.e. every kernel a
rank of `bench.py --gpus N --config 4` runs, with the K all-reduce
((m+2)^2 doubles, ~0.5 MB: a few us over NVLink) stood in for by a device copy
of the full K (so the projection and KKT see the matrix a real all-reduce
gives; rank 0's partial K alone is rank-deficient and sends the KKT down its
LU fallback).  Prints ms per call
(device-timed, steady state) for each N in argv (default 1 2 4 8)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json

import torch

from paper_2510_04094_b200 import dist as DI, linear as L, workloads as W
from paper_2510_04094_b200.problems import ivp

cfg = W.CONFIGS[4]
bt = W.linear_batch(cfg, 0, 1)
cond = ivp(bt.instances[0].conditions())
pts = torch.as_tensor(bt.pts, device="cuda")
coef = torch.as_tensor(bt.coef[0], device="cuda")
forc = torch.as_tensor(bt.forcing[0], device="cuda")
ev0 = torch.cuda.Event()
ev0.record()
steps = int(os.environ.get("STEPS", "60"))
full = L.SingleSolvePipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond)
full.run_device(pts, coef, forc, input_event=ev0)
torch.cuda.synchronize()
K_full = full._kcur.clone()
del full
DI.allreduce_sum = lambda t, group=None: t.copy_(K_full)
for world in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    rows = DI.row_ranges(bt.pts.size, world)[0] if world > 1 else None
    pipe = L.SingleSolvePipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond,
                                 rows=rows)
    for _ in range(8):
        x, info = pipe.run_device(pts, coef, forc, input_event=ev0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        x, info = pipe.run_device(pts, coef, forc, input_event=ev0)
    b.record()
    torch.cuda.synchronize()
    pipe.model()
    ms = a.elapsed_time(b) / steps
    print(json.dumps({"world": world, "rows": rows, "eig_streams": pipe._n_eig_streams(),
                      "gram_ctas": pipe._kctas, "ms_per_call": round(ms, 4),
                      "info": int(info[0])}), flush=True)
    del pipe
    torch.cuda.synchronize()
