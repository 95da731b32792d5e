"""Time the device leverage-score sweep (CUDA events, graph-free) at n."""
import sys
import time

import numpy as np
import torch

from paper_2510_04094_b200 import _lib
from paper_2510_04094_b200 import nystrom as N
from paper_2510_04094_b200.kernel import RbfKernel

for n in [int(a) for a in sys.argv[1:]] or [1000, 4000]:
    grid = np.linspace(0.0, 1.0, n)
    lib, _ = _lib.require_device()
    dev = torch.device("cuda")
    d_grid = _lib.as_f64(grid, dev)
    sc = torch.empty(n, dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    wsb = lib.nys_leverage_workspace_bytes(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def run():
        _lib.call("nys_leverage_scores_f64", d_grid.data_ptr(), n, 0.01, 1e-6, sc.data_ptr(),
                  info.data_ptr(), ws.data_ptr(), wsb, st)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nt = (n + 63) // 64
    flops = 2 * (nt * 64) ** 3 / 3
    t0 = time.perf_counter()
    from oracle import nys_port as O
    ref = O.leverage_scores(0.01, grid, 1e-6) if n <= 4000 else None
    tc = time.perf_counter() - t0
    err = float(np.max(np.abs(sc.cpu().numpy() / ref - 1))) if ref is not None else -1
    print(f"n={n} device {ms:.3f} ms  ({flops / ms / 1e9:.2f} TF/s on 2n^3/3)  cpu {tc*1e3:.1f} ms"
          f"  maxrel {err:.2e} info {int(info.item())}")

# sketch branch timing (n > 4000) through the Python mirror (includes the rank read-back)
for n in [6000, 10000, 100000]:
    grid = np.linspace(0.0, 1.0, n)
    k = RbfKernel(0.01)
    for _ in range(2):
        N.ridge_leverage_scores(k, grid, 1e-6)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        N.ridge_leverage_scores(k, grid, 1e-6)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    from oracle import nys_port as O
    ref = O.leverage_scores(0.01, grid, 1e-6) if n <= 10000 else None
    tc = time.perf_counter() - t0
    print(f"sketch n={n}: device+host {dt*1e3:.2f} ms   cpu {tc*1e3:.1f} ms")
