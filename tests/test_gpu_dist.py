"""Row-sharded config 4 through the product pipeline with a real process group.

Two processes (world size 2, gloo -- this run has one GPU, and NCCL refuses
two ranks on one device) each run ``SingleSolvePipeline(rows=<its slab>)``
end to end: its slab of the kernel-space Gram on cuda:0, the pipeline's own
all-reduce of K over the group (dist.allreduce_sum), projection, KKT.  Both
ranks must return the single-rank solution (row sums reassociate:
SURVEY.md A1, <= 1.5e-14 on config-4 shapes).  The ranks' kernels never wait
on each other; the exchange is the host-side gloo all-reduce.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_ROWS = (1 << 20) + 1


def _problem():
    from paper_2510_04094_b200 import workloads as W

    cfg = W.scaled(W.CONFIGS[4], n=N_ROWS)
    return cfg, W.linear_batch(cfg, 0, 1)


def _solve(rows):
    from paper_2510_04094_b200 import linear as L
    from paper_2510_04094_b200.problems import ivp

    cfg, bt = _problem()
    dev = torch.device("cuda", 0)
    pipe = L.SingleSolvePipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order,
                                 ivp(bt.instances[0].conditions()), device=dev, rows=rows)
    pts = torch.as_tensor(bt.pts, device=dev)
    coef = torch.as_tensor(bt.coef[0], device=dev)
    forc = torch.as_tensor(bt.forcing[0], device=dev)
    out = None
    for _ in range(2):
        x, info = pipe.run_device(pts, coef, forc)
        torch.cuda.synchronize()
        assert int(info[0]) == 0
        out = x.cpu().numpy().copy() if out is None else out
        assert np.array_equal(out, x.cpu().numpy())
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_04094_b200 import dist as DI

        rows = DI.row_ranges(N_ROWS - 1, world)[rank]
        q.put((rank, _solve(rows)))
    finally:
        dist.destroy_process_group()


def test_row_sharded_pipeline_two_ranks_matches_single():
    single = _solve(None)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(res[0], res[1])          # redundant KKT: identical on every rank
    d = np.linalg.norm(res[0] - single) / np.linalg.norm(single)
    assert d <= 1e-11, d
