"""Multi-process (gloo, world_size 2) coverage of the sharding logic on CPU:
row-sharded partial Grams + one all-reduce reproduce the full extended Gram,
and instance slabs tile the batch.  The per-rank partial Gram is computed by
the oracle here (no GPU in this container); the GPU test covers the kernel's
row_begin/row_end contract."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_04094_b200 import dist as D


def test_instance_and_row_ranges_tile():
    for B, w in [(4096, 8), (4095, 3), (7, 4), (1, 2)]:
        rs = [D.instance_range(B, w, r) for r in range(w)]
        assert rs[0][0] == 0 and rs[-1][1] == B
        assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
        assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
    for n, w in [(4194303, 8), (999, 2), (31, 4)]:
        rr = D.row_ranges(n, w)
        assert rr[0][0] == 0 and rr[-1][1] == n
        assert all(rr[i][1] == rr[i + 1][0] for i in range(w - 1))
        assert all(lo % 32 == 0 or lo == n for lo, _ in rr)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import nys_port as O
    from paper_2510_04094_b200 import workloads as W

    cfg = W.scaled(W.CONFIGS[4], n=4097)
    bt = W.linear_batch(cfg, 0, 1)
    s, v = O.eig_landmarks(cfg.sigma2, bt.landmarks)
    Wb = O.scaled_basis(s, v)
    lo, hi = D.row_ranges(bt.pts.size, world)[rank]
    pts = bt.pts[lo:hi]
    Dm = O.features(cfg.sigma2, bt.landmarks, Wb, 2, pts)
    Dm = Dm - bt.coef[0, 0, lo:hi, None] * O.features(cfg.sigma2, bt.landmarks, Wb, 1, pts)
    Dm = Dm - bt.coef[0, 1, lo:hi, None] * O.features(cfg.sigma2, bt.landmarks, Wb, 0, pts)
    X = np.column_stack([Dm, -bt.coef[0, 1, lo:hi], bt.forcing[0, lo:hi]])
    E = torch.as_tensor(X.T @ X)
    D.allreduce_sum(E)
    if rank == 0:
        out.put(E.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_row_sharded_allreduce_matches_full_gram():
    from oracle import nys_port as O
    from paper_2510_04094_b200 import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    E = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = W.scaled(W.CONFIGS[4], n=4097)
    bt = W.linear_batch(cfg, 0, 1)
    s, v = O.eig_landmarks(cfg.sigma2, bt.landmarks)
    Wb = O.scaled_basis(s, v)
    sy = O.assemble(2, list(bt.coef[0]), bt.forcing[0], bt.instances[0].conditions(), bt.grid,
                    cfg.gamma, cfg.sigma2, bt.landmarks, Wb)
    X = np.column_stack([sy["D"], sy["g"], sy["r"]])
    Ef = X.T @ X
    np.testing.assert_allclose(E, Ef, rtol=0, atol=1e-12 * np.abs(Ef).max())
    # the KKT block layout built from the reduced E equals the full assembly
    me = Wb.shape[1]
    np.testing.assert_allclose(E[:me, :me] + np.eye(me) / cfg.gamma, sy["M"][:me, :me],
                               rtol=0, atol=1e-12 * np.abs(sy["M"]).max())
