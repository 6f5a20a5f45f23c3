"""N>1 path on CPU: world_size-2 gloo processes shard the batch exactly as the multi-GPU
bench does (contiguous slices, no data-path collective), solve their slices (the oracle
stands in for the per-rank GPU solve here — this test covers the host-side sharding,
gathering and max-over-ranks logic) and all_gather the results for verification."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_29155_b200 import DynModel, problems, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import oracle

    pb = problems.random_problem(DynModel.quadrotor(), B, 6, seed=9)
    lo, hi = shard.shard_range(B, rank, world)
    o = oracle.forward(pb.model, pb.settings, pb.x0[lo:hi], pb.dense_C()[lo:hi], pb.c[lo:hi],
                       pb.U_warm[lo:hi])
    U = shard.all_gather_batch(torch.from_numpy(o["U"]), B)
    it = shard.all_gather_batch(torch.from_numpy(o["iters"].astype(np.int64)), B)
    mx = shard.max_over_ranks(float(rank + 1))
    if rank == 0:
        out_q.put((U.numpy(), it.numpy(), mx))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    for B in (1, 7, 16, 16385):
        for W in (1, 2, 3, 8):
            r = [shard.shard_range(B, k, W) for k in range(W)]
            assert r[0][0] == 0 and r[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert max(h - l for l, h in r) - min(h - l for l, h in r) <= 1
    with pytest.raises(ValueError):
        shard.shard_range(4, 2, 2)


def test_two_rank_gloo_sharded_solve_matches_single_process():
    B, world = 9, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    U, iters, mx = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle

    pb = problems.random_problem(DynModel.quadrotor(), B, 6, seed=9)
    ref = oracle.forward(pb.model, pb.settings, pb.x0, pb.dense_C(), pb.c, pb.U_warm)
    assert np.array_equal(U, ref["U"])
    assert np.array_equal(iters, ref["iters"])
    assert mx == 2.0
