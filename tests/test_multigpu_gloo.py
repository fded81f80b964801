"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path: each rank
computes its shard of one seeded global batch (bench.shard_rows); gathered on
rank 0 the shards equal the single-process result bit for bit.  The per-rank
compute here is the oracle (no GPU in CI); on the B200 box the same sharding
feeds the engine (bench.py under torchrun)."""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, per, out_path):
    import torch
    import torch.distributed as dist

    import bench
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, B = make_cyclic_inputs(n, per * world)
    sl = bench.shard_rows(rank, world, per)
    C = c_mul_cyclic(A[sl], B[sl], n, threads=1)
    t = torch.from_numpy(C.view(np.int64).copy())
    gathered = [torch.zeros_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, gathered, dst=0)
    # max-over-ranks reduction used for timing in bench.py
    tm = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = torch.cat(gathered).numpy().view(np.uint64)
        np.save(out_path, full)
        assert tm.item() == world
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_match_single_process(tmp_path):
    import sys

    import torch.multiprocessing as mp

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs

    n, per, world = 1000, 24, 2
    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(world, _free_port(), n, per, out), nprocs=world, join=True)
    A, B = make_cyclic_inputs(n, per * world)
    assert np.array_equal(np.load(out), c_mul_cyclic(A, B, n))


def test_shard_rows_partition():
    import bench

    for world in (1, 2, 4, 8):
        rows = []
        for r in range(world):
            sl = bench.shard_rows(r, world, 4096)
            rows.extend(range(sl.start, sl.stop))
        assert rows == list(range(4096 * world))
    with pytest.raises(ValueError):
        bench.shard_rows(2, 2, 10)
