"""Multi-process coverage of the N>1 bench path on CPU: the real shard
dispatchers (bench.shard_rows weak shards, bench.split_rows strong shards)
and the real rank coordinators (bench.GlooSync over gloo/TCP, the torchrun
path; bench.launch_spawned + SpawnSync, the `--gpus N` path without
torchrun) at world size 2.  Each rank computes its shard (the oracle stands
in for the engine: no GPU here); gathered, the shards equal the
single-process result bit for bit, and the max-over-ranks timing reduction
returns the slowest rank.  No NCCL anywhere.  The GPU form is
tests/test_gpu_parity.py::test_bench_two_gpus_spawned (skipped with < 2
devices)."""

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_body(sync, rank, n, per, total, out_dir):
    """What gpu_arm does per rank, with the oracle as the compute."""
    import bench
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs

    world = sync.world
    A, B = make_cyclic_inputs(n, max(per * world, total))
    weak = bench.shard_rows(rank, world, per)
    strong = bench.split_rows(rank, world, total)
    sync.barrier()
    np.save(os.path.join(out_dir, f"weak{rank}.npy"), c_mul_cyclic(A[weak], B[weak], n, threads=1))
    np.save(os.path.join(out_dir, f"strong{rank}.npy"), c_mul_cyclic(A[strong], B[strong], n, threads=1))
    # the timing reduction: every rank must see the slowest rank's numbers
    got = sync.max([float(rank + 1), 10.0 - rank, 0.0])
    assert got == [float(world), 10.0, 0.0], got
    sync.barrier()


def _gloo_worker(rank, world, port, n, per, total, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    import bench

    sync = bench.GlooSync(rank, world)
    try:
        _rank_body(sync, rank, n, per, total, out_dir)
    finally:
        sync.close()


def _check(out_dir, n, per, total, world):
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs

    A, B = make_cyclic_inputs(n, max(per * world, total))
    weak = np.concatenate([np.load(os.path.join(out_dir, f"weak{r}.npy")) for r in range(world)])
    strong = np.concatenate([np.load(os.path.join(out_dir, f"strong{r}.npy")) for r in range(world)])
    assert np.array_equal(weak, c_mul_cyclic(A[: per * world], B[: per * world], n))
    assert np.array_equal(strong, c_mul_cyclic(A[:total], B[:total], n))


def test_gloo_ranks_shards_match_single_process(tmp_path):
    import torch.multiprocessing as mp

    n, per, total, world = 1000, 24, 70, 2
    mp.spawn(_gloo_worker, args=(world, _free_port(), n, per, total, str(tmp_path)), nprocs=world, join=True)
    _check(str(tmp_path), n, per, total, world)


def test_spawned_ranks_shards_match_single_process(tmp_path):
    import bench

    n, per, total, world = 1000, 24, 70, 2
    codes = bench.launch_spawned(world, _rank_body, n, per, total, str(tmp_path), timeout_s=120)
    assert codes == [0, 0]
    _check(str(tmp_path), n, per, total, world)


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


@pytest.mark.parametrize("total", [16384, 70, 32, 1, 100000])
def test_split_rows_strong_partition(total):
    """configs[3] split 16384/G: contiguous, whole 32-row groups except the
    tail, balanced to one group, covering every row exactly once."""
    import bench

    for world in (1, 2, 4, 8):
        rows, sizes = [], []
        for r in range(world):
            sl = bench.split_rows(r, world, total)
            assert sl.start % 32 == 0
            rows.extend(range(sl.start, sl.stop))
            sizes.append(sl.stop - sl.start)
        assert rows == list(range(total))
        if total >= 32 * world:
            assert max(sizes) - min(sizes) <= 32
    assert [bench.split_rows(r, 8, 16384).stop - bench.split_rows(r, 8, 16384).start for r in range(8)] == [2048] * 8


def test_parity_rows_cover_edges():
    import bench

    assert bench.parity_rows(100) == list(range(100))
    r = bench.parity_rows(16384)
    assert len(r) == 256 and r[:32] == list(range(32)) and r[-32:] == list(range(16352, 16384))
    assert sorted(set(r)) == r
