"""GPU parity at EXACTLY the BASELINE.json batches (the sizes bench.py
reports), through the C ABI, against the C oracle:

* configs[0] n=12323 x 256: every row;
* configs[1] n=17669 x 4096, configs[2] n=35851 x 4096, configs[3]
  n=57637 x 16384: a 256-row subsample (bench.parity_rows: the first and last
  32-row groups + an even stride) plus commutativity over the WHOLE batch;
* configs[4] d-sweep, 1024..65536 bits at ~1 GB of operands per size (the
  8 GiB workspace budget row-chunks d=65536): subsample + commutativity;
* very large single products (t = 16384 .. 131072 words) with few rows --
  the Toom interpolation's sequential fallback for few products -- against
  the oracle (t=16384) and through bilinearity / commutativity beyond.
Bit-exact everywhere (integer path, no tolerance)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(x, cuda):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64).view(np.int64)).to(cuda)


def _np(x):
    return x.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("n,batch", [(12323, 256), (17669, 4096), (35851, 4096), (57637, 16384)])
def test_ring_config_exact_batch(n, batch, cuda):
    import torch

    import bench
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import mul_cyclic

    A, B = make_cyclic_inputs(n, batch)
    dA, dB = _dev(A, cuda), _dev(B, cuda)
    C = mul_cyclic(dA, dB, n)
    rows = bench.parity_rows(batch)
    got = _np(C)[rows]
    assert np.array_equal(got, c_mul_cyclic(A[rows], B[rows], n))
    assert torch.equal(C, mul_cyclic(dB, dA, n))
    if batch <= 256:
        assert len(rows) == batch


@pytest.mark.parametrize("d", [1024, 4096, 8192, 16384, 32768, 65536])
def test_dsweep_exact_batch(d, cuda):
    import torch

    import bench
    from oracle import c_mul_full
    from paper_2201_10473_b200 import mul_full

    t = d // 64
    batch = bench.DSWEEP_OPERAND_BYTES // (2 * 8 * t)
    dA = bench.device_words(torch, batch, t, 0xF2F2 + 2 * d, cuda)
    dB = bench.device_words(torch, batch, t, 0xF2F2 + 2 * d + 1, cuda)
    C = mul_full(dA, dB)
    rows = bench.parity_rows(batch)
    idx = torch.tensor(rows, device=cuda)
    A, B = _np(dA[idx]), _np(dB[idx])
    assert np.array_equal(_np(C[idx]), c_mul_full(A, B))
    assert torch.equal(C, mul_full(dB, dA))


@pytest.mark.parametrize("t,batch", [(16384, 2), (16384, 40)])
def test_very_large_full_vs_oracle(t, batch, cuda):
    from oracle import c_mul_full
    from oracle.f2x_oracle import make_full_inputs
    from paper_2201_10473_b200 import mul_full

    A, B = make_full_inputs(t, batch, words=True)
    out = _np(mul_full(_dev(A, cuda), _dev(B, cuda)))
    rows = list(range(min(batch, 2)))
    assert np.array_equal(out[rows], c_mul_full(A[rows], B[rows]))


@pytest.mark.parametrize("t", [32768, 65536, 131072])
def test_very_large_full_properties(t, cuda):
    import torch

    from oracle.f2x_oracle import make_full_inputs
    from paper_2201_10473_b200 import mul_full

    A, B = make_full_inputs(t, 3, words=True)
    dA, dB = _dev(A, cuda), _dev(B, cuda)
    C = mul_full(dA, dB)
    assert torch.equal(C, mul_full(dB, dA))
    D = torch.roll(dB, 1, 0)
    assert torch.equal(mul_full(dA, dB ^ D), C ^ mul_full(dA, D))
    # X^k shift: A * X^(64 j) = A shifted by j words
    sh = np.zeros_like(A)
    sh[:, 7] = 1
    S = _np(mul_full(dA, _dev(sh, cuda)))
    want = np.zeros((3, 2 * t), dtype=np.uint64)
    want[:, 7:7 + t] = A
    assert np.array_equal(S, want)


def test_odd_offset_row_views(cuda):
    """mul_cyclic(A[1:], B[1:], n) at the odd-t config sizes: 8-byte aligned
    row views are accepted and exact (the reference takes any row)."""
    from oracle import c_mul_cyclic, c_mul_full
    from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
    from paper_2201_10473_b200 import mul_cyclic, mul_full

    for n in (12323, 17669, 35851, 57637):
        A, B = make_cyclic_inputs(n, 41)
        dA, dB = _dev(A, cuda), _dev(B, cuda)
        assert dA[1:].data_ptr() % 16 == 8
        assert np.array_equal(_np(mul_cyclic(dA[1:], dB[1:], n)), c_mul_cyclic(A[1:], B[1:], n))
    A, B = make_full_inputs(3, 9, words=True)
    dA, dB = _dev(A, cuda), _dev(B, cuda)
    assert np.array_equal(_np(mul_full(dA[1:], dB[1:])), c_mul_full(A[1:], B[1:]))
    # strided (non-contiguous) views are copied, not rejected
    A, B = make_full_inputs(8, 10, words=True)
    dA, dB = _dev(A, cuda), _dev(B, cuda)
    assert np.array_equal(_np(mul_full(dA[:, :4], dB[:, :4])), c_mul_full(A[:, :4], B[:, :4]))


def test_bench_two_ranks_spawned_functional(cuda):
    """The `--gpus 2` spawned-rank path end to end on ONE device
    (`--share-device`: both ranks on cuda:0; a functional test of the N-rank
    code -- barrier, max-over-ranks, shard dispatch, scaling block, parity --
    not a measurement), with no NCCL in the process tree."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NCCL_DEBUG="INFO")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--share-device", "--steps", "5", "--warmup",
                        "3", "--no-cpu", "--no-dsweep", "--e2e-chunks", "1", "--e2e-lanes", "1", "--batch", "1024"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["parity"]["ok"] and line["parity_all_ok"], line
    assert line["config"]["global_batch"] == 2048 and "functional_test_only" in line
    sc = line["scaling_57637"]
    assert sc["n_gpus"] == 2 and [g["rows"] for g in sc["per_gpu"]] == [8192, 8192] and sc["parity"]["ok"]
    assert "NCCL INFO" not in r.stdout + r.stderr  # no NCCL communicator was created


def test_bench_two_ranks_torchrun_functional(cuda):
    """The torchrun form (the driver's N > 1 launch): two ranks joined by a
    gloo group for the barrier and the max -- on ONE device
    (`--share-device`, functional test, not a measurement), no NCCL."""
    import json
    import os
    import socket
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NCCL_DEBUG="INFO")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                        "--share-device", "--steps", "5", "--warmup", "3", "--no-cpu", "--no-dsweep",
                        "--e2e-chunks", "1", "--e2e-lanes", "1", "--batch", "1024"], cwd=root, env=env, capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["parity_all_ok"] and "GlooSync" in line["config"]["parallelism"]
    assert "NCCL INFO" not in r.stdout + r.stderr


def test_bench_two_gpus_spawned(cuda):
    """`bench.py --gpus 2` without torchrun: two spawned ranks, no NCCL."""
    import json
    import os
    import subprocess
    import sys

    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun boxes have one)")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NCCL_DEBUG="INFO")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3",
                        "--quick", "--no-cpu"], cwd=root, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["parity"]["ok"]
    assert "NCCL INFO" not in r.stdout + r.stderr  # no NCCL communicator was created


def _random_cases():
    """(kind, size, batch) draws of test_random_sizes_vs_oracle: small batches
    (Karatsuba-only plans: the Toom passes cannot fill the GPU) and batches
    of 1000-4200 rows (the planner's Toom depths)."""
    rng = np.random.default_rng(0x5EED)
    cases = []
    for i in range(28):
        n = int(rng.integers(1, 70000))
        batch = int(rng.integers(1, 48)) if i % 2 == 0 else int(rng.integers(1000, 4200))
        cases.append(("cyclic", n, batch))
    for i in range(16):
        t = int(rng.integers(1, 1536))
        batch = int(rng.integers(1, 40)) if i % 2 == 0 else int(rng.integers(1000, 2100))
        cases.append(("full", t, batch))
    return cases


def test_random_cases_reach_every_toom_depth():
    """The seeded draws cover Karatsuba-only plans and 1, 2 and 3 Toom-3 levels
    (the plan is host-only: checked without a GPU too)."""
    from paper_2201_10473_b200 import plan

    seen = {plan(kind, batch, size)["toom_levels"] for kind, size, batch in _random_cases()}
    assert seen == {0, 1, 2, 3}, seen


def test_random_sizes_vs_oracle(cuda):
    """Seeded random ring sizes (1 .. 70000 bits, every Toom / leaf / chunk
    regime the planner reaches) and full-product sizes (1 .. 1536 words)
    with random batch sizes, against the C oracle (all rows of the small
    batches; the first and last 8 rows and 16 random rows of the large)."""
    from oracle import c_mul_cyclic, c_mul_full
    from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
    from paper_2201_10473_b200 import mul_cyclic, mul_full

    rng = np.random.default_rng(0xC0FFEE)
    for kind, size, batch in _random_cases():
        if kind == "cyclic":
            A, B = make_cyclic_inputs(size, batch)
            got = _np(mul_cyclic(_dev(A, cuda), _dev(B, cuda), size))
        else:
            A, B = make_full_inputs(size, batch, words=True)
            got = _np(mul_full(_dev(A, cuda), _dev(B, cuda)))
        rows = np.arange(batch) if batch <= 48 else np.unique(np.r_[0:8, batch - 8:batch,
                                                                     rng.integers(0, batch, 16)])
        want = c_mul_cyclic(A[rows], B[rows], size) if kind == "cyclic" else c_mul_full(A[rows], B[rows])
        assert np.array_equal(got[rows], want), (kind, size, batch)


@pytest.mark.parametrize("tl,n,batch", [(1, 12323, 4096), (2, 17669, 4096), (2, 20000, 4096), (2, 35851, 4096),
                                         (3, 28000, 3072), (3, 57637, 1024), (2, 1000, 4000)])
def test_innermost_point_x8_vs_oracle(cuda, tl, n, batch):
    """The innermost Toom level at x = X^8 (F2X_TOOM_WLAST=8, read once per
    process: subprocess) for every interpolation form it can take -- resident
    roots with 2048 / 2304 blocks, plain roots, the 512-thread form, 1..3
    levels -- against the C oracle on the first / last 8 and 48 random rows."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
n, batch, tl = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
from oracle import c_mul_cyclic
from oracle.f2x_oracle import make_cyclic_inputs
from paper_2201_10473_b200 import mul_cyclic, plan
p = plan("cyclic", batch, n)
assert p["toom_levels"] == tl and p["toom_w_last"] == 8, p
assert p["leaf_words"] << p["levels"] >= p["toom_M"][-1] + 16
A, B = make_cyclic_inputs(n, batch)
d = lambda x: torch.from_numpy(x.view(np.int64)).cuda()
got = mul_cyclic(d(A), d(B), n).cpu().numpy().view(np.uint64)
rows = np.unique(np.r_[0:8, batch - 8:batch, np.random.default_rng(n).integers(0, batch, 48)])
assert np.array_equal(got[rows], c_mul_cyclic(A[rows], B[rows], n))
print("ok")
"""
    env = dict(os.environ, F2X_TOOM_WLAST="8", F2X_TOOM=str(tl))
    r = subprocess.run([sys.executable, "-c", script, root, str(n), str(batch), str(tl)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]


def test_oversize_root_keeps_the_separate_pass(cuda):
    """n=54718 on three Toom levels: M_3 = 2044 but the node problem is 33 * 64
    = 2112 coefficients, so its 4224-word product does not fit the resident
    span (2 x 2048 + 3w slots) of the resident-root interpolation -- found by
    tools/stress_parity.py as an illegal shared-memory access.  The plan must
    keep the separate k3_interp<1> pass there, and the product must match."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import c_mul_cyclic
from oracle.f2x_oracle import make_cyclic_inputs
from paper_2201_10473_b200 import mul_cyclic, plan
n, batch = 54718, 942
p = plan("cyclic", batch, n)
assert p["toom_levels"] == 3 and p["leaf_words"] << p["levels"] == 2112 and p["toom_M"][-1] == 2044, p
assert p["launches"] == 3 + p["num_passes"] + 2 * 3, p  # not folded
A, B = make_cyclic_inputs(n, batch)
d = lambda x: torch.from_numpy(x.view(np.int64)).cuda()
got = mul_cyclic(d(A), d(B), n).cpu().numpy().view(np.uint64)
rows = np.r_[0:16, batch - 16:batch]
assert np.array_equal(got[rows], c_mul_cyclic(A[rows], B[rows], n))
print("ok")
"""
    env = dict(os.environ, F2X_TOOM="3", F2X_TOOM_WLAST="16")
    r = subprocess.run([sys.executable, "-c", script, root], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
