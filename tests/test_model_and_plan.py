"""CPU checks of the GPU algorithm's index math and of the host planner.

``model_bitsliced`` executes the kernels' exact layout/index arithmetic in
numpy; it is compared with the oracle here, so plan/layout bugs show up
without a GPU.  The planner is exercised through the real C ABI (libf2x.so
loads and plans without a device).
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest

import model_bitsliced as mb
from oracle import f2x_oracle as o

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kind,t,n,LF,K,KC,batch", [
    ("full", 1, 0, 16, 2, 2, 5),
    ("full", 2, 0, 17, 3, 2, 33),
    ("full", 4, 0, 19, 4, 2, 40),
    ("full", 8, 0, 16, 5, 1, 2),       # GL=4: passes [3, 1]
    ("cyc", 0, 100, 16, 3, 1, 3),
    ("cyc", 0, 129, 13, 4, 2, 3),
    ("cyc", 0, 300, 10, 5, 3, 7),
    ("cyc", 0, 300, 10, 5, 0, 2),      # GL=5: passes [3, 2]
    ("full", 4, 0, 2, 7, 0, 1),        # GL=7: passes [3, 3, 1]
    ("full", 4, 0, 9, 5, 5, 2),        # KC=5: eval pairs (0,1),(2,3); interp pairs 3,1 + level 0
    ("full", 4, 0, 9, 5, 4, 2),        # KC=4: eval pair + single; interp pairs 2,0
    ("full", 8, 0, 17, 5, 4, 1),
])
def test_model_matches_oracle(kind, t, n, LF, K, KC, batch):
    rng = np.random.default_rng(LF * 1000 + K)
    if kind == "full":
        A = rng.integers(0, 1 << 64, (batch, t), dtype=np.uint64)
        B = rng.integers(0, 1 << 64, (batch, t), dtype=np.uint64)
        p = mb.Plan(LF, K, KC, kind="full", t=t, n=0, batch=batch)
        ref = o.mul_full(A, B)
    else:
        A, B = o.make_cyclic_inputs(n, batch)
        t = A.shape[1]
        p = mb.Plan(LF, K, KC, kind="cyc", t=t, n=n, batch=batch)
        ref = o.mul_cyclic(A, B, n)
    assert np.array_equal(mb.run(p, A, B), ref)
    assert np.array_equal(mb.run_v2(p, A, B), ref)  # the kernels' current schedule
    for el in range(1, min(2, p.GL) + 1):  # slicing kernel pre-evaluates el levels
        assert np.array_equal(mb.run_v3(p, A, B, el), ref), el


def test_position_table_matches_generator():
    """The kernels' precomputed table (gen_instances.py) equals the model's."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "gen", os.path.join(ROOT, "paper_2201_10473_b200", "csrc", "gen_instances.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    for KC in range(6):
        plan = mb.Plan(1, KC, KC, kind="full", t=0, n=0, batch=1)
        plan.LFS = 1  # positions in chunks
        flat = [x for lvl in mb.leaf_positions(plan) for x in lvl]
        assert gen.pos_table(KC) == flat


def test_transpose_model():
    rng = np.random.default_rng(3)
    x = rng.integers(0, 1 << 32, 32, dtype=np.uint64).astype(np.uint32)
    y = mb.transpose32(x)
    for i in range(32):
        for p in range(32):
            assert (int(y[i]) >> p) & 1 == (int(x[p]) >> i) & 1


# ----------------------------------------------------------- C ABI on CPU

@pytest.fixture(scope="module")
def lib():
    from paper_2201_10473_b200 import _lib

    try:
        return _lib.load()
    except ImportError:
        from paper_2201_10473_b200 import build

        build.build()
        return _lib.load()


def test_abi_exports_every_declared_symbol(lib):
    from paper_2201_10473_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "f2x.h")).read()
    import re

    declared = set(re.findall(r"F2X_API\s+[\w\s\*]+?\b(f2x_\w+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert declared <= exported, declared - exported
    for name in declared:
        assert hasattr(lib, name)


def test_plan_struct_size_matches_header(lib):
    """ctypes mirror of f2x_plan must have the C layout (field offsets)."""
    from paper_2201_10473_b200 import _lib

    pl = _lib.make_plan(_lib.KIND_CYCLIC, 2048, 17669)  # 64 groups: Karatsuba only
    assert pl.t == 277 and pl.n == 17669 and pl.groups == 64 and pl.toom_levels == 0
    assert pl.N >= 64 * 277 and pl.N == pl.leaf_words << pl.levels
    assert pl.levels == pl.cta_levels + pl.global_levels
    assert sum(pl.pass_levels[: pl.num_passes]) == pl.global_levels
    assert pl.launches == 3 + pl.num_passes
    assert pl.workspace_bytes > 0
    pl = _lib.make_plan(_lib.KIND_CYCLIC, 4096, 17669)  # 128 groups: two Toom-3 levels
    assert pl.t == 277 and pl.groups == 128 and pl.toom_levels == 2 and pl.toom_w == 16
    assert pl.N == 3 * pl.toom_M[0] >= 64 * 277
    assert pl.leaf_words << pl.levels >= pl.toom_M[1] + 2 * pl.toom_w_last
    assert pl.node_ctas == 128 * 25 * 3 ** pl.global_levels
    # one global level, folded into the resident-root interpolation
    assert pl.global_levels == 1 and pl.launches == 3 + 1 + 2 * 2 - 1


# (kind, batch, t_or_n) -> Toom-3 levels measured fastest on B200 (DESIGN §7b
# "planner regret"; tools/runs/toomgrid2.sh, toomgate.sh, toomsmall.sh): the
# depth depends on the batch -- the Toom passes add ~10 us of latency per level
# and call, so small batches stay Karatsuba-only
PLANNER_PINS = [
    (1, 256, 12323, 0), (1, 2048, 12323, 0), (1, 3072, 12323, 1), (1, 4096, 12323, 1),
    (1, 256, 17669, 0), (1, 2048, 17669, 0), (1, 3072, 17669, 2), (1, 4096, 17669, 2),
    (1, 16384, 17669, 2), (1, 4096, 9000, 0), (1, 4096, 14000, 2), (1, 1024, 20000, 2),
    (1, 4096, 20000, 2), (1, 1024, 24000, 1), (1, 4096, 22000, 3), (1, 2048, 28000, 3),
    (1, 4096, 28000, 3), (1, 4096, 30000, 3), (1, 32, 35851, 0), (1, 256, 35851, 0),
    (1, 1024, 35851, 2), (1, 4096, 35851, 2), (1, 32, 57637, 0), (1, 256, 57637, 3),
    (1, 16384, 57637, 3), (0, 1 << 20, 64, 0), (0, 1 << 19, 128, 0), (0, 1 << 18, 256, 2),
    (0, 1 << 17, 512, 2), (0, 1 << 16, 1024, 2),
]


def test_planner_innermost_point_pins(lib):
    """The innermost Toom level evaluates at x = X^8 where that saves a leaf
    word (measured: n=57637 x 16384 6583 -> 6402 us with LF 35 -> 34, n=30000
    729 -> 631, n=32000 846 -> 763) and stays at X^16 elsewhere (d=32768:
    25.4 vs 26.4 ms); never with the two-kernel interpolation of small levels."""
    from paper_2201_10473_b200 import _lib

    for kind, batch, size, wl, lf in ((1, 16384, 57637, 8, 34), (1, 4096, 30000, 8, 36), (1, 4096, 32000, 8, 28),
                                      (1, 4096, 17669, 16, 32), (1, 4096, 35851, 16, 32), (0, 1 << 17, 512, 16, 29),
                                      (0, 1 << 18, 256, 8, 29)):
        pl = _lib.make_plan(kind, batch, size)
        assert (pl.toom_w_last, pl.leaf_words) == (wl, lf), (kind, batch, size)
        assert pl.leaf_words << pl.levels >= pl.toom_M[pl.toom_levels - 1] + 2 * pl.toom_w_last
    assert _lib.make_plan(1, 2048, 17669).toom_w_last == 0  # no Toom level


@pytest.mark.parametrize("kind,batch,size,tl", PLANNER_PINS)
def test_planner_toom_depth_pins(lib, kind, batch, size, tl):
    from paper_2201_10473_b200 import _lib

    pl = _lib.make_plan(kind, batch, size)
    assert pl.toom_levels == tl
    # the pick is the cheapest modelled depth among those considered
    costs = [lib.f2x_plan_cost(kind, batch, size, k) for k in range(4)]
    assert all(c > 0 for c in costs)
    assert costs[tl] == min(costs) or tl == 0
    assert lib.f2x_plan_cost(kind, batch, size, 4) < 0 and lib.f2x_plan_cost(5, batch, size, 0) < 0


@pytest.mark.parametrize("t", list(range(1, 70)) + [100, 128, 193, 256, 277, 512, 561, 901, 1024, 2048])
def test_plan_covers_every_size(lib, t):
    from paper_2201_10473_b200 import _lib

    pl = _lib.make_plan(_lib.KIND_FULL, 33, t)
    assert pl.N >= 64 * t
    assert pl.N <= 64 * t * 1.25 + 64 * 16  # no pathological padding
    assert 16 <= pl.leaf_words <= 40
    assert pl.leaf_stride % 4 == 0 and (pl.leaf_stride // 4) % 2 == 1
    assert pl.leaf_stride - pl.leaf_words < 8


def test_plan_errors(lib):
    from paper_2201_10473_b200 import _lib

    with pytest.raises(ValueError):
        _lib.make_plan(_lib.KIND_FULL, 0, 5)
    with pytest.raises(ValueError):
        _lib.make_plan(_lib.KIND_FULL, 1, 0)
    with pytest.raises(ValueError):
        _lib.make_plan(7, 1, 5)
    with pytest.raises(ValueError):
        _lib.make_plan(_lib.KIND_FULL, 1, 1 << 22)  # outside the envelope
    assert "workspace" in _lib.strerror(_lib.F2X_ENOSPC)


def test_null_pointer_rejected_without_gpu(lib):
    rc = lib.f2x_mul_full(None, None, None, 1, 1, None, 0, 0, None)
    assert rc == -22
    rc = lib.f2x_mul_cyclic(None, None, None, 1, 100, None, 0, 0, None, None)
    assert rc == -22


def test_workspace_query(lib):
    a = lib.f2x_workspace_bytes(1, 4096, 17669, 0)
    b = lib.f2x_workspace_bytes(1, 8192, 17669, 0)
    assert 0 < a < b
    assert lib.f2x_workspace_bytes(1, 4096, 17669, 18) > 0


def _pos_chunks_port(KC, j, nu):
    """Digit-walk derivation of pos_j(nu) (top-down, MS digit first), an
    independent construction of the kernels' kPosChunks table."""
    digs, v = 0, nu
    for l in range(j):
        digs |= (v % 3) << (2 * l)
        v //= 3
    pos = prefix = 0
    p3 = 1
    for l in range(j):
        d = (digs >> (2 * (j - 1 - l))) & 3
        h = 1 << (KC - l - 1)
        R = (1 << (KC - l)) * p3
        pos = pos if d == 0 else (pos + h if d == 1 else R + prefix * h)
        prefix = prefix * 3 + d
        p3 *= 3
    return pos


def test_arithmetic_positions_match_table():
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "gen", os.path.join(ROOT, "paper_2201_10473_b200", "csrc", "gen_instances.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    for KC in range(1, 6):
        flat = [_pos_chunks_port(KC, j, nu) for j in range(KC + 1) for nu in range(3 ** j)]
        assert flat == gen.pos_table(KC)


@pytest.mark.parametrize("kind,size", [(1, 17669), (1, 35851), (1, 57637), (0, 16), (0, 1024)])
def test_plan_counts_match_closed_forms(lib, kind, size):
    """Counter conservation (Table 1): the plan's analytic counts
    follow the KaratRec closed forms -- 3^K leaf products of LF x LF
    coefficients (LF^2/32 LOP3 each per product, bitsliced over 32), and
    eval+interp XOR work sum_j 3^j * 5 * LF*2^(K-j-1) / 32 per product; with
    Toom-3 levels on top, 5^toom_levels node problems per product."""
    from paper_2201_10473_b200 import _lib

    pl = _lib.make_plan(kind, 4096, size)
    LF, K, T = pl.leaf_words, pl.levels, 5 ** pl.toom_levels
    assert pl.leaf_ops_per_product == pytest.approx(T * 3 ** K * LF * LF / 32)
    xors = sum(3 ** j * 5 * (LF << (K - j - 1)) for j in range(K)) / 32
    assert pl.karatsuba_ops_per_product == pytest.approx(T * xors)
    # KaratRec base-multiplication count for 2^K leaves is 3^K (Table 1, t^log2(3))
    assert round((2 ** K) ** np.log2(3)) == 3 ** K


def _byte_perm(x, y, sel):
    b = [(x >> (8 * i)) & 255 for i in range(4)] + [(y >> (8 * i)) & 255 for i in range(4)]
    return sum(b[(sel >> (4 * i)) & 7] << (8 * i) for i in range(4))


def test_transpose_prmt_selectors():
    """The byte-permute form of the 16/8-bit transpose stages
    (f2x_kernels.cuh tstage_prmt) equals the masked-swap form."""
    rng = np.random.default_rng(7)
    for a, c in rng.integers(0, 1 << 32, size=(500, 2), dtype=np.uint64).tolist():
        for J, m, sx, sy in ((16, 0x0000FFFF, 0x5410, 0x7632), (8, 0x00FF00FF, 0x6240, 0x7351)):
            s = ((a >> J) ^ c) & m
            assert _byte_perm(a, c, sx) == (a ^ (s << J)) & 0xFFFFFFFF
            assert _byte_perm(a, c, sy) == c ^ s


@pytest.mark.parametrize("kind,size", [("cyclic", 12323), ("cyclic", 17669), ("cyclic", 35851),
                                       ("cyclic", 57637), ("full", 1), ("full", 16), ("full", 64),
                                       ("full", 100), ("full", 1024)])
def test_plan_eval_levels(kind, size):
    """The slicing kernel pre-evaluates at most 2 top global levels, only
    where each part is whole operand words (k1_slice_eval's tiling)."""
    from paper_2201_10473_b200 import plan

    if os.environ.get("F2X_EVAL_LEVELS"):
        pytest.skip("override set")
    p = plan(kind, 4096, size)
    el = p["eval_levels"]
    assert 0 <= el <= min(2, p["global_levels"])
    if p["toom_levels"]:  # Toom plans slice plainly; the node kernel walks its levels
        assert el == 0
        return
    assert (p["N"] >> el) % 64 == 0
    if kind == "cyclic":
        assert el == 2


def _phase_wavefronts(addrs):
    """Shared-memory wavefronts of 16-byte accesses: a warp's request is
    served in 8-thread phases, each costing the largest number of threads
    that hit the same 16-byte bank group (quad index mod 8)."""
    import collections

    w = 0
    for b in range(0, len(addrs), 8):
        c = collections.Counter(a % 8 for a in addrs[b:b + 8] if a is not None)
        if c:
            w += max(c.values())
    return w


def test_mid_perm_bank_phases():
    """gen_instances.MID_PERM is a permutation of the 81 mid leaves (KC=5)
    that, with odd threads reading the parent's hi chunk first, makes the
    mid leaves' parent reads conflict-free (1620 -> 648 weighted wavefronts,
    9-quad chunks) and lowers the level-3/4 interpolation's mid-product reads
    (324 -> 202), as the generator states."""
    sigma = mb.mid_perm(5)
    assert sorted(sigma) == list(range(81))
    inv = [sigma.index(m) for m in range(81)]
    p = mb.Plan(35, 9, 5, kind="full", t=280, n=0, batch=32)
    Q, RM = p.LFS // 4, 162
    P4 = [x // p.LFS for x in mb.leaf_positions(p)[4]]   # chunks
    P3 = mb.leaf_positions(p)[3]

    def leaf(sig, stagger):
        tot = 0
        for q in range(Q):
            for k in (0, 1):  # first / second load instruction
                addrs = [None if t >= 243 else
                         (t * Q + q if t < RM else (P4[sig[t - RM]] + (k ^ (t & 1) if stagger else k)) * Q + q)
                         for t in range(160, 256)]
                tot += 3 * _phase_wavefronts(addrs)
        return tot

    def interp(iv):
        tot = 0
        for c in range(3):
            addrs = [None if it >= 27 * Q else (RM + iv[3 * (it // Q) + c]) * Q + it % Q for it in range(256)]
            tot += 2 * _phase_wavefronts(addrs)
        return tot

    ident = list(range(81))
    assert (leaf(ident, False), interp(ident)) == (1620, 324)
    assert (leaf(sigma, True), interp(inv)) == (648, 202)
    assert len(P3) == 27


@pytest.mark.parametrize("levels_spec", [[(20, 3)], [(37, 8)], [(64, 16)], [(50, 1)],
                                         [(60, 4), None], [(40, 2), None, None]])
def test_toom_model_matches_oracle(levels_spec):
    """tests/model_toom.py: bitsliced Toom-3 (points 0, 1, x, x+1, inf with
    x = X^w, SURVEY Appx A.2 grouped numerators, exact divisions asserted)
    over 1-3 levels equals the oracle product for 32 random products."""
    import model_toom as mt

    M1, w = levels_spec[0]
    levels = []
    M = M1
    for i in range(len(levels_spec)):
        S = M + 2 * w
        if i + 1 < len(levels_spec):
            S = 3 * (-(-S // 3))
        levels.append((M, w, S))
        M = S // 3
    rng = np.random.default_rng(M1 * 7 + w)
    t = (3 * M1) // 64 + 1
    A = rng.integers(0, 1 << 64, (32, t), dtype=np.uint64)
    B = rng.integers(0, 1 << 64, (32, t), dtype=np.uint64)
    a, b = mt.slice32(A, 3 * M1), mt.slice32(B, 3 * M1)
    ref = o.mul_full(mt.unslice32(a, 32, t), mt.unslice32(b, 32, t))
    assert np.array_equal(mt.unslice32(mt.toom_mul(a, b, levels), 32, 2 * t), ref)


@pytest.mark.parametrize("kind,size", [("cyclic", 17669), ("cyclic", 57637), ("full", 1024)])
@pytest.mark.parametrize("tl", [1, 2, 3])
def test_toom_plan_sizes(kind, size, tl):
    """Forced Toom plans (F2X_TOOM is read once per process, so the sizes are
    recomputed here from the same rule): 3 M_1 >= 64 t, S_l = 3 M_{l+1} >=
    M_l + 2w, and the node problem LF 2^K >= M_tl + 2w."""
    t = (size + 63) // 64 if kind == "cyclic" else size
    w = 16
    M = [0, -(-64 * t // 3)]
    for _ in range(1, tl):
        M.append(-(-(M[-1] + 2 * w) // 3))
    assert 3 * M[1] >= 64 * t
    for l in range(1, tl):
        assert 3 * M[l + 1] >= M[l] + 2 * w
    from paper_2201_10473_b200 import plan

    p = plan(kind, 4096, size)
    if p["toom_levels"]:
        Ms = p["toom_M"]
        assert 3 * Ms[0] >= 64 * t and len(Ms) == p["toom_levels"]
        assert p["toom_w_last"] in (8, p["toom_w"])
        assert p["leaf_words"] << p["levels"] >= Ms[-1] + 2 * p["toom_w_last"]


def test_row_chunks_bound_workspace(monkeypatch):
    """Batches whose scratch exceeds the budget run as whole-group row
    chunks, each within the budget, covering every row once."""
    from paper_2201_10473_b200 import _lib, engine

    lib = _lib.load()
    full = int(lib.f2x_workspace_bytes(_lib.KIND_CYCLIC, 100_000, 17669, 0))
    monkeypatch.setattr(engine, "_WS_BUDGET", full // 7)
    chunks, need = engine._row_chunks(lib, _lib.KIND_CYCLIC, 100_000, 17669, 0)
    assert len(chunks) >= 7 and need <= full // 7
    assert chunks[0][0] == 0 and chunks[-1][1] == 100_000
    for (a, b), (c, _) in zip(chunks, chunks[1:]):
        assert b == c and (b - a) % 32 == 0
    monkeypatch.setattr(engine, "_WS_BUDGET", 8 << 30)
    assert engine._row_chunks(lib, _lib.KIND_CYCLIC, 4096, 17669, 0)[0] == [(0, 4096)]


def test_release_workspaces_drops_cached_scratch():
    """engine.release_workspaces empties the grow-only per-(device, stream)
    scratch cache (all devices or one) and reports the bytes dropped."""
    import torch

    from paper_2201_10473_b200 import engine

    saved = dict(engine._workspaces)
    try:
        engine._workspaces.clear()
        engine._workspaces[(0, 1)] = torch.empty(100, dtype=torch.uint8)
        engine._workspaces[(1, 7)] = torch.empty(30, dtype=torch.uint8)
        if not torch.cuda.is_available():
            assert engine.release_workspaces(1) == 30 and list(engine._workspaces) == [(0, 1)]
            assert engine.release_workspaces() == 100 and not engine._workspaces
    finally:
        engine._workspaces.clear()
        engine._workspaces.update(saved)


def test_plan_resident_root_launches(lib):
    """The last global Karatsuba pass of a Toom plan (one level into the
    node-problem root) is folded into the innermost Toom interpolation
    (resident roots) when that level runs one CTA per product (>= 96
    products): one launch fewer.  n=35851's last pass has two levels."""
    from paper_2201_10473_b200 import _lib

    for batch in (16384, 1024, 256):
        pl = _lib.make_plan(_lib.KIND_CYCLIC, batch, 57637)
        assert pl.toom_levels == 3 and pl.num_passes == 1 and pl.pass_levels[0] == 1
        assert pl.launches == 3 + pl.num_passes + 2 * pl.toom_levels - 1, batch
    # (batches whose innermost level has < 96 products take no Toom level at all)
    assert _lib.make_plan(_lib.KIND_CYCLIC, 40, 57637).toom_levels == 0
    pl = _lib.make_plan(_lib.KIND_CYCLIC, 4096, 35851)
    assert pl.launches == 3 + pl.num_passes + 2 * pl.toom_levels


def test_plan_k34_fusion_launches(lib):
    """The last global pass is fused with the unslicing kernel (k34) for
    Karatsuba-only plans with >= 1024 groups, a last pass of <= 3 levels and
    a root stage of <= 72 KB: d-sweep d=4096 / 8192 yes, d=4096 x 4096 (128
    groups) and n=17669 x 2048 (64 groups, 4 levels) no."""
    from paper_2201_10473_b200 import _lib

    for t, batch, fused in ((64, 1 << 20, True), (128, 1 << 19, True), (64, 4096, False)):
        pl = _lib.make_plan(_lib.KIND_FULL, batch, t)
        assert pl.toom_levels == 0
        assert pl.launches == 3 + pl.num_passes - (1 if fused else 0), (t, batch)
    pl = _lib.make_plan(_lib.KIND_CYCLIC, 2048, 17669)
    assert pl.toom_levels == 0 and pl.launches == 3 + pl.num_passes


def test_plan_fused_last_pass_needs_no_pingpong_buffer(lib):
    """When the only global pass is folded into a later kernel (resident-root
    interpolation at n=57637, k34 at d=4096) the plan does not reserve the
    pass's output buffer: F2X_KROOT / F2X_K34 are read once per process, so
    compare against the closed-form size of that buffer instead."""
    from paper_2201_10473_b200 import _lib

    pl = _lib.make_plan(_lib.KIND_CYCLIC, 16384, 57637)
    assert pl.num_passes == 1 and pl.launches == 2 + pl.num_passes + 2 * pl.toom_levels
    assert pl.workspace_bytes < 4.5 * 2 ** 30  # 5.27 GiB with the pass output buffer
    pl = _lib.make_plan(_lib.KIND_FULL, 1 << 20, 64)
    assert pl.num_passes == 1 and pl.launches == 2 + pl.num_passes
    assert pl.workspace_bytes < 5.5 * 2 ** 30  # 6.19 GiB with it
