"""Shared-memory race model of the node kernel (racecheck substitute;
compute-sanitizer is closed on this pool).

For every barrier phase of ``k2_node_mul`` at KC = 5 (the compiled
schedule: fused load + eval(0,1) | eval_pair<2> | leaf b-load | leaf passes |
leaf lo store | interp_pair<3> | interp_pair<1> | level-0 interpolation +
store), this test rebuilds each thread-item's shared-memory read and write
sets with the kernel's own index formulas (f2x_kernels.cuh: node_load_eval0,
item_node_quad, eval_pair, node_leaves, interp_pair, node_level0_store; the
position table and mid-leaf permutation from gen_instances.py) and checks:

* no two items write the same quad in one phase (write-write race);
* no item reads a quad another item writes in the same phase (read-write
  race);
* every quad a phase reads was written by the load phase or an earlier
  phase (no read of uninitialised shared memory).

CPU only; chunk sizes Q = 5, 9, 11 quads (LF 17-20, 33-36, 37-40)."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2201_10473_b200", "csrc"))

KC = 5
NT = 256


def gen():
    import gen_instances

    return gen_instances


def item_node_quad(nodes, q, it):
    qa = q & ~7
    qt = q - qa
    if qa > 0 and it < nodes * qa:
        nu = it // qa
        return nu, it - nu * qa
    r = it - nodes * qa
    nu = r // qt if qt > 0 else 0
    return nu, qa + r - nu * qt


def phases(Q):
    g = gen()
    flat = g.pos_table(KC)
    P = []
    off = 0
    for j in range(KC + 1):
        P.append([x * Q for x in flat[off:off + 3 ** j]])
        off += 3 ** j
    perm, inv = g.MID_PERM, g.MID_INV
    SQ = Q << KC
    out = []  # (name, [(reads, writes) per item]) with accesses ("A"|"B", quad)

    # load + eval(0,1): item (op, w), w < q
    q = Q << (KC - 2)
    Rj1 = Q * (1 << (KC - 1)) * 3
    items = []
    for op in "AB":
        for w in range(q):
            wr = [w + k * q for k in range(4)] + [SQ + w, SQ + q + w, Rj1 + w, Rj1 + q + w, Rj1 + 2 * q + w]
            items.append((set(), {(op, x) for x in wr}))
    out.append(("load_eval01", items))

    # eval_pair<2>
    J = 2
    q = Q << (KC - J - 2)
    Rj = Q * (1 << (KC - J)) * 3 ** J
    Rj1 = Q * (1 << (KC - J - 1)) * 3 ** (J + 1)
    items = []
    for it in range(3 ** J * q):
        nu, w = item_node_quad(3 ** J, q, it)
        p = P[J][nu] + w
        m = Rj + nu * 2 * q + w
        c = Rj1 + 3 * nu * q + w
        rd = {(op, p + k * q) for op in "AB" for k in range(4)}
        wr = {(op, x) for op in "AB" for x in (m, m + q, c, c + q, c + 2 * q)}
        items.append((rd, wr))
    out.append(("eval_pair2", items))

    # leaves: thread t < 243 owns chunk t; mids (t >= RM) read their parent's
    # lo/hi chunks (parent = level-4 node perm[t - RM])
    NLEAF, RM = 3 ** KC, 3 ** KC - 3 ** (KC - 1)
    src = []
    for t in range(NLEAF):
        own = t * Q
        if t >= RM:
            par = P[KC - 1][perm[t - RM]]
            src.append((own, [par, par + Q]))
        else:
            src.append((own, [own]))
    out.append(("leaf_b_load", [({("B", s + k) for s in ss for k in range(Q)}, set()) for own, ss in src]))
    out.append(("leaf_passes", [({("A", s + k) for s in ss for k in range(Q)},
                                 {("B", own + k) for k in range(Q)}) for own, ss in src]))
    out.append(("leaf_lo_store", [(set(), {("A", own + k) for k in range(Q)}) for own, ss in src]))

    # interp_pair<J> for J = 3, 1 (in place; level-KC mid products permuted)
    for J in (3, 1):
        q = Q << (KC - J - 2)
        RJ = Q * (1 << (KC - J)) * 3 ** J
        RJ1 = Q * (1 << (KC - J - 1)) * 3 ** (J + 1)
        items = []
        for it in range(3 ** J * q):
            nu, w = item_node_quad(3 ** J, q, it)
            p = P[J][nu] + w
            pc = [p, p + 2 * q, RJ + 2 * q * nu + w]
            rd = set()
            for c in range(3):
                m = inv[3 * nu + c] if J == KC - 2 else 3 * nu + c
                for x in (pc[c], pc[c] + q, RJ1 + q * m + w):
                    rd |= {("A", x), ("B", x)}
            p0, p1 = pc[0], pc[1]
            wr = {("A", p0 + q), ("A", p1), ("A", p1 + q), ("B", p0), ("B", p0 + q), ("B", p1)}
            items.append((rd, wr))
        out.append((f"interp_pair{J}", items))

    # level 0 + store: reads only
    hq = SQ // 2
    out.append(("level0_store", [({("A", it), ("B", it), ("A", it + hq), ("B", it + hq), ("A", SQ + it),
                                   ("B", SQ + it)}, set()) for it in range(hq)]))
    return out


@pytest.mark.parametrize("Q", [5, 9, 11])
def test_node_kernel_phases_are_race_free(Q):
    RQ = Q * 3 ** KC
    written = set()
    for name, items in phases(Q):
        owner = {}
        for i, (rd, wr) in enumerate(items):
            for x in wr:
                assert 0 <= x[1] < RQ, (name, x)
                assert x not in owner, f"{name}: write-write race on {x} (items {owner[x]} and {i})"
                owner[x] = i
        for i, (rd, wr) in enumerate(items):
            for x in rd:
                assert 0 <= x[1] < RQ, (name, x)
                assert x in written, f"{name}: item {i} reads {x}, never written before this phase"
                j = owner.get(x)
                assert j is None or j == i, f"{name}: read-write race on {x} (reader {i}, writer {j})"
        written |= set(owner)


def test_item_maps_are_bijective():
    """item_node_quad covers every (node, quad) exactly once."""
    for nodes in (1, 3, 9, 27, 81):
        for q in (5, 8, 9, 11, 18, 36, 72):
            seen = {item_node_quad(nodes, q, it) for it in range(nodes * q)}
            assert seen == {(nu, w) for nu in range(nodes) for w in range(q)}
