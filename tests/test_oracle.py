"""Pin the oracle before trusting it (CPU only).

The numpy and C restatements must reproduce the golden vectors produced by
the real reference (tests/golden/make_golden.py) and the reference's own
known-answer tests (test_poly.py:134-143, 219-225).  The cyclic fold is pinned
against the rotation-sum definition of the ring product.
"""

import numpy as np
import pytest

from conftest import int_clmul

import oracle
from oracle import f2x_oracle as o


def test_clmul_known_answers():
    # test_poly.py:134-143
    assert o.clmul64_shift_xor(0x0, 0xDEADBEEF) == 0
    assert o.clmul64_shift_xor(0x1, 0xFEDCBA9876543210) == 0xFEDCBA9876543210
    assert o.clmul64_shift_xor(0x5, 0x3) == 0xF
    assert o.clmul64_int_mul(0x5, 0x3) == 0xF


def test_clmul_recipes_agree_vs_bitwise(rng):
    a = rng.integers(0, 1 << 64, 200, dtype=np.uint64)
    b = rng.integers(0, 1 << 64, 200, dtype=np.uint64)
    lo, hi = o.clmul64_lanes(a, b)
    clo, chi = oracle.c_clmul64(a, b)
    plo, phi = oracle.c_clmul64(a, b, portable=True)
    for i in range(200):
        want = int_clmul(int(a[i]), int(b[i]))
        assert o.clmul64_shift_xor(int(a[i]), int(b[i])) == want
        assert o.clmul64_int_mul(int(a[i]), int(b[i])) == want
        assert int(lo[i]) | int(hi[i]) << 64 == want
    assert np.array_equal(lo, clo) and np.array_equal(hi, chi)
    assert np.array_equal(lo, plo) and np.array_equal(hi, phi)


def test_golden_clmul(golden):
    lo, hi = o.clmul64_lanes(golden["clmul_a"], golden["clmul_b"])
    assert np.array_equal(lo, golden["clmul_lo"]) and np.array_equal(hi, golden["clmul_hi"])
    lo, hi = oracle.c_clmul64(golden["clmul_a"], golden["clmul_b"])
    assert np.array_equal(lo, golden["clmul_lo"]) and np.array_equal(hi, golden["clmul_hi"])


def test_golden_full_products(golden):
    for t in golden["full_ts"]:
        A, B, C = golden[f"full_t{t}_A"], golden[f"full_t{t}_B"], golden[f"full_t{t}_C"]
        assert np.array_equal(oracle.c_mul_full(A, B), C), t
        if t <= 256:
            assert np.array_equal(o.mul_full(A, B), C), t


def test_golden_both_routes(golden):
    """spread (reference default for t > 48) and convolution routes agree,
    as the reference asserts at test_poly.py:269-284."""
    for t in (49, 64, 100, 193, 256):
        A, B, C = golden[f"full_t{t}_A"], golden[f"full_t{t}_B"], golden[f"full_t{t}_C"]
        for r in range(A.shape[0]):
            assert np.array_equal(o.mul_spread(A[r], B[r]), C[r])
            assert np.array_equal(o.mul_convolution(A[r], B[r]), C[r])


def test_golden_cyclic(golden):
    for n in golden["cyc_ns"]:
        n = int(n)
        A, B, C = golden[f"cyc_n{n}_A"], golden[f"cyc_n{n}_B"], golden[f"cyc_n{n}_C"]
        assert np.array_equal(oracle.c_mul_cyclic(A, B, n), C), n
        if n <= 20000:
            assert np.array_equal(o.mul_cyclic(A, B, n), C), n


@pytest.mark.parametrize("n", [1, 5, 63, 64, 65, 130, 200])
def test_fold_matches_rotation_sum(n, rng):
    """R = sum_i a_i X^i * B rotated: the ring product by definition."""
    t = (n + 63) // 64
    for _ in range(3):
        a = int(rng.integers(0, 1 << 62)) ** 4 % (1 << n)
        b = int(rng.integers(0, 1 << 62)) ** 3 % (1 << n)
        want = 0
        for i in range(n):
            if a >> i & 1:
                rot = ((b << i) | (b >> (n - i))) & ((1 << n) - 1) if i else b
                want ^= rot
        A = np.frombuffer(a.to_bytes(8 * t, "little"), dtype=np.uint64).reshape(1, t)
        B = np.frombuffer(b.to_bytes(8 * t, "little"), dtype=np.uint64).reshape(1, t)
        got = o.mul_cyclic(A, B, n)
        assert int.from_bytes(got.tobytes(), "little") == want
        assert np.array_equal(oracle.c_mul_cyclic(A, B, n), got)


def test_ring_identities():
    # SPEC.md:351-352
    for n in (17669, 35851):
        t = (n + 63) // 64
        A, _ = o.make_cyclic_inputs(n, 2)
        one = np.zeros_like(A)
        one[:, 0] = 1
        assert np.array_equal(oracle.c_mul_cyclic(A, one, n), A)
        x = np.zeros((1, t), dtype=np.uint64)
        x[0, 0] = 2
        xn1 = np.zeros((1, t), dtype=np.uint64)
        xn1[0, (n - 1) // 64] = np.uint64(1 << ((n - 1) % 64))
        r = oracle.c_mul_cyclic(xn1, x, n)
        assert int(r[0, 0]) == 1 and not r[0, 1:].any()


def test_top_bits_rejected():
    A, B = o.make_cyclic_inputs(1000, 2)
    B[1, -1] |= np.uint64(1 << (1000 % 64))
    with pytest.raises(ValueError):
        o.mul_cyclic(A, B, 1000)
    with pytest.raises(ValueError):
        oracle.c_mul_cyclic(A, B, 1000)


def test_hex_round_trip_and_format():
    # test_poly.py:120-127
    assert o.to_hex(np.array([1, 2], dtype=np.uint64)) == "0000000000000002" "0000000000000001"
    w = np.array([0xDEADBEEF, 0, 1 << 63], dtype=np.uint64)
    assert np.array_equal(o.from_hex(o.to_hex(w)), w)
    for bad in ("", "123", "0000000000000001Z000000000000000", "000000000000000A" * 2):
        with pytest.raises(ValueError):
            o.from_hex(bad)


def test_generator_matches_reference_fixture_recipe():
    """make_*_inputs follow conftest.py:40-46 (rng.integers(0, 1<<64, ...)) keyed
    by [0xF2F2, size]; cyclic rows have bits >= n cleared."""
    A, B = o.make_cyclic_inputs(17669, 8)
    rng = np.random.default_rng([0xF2F2, 17669])
    A2 = rng.integers(0, 1 << 64, size=(8, 277), dtype=np.uint64)
    A2[:, -1] &= np.uint64((1 << (17669 - 64 * 276)) - 1)
    assert np.array_equal(A, A2)
    assert not (B[:, -1] >> np.uint64(17669 - 64 * 276)).any()
