"""Constant-time check: the leaky positive control fails on
CPU; the GPU ring product passes the fixed-vs-random Welch test."""

import pytest


def test_leaky_control_fails():
    from paper_2201_10473_b200.ct_check import ct_check_leaky

    assert ct_check_leaky()["verdict"] == "fail"


def test_welch_identical_distributions_pass():
    import numpy as np

    from paper_2201_10473_b200.ct_check import THRESHOLD, welch_t

    rng = np.random.default_rng(1)
    assert abs(welch_t(rng.normal(size=5000), rng.normal(size=5000))) < THRESHOLD


def test_leaky_mul_is_correct():
    from oracle.f2x_oracle import make_cyclic_inputs, mul_cyclic
    from paper_2201_10473_b200.ct_check import leaky_mul

    n = 300
    A, B = make_cyclic_inputs(n, 2)
    a = int.from_bytes(A[0].tobytes(), "little")
    b = int.from_bytes(B[0].tobytes(), "little")
    want = int.from_bytes(mul_cyclic(A[:1], B[:1], n).tobytes(), "little")
    assert leaky_mul(a, b, n) == want


@pytest.mark.gpu
def test_gpu_ring_mul_constant_time(cuda):
    from paper_2201_10473_b200.ct_check import ct_check

    r = ct_check(n=17669, weight=75, trials=1500)
    if r["verdict"] != "pass":  # flaky-tolerant: one retry
        r = ct_check(n=17669, weight=75, trials=1500, seed=0xC9)
    assert r["verdict"] == "pass", r
