"""CPU ORACLE package -- test infrastructure, never the product path.

``f2x_oracle`` (numpy / Python int) restates the reference's multiply path
(poly.py) and the SPEC ring fold; ``c_oracle`` binds the C restatement in
``f2x_oracle.c`` (built by ``make -C oracle``) for fast checking of large
batches and for the timed CPU baseline.  Only tests/, __graft_entry__.smoke()
and bench.py's CPU legs may import this package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import f2x_oracle  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libf2x_oracle.so")
_lib = None


def build() -> str:
    src = os.path.join(_HERE, "f2x_oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


REF_ROOT = "/root/reference"
REF_TESTS = os.path.join(_HERE, "_ref", "ref_tests")


def stage_reference_tests() -> str | None:
    """Stage the reference's OWN unit tests (pkg/tests/conftest.py,
    test_poly.py), unmodified, into oracle/_ref/ref_tests/ when the reference
    tree is present (this container).  oracle/_ref/ is git-ignored (kept out
    of history) but travels to the GPU box with the snapshot, where
    tests/test_reference_suite.py runs them against the drop-in through
    tests/ref_shim/f2xmul.  Returns the staged directory or None."""
    import shutil

    src = os.path.join(REF_ROOT, "pkg", "tests")
    if not os.path.isdir(src):
        return REF_TESTS if os.path.isdir(REF_TESTS) else None
    os.makedirs(REF_TESTS, exist_ok=True)
    for f in ("conftest.py", "test_poly.py"):
        shutil.copyfile(os.path.join(src, f), os.path.join(REF_TESTS, f))
    return REF_TESTS


def c_oracle():
    """Load (building if needed) the C oracle library."""
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        p = ctypes.c_void_p
        lib.f2x_oracle_mul_full.argtypes = [p, p, p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
        lib.f2x_oracle_mul_cyclic.argtypes = [p, p, p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
        lib.f2x_oracle_clmul64.argtypes = [p, p, p, p, ctypes.c_int64, ctypes.c_int]
        lib.f2x_oracle_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def c_mul_full(A: np.ndarray, B: np.ndarray, threads: int = 0) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint64)
    B = np.ascontiguousarray(B, dtype=np.uint64)
    if A.ndim != 2 or A.shape != B.shape or A.shape[1] < 1:
        raise ValueError("A and B must be equal-shape uint64[batch][t], t >= 1")
    C = np.zeros((A.shape[0], 2 * A.shape[1]), dtype=np.uint64)
    rc = c_oracle().f2x_oracle_mul_full(_ptr(A), _ptr(B), _ptr(C), A.shape[0], A.shape[1], threads)
    if rc:
        raise ValueError(f"oracle mul_full failed ({rc})")
    return C


def c_mul_cyclic(A: np.ndarray, B: np.ndarray, n: int, threads: int = 0) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint64)
    B = np.ascontiguousarray(B, dtype=np.uint64)
    t = (n + 63) // 64
    if A.ndim != 2 or A.shape != B.shape or A.shape[1] != t:
        raise ValueError(f"A and B must be equal-shape uint64[batch][{t}]")
    C = np.zeros_like(A)
    rc = c_oracle().f2x_oracle_mul_cyclic(_ptr(A), _ptr(B), _ptr(C), A.shape[0], n, threads)
    if rc == -2:
        raise ValueError("operand has bits set at or above n")
    if rc:
        raise ValueError(f"oracle mul_cyclic failed ({rc})")
    return C


def c_clmul64(a: np.ndarray, b: np.ndarray, portable: bool = False):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    lo = np.zeros_like(a)
    hi = np.zeros_like(a)
    c_oracle().f2x_oracle_clmul64(_ptr(a), _ptr(b), _ptr(lo), _ptr(hi), a.size, int(portable))
    return lo, hi
