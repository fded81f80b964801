"""ctypes binding of the C ABI in include/f2x.h (libf2x.so, built in-tree).

There is no fallback: if the library is missing or fails to load, every
entry point raises.  The library is the only compute path of this package.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libf2x.so")
# F2X_LIB_VARIANT=leaky|checked loads a TEST FIXTURE built from the same
# sources (build.py VARIANTS) instead: used only by the constant-time
# positive control and the shared-memory initcheck tests, each in its own
# process
_VARIANT = os.environ.get("F2X_LIB_VARIANT")
if _VARIANT in ("leaky", "checked"):
    LIB_PATH = os.path.join(HERE, f"_build_{_VARIANT}", f"libf2x_{_VARIANT}.so")

F2X_OK = 0
F2X_EINVAL = -22
F2X_ENOSPC = -28
F2X_ERANGE = -34
F2X_ECUDA = -1000
KIND_FULL = 0
KIND_CYCLIC = 1

EXPORTS = (
    "f2x_make_plan",
    "f2x_plan_cost",
    "f2x_workspace_bytes",
    "f2x_mul_full",
    "f2x_mul_cyclic",
    "f2x_clmul64",
    "f2x_set_node_events",
    "f2x_bench_lop3",
    "f2x_strerror",
    "f2x_version",
)


class F2xPlan(ctypes.Structure):
    """Mirror of ``struct f2x_plan`` (include/f2x.h)."""

    _fields_ = [
        ("kind", ctypes.c_int32),
        ("t", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("N", ctypes.c_int32),
        ("batch", ctypes.c_int64),
        ("groups", ctypes.c_int64),
        ("leaf_words", ctypes.c_int32),
        ("leaf_stride", ctypes.c_int32),
        ("levels", ctypes.c_int32),
        ("cta_levels", ctypes.c_int32),
        ("global_levels", ctypes.c_int32),
        ("num_passes", ctypes.c_int32),
        ("pass_levels", ctypes.c_int32 * 8),
        ("launches", ctypes.c_int32),
        ("cta_threads", ctypes.c_int32),
        ("node_ctas", ctypes.c_int64),
        ("node_smem_bytes", ctypes.c_int64),
        ("workspace_bytes", ctypes.c_int64),
        ("leaf_ops_per_product", ctypes.c_double),
        ("karatsuba_ops_per_product", ctypes.c_double),
        ("eval_levels", ctypes.c_int32),
        ("toom_levels", ctypes.c_int32),
        ("toom_w", ctypes.c_int32),
        ("toom_M", ctypes.c_int32 * 4),
        ("toom_w_last", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_}
        d["pass_levels"] = list(self.pass_levels)[: self.num_passes]
        d["toom_M"] = list(self.toom_M)[: self.toom_levels]
        return d


_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libf2x.so; raises ImportError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2201_10473_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        lib.f2x_make_plan.argtypes = [i32, i64, i32, i32, ctypes.POINTER(F2xPlan)]
        lib.f2x_make_plan.restype = ctypes.c_int
        lib.f2x_plan_cost.argtypes = [i32, i64, i32, i32]
        lib.f2x_plan_cost.restype = ctypes.c_double
        lib.f2x_workspace_bytes.argtypes = [i32, i64, i32, i32]
        lib.f2x_workspace_bytes.restype = i64
        lib.f2x_mul_full.argtypes = [vp, vp, vp, i64, i32, vp, sz, i32, vp]
        lib.f2x_mul_full.restype = ctypes.c_int
        lib.f2x_mul_cyclic.argtypes = [vp, vp, vp, i64, i32, vp, sz, i32, vp, vp]
        lib.f2x_mul_cyclic.restype = ctypes.c_int
        lib.f2x_clmul64.argtypes = [vp, vp, vp, i64, vp, sz, vp]
        lib.f2x_clmul64.restype = ctypes.c_int
        lib.f2x_set_node_events.argtypes = [vp, vp]
        lib.f2x_set_node_events.restype = ctypes.c_int
        lib.f2x_bench_lop3.argtypes = [vp, i32, i32, vp]
        lib.f2x_bench_lop3.restype = ctypes.c_int
        lib.f2x_strerror.argtypes = [ctypes.c_int]
        lib.f2x_strerror.restype = ctypes.c_char_p
        lib.f2x_version.argtypes = []
        lib.f2x_version.restype = ctypes.c_int
        _lib = lib
    return _lib


def strerror(code: int) -> str:
    return load().f2x_strerror(int(code)).decode()


def check(code: int, what: str) -> None:
    if code == F2X_OK:
        return
    msg = f"{what}: {strerror(code)} (code {code})"
    if code in (F2X_EINVAL, F2X_ERANGE):
        raise ValueError(msg)
    raise RuntimeError(msg)


def make_plan(kind: int, batch: int, t_or_n: int, leaf: int = 0) -> F2xPlan:
    pl = F2xPlan()
    check(load().f2x_make_plan(kind, batch, t_or_n, leaf, ctypes.byref(pl)), "f2x_make_plan")
    return pl
