"""B200-native batched constant-time dense GF(2)[X] multiplication.

Drop-in for the multiply path of the reference package ``f2xmul``
(/root/reference/pkg/src/f2xmul/__init__.py:9-21): same value types, entry
points and packed little-endian uint64 layout, computed by hand-written
sm_100a kernels (libf2x.so, C ABI in include/f2x.h).  Batched device API:
``mul_full`` / ``mul_cyclic`` over torch CUDA tensors.
"""

from .poly import (
    BackendId,
    MulCounters,
    PolyWords,
    WideProduct,
    backend_select,
    clmul64,
    clmul64_batch,
    from_hex,
    schoolbook_mul,
    to_hex,
)
from .ring import RingParams, preset, ring_mul, ring_mul_batch, sparse_to_dense

__version__ = "0.1.0"

__all__ = [
    "BackendId",
    "MulCounters",
    "PolyWords",
    "WideProduct",
    "backend_select",
    "clmul64",
    "clmul64_batch",
    "from_hex",
    "schoolbook_mul",
    "to_hex",
    "RingParams",
    "preset",
    "ring_mul",
    "ring_mul_batch",
    "sparse_to_dense",
    "mul_full",
    "mul_cyclic",
    "plan",
]


def __getattr__(name):
    # engine pulls in torch; import lazily so value types work without it
    if name in ("mul_full", "mul_cyclic", "plan", "clmul64_lanes"):
        from . import engine

        return getattr(engine, name)
    raise AttributeError(name)
