"""Ring multiplication mod X^N - 1 (SPEC ``ring`` module).

The reference package does not ship this module; its contract is restated
from the SPEC: dense product then ONE fold (deg <= 2N-2), inputs with bits
>= N rejected (never masked), output bits >= N zero, HQC presets at
N in {17669, 35851, 57637}.  Here the fold is fused into the GPU kernel that
transposes the product back to packed words (k4_unslice), and the top-bit
check into the kernel that slices the inputs (k1_slice).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .poly import PolyWords

__all__ = ["RingParams", "preset", "ring_mul", "ring_mul_batch", "sparse_to_dense", "PRESETS"]

# SPEC.md:354-360 / PAPER Table 8: level -> (N, paper plan size, w) per backend class
PRESETS = {
    "hqc-128": {"N": 17669, "paper_plan": {"128-lane": (18048, 64), "multi-lane": (18048, 64)}},
    "hqc-192": {"N": 35851, "paper_plan": {"128-lane": (36480, 64), "multi-lane": (36480, 64)}},
    "hqc-256": {"N": 57637, "paper_plan": {"128-lane": (59904, 256), "multi-lane": (58368, 512)}},
}


@dataclass(frozen=True)
class RingParams:
    """N: ring degree; words = ceil(N/64); paper_plan: the SPEC/Table-8 CPU
    plan text for reference; engine_plan: what the GPU executes for one
    product (leaf size, Karatsuba levels, padded N)."""

    N: int
    words: int
    paper_plan: str = ""
    engine_plan: dict = field(default_factory=dict, compare=False, hash=False)

    @classmethod
    def for_degree(cls, N: int) -> "RingParams":
        if N < 1:
            raise ValueError("ring degree must be >= 1")
        return cls(N=N, words=(N + 63) // 64)


def preset(level: str, backend_class: str = "multi-lane") -> RingParams:
    """HQC presets."""
    if level not in PRESETS:
        raise ValueError(f"unknown preset {level!r}; expected one of {sorted(PRESETS)}")
    if backend_class not in ("128-lane", "multi-lane"):
        raise ValueError("backend_class must be '128-lane' or 'multi-lane'")
    N = PRESETS[level]["N"]
    size, w = PRESETS[level]["paper_plan"][backend_class]
    elem = "karat5" if level == "hqc-256" else "karat3"
    text = f"toom3[w={w}]({elem}(karatrec(kernel:karat512_sb)))@{size}"
    try:
        from .engine import plan

        eplan = plan("cyclic", 1, N)
    except Exception:  # library not built: presets still describe the ring
        eplan = {}
    return RingParams(N=N, words=(N + 63) // 64, paper_plan=text, engine_plan=eplan)


def _params(p) -> RingParams:
    if isinstance(p, RingParams):
        return p
    return RingParams.for_degree(int(p))


def ring_mul(A: PolyWords, B: PolyWords, p) -> PolyWords:
    """A * B mod X^N - 1 for one pair of ceil(N/64)-word operands."""
    from .engine import one_product
    from .poly import _device

    rp = _params(p)
    if A.word_len != rp.words or B.word_len != rp.words:
        raise ValueError(f"ring operands need {rp.words} words for N={rp.N}")
    return PolyWords(one_product("cyclic", A.words, B.words, rp.N, _device()))


def ring_mul_batch(A, B, p):
    """Batched form over torch CUDA word tensors [batch, ceil(N/64)]."""
    from .engine import mul_cyclic

    return mul_cyclic(A, B, _params(p).N)


def sparse_to_dense(support, N: int) -> PolyWords:
    """Support list -> dense ring element.  Every index updates every word
    through a mask, so the touched memory depends only on (weight, N)."""
    words = (N + 63) // 64
    out = np.zeros(words, dtype=np.uint64)
    idx = np.arange(words, dtype=np.int64)
    for s in support:
        s = int(s)
        if not 0 <= s < N:
            raise ValueError("support index outside [0, N)")
        sel = (idx == (s >> 6)).astype(np.uint64)
        out |= sel * np.uint64(1 << (s & 63))
    return PolyWords(out)
