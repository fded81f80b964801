"""Reference-compatible value types and per-call entry points.

Mirrors the public surface of ``f2xmul.poly`` (/root/reference/pkg/src/
f2xmul/poly.py:47-59) with the same names, argument meaning and error
behaviour, so code written against the reference switches by import:

* ``PolyWords`` / ``WideProduct`` -- immutable little-endian uint64 word
  polynomials with explicit length, padding-insensitive equality
  (poly.py:70-175);
* ``schoolbook_mul(a, b)`` -> ``WideProduct`` of 2t words (poly.py:547-561);
* ``clmul64`` / ``clmul64_batch`` (poly.py:311-327, 451-480);
* ``to_hex`` / ``from_hex`` (poly.py:569-584).

Every multiply runs on the GPU through libf2x.so (one batched launch
sequence per call; per-product calls are a batch of one).  There is no CPU
arithmetic path.  The reference's lane-level backend seam (``BackendId``,
``backend_select``, ``set_backend_override``, ``F2XMUL_BACKEND``,
poly.py:208-253) selects between bit-identical CPU recipes; here the
selection logic is kept verbatim in behaviour (override, then environment,
then the two machine probes) but every name maps to the single device path.
``MulCounters`` keeps the reference's accounting (poly.py:451-514: one base
multiplication per 64x64 lane, t*t of them and 2 t^2 word XORs per counted
t-word product); the work the GPU plan actually executes is reported by
``engine.plan`` (``leaf_ops_per_product``, ``karatsuba_ops_per_product``).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Optional, Sequence, Union

import numpy as np
import os

__all__ = [
    "PolyWords",
    "WideProduct",
    "MulCounters",
    "BackendId",
    "backend_select",
    "set_backend_override",
    "clmul64",
    "clmul64_batch",
    "schoolbook_mul",
    "to_hex",
    "from_hex",
]

_MASK64 = (1 << 64) - 1


class PolyWords:
    """Dense F2[X] polynomial with an explicit word length (t >= 1).

    Value semantics follow poly.py:70-171: immutable read-only backing array,
    equality after zero-extension, hash on the trimmed words.
    """

    __slots__ = ("words",)

    def __init__(self, words: Union[Sequence[int], np.ndarray]):
        arr = np.array(words, dtype=np.uint64)  # always a private copy
        if arr.ndim != 1:
            raise ValueError("words must be one-dimensional")
        if arr.size == 0:
            raise ValueError("zero-length polynomials are rejected; need t >= 1")
        arr.flags.writeable = False
        object.__setattr__(self, "words", arr)

    def __setattr__(self, name, value):
        raise AttributeError("PolyWords is immutable")

    @property
    def word_len(self) -> int:
        return int(self.words.size)

    @property
    def bit_capacity(self) -> int:
        return 64 * self.word_len

    @classmethod
    def zero(cls, word_len: int) -> "PolyWords":
        return cls(np.zeros(word_len, dtype=np.uint64))

    @classmethod
    def one(cls, word_len: int = 1) -> "PolyWords":
        w = np.zeros(word_len, dtype=np.uint64)
        w[0] = 1
        return cls(w)

    @classmethod
    def from_int(cls, value: int, word_len: Optional[int] = None) -> "PolyWords":
        if value < 0:
            raise ValueError("polynomial integers are non-negative")
        need = max(1, -(-value.bit_length() // 64))
        if word_len is None:
            word_len = need
        if word_len < need:
            raise ValueError(f"value needs {need} words, got word_len={word_len}")
        return cls(np.frombuffer(value.to_bytes(8 * word_len, "little"), dtype=np.uint64))

    def to_int(self) -> int:
        return int.from_bytes(self.words.tobytes(), "little")

    def degree(self) -> int:
        """Degree, or -1 for the zero polynomial."""
        nz = np.nonzero(self.words)[0]
        if nz.size == 0:
            return -1
        top = int(nz[-1])
        return 64 * top + int(self.words[top]).bit_length() - 1

    def padded(self, word_len: int) -> "PolyWords":
        if word_len < self.word_len:
            raise ValueError("padded() cannot shrink; use truncated()")
        w = np.zeros(word_len, dtype=np.uint64)
        w[: self.word_len] = self.words
        return type(self)(w)

    def truncated(self, word_len: int) -> "PolyWords":
        """Drop words at and above word_len; they must all be zero."""
        if word_len >= self.word_len:
            return self.padded(word_len)
        if self.words[word_len:].any():
            raise ValueError("truncation would drop nonzero words")
        return type(self)(self.words[:word_len])

    def __xor__(self, other: "PolyWords") -> "PolyWords":
        m = max(self.word_len, other.word_len)
        w = np.zeros(m, dtype=np.uint64)
        w[: self.word_len] ^= self.words
        w[: other.word_len] ^= other.words
        return PolyWords(w)

    def __eq__(self, other) -> bool:
        if not isinstance(other, PolyWords):
            return NotImplemented
        a, b = self.words, other.words
        k = min(a.size, b.size)
        return bool(np.array_equal(a[:k], b[:k]) and not a[k:].any() and not b[k:].any())

    def __hash__(self):
        nz = np.nonzero(self.words)[0]
        end = int(nz[-1]) + 1 if nz.size else 0
        return hash(self.words[:end].tobytes())

    def __repr__(self):
        return f"PolyWords(t={self.word_len}, hex={to_hex(self)})"


class WideProduct(PolyWords):
    """A product: 2t words for t-word operands."""


@dataclass
class MulCounters:
    """Per-call work record with the reference's semantics (poly.py:178-200):
    ``base_mul_count`` = 64x64 word products of the schoolbook convolution
    (t*t per t-word product, one per clmul lane), ``xor64_count`` = its 2 t^2
    word XORs."""

    base_mul_count: int = 0
    xor64_count: int = 0

    def reset(self) -> None:
        self.base_mul_count = 0
        self.xor64_count = 0

    def add_muls(self, n: int) -> None:
        self.base_mul_count += int(n)

    def add_xors(self, n: int) -> None:
        self.xor64_count += int(n)


class BackendId(Enum):
    """Backend names of poly.py:208-211.  All reference backends are
    bit-identical by contract (test_poly.py:156-164); every name selects the
    single device path of this package."""

    PORTABLE = "portable"
    CLMUL = "clmul"
    MULTILANE = "multilane"


_BACKEND_ENV = "F2XMUL_BACKEND"
_backend_override: Optional[BackendId] = None


def set_backend_override(backend: Optional[Union[BackendId, str]]) -> None:
    """Force a backend name for subsequent operations (None restores
    detection), as poly.py:217-223; unknown names raise ValueError."""
    global _backend_override
    if backend is None:
        _backend_override = None
    else:
        _backend_override = backend if isinstance(backend, BackendId) else BackendId(backend)


def _machine_supports_wide_mul() -> bool:
    """Probe seam (poly.py:226-231): the batched lane machinery here is the
    GPU engine, always present when the package imports."""
    return True


def _int_mul_selfcheck() -> bool:
    """Probe seam (poly.py:300-303).  The device leaf has no integer-multiply
    recipe to self-check; kept so callers and tests can patch it."""
    return True


def backend_select() -> BackendId:
    """Backend name with the reference's priority (poly.py:234-246): explicit
    override, then ``F2XMUL_BACKEND`` (portable/clmul/multilane/auto), then
    the machine probes.  The name does not change the arithmetic."""
    if _backend_override is not None:
        return _backend_override
    env = os.environ.get(_BACKEND_ENV, "").strip().lower()
    if env and env != "auto":
        return BackendId(env)
    if _machine_supports_wide_mul():
        return BackendId.MULTILANE
    return BackendId.CLMUL if _int_mul_selfcheck() else BackendId.PORTABLE


def _validate_backend(backend) -> None:
    if backend is None:
        backend_select()  # an invalid F2XMUL_BACKEND raises ValueError, as poly.py:249-253
    elif not isinstance(backend, BackendId):
        BackendId(backend)  # raises ValueError on unknown names


def _device():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: this package only computes on the GPU")
    return torch.device("cuda", torch.cuda.current_device())


def _count_convolution(counters: Optional[MulCounters], t: int, batch: int = 1) -> None:
    """The reference's counted-path accounting (poly.py:493-514): t*t lane
    products and 2 t^2 word XORs per t-word product."""
    if counters is None:
        return
    counters.add_muls(batch * t * t)
    counters.add_xors(batch * 2 * t * t)


def clmul64(a: int, b: int, counters: Optional[MulCounters] = None,
            backend: Optional[Union[BackendId, str]] = None) -> tuple[int, int]:
    """Carry-less 64x64 -> 128 product as (low word, high word) (poly.py:311-327)."""
    if not (0 <= a <= _MASK64 and 0 <= b <= _MASK64):
        raise ValueError("operands must be 64-bit words")
    _validate_backend(backend)
    lo, hi = clmul64_batch(np.array([a], dtype=np.uint64), np.array([b], dtype=np.uint64))
    if counters is not None:
        counters.add_muls(1)
    return int(lo[0]), int(hi[0])


def clmul64_batch(a: np.ndarray, b: np.ndarray, counters: Optional[MulCounters] = None,
                  backend: Optional[Union[BackendId, str]] = None
                  ) -> tuple[np.ndarray, np.ndarray]:
    """Lane-wise carry-less products of equal-length uint64 arrays
    (poly.py:451-480); one GPU batch of t = 1 full products."""
    import torch

    from .engine import clmul64_lanes

    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    if a.shape != b.shape or a.ndim != 1:
        raise ValueError("lane arrays must be equal-length 1-D")
    _validate_backend(backend)
    if counters is not None:
        counters.add_muls(a.shape[0])
    if a.size == 0:
        return a.copy(), a.copy()
    dev = _device()
    lo, hi = clmul64_lanes(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev))
    return lo.cpu().numpy().copy(), hi.cpu().numpy().copy()


def _mul_words(aw: np.ndarray, bw: np.ndarray) -> np.ndarray:
    """One t-word product on the device (a cached captured call per t:
    engine.one_product); returns 2t uint64 words."""
    from .engine import one_product

    aw = np.ascontiguousarray(aw, dtype=np.uint64)
    bw = np.ascontiguousarray(bw, dtype=np.uint64)
    return one_product("full", aw, bw, aw.shape[0], _device())


def _convolution_mul_arrays(aw: np.ndarray, bw: np.ndarray, counters: Optional[MulCounters],
                            backend: Optional[Union[BackendId, str]]) -> np.ndarray:
    """The reference's counted route (poly.py:493-514) as a name: the device
    product, with the convolution's t*t / 2 t^2 accounting."""
    _validate_backend(backend)
    out = _mul_words(aw, bw)
    _count_convolution(counters, int(np.asarray(aw).shape[0]))
    return out


def _spread_mul_arrays(aw: np.ndarray, bw: np.ndarray) -> np.ndarray:
    """The reference's uncounted route (poly.py:517-544) as a name: the same
    device product (one path here; the two reference routes are
    bit-identical by contract, test_poly.py:225-239)."""
    return _mul_words(aw, bw)


def schoolbook_mul(a: PolyWords, b: PolyWords, counters: Optional[MulCounters] = None,
                   backend: Optional[Union[BackendId, str]] = None) -> WideProduct:
    """Exact F2[X] product of equal-length operands, 2t words (poly.py:547-561).
    With ``counters`` the reference's accounting is added: t*t base
    multiplications and 2 t^2 word XORs."""
    if a.word_len != b.word_len:
        raise ValueError(
            f"schoolbook_mul needs equal lengths, got {a.word_len} and {b.word_len}")
    _validate_backend(backend)
    out = _mul_words(a.words, b.words)
    _count_convolution(counters, a.word_len)
    return WideProduct(out)


def to_hex(p: PolyWords) -> str:
    """Lowercase hex, most-significant word first, 16 digits per word."""
    return "".join(format(int(w), "016x") for w in reversed(p.words))


def from_hex(s: str) -> PolyWords:
    """Inverse of ``to_hex``; rejects empty, ragged, upper-case or non-hex input."""
    s = s.strip()
    if len(s) == 0 or len(s) % 16 != 0:
        raise ValueError("hex length must be a positive multiple of 16")
    if any(ch not in "0123456789abcdef" for ch in s):
        raise ValueError("hex polynomials must be lowercase, fixed width")
    words = [int(s[i:i + 16], 16) for i in range(0, len(s), 16)]
    return PolyWords(words[::-1])
