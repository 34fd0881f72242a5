"""Oracle 32->16->32 lossy codec.  TEST INFRASTRUCTURE ONLY.

PAPER.md §5.5 (:813-821): "convert 32-bit floating point representations into
a 16-bit floating point representation (not the proposed IEEE 16-bit floating
point standard, but rather just a 32-bit IEEE 794 float format, but with 16 bits
less precision in the mantissa), and then convert back to a 32-bit
representation on the other side of the communication channel (by just filling
in zeroes for the lost portion of the mantissa ...)".

Reading A5: keep the high half-word (1 sign, 8 exponent, 7 mantissa bits) —
truncation toward zero in magnitude; expansion zero-fills.  Reading A8: pure
bit operations, so +-Inf, -0 and subnormal top bits are kept; a NaN whose
payload lies only in the low 16 bits becomes +-Inf.
Parity: pinned by tests/test_oracle_codec.py (P1 worked values, P3
invariants, exhaustive 2^16 expansion round trip).

Stochastic rounding (PAPER.md:819-821 names it: "the
mathematically correct probabilistic rounding" the paper chose not to do).
Reading A26: with u = bits(x) and r uniform on [0, 2^16), q = (u + r) >> 16
rounds |x| up to the next 16-bit value with probability (u & 0xFFFF) / 2^16 and
down otherwise, so E[expand(q)] = x (a carry into the exponent is the next
binade, as it should be).  Non-finite inputs (exponent all ones) are truncated
as in TRUNC16.  Reading A27: r comes from a counter-based generator both sides
implement independently — mix32 (an xorshift-multiply 32-bit mixer) of
(bucket index XOR key), upper 16 bits; key = mix32 chain of (seed, step, layer,
stage, rank).  Pinned by tests/test_oracle_codec.py (P20: r = 0 is truncation,
exhaustive-r round-up counts, exact unbiasedness; generator uniformity).
"""
from __future__ import annotations

import numpy as np


def truncate16(x) -> np.ndarray:
    """float32 array -> uint16 array: bits(x) >> 16."""
    bits = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return (bits >> np.uint32(16)).astype(np.uint16)


def expand16(q) -> np.ndarray:
    """uint16 array -> float32 array: bits = q << 16 (zero-filled low mantissa)."""
    return (np.asarray(q, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def roundtrip(x) -> np.ndarray:
    return expand16(truncate16(x))


# ---------------------------------------------------------------- stochastic rounding
_M32 = 0xFFFFFFFF


def mix32(x):
    """32-bit mixer on uint32 (numpy array or int), wrap-around arithmetic:
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16."""
    if isinstance(x, (int, np.integer)):
        x = int(x) & _M32
        x ^= x >> 16
        x = (x * 0x7FEB352D) & _M32
        x ^= x >> 15
        x = (x * 0x846CA68B) & _M32
        x ^= x >> 16
        return x
    x = np.asarray(x, dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint32(16)
        x *= np.uint32(0x7FEB352D)
        x ^= x >> np.uint32(15)
        x *= np.uint32(0x846CA68B)
        x ^= x >> np.uint32(16)
    return x


def sr_key(seed: int, step: int, layer: int, stage: int, rank: int) -> int:
    """Stream key of one compression point (reading A27): stage 0 = the sender's
    compression of its gradient (rank = sender), stage 1 = the owner's compression
    of the mean (rank = owner); step = 1-based exchange counter; layer = bucket id."""
    k = mix32((stage * 256 + rank) & _M32)
    k = mix32((layer & _M32) ^ k)
    k = mix32((step & _M32) ^ k)
    return mix32((seed & _M32) ^ k)


def sr_random(key: int, idx) -> np.ndarray:
    """The 16-bit uniform draw for bucket positions idx under `key`."""
    idx = np.asarray(idx, dtype=np.uint64).astype(np.uint32)
    return (mix32(idx ^ np.uint32(key)) >> np.uint32(16)).astype(np.uint32)


def sr16(x, r) -> np.ndarray:
    """float32 array, uint16-range randoms r -> uint16: (bits(x) + r) >> 16 for finite x,
    bits(x) >> 16 for +-Inf / NaN (reading A26)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = np.asarray(r, dtype=np.uint64)
    finite = (u & 0x7F800000) != 0x7F800000
    v = np.where(finite, u + r, u)
    return (v >> 16).astype(np.uint16)
