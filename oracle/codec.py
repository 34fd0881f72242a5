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
