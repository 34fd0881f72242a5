"""Pins for oracle.codec (P1, P2-subset, P3, A8).  CPU only."""
import math
import os
import struct

import numpy as np
import pytest

from oracle.codec import expand16, roundtrip, truncate16
from synth import random_f32_bits

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "codec_worked_values.txt")


def _golden():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        a, b, c = line.split()
        rows.append((int(a, 16), int(b, 16), float(c)))
    return rows


def test_p1_worked_values():
    for bits, q, val in _golden():
        x = np.array([bits], dtype=np.uint32).view(np.float32)
        assert int(truncate16(x)[0]) == q, hex(bits)
        r = float(expand16(np.array([q], np.uint16))[0])
        assert r == val and math.copysign(1, r) == math.copysign(1, val), hex(bits)


def test_p1_pi_and_decimal():
    # SPEC.md:688 "3.1415927 -> 3.140625"
    assert float(roundtrip(np.array([3.1415927], np.float32))[0]) == 3.140625


def test_powers_of_two_exact():
    # SPEC.md:687 "1.0 and every power of two round-trip exactly"
    # (normals and the subnormals whose set bit lies in the kept top 7 mantissa
    # bits, i.e. >= 2^-133; smaller ones truncate to zero, reading A8)
    e = np.arange(-133, 128)
    x = np.ldexp(1.0, e).astype(np.float32)
    assert np.array_equal(roundtrip(x), x)
    assert np.array_equal(roundtrip(-x), -x)
    tiny = np.ldexp(1.0, np.arange(-149, -133)).astype(np.float32)
    assert np.all(roundtrip(tiny) == 0)


def test_exhaustive_u16_expand_then_truncate_is_identity():
    q = np.arange(2 ** 16, dtype=np.uint32).astype(np.uint16)
    assert np.array_equal(truncate16(expand16(q)), q)


def _struct_trunc(v: float) -> int:
    """Independent route: high two bytes of the big-endian binary32 encoding."""
    b = struct.pack(">f", v)
    return (b[0] << 8) | b[1]


def test_matches_byte_level_definition_on_random_patterns():
    x = random_f32_bits(20000)
    ours = truncate16(x)
    for v, q in zip(x[:20000], ours[:20000]):
        if np.isnan(v):
            continue  # struct may canonicalise NaN payloads
        assert _struct_trunc(float(v)) == int(q)


def test_p3_invariants_on_normals():
    # |rt(x) - x| / |x| < 2^-7 for finite normals; |rt(x)| <= |x|; same sign.
    x = random_f32_bits(1 << 20)
    finite = np.isfinite(x) & (np.abs(x) >= np.float32(2.0 ** -126))
    x = x[finite].astype(np.float64)
    r = roundtrip(x.astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(r) <= np.abs(x))
    assert np.all(np.sign(r) == np.sign(x))
    assert np.all(np.abs(r - x) < 2.0 ** -7 * np.abs(x))


def test_a8_special_values():
    nan_low = np.array([0x7F800001], np.uint32).view(np.float32)   # NaN with low-only payload
    nan_gpu = np.array([0x7FFFFFFF], np.uint32).view(np.float32)
    assert int(truncate16(nan_low)[0]) == 0x7F80 and np.isinf(roundtrip(nan_low)[0])
    assert np.isnan(roundtrip(nan_gpu)[0])
    assert int(truncate16(np.array([1e-45], np.float32))[0]) == 0x0000
    sub = np.array([0x00400000], np.uint32).view(np.float32)          # subnormal keeps top bits
    assert int(truncate16(sub)[0]) == 0x0040 and roundtrip(sub)[0] == sub[0]
