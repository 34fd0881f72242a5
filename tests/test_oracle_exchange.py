"""Pins for oracle.exchange (A6, A7, P18, P19).  CPU only."""
import numpy as np

from oracle.codec import roundtrip
from oracle.exchange import combine, owner_reduce_trunc16
from synth import rng


def test_n1_is_identity_no_codec():
    # Reading A6: N = 1 has no channel, hence no compression.
    g = rng(1).standard_normal(1000).astype(np.float32)
    assert np.array_equal(combine([g], "TRUNC16"), g)
    assert np.array_equal(combine([g], "FP32"), g)


def test_trunc16_hand_values():
    # Worked by hand from PAPER.md:813-821 with reading A6 (two truncations):
    #  elem0: g = (1.0, 3.0): both exact in 7 mantissa bits -> mean 2.0 -> 2.0
    #  elem1: g = (pi, 1.0): trunc(pi) = 3.140625; (3.140625 + 1)/2 = 2.0703125
    #         = 2 * (1 + 9/256); 9/256 needs 8 mantissa bits -> truncates to 2 * (1 + 8/256) = 2.0625
    #  elem2: g = (-0.5, 0.25): (-0.25)/2 = -0.125 exact
    g0 = np.array([1.0, 3.1415927, -0.5], np.float32)
    g1 = np.array([3.0, 1.0, 0.25], np.float32)
    assert combine([g0, g1], "TRUNC16").tolist() == [2.0, 2.0625, -0.125]
    # FP32 combine keeps full precision: (pi + 1)/2 in fp32
    assert combine([g0, g1], "FP32")[1] == np.float32(np.float32(3.1415927) + np.float32(1.0)) * np.float32(0.5)


def test_trunc16_result_is_always_on_the_16bit_grid():
    gs = [rng(10 + r).standard_normal(4096).astype(np.float32) for r in range(4)]
    out = combine(gs, "TRUNC16")
    assert np.array_equal(roundtrip(out), out)


def test_p19_scale_by_reciprocal_equals_division():
    # fl32(s * (1/N)) == fl32(s / N) for N = 2, 4, 8 (power-of-two N, no underflow)
    s = rng(2).standard_normal(1_000_000).astype(np.float32)
    for n in (2, 4, 8):
        assert np.array_equal((s * np.float32(1.0 / n)).astype(np.float32), (s / np.float32(n)).astype(np.float32))


def test_trunc16_exact_when_sums_are_representable():
    # Values on a coarse grid: every fp32 partial sum is exact, so the result is
    # the exact mean, truncated (independent route: Python fractions).
    from fractions import Fraction
    g = rng(4)
    gs = [(g.integers(-64, 64, 512) * 2.0 ** -6).astype(np.float32) for _ in range(4)]
    out = combine(gs, "TRUNC16")
    exact = [sum(Fraction(float(v[i])) for v in gs) / 4 for i in range(512)]
    trunc_exact = roundtrip(np.array([float(e) for e in exact], np.float32))
    assert np.array_equal(out, trunc_exact)


def test_p18_truncation_statistical_signature():
    # One truncation stage has mean relative error -2^-8 E[1/m] ~ -2.82e-3 for
    # log-uniform magnitudes (m = significand in [1,2)); RNE would give ~0.
    g = rng(3)
    mag = np.exp(g.uniform(np.log(1e-6), np.log(1e2), 1_000_000)).astype(np.float32)
    x = mag * np.where(g.random(mag.size) < 0.5, -1, 1).astype(np.float32)
    rel = (roundtrip(x).astype(np.float64) - x) / np.abs(x.astype(np.float64))
    # sign-aware: truncation moves toward zero, so rel error on |x| is negative
    rel_mag = (np.abs(roundtrip(x)).astype(np.float64) - np.abs(x)) / np.abs(x)
    assert -3.0e-3 < rel_mag.mean() < -2.6e-3
    # Two stages (N = 8 exchange) vs the exact f64 mean:
    gs = [(x[i::8][:100000] * (1 + 0.01 * r)).astype(np.float32) for i, r in zip(range(8), range(8))]
    gs = [np.abs(v) for v in gs]
    out = combine(gs, "TRUNC16").astype(np.float64)
    exact = np.mean([v.astype(np.float64) for v in gs], axis=0)
    r2 = (out - exact) / exact
    assert -6.5e-3 < r2.mean() < -4.0e-3
    assert np.max(np.abs(r2)) < 2 * 2.0 ** -7 + 1e-6
