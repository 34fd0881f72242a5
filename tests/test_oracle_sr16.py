"""Pins for the stochastic-rounding codec (f2; readings A26-A28).  CPU only.

PAPER.md:819-821 names the alternative the paper declined: "the mathematically
correct probabilistic rounding".  Its definition fixes, for every finite x with
u = bits(x): the result is trunc16(x) or the next 16-bit value up in magnitude,
the round-up happens for exactly (u & 0xFFFF) of the 2^16 equally likely draws,
and so the expectation is x exactly.  These tests check the oracle against those
consequences, not against its own formula.
"""
from fractions import Fraction

import numpy as np

from oracle.codec import expand16, mix32, roundtrip, sr16, sr_key, sr_random, truncate16
from oracle.exchange import combine
from synth import random_f32_bits, rng

ALL_R = np.arange(1 << 16, dtype=np.uint32)


def _finite_samples(n=64):
    x = random_f32_bits(4 * n)
    x = x[np.isfinite(x)][:n]
    extra = np.array([1.0, -1.0, 2.0 ** -126, 2.0 ** -140, 3.1415927, 0.1, -0.0, 0.0], np.float32)
    edge = np.array([0x3FFFFFFF, 0x3F80FFFF, 0xBF80FFFF, 0x00008001, 0x7F7F7FFF], np.uint32).view(np.float32)
    return np.concatenate([x, extra, edge])


def test_p20_zero_draw_is_truncation():
    x = random_f32_bits(1 << 16)
    assert np.array_equal(sr16(x, np.zeros(x.size, np.uint32)), truncate16(x))


def test_p20_round_up_count_is_the_discarded_fraction_exhaustive_over_draws():
    for v in _finite_samples():
        u = int(np.array([v], np.float32).view(np.uint32)[0])
        q = sr16(np.full(ALL_R.size, v, np.float32), ALL_R).astype(np.int64)
        lo = u >> 16
        assert set(np.unique(q)).issubset({lo, lo + 1}), hex(u)
        assert int(np.count_nonzero(q == lo + 1)) == (u & 0xFFFF), hex(u)
        # the round-up value is the next 16-bit value in magnitude (same sign): |up| > |x| >= |down|
        if u & 0xFFFF:
            up = expand16(np.array([lo + 1], np.uint16))[0]
            assert abs(float(up)) > abs(float(v)) >= abs(float(roundtrip(np.array([v], np.float32))[0]))


def test_p20_unbiased_exactly_over_all_draws():
    # E_r[expand(sr16(x, r))] = x, checked in exact rational arithmetic (x below the
    # largest binade, so a round-up never overflows to Inf)
    for v in _finite_samples():
        if not np.isfinite(v) or abs(float(v)) >= 2.0 ** 127:
            continue
        q = sr16(np.full(ALL_R.size, v, np.float32), ALL_R)
        vals, counts = np.unique(q, return_counts=True)
        total = sum(Fraction(float(expand16(np.array([a], np.uint16))[0])) * int(c) for a, c in zip(vals, counts))
        assert total / (1 << 16) == Fraction(float(v)), float(v)


def test_p20_non_finite_is_truncated():
    specials = np.array([0x7F800000, 0xFF800000, 0x7FC00000, 0x7F800001, 0x7FFFFFFF], np.uint32).view(np.float32)
    for v in specials:
        q = sr16(np.full(ALL_R.size, v, np.float32), ALL_R)
        assert np.all(q == truncate16(np.array([v], np.float32))[0])


def test_p20_values_on_the_16bit_grid_are_unchanged():
    x = roundtrip(random_f32_bits(1 << 16))
    r = rng(7).integers(0, 1 << 16, x.size).astype(np.uint32)
    assert np.array_equal(sr16(x, r), truncate16(x))


def test_generator_uniform_and_decorrelated():
    r = sr_random(sr_key(1234, 1, 0, 0, 0), np.arange(1 << 20))
    assert r.min() >= 0 and r.max() < (1 << 16)
    hist = np.bincount(r >> 8, minlength=256).astype(np.float64)
    exp = r.size / 256
    chi2 = float(np.sum((hist - exp) ** 2 / exp))
    assert chi2 < 400, chi2  # 255 dof: mean 255, sd 22.6
    a, b = r[:-1].astype(np.float64), r[1:].astype(np.float64)
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.01
    # streams of different (step, layer, stage, rank) keys are unrelated
    keys = {sr_key(1234, s, l, st, k) for s in range(4) for l in range(4) for st in range(2) for k in range(8)}
    assert len(keys) == 4 * 4 * 2 * 8
    r2 = sr_random(sr_key(1234, 2, 0, 0, 0), np.arange(1 << 20))
    assert np.count_nonzero(r == r2) < 64


def test_mix32_is_a_bijection_on_a_slice():
    x = np.arange(1 << 22, dtype=np.uint32) * np.uint32(977)
    assert np.unique(mix32(x)).size == x.size
    assert mix32(0) == 0 and mix32(np.array([0], np.uint32))[0] == 0


def test_sr16_statistical_signature_vs_truncation():
    # P18's counterpart: truncation has mean relative error ~ -2.82e-3 per stage; the
    # probabilistic rounding's is ~0 (the paper's "mathematically correct" variant)
    g = rng(3)
    mag = np.exp(g.uniform(np.log(1e-6), np.log(1e2), 1_000_000)).astype(np.float32)
    x = mag * np.where(g.random(mag.size) < 0.5, -1, 1).astype(np.float32)
    r = sr_random(sr_key(99, 1, 0, 0, 0), np.arange(x.size))
    rel = (expand16(sr16(x, r)).astype(np.float64) - x) / x.astype(np.float64)
    rel_t = (roundtrip(x).astype(np.float64) - x) / x.astype(np.float64)
    assert abs(rel.mean()) < 2e-5, rel.mean()
    assert rel_t.mean() < -2.5e-3
    assert np.max(np.abs(rel)) < 2.0 ** -7


def test_sr16_combine_n1_identity_and_grid():
    g = rng(1).standard_normal(1000).astype(np.float32)
    assert np.array_equal(combine([g], "SR16", sr=(5, 1, 0)), g)  # reading A6: N = 1 has no channel
    gs = [rng(10 + r).standard_normal(4099).astype(np.float32) for r in range(4)]
    out = combine(gs, "SR16", sr=(5, 1, 0))
    assert np.array_equal(roundtrip(out), out)


def test_sr16_combine_equals_trunc16_when_everything_is_on_the_grid():
    # inputs on a coarse grid whose mean is exactly representable in 16 bits: no draw can
    # change anything (P12-style exact regime)
    g = rng(4)
    gs = [(g.integers(-64, 64, 512) * 2.0 ** -6).astype(np.float32) for _ in range(4)]
    assert np.array_equal(combine(gs, "SR16", sr=(5, 3, 1)), combine(gs, "TRUNC16"))


def test_sr16_combine_two_stages_unbiased():
    # two stochastic stages (sender, owner): mean relative error of g_hat vs the exact
    # f64 mean ~ 0, against ~ -5.3e-3 for TRUNC16 (P18, N = 4)
    g = rng(8)
    n = 4
    base = np.exp(g.uniform(np.log(1e-4), np.log(1e1), 250_000))
    gs = [(base * (1 + 0.1 * g.standard_normal(base.size))).astype(np.float32) for _ in range(n)]
    exact = np.mean([x.astype(np.float64) for x in gs], axis=0)
    sr = (combine(gs, "SR16", sr=(11, 1, 0)).astype(np.float64) - exact) / np.abs(exact)
    tr = (combine(gs, "TRUNC16").astype(np.float64) - exact) / np.abs(exact)
    assert abs(sr.mean()) < 1e-4, sr.mean()
    assert tr.mean() < -4e-3, tr.mean()


def test_sr16_combine_uses_the_owner_stream_per_shard():
    # the owner's draw depends on who owns the element: shard = ceil(P / 8N) * 8
    n, p = 2, 1000
    gs = [rng(20 + r).standard_normal(p).astype(np.float32) for r in range(n)]
    a = combine(gs, "SR16", sr=(1, 1, 0))
    b = combine(gs, "SR16", sr=(1, 2, 0))  # another step: other draws
    assert not np.array_equal(a, b)
    # both within two 16-bit stages of the exact mean: |a - b| <= 2^-6 (|g0| + |g1|) / 2
    scale = (np.abs(gs[0]).astype(np.float64) + np.abs(gs[1])) / 2
    assert np.all(np.abs(a.astype(np.float64) - b) <= 2.0 ** -6 * scale + 1e-30)


def test_train_step_sr16_two_replicas():
    # a whole oracle step with the SR16 channel: W moves by g_hat on the 16-bit grid, close
    # to the FP32-exchange step, and a different step counter draws other roundings
    from oracle.mlp import build_mlp, train_step
    import synth
    w = synth.with_batch(synth.C2, 64)
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w)
    mg = build_mlp(w.dims, "MSE", w.lr)
    a = train_step(mg, Ws, bs, X, Y, 2, "SR16", sr_seed=3, step=1)
    f = train_step(mg, Ws, bs, X, Y, 2, "FP32")
    c = train_step(mg, Ws, bs, X, Y, 2, "SR16", sr_seed=3, step=2)
    for v, g in a["ghat"].items():
        assert np.array_equal(roundtrip(g), g)
        ref = f["ghat"][v].astype(np.float64)
        # two stages, each within one 16-bit ulp (2^-7 relative) of its input
        mag = np.mean([np.abs(p[v]).astype(np.float64) for p in a["per_replica"]], axis=0)
        assert np.all(np.abs(g - ref) <= 2.0 ** -7 * (mag + np.abs(ref)) * (1 + 1e-6) + 1e-30)
    assert any(not np.array_equal(a["ghat"][v], c["ghat"][v]) for v in a["ghat"])
