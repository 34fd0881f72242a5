"""Pins for oracle.async_dp (f3; readings A29-A31).  CPU only."""
import numpy as np

import synth
from oracle import kernels as K
from oracle.async_dp import coded_gradient, push, sequential, shard_of
from oracle.codec import roundtrip
from oracle.mlp import build_mlp, train_step
from synth import rng


def _small():
    w = synth.with_batch(synth.C2, 32)
    Ws, bs = synth.init_params(w)
    return w, Ws, bs, build_mlp(w.dims, "MSE", w.lr)


def test_fp32_channel_is_sequential_single_replica_sgd():
    # A29: with no coding, replica steps serialised in a schedule are plain SGD steps with
    # batch b in that order: each equals the synchronous oracle's N = 1 step
    w, Ws, bs, mg = _small()
    events = []
    for k in range(3):
        X, Y = synth.batch(w, step=k)
        events.append((k % 2, k, X, Y))
    Wa, ba, _ = sequential(mg, Ws, bs, events, 2, "FP32")
    Wr, br = Ws, bs
    for _, _, X, Y in events:
        r = train_step(mg, Wr, br, X, Y, 1, "FP32")
        Wr, br = r["W"], r["b"]
    for a, b in zip(Wa + ba, Wr + br):
        assert np.array_equal(a, b)


def test_world1_push_is_the_synchronous_step():
    w, Ws, bs, mg = _small()
    X, Y = synth.batch(w)
    Wa, ba, _ = sequential(mg, Ws, bs, [(0, 1, X, Y)], 1, "TRUNC16")
    r = train_step(mg, Ws, bs, X, Y, 1, "TRUNC16")
    for a, b in zip(Wa + ba, r["W"] + r["b"]):
        assert np.array_equal(a, b)


def test_coding_applies_to_cross_device_elements_only():
    # A30 with P = 20, N = 2: shard = ceil(20 / 16) * 8 = 16 -> rank 0 owns 0..15, rank 1 16..19
    assert shard_of(20, 2) == 16 and shard_of(16, 2) == 8 and shard_of(17, 4) == 8
    g = rng(3).standard_normal(20).astype(np.float32)
    for sender in (0, 1):
        gh = coded_gradient(g, sender, 2, "TRUNC16")
        own = (np.arange(20) // 16) == sender
        assert np.array_equal(gh[own], g[own])
        assert np.array_equal(gh[~own], roundtrip(g[~own]))
    assert np.array_equal(coded_gradient(g, 1, 2, "FP32"), g)
    # SR16: cross-device elements land on the 16-bit grid, own elements stay exact
    gs = coded_gradient(g, 0, 2, "SR16", (5, 1, 0))
    assert np.array_equal(gs[:16], g[:16]) and np.array_equal(roundtrip(gs[16:]), gs[16:])


def test_two_updates_from_one_point_commute_up_to_one_rounding():
    # A31: two replicas' deltas on one element applied in either order differ by rounding
    # only: at most one ulp of the largest intermediate (|w| + |a| + |b|)
    g = rng(9)
    W = g.standard_normal(5000).astype(np.float32)
    bz = np.zeros(0, np.float32)
    gA = g.standard_normal(5000).astype(np.float32)
    gB = g.standard_normal(5000).astype(np.float32)
    lr = 0.25
    ab = push(push(W, bz, gA, bz, lr, 0, 2, "TRUNC16")[0], bz, gB, bz, lr, 1, 2, "TRUNC16")[0]
    ba = push(push(W, bz, gB, bz, lr, 1, 2, "TRUNC16")[0], bz, gA, bz, lr, 0, 2, "TRUNC16")[0]
    ulp = np.spacing((np.abs(W) + lr * np.abs(gA) + lr * np.abs(gB)).astype(np.float32))
    assert np.all(np.abs(ab.astype(np.float64) - ba) <= ulp)
    # and each single push is the reading-A9 update of the coded gradient
    one = push(W, bz, gA, bz, lr, 0, 2, "TRUNC16")[0]
    assert np.array_equal(one, K.apply_gradient_descent(W, lr, coded_gradient(gA, 0, 2, "TRUNC16"), "f32"))
