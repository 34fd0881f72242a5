"""Oracle cross-replica gradient combine.  TEST INFRASTRUCTURE ONLY.

PAPER.md §7 (:934-941): replicas "compute the gradient for 100 elements, and
then combine the gradients and apply updates to the parameters synchronously,
in order to behave exactly as if we were running the sequential SGD algorithm
with a batch size of 1000 elements."  Combine = MEAN (reading A3), as an fp32
left fold over ranks 0..N-1 then multiplication by 1/N (reading A7).

TRUNC16 (reading A6): every cross-device gradient transfer is
compressed — the replica->owner leg AND the owner->replica leg, so each value
is truncated twice.  N = 1: no channel, no codec.

    q_r = trunc(g_r);  e_r = expand(q_r);  s = e_0;  s = fl32(s + e_r), r=1..N-1
    a   = fl32(s * (1/N));  g_hat = expand(trunc(a))

FP32:  g_hat = fl32(fl32(sum_r g_r) * (1/N)), same left fold.

SR16 (f2, readings A26-A28): TRUNC16's schedule with both compressions replaced by
stochastic rounding.  The bucket of one layer (P elements) is padded to
P_pad = ceil(P / 8N) * 8N and split into N shards of P_pad / N; element idx is
owned by rank idx // shard.  Sender r rounds with key(seed, step, layer, 0, r),
the owner o rounds the mean with key(seed, step, layer, 1, o); the draw for an
element is sr_random(key, idx) with idx its bucket position.
Parity: pinned by tests/test_oracle_exchange.py (closed form on hand values,
P19 scaling identity, P18 truncation signature, N=1 identity).
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from .codec import expand16, sr16, sr_key, sr_random, truncate16


def owner_reduce_trunc16(q_shards: Sequence[np.ndarray]) -> np.ndarray:
    """Owner step a8: N truncated shards (rank order) -> truncated mean."""
    n = len(q_shards)
    s = expand16(q_shards[0]).astype(np.float32)
    for q in q_shards[1:]:
        s = (s + expand16(q)).astype(np.float32)
    a = (s * np.float32(1.0 / n)).astype(np.float32)
    return truncate16(a)


def combine(grads: Sequence[np.ndarray], exchange: str, sr: tuple | None = None) -> np.ndarray:
    """Combine per-replica fp32 gradients of one tensor -> the g_hat every replica applies.
    SR16 needs sr = (seed, step, layer) and the grads as whole flat layer buckets."""
    n = len(grads)
    grads = [np.asarray(g, dtype=np.float32) for g in grads]
    if n == 1 or exchange == "NONE_N1":
        return grads[0].copy()
    if exchange == "FP32":
        s = grads[0].copy()
        for g in grads[1:]:
            s = (s + g).astype(np.float32)
        return (s * np.float32(1.0 / n)).astype(np.float32)
    if exchange == "TRUNC16":
        q = [truncate16(g) for g in grads]
        return expand16(owner_reduce_trunc16(q)).reshape(grads[0].shape)
    if exchange == "SR16":
        seed, step, layer = sr
        p = grads[0].size
        idx = np.arange(p, dtype=np.int64)
        shard = -(-p // (8 * n)) * 8  # P_pad / N
        q = [sr16(g.ravel(), sr_random(sr_key(seed, step, layer, 0, r), idx)) for r, g in enumerate(grads)]
        s = expand16(q[0]).astype(np.float32)
        for qr in q[1:]:
            s = (s + expand16(qr)).astype(np.float32)
        a = (s * np.float32(1.0 / n)).astype(np.float32)
        owner = idx // shard
        rr = np.zeros(p, np.uint32)
        for o in range(n):
            sel = owner == o
            rr[sel] = sr_random(sr_key(seed, step, layer, 1, o), idx[sel])
        return expand16(sr16(a, rr)).reshape(grads[0].shape)
    raise ValueError(f"unknown exchange {exchange}")


def combine_f64(grads: Sequence[np.ndarray]) -> np.ndarray:
    """Pure-f64 mean (for the P10 data-parallel invariant)."""
    acc = np.zeros_like(np.asarray(grads[0], np.float64))
    for g in grads:
        acc = acc + np.asarray(g, np.float64)
    return acc / len(grads)
