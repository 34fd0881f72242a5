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
Parity: pinned by tests/test_oracle_exchange.py (closed form on hand values,
P19 scaling identity, P18 truncation signature, N=1 identity).
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from .codec import expand16, truncate16


def owner_reduce_trunc16(q_shards: Sequence[np.ndarray]) -> np.ndarray:
    """Owner step a8: N truncated shards (rank order) -> truncated mean."""
    n = len(q_shards)
    s = expand16(q_shards[0]).astype(np.float32)
    for q in q_shards[1:]:
        s = (s + expand16(q)).astype(np.float32)
    a = (s * np.float32(1.0 / n)).astype(np.float32)
    return truncate16(a)


def combine(grads: Sequence[np.ndarray], exchange: str) -> np.ndarray:
    """Combine per-replica fp32 gradients of one tensor -> the g_hat every replica applies."""
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
    raise ValueError(f"unknown exchange {exchange}")


def combine_f64(grads: Sequence[np.ndarray]) -> np.ndarray:
    """Pure-f64 mean (for the P10 data-parallel invariant)."""
    acc = np.zeros_like(np.asarray(grads[0], np.float64))
    for g in grads:
        acc = acc + np.asarray(g, np.float64)
    return acc / len(grads)
