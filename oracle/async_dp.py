"""Oracle asynchronous data parallelism.  TEST INFRASTRUCTURE ONLY.

PAPER.md §7 (:948-955, Fig.7 bottom): "This approach can also be made
asynchronous, where the TensorFlow graph has many replicas of the portion of
the graph that does the bulk of the model computation, and each one of these
replicas also applies the parameter updates to the model parameters
asynchronously.  In this configuration, there is one client thread for each of
the graph replicas."  (Dean et al. 2012, Downpour SGD.)

Readings (A29-A31):
* A29  The shared parameters live once, sharded by bucket position exactly as
       the synchronous exchange shards them (P_pad = ceil(P/8N)*8N per layer
       bucket [W_l ; b_l], element idx owned by rank idx // (P_pad/N)).  A
       replica's step: read ("pull") the current parameters, compute its
       gradient on its own b rows, and apply it — no mean over replicas (each
       replica's gradient is a full SGD update), no barrier.
* A30  Every cross-device gradient transfer is coded (reading A6): a replica's
       gradient for elements another rank owns is coded (TRUNC16 / SR16 with
       the stage-0 stream of (seed, step, layer, sender)); for elements it owns
       itself nothing crosses a device and it applies g unchanged.  FP32: no
       coding anywhere.
* A31  Each element's update is W <- fl(W - fl(lr * g_hat)) (reading A9),
       applied atomically; updates of different replicas to one element
       happen in some order, each exactly this formula.

So with the replicas' steps serialised in a given order the result is
sequential SGD over their batches in that order (with per-element coding) —
what `sequential` computes.  Parity: pinned by tests/test_oracle_async.py
(FP32 channel == sequential single-replica SGD steps; N = 1 == the
synchronous step; two updates from one W commute up to one rounding).
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np

from . import kernels as K
from .codec import expand16, sr16, sr_key, sr_random, truncate16
from .mlp import MLPGraph, replica_gradients


def shard_of(p: int, world: int) -> int:
    """Shard length of a P-element bucket over `world` owners (reading A28 / A29)."""
    return -(-p // (8 * world)) * 8


def coded_gradient(g: np.ndarray, sender: int, world: int, exchange: str, sr: Tuple[int, int, int] = (0, 1, 0)):
    """g_hat of one replica's flat layer bucket as its owners receive it (A30)."""
    g = np.asarray(g, np.float32).ravel()
    if exchange == "FP32" or world == 1:
        return g.copy()
    p = g.size
    idx = np.arange(p, dtype=np.int64)
    own = (idx // shard_of(p, world)) == sender
    if exchange == "TRUNC16":
        coded = expand16(truncate16(g))
    elif exchange == "SR16":
        seed, step, layer = sr
        coded = expand16(sr16(g, sr_random(sr_key(seed, step, layer, 0, sender), idx)))
    else:
        raise ValueError(exchange)
    return np.where(own, g, coded).astype(np.float32)


def push(W: np.ndarray, b: np.ndarray, gW: np.ndarray, gb: np.ndarray, lr: float, sender: int, world: int,
         exchange: str, sr: Tuple[int, int, int] = (0, 1, 0)):
    """Apply one replica's layer gradient to the shared W, b (A29-A31): returns new W, b."""
    bucket = np.concatenate([np.asarray(gW, np.float32).ravel(), np.asarray(gb, np.float32).ravel()])
    ghat = coded_gradient(bucket, sender, world, exchange, sr)
    nw = W.size
    Wn = K.apply_gradient_descent(np.asarray(W, np.float32), lr, ghat[:nw].reshape(W.shape), "f32")
    bn = K.apply_gradient_descent(np.asarray(b, np.float32), lr, ghat[nw:].reshape(b.shape), "f32")
    return Wn, bn


def sequential(mg: MLPGraph, Ws, bs, schedule: Sequence[tuple], world: int, exchange: str, sr_seed: int = 0):
    """Replica steps applied one after another.  schedule: (rank, step, X_r, Y_r) events;
    each pulls the current parameters, computes its gradient and pushes it (SR16 draws of
    that replica's `step`).  Returns (Ws, bs, losses)."""
    Ws = [np.asarray(w, np.float32).copy() for w in Ws]
    bs = [np.asarray(v, np.float32).copy() for v in bs]
    losses = []
    for rank, step, X, Y in schedule:
        res = replica_gradients(mg, Ws, bs, X, Y, "f32")
        losses.append(float(res["C"]))
        for l, (wv, bv) in enumerate(zip(mg.weights, mg.biases)):
            Ws[l], bs[l] = push(Ws[l], bs[l], res[wv], res[bv], mg.lr, rank, world, exchange, (sr_seed, step, l))
    return Ws, bs, losses
