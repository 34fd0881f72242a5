"""Seeded input generators (no arithmetic of the method lives here).

See the package docstring for the recipe.  Every function returns numpy
arrays on the host; callers move them to the device themselves.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import numpy as np

SEED = 1603
STREAM_X, STREAM_Y = 0, 1


def rng(stream: int) -> np.random.Generator:
    """Counter-style seeded generator: stream ids per SURVEY.md §8(d)."""
    return np.random.default_rng(np.random.SeedSequence([SEED, int(stream)]))


@dataclasses.dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration (shapes, loss, learning rate, init)."""

    name: str
    dims: Tuple[int, ...]          # (in_1, out_1 = in_2, ..., out_L)
    batch: int                     # GLOBAL batch B
    loss: str                      # "MSE" | "SUM"
    lr: float                      # constant, a power of two (reading A12)
    init: str                      # "fig1" | "fig1_bias" | "he"
    precision: str = "bf16"        # "bf16" | "3xtf32"
    steps: int = 1

    @property
    def layers(self) -> int:
        return len(self.dims) - 1

    @property
    def params(self) -> int:
        return sum(self.dims[i] * self.dims[i + 1] + self.dims[i + 1] for i in range(self.layers))

    def flops_per_example(self) -> float:
        """Algorithmic FLOPs per example: forward + dW for every
        layer, dX for layers 2..L, 2*in*out each."""
        f = 0.0
        for l in range(self.layers):
            io = self.dims[l] * self.dims[l + 1]
            f += 2 * io * (3 if l > 0 else 2)
        return f


# BASELINE.json "configs" (index 0..4 -> C1..C5); see DESIGN.md for readings.
C1 = Workload("C1_fig1_784x100_b100", (784, 100), 100, "SUM", 2.0 ** -7, "fig1", "3xtf32")
C1_BIAS = Workload("C1b_fig1_bias", (784, 100), 100, "SUM", 2.0 ** -7, "fig1_bias", "3xtf32")
C2 = Workload("C2_mnist_784-1024-1024-10_b256", (784, 1024, 1024, 10), 256, "MSE", 2.0 ** -5, "he",
              "bf16", steps=100)
C3 = Workload("C3_wide_4x8192_b32768", (8192,) * 5, 32768, "MSE", 2.0 ** -2, "he", "bf16")
C5 = Workload("C5_deep_16x4096_b65536", (4096,) * 17, 65536, "MSE", 2.0 ** -2, "he", "3xtf32")
CONFIGS = {"C1": C1, "C1b": C1_BIAS, "C2": C2, "C3": C3, "C5": C5}


def with_batch(w: Workload, batch: int) -> Workload:
    return dataclasses.replace(w, batch=batch)


def init_params(w: Workload) -> Tuple[List[np.ndarray], List[np.ndarray]]:
    """W_l [in,out] and b_l [out], float32 (reading A11)."""
    Ws, bs = [], []
    for l in range(w.layers):
        fan_in, fan_out = w.dims[l], w.dims[l + 1]
        g = rng(10 + l)
        if w.init in ("fig1", "fig1_bias"):
            # PAPER.md:103 tf.random_uniform([784,100],-1,1)
            W = g.uniform(-1.0, 1.0, size=(fan_in, fan_out))
        else:
            a = np.sqrt(6.0 / fan_in)
            W = g.uniform(-a, a, size=(fan_in, fan_out))
        gb = rng(100 + l)
        if w.init == "fig1":
            b = np.zeros(fan_out)  # PAPER.md:102 tf.zeros([100])
        else:
            b = gb.uniform(-0.1, 0.1, size=(fan_out,))
        Ws.append(W.astype(np.float32))
        bs.append(b.astype(np.float32))
    return Ws, bs


def batch(w: Workload, step: Optional[int] = None, rows: Optional[int] = None,
          row0: int = 0) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """X [rows, in] ~ U[0,1) and Y [rows, out_L] ~ U[0,1) (None for SUM loss).

    ``step`` None uses streams 0/1 (the fixed batch); otherwise stream
    1000+step draws (X, Y) for that step.  ``rows``/``row0`` select a
    contiguous block of the global batch without drawing the rest
    (generated block-wise so a sample of a huge batch stays cheap).
    """
    rows = w.batch if rows is None else rows
    din, dout = w.dims[0], w.dims[-1]
    X = _uniform_rows(STREAM_X if step is None else 1000 + step, 0, row0, rows, din)
    Y = None
    if w.loss == "MSE":
        Y = _uniform_rows(STREAM_Y if step is None else 1000 + step, 1, row0, rows, dout)
    return X, Y


_BLOCK = 256


def _uniform_rows(stream: int, sub: int, row0: int, rows: int, cols: int) -> np.ndarray:
    """Rows [row0, row0+rows) of a U[0,1) float32 matrix, drawn in 256-row blocks
    (block k from SeedSequence([1603, stream, sub, k])) so any row range is cheap
    to regenerate identically."""
    out = np.empty((rows, cols), dtype=np.float32)
    k0, k1 = row0 // _BLOCK, (row0 + rows - 1) // _BLOCK if rows else row0 // _BLOCK - 1
    for k in range(k0, k1 + 1):
        g = np.random.default_rng(np.random.SeedSequence([SEED, int(stream), sub, k]))
        blk = g.random((_BLOCK, cols), dtype=np.float32)
        lo, hi = max(row0, k * _BLOCK), min(row0 + rows, (k + 1) * _BLOCK)
        out[lo - row0:hi - row0] = blk[lo - k * _BLOCK:hi - k * _BLOCK]
    return out


# ---------------------------------------------------------------------------
# P12 exact-arithmetic regime: every stored intermediate
# is a small-integer multiple of a power of two, so bf16 storage and any fp32
# summation order are exact.
# ---------------------------------------------------------------------------
EXACT_DIMS = (784, 1024, 1024, 16)
EXACT_BATCH = 256
EXACT_LR = 2.0 ** -4
EXACT_SHIFTS = (3, 2, 1)


def exact_regime(seed_stream: int = 7, batch_rows: int = EXACT_BATCH, dims=EXACT_DIMS):
    """Returns (X, Y, Ws, bs, lr).  X in {0,1} with exactly 15 ones per row;
    W_l a signed partial permutation (<=1 nonzero per row, <=2 per column)
    times 2^-s_l; b_l in {-2..2} * 2^-s_l; Y in {0..7} * 2^-2."""
    g = rng(50000 + seed_stream)
    din = dims[0]
    X = np.zeros((batch_rows, din), dtype=np.float32)
    for i in range(batch_rows):
        X[i, g.choice(din, size=15, replace=False)] = 1.0
    Ws, bs = [], []
    for l in range(len(dims) - 1):
        fi, fo = dims[l], dims[l + 1]
        s = EXACT_SHIFTS[l % len(EXACT_SHIFTS)]
        W = np.zeros((fi, fo), dtype=np.float32)
        slots = np.repeat(np.arange(fo), 2)
        g.shuffle(slots)
        n_used = min(fi, len(slots)) * 3 // 4
        rows = g.choice(fi, size=n_used, replace=False)
        for r, c in zip(rows, slots[:n_used]):
            W[r, c] = (1.0 if g.random() < 0.5 else -1.0) * 2.0 ** -s
        b = (g.integers(-2, 3, size=fo) * 2.0 ** -s).astype(np.float32)
        Ws.append(W)
        bs.append(b)
    Y = (g.integers(0, 8, size=(batch_rows, dims[-1])) * 0.25).astype(np.float32)
    return X, Y, Ws, bs, EXACT_LR


def finite_difference_mlp(seed_stream: int = 3, dims=(3, 5, 4, 2), batch_rows: int = 3):
    """Tiny float64 problem for the P7 finite-difference pin."""
    g = rng(60000 + seed_stream)
    X = g.uniform(0.0, 1.0, size=(batch_rows, dims[0]))
    Y = g.uniform(0.0, 1.0, size=(batch_rows, dims[-1]))
    Ws = [g.uniform(-1.0, 1.0, size=(dims[i], dims[i + 1])) for i in range(len(dims) - 1)]
    bs = [g.uniform(-0.5, 0.5, size=(dims[i + 1],)) for i in range(len(dims) - 1)]
    return X, Y, Ws, bs


def random_f32_bits(n: int, stream: int = 70000) -> np.ndarray:
    """Uniformly random 32-bit patterns viewed as float32 (codec tests)."""
    return rng(stream).integers(0, 2 ** 32, size=n, dtype=np.uint64).astype(np.uint32).view(np.float32)
