"""Oracle op kernels (float64).  TEST INFRASTRUCTURE ONLY.

Two precision modes:
  * "f32"  (fp32-boundary, default): every op computes in float64 from its
    float32 inputs and rounds its output to float32 at the op boundary —
    tensors are fp32 as in the paper, float64 arithmetic isolates GPU error.
  * "f64"  (pure-f64): no rounding anywhere (finite differences P7, the
    data-parallel invariant P10).

Each kernel cites the passage defining the op.  A library primitive
(numpy's matmul, sum) serves as a step; there is no blocking or fusion.
Mask-locked mode (reading A22): ``masks[relu_node]`` (bool array) replaces
the forward's own 1[z>0] in Relu and in the ReluGrad that consumes it.
"""
from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np


def _out(x: np.ndarray, mode: str) -> np.ndarray:
    return x.astype(np.float32) if mode == "f32" else x.astype(np.float64)


def matmul(a, b, transpose_a: int, transpose_b: int, mode: str):
    """MatMul (Table 1): c[i,j] = sum_p op(a)[i,p] op(b)[p,j]."""
    A = np.asarray(a, dtype=np.float64)
    B = np.asarray(b, dtype=np.float64)
    if transpose_a:
        A = A.T
    if transpose_b:
        B = B.T
    return _out(A @ B, mode)


def add(a, b, mode: str):
    """Add with rank-1 broadcast over rows (Fig.1 "Wx+b")."""
    return _out(np.asarray(a, np.float64) + np.asarray(b, np.float64), mode)


def relu(z, mode: str, mask: Optional[np.ndarray] = None):
    """Relu: max(z, 0).  Mask-locked: z * m (reading A22)."""
    Z = np.asarray(z, np.float64)
    if mask is not None:
        return _out(np.where(mask, Z, 0.0), mode)
    return _out(np.maximum(Z, 0.0), mode)


def relu_grad(g, y, mode: str, mask: Optional[np.ndarray] = None):
    """Gradient function of Relu: g * 1[y > 0], y the forward
    output; Relu'(0) = 0 (reading A10)."""
    m = (np.asarray(y) > 0) if mask is None else mask
    return _out(np.where(m, np.asarray(g, np.float64), 0.0), mode)


def reduce_sum0(g, mode: str):
    """Gradient of the broadcast operand of Add: sum over the broadcast (row) axis."""
    return _out(np.asarray(g, np.float64).sum(axis=0), mode)


def add_n(parts: List[np.ndarray], mode: str):
    acc = np.zeros_like(np.asarray(parts[0], np.float64))
    for p in parts:
        acc = acc + np.asarray(p, np.float64)
    return _out(acc, mode)


def zeros_like(x, mode: str):
    return _out(np.zeros(np.shape(x)), mode)


def loss(kind: str, pred, target, mode: str):
    """Cost C (reading A2).  MSE: sum((a-y)^2) / (2*rows*cols).  SUM: sum(a) / rows."""
    P = np.asarray(pred, np.float64)
    rows, cols = P.shape
    if kind == "MSE":
        D = P - np.asarray(target, np.float64)
        c = np.sum(D * D) / (2.0 * rows * cols)
    else:
        c = np.sum(P) / rows
    return _out(np.asarray(c), mode)


def loss_grad(kind: str, pred, target, mode: str):
    """dC/dpred (the gradient function of the cost, seeded with dC/dC = 1).
    MSE: (a-y)/(rows*cols).  SUM: 1/rows (IEEE division, reading A20)."""
    P = np.asarray(pred, np.float64)
    rows, cols = P.shape
    if kind == "MSE":
        return _out((P - np.asarray(target, np.float64)) / float(rows * cols), mode)
    return _out(np.full(P.shape, 1.0 / rows), mode)


def apply_gradient_descent(var, lr: float, grad, mode: str):
    """ApplyGradientDescent: W <- W - lr*g.
    f32 mode rounds twice, fl(W - fl(lr*g)) (reading A9)."""
    if mode == "f32":
        V = np.asarray(var, np.float32)
        step = (np.float32(lr) * np.asarray(grad, np.float32)).astype(np.float32)
        return (V - step).astype(np.float32)
    return np.asarray(var, np.float64) - lr * np.asarray(grad, np.float64)
