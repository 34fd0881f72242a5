"""Oracle stacked Relu(XW+b) MLP and its synchronous replicated train step.
TEST INFRASTRUCTURE ONLY.

Graph (Fig.1, stacked; reading A1: Z = X W + b with X
[rows, in] row-major, W [in, out]):  x -> MatMul(x, W1) -> Add(., b1) -> Relu
-> ... -> Relu -> Loss C.  Its gradient graph is built by Graph.gradients
 and ApplyGradientDescent nodes are added per variable.

Replicated step (Fig.7 top):
rows [r*b, (r+1)*b) go to replica r (reading A4); every replica runs the
forward + gradient subgraph with identical W, b through the dependency-counting
executor; the per-replica fp32 gradients are combined (oracle.exchange) and
every variable is updated once with W <- fl(W - fl(lr*g_hat)).
Reported cost: C = mean_r C_r.
Parity: pinned by tests/test_oracle_mlp.py (P8 closed forms, P9 lr=0,
P10 N-replica invariant, P12 exact regime, P14 error-magnitude bands).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import kernels as K
from .exchange import combine, combine_f64
from .executor import execute
from .graph import BATCH, Graph, GraphError, INVALID_ARGUMENT


@dataclasses.dataclass
class MLPGraph:
    graph: Graph
    dims: tuple
    loss: str
    lr: float
    weights: List[str]
    biases: List[str]
    pre: List[str]       # Add outputs z_l
    acts: List[str]      # Relu outputs a_l
    cost: str
    grads: Dict[str, str]  # variable (or "x") -> gradient node
    applies: List[str]


def build_mlp(dims: Sequence[int], loss: str, lr: float, with_dx: bool = False) -> MLPGraph:
    """Builds the graph.  One layer uses Fig.1's names {b, W, x, MatMul, Add,
    ReLU, C} in Fig.1's order; deeper nets use x, y,
    W<l>, b<l>, layer<l>/{MatMul,Add,Relu}, C."""
    g = Graph()
    L = len(dims) - 1
    Ws, bs, pre, acts = [], [], [], []
    if L == 1:
        bs.append(g.variable("b", "f32", (dims[1],)))
        Ws.append(g.variable("W", "f32", (dims[0], dims[1])))
        x = g.placeholder("x", "f32", (BATCH, dims[0]))
        y = g.placeholder("y", "f32", (BATCH, dims[1])) if loss == "MSE" else None
        mm = g.matmul("MatMul", x, Ws[0])
        pre.append(g.add("Add", mm, bs[0]))
        acts.append(g.relu("ReLU", pre[0]))
    else:
        x = g.placeholder("x", "f32", (BATCH, dims[0]))
        y = g.placeholder("y", "f32", (BATCH, dims[-1])) if loss == "MSE" else None
        a = x
        for l in range(1, L + 1):
            Ws.append(g.variable(f"W{l}", "f32", (dims[l - 1], dims[l])))
            bs.append(g.variable(f"b{l}", "f32", (dims[l],)))
            mm = g.matmul(f"layer{l}/MatMul", a, Ws[-1])
            pre.append(g.add(f"layer{l}/Add", mm, bs[-1]))
            a = g.relu(f"layer{l}/Relu", pre[-1])
            acts.append(a)
    cost = g.loss("C", loss, acts[-1], y)
    xs: List[str] = []
    for W, b in zip(Ws, bs):
        xs += [W, b]
    if with_dx:
        xs.append(x)
    grad_nodes = g.gradients(cost, xs)
    grads = dict(zip(xs, grad_nodes))
    applies = [g.apply_gradient_descent(f"update/{v}", v, lr, grads[v]) for v in xs if v != x]
    return MLPGraph(g, tuple(dims), loss, lr, Ws, bs, pre, acts, cost, grads, applies)


def _variables(mg: MLPGraph, Ws, bs, mode: str) -> Dict[str, np.ndarray]:
    dt = np.float32 if mode == "f32" else np.float64
    v = {}
    for name, W in zip(mg.weights, Ws):
        v[name] = np.array(W, dtype=dt)
    for name, b in zip(mg.biases, bs):
        v[name] = np.array(b, dtype=dt)
    return v


def _feeds(mg: MLPGraph, X, Y):
    f = {"x": X}
    if mg.loss == "MSE":
        f["y"] = Y
    return f


def forward(mg: MLPGraph, Ws, bs, X, Y=None, fetch: Optional[Sequence[str]] = None,
            mode: str = "f32") -> Dict[str, np.ndarray]:
    """Session.Run(fetch, feeds) without an update."""
    fetch = list(fetch or [mg.cost])
    return execute(mg.graph, _feeds(mg, X, Y), fetch, _variables(mg, Ws, bs, mode), mode)


def replica_gradients(mg: MLPGraph, Ws, bs, X, Y=None, mode: str = "f32",
                      masks: Optional[Dict[str, np.ndarray]] = None,
                      extra: Sequence[str] = ()) -> Dict[str, np.ndarray]:
    """One replica's forward + gradient subgraph: {var: grad, cost: C_r, ...}."""
    fetch = [mg.grads[v] for v in mg.weights + mg.biases] + [mg.cost] + list(extra)
    if "x" in mg.grads:
        fetch.append(mg.grads["x"])
    out = execute(mg.graph, _feeds(mg, X, Y), fetch, _variables(mg, Ws, bs, mode), mode, masks)
    res = {v: out[mg.grads[v]] for v in mg.weights + mg.biases}
    res["C"] = out[mg.cost]
    if "x" in mg.grads:
        res["dx"] = out[mg.grads["x"]]
    for e in extra:
        res[e] = out[e]
    return res


def train_step(mg: MLPGraph, Ws, bs, X, Y=None, n_replicas: int = 1, exchange: str = "TRUNC16",
               mode: str = "f32", masks: Optional[Sequence[Dict[str, np.ndarray]]] = None,
               sr_seed: int = 0, step: int = 1) -> dict:
    """One synchronous replicated SGD step.  Returns W/b after the step, the
    mean cost, per-replica gradients, the combined g_hat, and (when ``masks``
    is given: mask-locked mode) the number of Relu mask flips per layer.
    SR16 combines each layer's bucket [dW_l ; db_l] (reading A28) with the
    stochastic-rounding streams of (sr_seed, step, layer)."""
    B = X.shape[0]
    if B % n_replicas:
        raise GraphError(INVALID_ARGUMENT, f"batch {B} not divisible by {n_replicas} replicas")
    b = B // n_replicas
    per = []
    flips = [0] * len(mg.pre)
    for r in range(n_replicas):
        Xr = X[r * b:(r + 1) * b]
        Yr = None if Y is None else Y[r * b:(r + 1) * b]
        m = None if masks is None else masks[r]
        extra = list(mg.pre) if m is not None else []
        res = replica_gradients(mg, Ws, bs, Xr, Yr, mode, m, extra)
        if m is not None:
            for l, (z, a) in enumerate(zip(mg.pre, mg.acts)):
                flips[l] += int(np.count_nonzero((res[z] > 0) != m[a]))
        per.append(res)
    variables = _variables(mg, Ws, bs, mode)
    ghat = {}
    if exchange == "SR16" and n_replicas > 1 and mode != "f64":
        for l, (wv, bv) in enumerate(zip(mg.weights, mg.biases)):
            gs = [np.concatenate([p[wv].ravel(), p[bv].ravel()]).astype(np.float32) for p in per]
            g = combine(gs, "SR16", sr=(sr_seed, step, l))
            nw = per[0][wv].size
            ghat[wv] = g[:nw].reshape(per[0][wv].shape)
            ghat[bv] = g[nw:].reshape(per[0][bv].shape)
    for v in mg.weights + mg.biases:
        if v in ghat:
            variables[v] = K.apply_gradient_descent(variables[v], mg.lr, ghat[v], mode)
            continue
        gs = [p[v] for p in per]
        if mode == "f64":
            if exchange not in ("FP32",) and n_replicas > 1:
                raise GraphError(INVALID_ARGUMENT, "pure-f64 mode supports the FP32 combine only")
            ghat[v] = combine_f64(gs)
        else:
            ghat[v] = combine(gs, exchange)
        variables[v] = K.apply_gradient_descent(variables[v], mg.lr, ghat[v], mode)
    cost = float(np.mean([float(p["C"]) for p in per]))
    return {
        "W": [variables[v] for v in mg.weights],
        "b": [variables[v] for v in mg.biases],
        "loss": cost,
        "per_replica": per,
        "ghat": ghat,
        "flips": flips,
    }
