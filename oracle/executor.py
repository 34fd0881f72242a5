"""Oracle single-device executor.  TEST INFRASTRUCTURE ONLY.

PAPER.md §3.1 (:335-344): "We keep track of a count per node of the number of
dependencies of that node that have not yet been executed.  Once this count
drops to zero, the node is eligible for execution and is added to a ready
queue."  Ties are broken by construction order.

Partial execution (§4.2 :549-598): only the transitive closure of the
fetched/target nodes runs; fed endpoints are replaced by their fed values.
Parity: pinned by tests/test_oracle_executor.py (execution counts, pruning,
schedule-independence) and indirectly by every numeric pin.
"""
from __future__ import annotations

from collections import deque
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import kernels as K
from .codec import expand16, truncate16
from .graph import Graph, GraphError, INVALID_ARGUMENT


def closure(graph: Graph, targets: Sequence[str], fed: Sequence[str]) -> List[str]:
    """Transitive closure of ``targets`` over inputs, stopping at fed nodes."""
    need, stack = set(), list(targets)
    fed = set(fed)
    while stack:
        n = stack.pop()
        if n in need:
            continue
        need.add(n)
        if n in fed:
            continue
        stack.extend(graph.by_name[n].inputs)
    return [n.name for n in graph.nodes if n.name in need]


def execute(graph: Graph, feeds: Dict[str, np.ndarray], fetches: Sequence[str],
            variables: Dict[str, np.ndarray], mode: str = "f32",
            masks: Optional[Dict[str, np.ndarray]] = None,
            trace: Optional[List[str]] = None) -> Dict[str, np.ndarray]:
    """Run the subgraph needed for ``fetches``.  ``variables`` holds the
    persistent Variable values and is UPDATED in place by
    ApplyGradientDescent nodes that run.  Returns {fetch: value}."""
    masks = masks or {}
    for f in list(feeds) + list(fetches):
        if f not in graph.by_name:
            raise GraphError(INVALID_ARGUMENT, f"unknown endpoint {f}")
    run = closure(graph, fetches, feeds.keys())
    run_set = set(run)
    values: Dict[str, np.ndarray] = {}
    pending: Dict[str, int] = {}
    consumers: Dict[str, List[str]] = {n: [] for n in run}
    ready = deque()
    for name in run:
        node = graph.by_name[name]
        if name in feeds:
            deps = []
        else:
            deps = [i for i in dict.fromkeys(node.inputs) if i in run_set]
        pending[name] = len(deps)
        for d in deps:
            consumers[d].append(name)
        if not deps:
            ready.append(name)
    while ready:
        name = ready.popleft()
        if trace is not None:
            trace.append(name)
        values[name] = _run_node(graph, name, feeds, values, variables, mode, masks)
        for c in consumers[name]:  # consumers are in construction order
            pending[c] -= 1
            if pending[c] == 0:
                ready.append(c)
    return {f: values[f] for f in fetches}


def _run_node(graph, name, feeds, values, variables, mode, masks):
    if name in feeds:
        v = np.asarray(feeds[name])
        return v.astype(np.float32) if mode == "f32" else v.astype(np.float64)
    n = graph.by_name[name]
    ins = [values[i] for i in n.inputs]
    op = n.op
    if op == "Variable":
        return variables[name]
    if op == "Placeholder":
        raise GraphError(INVALID_ARGUMENT, f"placeholder {name} must be fed")
    if op == "MatMul":
        return K.matmul(ins[0], ins[1], n.attrs["transpose_a"], n.attrs["transpose_b"], mode)
    if op == "Add":
        return K.add(ins[0], ins[1], mode)
    if op == "Relu":
        return K.relu(ins[0], mode, masks.get(name))
    if op == "ReluGrad":
        return K.relu_grad(ins[0], ins[1], mode, masks.get(n.inputs[1]))
    if op == "ReduceSum":
        return K.reduce_sum0(ins[0], mode)
    if op == "AddN":
        return K.add_n(ins, mode)
    if op == "ZerosLike":
        return K.zeros_like(ins[0], mode)
    if op == "Loss":
        return K.loss(n.attrs["kind"], ins[0], ins[1] if len(ins) > 1 else None, mode)
    if op == "LossGrad":
        return K.loss_grad(n.attrs["kind"], ins[0], ins[1] if len(ins) > 1 else None, mode)
    if op == "Truncate16":  # channel codec (reading A5)
        return truncate16(np.asarray(ins[0], np.float32))
    if op == "Expand16":
        return expand16(ins[0]) if mode == "f32" else expand16(ins[0]).astype(np.float64)
    if op == "ApplyGradientDescent":
        new = K.apply_gradient_descent(ins[0], n.attrs["lr"], ins[1], mode)
        variables[n.inputs[0]] = new
        return new
    raise GraphError(INVALID_ARGUMENT, f"no kernel for {op}")
