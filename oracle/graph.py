"""Oracle dataflow graph IR and gradient-graph construction.  TEST INFRASTRUCTURE ONLY.

PAPER.md §2 (:159-185): "A TensorFlow computation is described by a directed
graph ... Each node has zero or more inputs and zero or more outputs, and
represents the instantiation of an operation."  Every hot-path op here has one
output (port 0), so an endpoint is just the producer's name.

PAPER.md §4.1 (:494-518): to compute dC/dI "it first finds the path in the
computation graph from I to C.  Then it backtracks from C to I, and for each
operation on the backward path it adds a node to the TensorFlow graph,
composing the partial gradients along the backwards path using the chain rule."
``Graph.gradients`` follows that text step by step.

Interface shapes follow SPEC.md (add_node :118-126, add_gradients :354-362,
naming ``grad/<forward-name>/<suffix>`` :379, AddN summation :380).
Parity: pinned by tests/test_oracle_graph.py (Fig.2 / Fig.5 structure,
P13) and tests/test_oracle_fd.py (finite differences, P7; closed forms, P8).
"""
from __future__ import annotations

import json
import re
from typing import Dict, List, Optional, Sequence, Tuple

# Status codes mirror include/dflow.h (values chosen independently there; tests
# compare the NAMES, not the numbers).
DUPLICATE_NAME = "DUPLICATE_NAME"
UNKNOWN_OP = "UNKNOWN_OP"
DANGLING_INPUT = "DANGLING_INPUT"
SHAPE_MISMATCH = "SHAPE_MISMATCH"
NON_DIFFERENTIABLE = "NON_DIFFERENTIABLE"
NON_SCALAR_TARGET = "NON_SCALAR_TARGET"
INVALID_ARGUMENT = "INVALID_ARGUMENT"

OPS = ("Placeholder", "Variable", "MatMul", "Add", "Relu", "Loss", "LossGrad", "ReluGrad",
       "ReduceSum", "AddN", "ZerosLike", "ApplyGradientDescent",
       # inserted by insert_exchange (the replicated graph's transfer nodes)
       "Truncate16", "CrossReplicaMeanT16", "Expand16", "CrossReplicaMean",
       # f2: the probabilistic-rounding variant of the same channel (reading A26)
       "StochasticRound16", "CrossReplicaMeanSR16",
       # f4: cross-device channel endpoints of a partitioned graph
       "Send", "Recv")
BATCH = -1  # unknown (batch) dimension, only allowed through Placeholder
_NAME_RE = re.compile(r"^[A-Za-z0-9_./]+$")


class GraphError(Exception):
    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


class Node:
    __slots__ = ("name", "op", "inputs", "attrs", "dtype", "shape", "index")

    def __init__(self, name, op, inputs, attrs, dtype, shape, index):
        self.name, self.op, self.inputs = name, op, list(inputs)
        self.attrs, self.dtype, self.shape, self.index = dict(attrs), dtype, tuple(shape), index

    def to_dict(self):
        return {"name": self.name, "op": self.op, "inputs": list(self.inputs),
                "attrs": dict(sorted(self.attrs.items())), "dtype": self.dtype,
                "shape": list(self.shape)}


def _dims_compatible(a: int, b: int) -> bool:
    return a == b or a == BATCH or b == BATCH


class Graph:
    """Append-only graph; a failed add leaves the graph unchanged."""

    def __init__(self):
        self.nodes: List[Node] = []
        self.by_name: Dict[str, Node] = {}

    # ------------------------------------------------------------------ build
    def _add(self, name: str, op: str, inputs: Sequence[str], attrs: dict, dtype: str,
             shape: Tuple[int, ...]) -> str:
        if op not in OPS:
            raise GraphError(UNKNOWN_OP, op)
        if not isinstance(name, str) or not _NAME_RE.match(name):
            raise GraphError(INVALID_ARGUMENT, f"bad node name {name!r}")
        if name in self.by_name:
            raise GraphError(DUPLICATE_NAME, name)
        n = Node(name, op, inputs, attrs, dtype, shape, len(self.nodes))
        self.nodes.append(n)
        self.by_name[name] = n
        return name

    def _get(self, name: str) -> Node:
        if name not in self.by_name:
            raise GraphError(DANGLING_INPUT, str(name))
        return self.by_name[name]

    def placeholder(self, name: str, dtype: str, shape: Sequence[int]) -> str:
        return self._add(name, "Placeholder", [], {}, dtype, tuple(shape))

    def variable(self, name: str, dtype: str, shape: Sequence[int]) -> str:
        if any(d == BATCH for d in shape):
            raise GraphError(SHAPE_MISMATCH, "variables need static shapes")
        return self._add(name, "Variable", [], {}, dtype, tuple(shape))

    def matmul(self, name: str, a: str, b: str, transpose_a: bool = False,
               transpose_b: bool = False) -> str:
        A, B = self._get(a), self._get(b)
        if len(A.shape) != 2 or len(B.shape) != 2:
            raise GraphError(SHAPE_MISMATCH, f"{name}: MatMul needs rank-2 inputs")
        m, ka = (A.shape[1], A.shape[0]) if transpose_a else A.shape
        kb, n = (B.shape[1], B.shape[0]) if transpose_b else B.shape
        if not _dims_compatible(ka, kb):
            raise GraphError(SHAPE_MISMATCH, f"{name}: inner dims {ka} vs {kb}")
        return self._add(name, "MatMul", [a, b],
                         {"transpose_a": int(bool(transpose_a)), "transpose_b": int(bool(transpose_b))},
                         A.dtype, (m, n))

    def add(self, name: str, a: str, b: str) -> str:
        A, B = self._get(a), self._get(b)
        if len(B.shape) == 1 and len(A.shape) == 2:
            if not _dims_compatible(A.shape[1], B.shape[0]):
                raise GraphError(SHAPE_MISMATCH, f"{name}: bias {B.shape} vs {A.shape}")
        elif len(A.shape) != len(B.shape) or not all(_dims_compatible(x, y) for x, y in zip(A.shape, B.shape)):
            raise GraphError(SHAPE_MISMATCH, f"{name}: {A.shape} + {B.shape}")
        return self._add(name, "Add", [a, b], {}, A.dtype, A.shape)

    def relu(self, name: str, x: str) -> str:
        X = self._get(x)
        return self._add(name, "Relu", [x], {}, X.dtype, X.shape)

    def loss(self, name: str, kind: str, pred: str, target: Optional[str] = None) -> str:
        """Cost C ("C = [...]", reading A2): MSE = sum((a-y)^2)/(2*rows*cols),
        SUM = sum(a)/rows."""
        P = self._get(pred)
        if kind not in ("MSE", "SUM"):
            raise GraphError(INVALID_ARGUMENT, f"loss kind {kind}")
        if len(P.shape) != 2:
            raise GraphError(SHAPE_MISMATCH, f"{name}: loss needs a rank-2 prediction")
        inputs = [pred]
        if kind == "MSE":
            if target is None:
                raise GraphError(INVALID_ARGUMENT, "MSE needs a target")
            T = self._get(target)
            if len(T.shape) != 2 or not all(_dims_compatible(x, y) for x, y in zip(P.shape, T.shape)):
                raise GraphError(SHAPE_MISMATCH, f"{name}: target {T.shape} vs {P.shape}")
            inputs.append(target)
        elif target is not None:
            raise GraphError(INVALID_ARGUMENT, "SUM takes no target")
        return self._add(name, "Loss", inputs, {"kind": kind}, P.dtype, ())

    def apply_gradient_descent(self, name: str, var: str, lr: float, grad: str) -> str:
        V, G = self._get(var), self._get(grad)
        if V.op != "Variable":
            raise GraphError(INVALID_ARGUMENT, f"{name}: {var} is not a Variable")
        if V.shape != G.shape:
            raise GraphError(SHAPE_MISMATCH, f"{name}: var {V.shape} grad {G.shape}")
        return self._add(name, "ApplyGradientDescent", [var, grad], {"lr": float(lr)}, V.dtype, V.shape)

    # -------------------------------------------------------------- gradients
    def consumers(self, name: str) -> List[Node]:
        return [n for n in self.nodes if name in n.inputs]

    def gradients(self, cost: str, xs: Sequence[str]) -> List[str]:
        """[dC/dx for x in xs] by PAPER.md:494-518.  Atomic: on error the graph is unchanged."""
        snapshot = (list(self.nodes), dict(self.by_name))
        try:
            return self._gradients(cost, xs)
        except GraphError:
            self.nodes, self.by_name = snapshot
            raise

    def _gradients(self, cost: str, xs: Sequence[str]) -> List[str]:
        C = self._get(cost)
        for x in xs:
            self._get(x)
        if C.shape != ():
            raise GraphError(NON_SCALAR_TARGET, cost)
        # 1. "finds the path in the computation graph from I to C": nodes that are
        #    reachable forward from some x AND reach C backward.
        fwd = set(xs)
        for n in self.nodes:  # construction order is a topological order
            if any(i in fwd for i in n.inputs):
                fwd.add(n.name)
        back = {cost}
        for n in reversed(self.nodes):
            if n.name in back:
                back.update(n.inputs)
        on_path = fwd & back
        # 2. "backtracks from C to I": reverse topological (= reverse construction) order.
        partials: Dict[str, List[str]] = {}
        total: Dict[str, str] = {}
        for n in reversed(list(self.nodes)):
            if n.name not in on_path:
                continue
            if n.name == cost:
                g = None  # dC/dC = 1 is folded into the loss gradient function
            else:
                g = self._sum_partials(n.name, partials.get(n.name, []))
                total[n.name] = g
            if n.op in ("Placeholder", "Variable"):
                continue
            for inp, grad_node in self._gradient_function(n, g, on_path):
                partials.setdefault(inp, []).append(grad_node)
        outs = []
        for x in xs:
            if x == cost:
                raise GraphError(NON_DIFFERENTIABLE, "gradient of C with respect to itself")
            if x in total:
                outs.append(total[x])
            elif x in on_path:
                outs.append(self._sum_partials(x, partials.get(x, [])))
                total[x] = outs[-1]
            else:
                # "C may only depend on some of them ... set to 0"
                X = self.by_name[x]
                outs.append(self._add(f"grad/{x}/zeros", "ZerosLike", [x], {}, X.dtype, X.shape))
                total[x] = outs[-1]
        return outs

    def _sum_partials(self, name: str, parts: List[str]) -> str:
        if not parts:
            raise GraphError(NON_DIFFERENTIABLE, f"no gradient reaches {name}")
        if len(parts) == 1:
            return parts[0]
        N = self.by_name[name]
        return self._add(f"grad/{name}/sum", "AddN", parts, {}, N.dtype, N.shape)

    def _gradient_function(self, n: Node, g: Optional[str], on_path) -> List[Tuple[str, str]]:
        """Registered gradient functions.  Returns
        [(forward input, partial-gradient node)] for inputs on the path only."""
        out = []
        if n.op == "Loss":
            pred = n.inputs[0]
            if len(n.inputs) > 1 and n.inputs[1] in on_path:
                raise GraphError(NON_DIFFERENTIABLE, f"{n.name}: gradient w.r.t. the loss target")
            if pred in on_path:
                P = self.by_name[pred]
                out.append((pred, self._add(f"grad/{n.name}/pred", "LossGrad", list(n.inputs),
                                            {"kind": n.attrs["kind"]}, P.dtype, P.shape)))
        elif n.op == "Relu":
            x = n.inputs[0]
            if x in on_path:
                # uses the forward OUTPUT (a "grey arrow" input)
                out.append((x, self._add(f"grad/{n.name}/x", "ReluGrad", [g, n.name], {},
                                         n.dtype, n.shape)))
        elif n.op == "Add":
            a, b = n.inputs
            A, B = self.by_name[a], self.by_name[b]
            if a in on_path:
                out.append((a, g))  # identity partial: no node
            if b in on_path:
                if len(B.shape) == 1 and len(A.shape) == 2:
                    out.append((b, self._add(f"grad/{n.name}/b", "ReduceSum", [g], {"axis": 0},
                                             B.dtype, B.shape)))
                else:
                    out.append((b, g))
        elif n.op == "MatMul":
            a, b = n.inputs
            ta, tb = n.attrs["transpose_a"], n.attrs["transpose_b"]
            # C = op(A) op(B);  dA, dB by the chain rule for each transpose case.
            rules = {
                (0, 0): ((g, b, 0, 1), (a, g, 1, 0)),
                (1, 0): ((b, g, 0, 1), (a, g, 0, 0)),
                (0, 1): ((g, b, 0, 0), (g, a, 1, 0)),
                (1, 1): ((b, g, 1, 1), (g, a, 1, 1)),
            }[(ta, tb)]
            for inp, suffix, (x, y, txa, txb) in ((a, "a", rules[0]), (b, "b", rules[1])):
                if inp in on_path:
                    out.append((inp, self.matmul(f"grad/{n.name}/{suffix}", x, y, txa, txb)))
        else:
            raise GraphError(NON_DIFFERENTIABLE, f"{n.name}: op {n.op} has no gradient function")
        return out

    # ------------------------------------------------------------------- misc
    def to_json(self) -> str:
        return json.dumps({"version": 1, "nodes": [n.to_dict() for n in self.nodes]}, sort_keys=True)


def insert_exchange(graph: Graph, world: int, exchange: str, asynchronous: bool = False) -> Graph:
    """Compression-insertion on the replica->combine transfer (PAPER.md :813-821 on the
    §7 :934-941 channel; SPEC.md:681-689 shape).  For world > 1, between every
    ApplyGradientDescent and its gradient: TRUNC16 -> Truncate16, CrossReplicaMeanT16
    (attr world), Expand16; SR16 -> StochasticRound16, CrossReplicaMeanSR16, Expand16;
    FP32 modes -> CrossReplicaMean.  asynchronous (f3): every replica
    applies its own coded gradient — the code and Expand16 nodes without the mean; FP32:
    nothing (no coding, no mean).  world == 1 or NONE: a copy
    (reading A6).  The replicas themselves are implicit (one per rank)."""
    out = Graph()
    active = world > 1 and exchange != "NONE" and not (asynchronous and exchange.startswith("FP32"))
    for n in graph.nodes:
        inputs = list(n.inputs)
        if active and n.op == "ApplyGradientDescent":
            var, g = inputs
            G = out.by_name[g]
            if exchange in ("TRUNC16", "SR16"):
                code, mean = (("trunc16", "Truncate16"), "CrossReplicaMeanT16") if exchange == "TRUNC16" else \
                    (("sround16", "StochasticRound16"), "CrossReplicaMeanSR16")
                t = out._add(f"xchg/{var}/{code[0]}", code[1], [g], {}, "u16", G.shape)
                if not asynchronous:
                    t = out._add(f"xchg/{var}/mean", mean, [t], {"world": world}, "u16", G.shape)
                inputs[1] = out._add(f"xchg/{var}/expand16", "Expand16", [t], {}, "f32", G.shape)
            else:
                inputs[1] = out._add(f"xchg/{var}/mean", "CrossReplicaMean", [g], {"world": world}, "f32", G.shape)
        out._add(n.name, n.op, inputs, n.attrs, n.dtype, n.shape)
    return out
