"""Pins for oracle.graph (P13 Fig.2 / Fig.5 structure, error codes).  CPU only."""
import json

import numpy as np
import pytest

from oracle import graph as G
from oracle.executor import execute
from oracle.mlp import build_mlp


def _nodes(g):
    return {n["name"]: n for n in json.loads(g.to_json())["nodes"]}


def test_fig2_forward_node_set_and_edges():
    # PAPER.md:102-106 (Fig.1) and :121 (Fig.2): {b, W, x, MatMul, Add, ReLU, C}
    mg = build_mlp((784, 100), "SUM", 2.0 ** -7, with_dx=True)
    nodes = _nodes(mg.graph)
    fwd = [n for n in nodes if not n.startswith("grad/") and not n.startswith("update/")]
    assert fwd == ["b", "W", "x", "MatMul", "Add", "ReLU", "C"]
    assert nodes["MatMul"]["inputs"] == ["x", "W"]
    assert nodes["Add"]["inputs"] == ["MatMul", "b"]
    assert nodes["ReLU"]["inputs"] == ["Add"]
    assert nodes["C"]["inputs"] == ["ReLU"]
    assert nodes["W"]["shape"] == [784, 100] and nodes["b"]["shape"] == [100]
    assert nodes["ReLU"]["shape"] == [-1, 100]


def test_fig5_gradient_structure():
    # PAPER.md:512 "[db,dW,dx] = tf.gradients(C, [b,W,x])", Fig.5 caption :521.
    g = G.Graph()
    b = g.variable("b", "f32", (100,))
    W = g.variable("W", "f32", (784, 100))
    x = g.placeholder("x", "f32", (-1, 784))
    r = g.relu("ReLU", g.add("Add", g.matmul("MatMul", x, W), b))
    C = g.loss("C", "SUM", r)
    db, dW, dx = g.gradients(C, [b, W, x])
    nodes = _nodes(g)
    grad_nodes = [n for n in nodes if n.startswith("grad/")]
    # backtracking order C -> ReLU -> Add -> MatMul (reverse topological)
    assert grad_nodes == ["grad/C/pred", "grad/ReLU/x", "grad/Add/b", "grad/MatMul/a", "grad/MatMul/b"]
    assert nodes["grad/C/pred"]["op"] == "LossGrad" and nodes["grad/C/pred"]["inputs"] == ["ReLU"]
    # ReluGrad takes the incoming partial and the forward OUTPUT (grey arrow)
    assert nodes["grad/ReLU/x"]["op"] == "ReluGrad"
    assert nodes["grad/ReLU/x"]["inputs"] == ["grad/C/pred", "ReLU"]
    assert nodes["grad/Add/b"]["op"] == "ReduceSum" and nodes["grad/Add/b"]["inputs"] == ["grad/ReLU/x"]
    # dx = g W^T, dW = x^T g
    assert nodes["grad/MatMul/a"]["inputs"] == ["grad/ReLU/x", "W"]
    assert nodes["grad/MatMul/a"]["attrs"] == {"transpose_a": 0, "transpose_b": 1}
    assert nodes["grad/MatMul/b"]["inputs"] == ["x", "grad/ReLU/x"]
    assert nodes["grad/MatMul/b"]["attrs"] == {"transpose_a": 1, "transpose_b": 0}
    assert (db, dW, dx) == ("grad/Add/b", "grad/MatMul/b", "grad/MatMul/a")
    assert nodes[dW]["shape"] == [784, 100] and nodes[db]["shape"] == [100] and nodes[dx]["shape"] == [-1, 784]


def test_train_graph_has_no_dx_for_first_layer():
    # x is not requested -> the MatMul gradient w.r.t. x is never built.
    mg = build_mlp((784, 1024, 1024, 10), "MSE", 2.0 ** -5)
    names = set(_nodes(mg.graph))
    assert "grad/layer1/MatMul/a" not in names
    assert "grad/layer2/MatMul/a" in names and "grad/layer3/MatMul/a" in names
    assert len(mg.applies) == 6


def test_zero_partial_for_unused_source():
    # an output C does not depend on gets a zero partial.
    g = G.Graph()
    W = g.variable("W", "f32", (3, 2))
    U = g.variable("U", "f32", (3, 2))
    x = g.placeholder("x", "f32", (-1, 3))
    C = g.loss("C", "SUM", g.relu("r", g.matmul("m", x, W)))
    dW, dU = g.gradients(C, [W, U])
    assert dU == "grad/U/zeros"
    out = execute(g, {"x": np.ones((2, 3), np.float32)}, [dU],
                  {"W": np.ones((3, 2), np.float32), "U": np.ones((3, 2), np.float32)})
    assert np.array_equal(out[dU], np.zeros((3, 2), np.float32))


def test_fanout_sums_partials():
    # SPEC.md:357 "when a node's output feeds multiple consumers, incoming partials are summed"
    g = G.Graph()
    W = g.variable("W", "f32", (3, 3))
    x = g.placeholder("x", "f32", (-1, 3))
    h = g.relu("h", g.matmul("m1", x, W))
    s = g.add("s", g.matmul("m2", h, W), h)       # h and W both fan out
    C = g.loss("C", "SUM", g.relu("r", s))
    (dW,) = g.gradients(C, [W])
    nodes = _nodes(g)
    assert nodes["grad/h/sum"]["op"] == "AddN" and dW == "grad/W/sum"
    assert set(nodes["grad/W/sum"]["inputs"]) == {"grad/m1/b", "grad/m2/b"}


def test_error_codes_leave_graph_unchanged():
    g = G.Graph()
    W = g.variable("W", "f32", (3, 2))
    x = g.placeholder("x", "f32", (-1, 3))
    before = g.to_json()
    cases = [
        (lambda: g.variable("W", "f32", (3, 2)), G.DUPLICATE_NAME),
        (lambda: g.relu("r", "ghost"), G.DANGLING_INPUT),
        (lambda: g.matmul("m", W, W), G.SHAPE_MISMATCH),
        (lambda: g._add("q", "Conv2D", [], {}, "f32", ()), G.UNKNOWN_OP),
        (lambda: g.gradients(x, [W]), G.NON_SCALAR_TARGET),
    ]
    for fn, code in cases:
        with pytest.raises(G.GraphError) as e:
            fn()
        assert e.value.code == code
        assert g.to_json() == before
    m = g.matmul("m", x, W)
    C = g.loss("C", "SUM", g.relu("r", m))
    upd = g.apply_gradient_descent("u", W, 0.5, g.gradients(C, [W])[0])
    C2 = g.loss("C2", "SUM", g.relu("r2", g.add("a2", m, upd)))  # path through ApplyGradientDescent
    before = g.to_json()
    with pytest.raises(G.GraphError) as e:
        g.gradients(C2, [W])
    assert e.value.code == G.NON_DIFFERENTIABLE
    assert g.to_json() == before


def test_json_round_trip_fields():
    mg = build_mlp((4, 3), "MSE", 0.25)
    d = json.loads(mg.graph.to_json())
    assert d["version"] == 1
    assert [n["name"] for n in d["nodes"]] == [n.name for n in mg.graph.nodes]
    assert d["nodes"][-1]["op"] == "ApplyGradientDescent" and d["nodes"][-1]["attrs"] == {"lr": 0.25}
