"""Pins for oracle.partition (f4; readings A32-A34).  CPU only."""
import json

import numpy as np

import synth
from oracle import kernels as K
from oracle.codec import roundtrip
from oracle.executor import execute
from oracle.graph import Graph
from oracle.mlp import _feeds, _variables, build_mlp, train_step
from oracle.partition import (cross_edges, partition, place_mlp, train_step_model_parallel,
                              with_channel_codec)


def _edges(g):
    return sorted((i, n.name) for n in g.nodes for i in n.inputs)


def test_single_device_is_the_identity():
    mg = build_mlp((8, 6, 4, 2), "MSE", 0.5)
    place = place_mlp(mg, 1)
    parts = partition(mg.graph, place)
    assert list(parts) == [0] and parts[0].to_json() == mg.graph.to_json()
    assert with_channel_codec(mg.graph, place).to_json() == mg.graph.to_json()


def test_fig4_one_receive_per_tensor_and_destination():
    # a tensor consumed by b and c on another device is sent once
    g = Graph()
    x = g.placeholder("x", "f32", (-1, 4))
    W = g.variable("W", "f32", (4, 3))
    v = g.variable("v", "f32", (3,))
    a = g.matmul("a", x, W)
    g.relu("b", a)
    g.add("c", a, v)
    place = {"x": 0, "W": 0, "a": 0, "v": 1, "b": 1, "c": 1}
    parts = partition(g, place)
    ops1 = [n.op for n in parts[1].nodes]
    ops0 = [n.op for n in parts[0].nodes]
    assert ops1.count("Recv") == 1 and ops0.count("Send") == 1
    assert ops0.count("Truncate16") == 1 and ops1.count("Expand16") == 1  # the channel codec (A33)
    assert [n.inputs for n in parts[1].nodes if n.name in ("b", "c")] == [["chan/a/0to1/expand16"],
                                                                          ["chan/a/0to1/expand16", "v"]]
    send = [n for n in parts[0].nodes if n.op == "Send"][0]
    assert send.attrs == {"tensor_name": "a", "send_device": 0, "recv_device": 1}


def test_reconstruction_contracts_back_to_the_original():
    mg = build_mlp((8, 6, 4, 2), "MSE", 0.5)
    for world in (2, 3):
        place = place_mlp(mg, world)
        parts = partition(mg.graph, place, compress=False)
        # contract Send/Recv: Recv(tensor) -> tensor
        nodes = {}
        for g in parts.values():
            for n in g.nodes:
                if n.op in ("Send", "Recv"):
                    continue
                nodes[n.name] = [i[len("recv/"):].split("/")[:-1] and "/".join(i[len("recv/"):].split("/")[:-1])
                                 if i.startswith("recv/") else i for i in n.inputs]
        assert sorted(nodes) == sorted(n.name for n in mg.graph.nodes)
        assert sorted((i, k) for k, ins in nodes.items() for i in ins) == _edges(mg.graph)


def test_mlp_channels_are_the_activation_forward_and_its_gradient_backward():
    # A32 on 3 layers over 3 devices: per boundary one forward channel (A_{l-1}, consumed by the
    # next layer's MatMul and its dW) and one backward channel (dA_{l-1}, consumed by ReluGrad)
    mg = build_mlp((8, 6, 4, 2), "MSE", 0.5)
    ch = {(x, s, d): sorted(c) for x, s, d, c in cross_edges(mg.graph, place_mlp(mg, 3))}
    assert ch == {("layer1/Relu", 0, 1): ["grad/layer2/MatMul/b", "layer2/MatMul"],
                  ("grad/layer2/MatMul/a", 1, 0): ["grad/layer1/Relu/x"],
                  ("layer2/Relu", 1, 2): ["grad/layer3/MatMul/b", "layer3/MatMul"],
                  ("grad/layer3/MatMul/a", 2, 1): ["grad/layer2/Relu/x"]}
    mg4 = build_mlp((8, 8, 8, 8, 8), "MSE", 0.5)
    assert sorted((x, s, d) for x, s, d, _ in cross_edges(mg4.graph, place_mlp(mg4, 2))) == \
        [("grad/layer3/MatMul/a", 1, 0), ("layer2/Relu", 0, 1)]


def test_codec_sits_on_the_channels_dW_uses_the_received_activation():
    w = synth.with_batch(synth.C2, 16)
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w)
    mg = build_mlp(w.dims, "MSE", w.lr)
    place = place_mlp(mg, 3)
    g = with_channel_codec(mg.graph, place)
    out = execute(g, _feeds(mg, X, Y), ["layer1/Relu", "grad/layer2/Relu/x", "grad/layer2/MatMul/b",
                                         "grad/layer2/MatMul/a", "grad/layer1/Relu/x"],
                  _variables(mg, Ws, bs, "f32"), "f32")
    A1, dZ2 = out["layer1/Relu"], out["grad/layer2/Relu/x"]
    # dW_2 on device 1 multiplies the RECEIVED (coded) A_1
    assert np.array_equal(out["grad/layer2/MatMul/b"], K.matmul(roundtrip(A1), dZ2, 1, 0, "f32"))
    assert not np.array_equal(out["grad/layer2/MatMul/b"], K.matmul(A1, dZ2, 1, 0, "f32"))
    # dZ_1 on device 0 masks the RECEIVED (coded) dA_1 with its own A_1
    assert np.array_equal(out["grad/layer1/Relu/x"], K.relu_grad(roundtrip(out["grad/layer2/MatMul/a"]), A1, "f32"))


def test_exact_regime_partitioned_step_equals_single_device_step():
    # every channel tensor is exactly representable in 16 bits there, so the codec is the
    # identity and the model-parallel step is the single-device step bit for bit
    X, Y, Ws, bs, lr = synth.exact_regime()
    dims = (X.shape[1],) + tuple(W.shape[1] for W in Ws)
    mg = build_mlp(dims, "MSE", lr)
    mp = train_step_model_parallel(mg, Ws, bs, X, Y, len(Ws))
    chans = [x for x, _, _, _ in cross_edges(mg.graph, mp["place"])]
    vals = execute(mg.graph, _feeds(mg, X, Y), chans, _variables(mg, Ws, bs, "f32"), "f32")
    assert all(np.array_equal(roundtrip(v), v) for v in vals.values())
    ref = train_step(mg, Ws, bs, X, Y, 1, "FP32")
    for a, b in zip(mp["W"] + mp["b"], ref["W"] + ref["b"]):
        assert np.array_equal(a, b)
    assert mp["loss"] == ref["loss"]


def test_partition_json_attrs_are_stable():
    mg = build_mlp((8, 6, 4, 2), "MSE", 0.5)
    parts = partition(mg.graph, place_mlp(mg, 2))
    s = json.loads(parts[0].to_json())
    names = [n["name"] for n in s["nodes"]]
    assert "send/layer2/Relu/1to0" not in names and "chan/grad/layer3/MatMul/a/1to0/expand16" in names
