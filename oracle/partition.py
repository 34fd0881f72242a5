"""Oracle placement, partitioning into per-device subgraphs with Send/Recv pairs, channel
compression, and the model-parallel MLP step.  TEST INFRASTRUCTURE ONLY.

PAPER.md §3.2.2 (:399-430): "Once the node placement has been computed, the graph is
partitioned into a set of subgraphs, one per device.  Any cross-device edge from x to y
is removed and replaced by an edge from x to a new Send node in x's subgraph and an edge
from a corresponding Receive node to y in y's subgraph ... we canonicalize all users of a
particular tensor on a particular device to use a single Receive node".
PAPER.md §5.5 (:813-821): data sent between devices is compressed 32 -> 16 bits and
expanded on the other side (SPEC.md:681-689 insert_compression: Compress before Send,
Decompress after Receive).
PAPER.md §7 (:958-972, Fig. 8): model-parallel training places different portions of the
model on different devices for the same batch.

Readings (A32-A34):
* A32  Layer-wise placement of the MLP over N devices: layer l (1-based) of L goes to
       device floor((l-1) N / L) with everything that belongs to it — W_l, b_l, its
       forward nodes, the gradient nodes named after them (grad/layer{l}/...), and its
       ApplyGradientDescent nodes; x on device 0; y, the loss and its gradient seed on the
       last layer's device.
* A33  Every cross-device channel carries fp32 data and is compressed (policy: all F32
       channels): Truncate16 before the Send, Expand16 after the Recv.
* A34  Executing the partition set is executing the graph with every Send/Recv pair
       contracted to a direct edge through Truncate16 -> Expand16 (`with_channel_codec`);
       the oracle step runs that graph through the dependency-counting executor.
Parity: pinned by tests/test_oracle_partition.py (single-device identity, the Fig. 4
canonicalisation, reconstruction, codec-free partitions == the unpartitioned step
bitwise, the MLP's channel set).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import kernels as K
from .executor import execute
from .graph import Graph
from .mlp import MLPGraph, _feeds, _variables


def place_mlp(mg: MLPGraph, world: int) -> Dict[str, int]:
    """Reading A32: node name -> device."""
    L = len(mg.weights)
    dev = {l: ((l - 1) * world) // L for l in range(1, L + 1)}
    place = {}
    for n in mg.graph.nodes:
        name = n.name
        d = None
        for l in range(1, L + 1):
            if name in (f"W{l}", f"b{l}", f"update/W{l}", f"update/b{l}") or name.startswith(f"layer{l}/") \
                    or name.startswith(f"grad/layer{l}/"):
                d = dev[l]
                break
        if d is None:
            d = 0 if name == "x" else dev[L]  # y, the loss and its seed with the last layer
        place[name] = d
    return place


def cross_edges(graph: Graph, place: Dict[str, int]) -> List[Tuple[str, int, int, List[str]]]:
    """Channels: (producer, src device, dst device, consumers on dst) in construction order,
    one per (producer, destination device) — the canonicalised Receive."""
    chans: Dict[Tuple[str, int], List[str]] = {}
    for n in graph.nodes:
        for i in dict.fromkeys(n.inputs):
            if place[i] != place[n.name]:
                chans.setdefault((i, place[n.name]), []).append(n.name)
    return [(x, place[x], d, cons) for (x, d), cons in chans.items()]


def partition(graph: Graph, place: Dict[str, int], compress: bool = True) -> Dict[int, Graph]:
    """Per-device subgraphs with Send/Recv pairs (+ the channel codec, reading A33)."""
    chans = {(x, d): (s, cons) for x, s, d, cons in cross_edges(graph, place)}
    out: Dict[int, Graph] = {}
    for d in sorted(set(place.values())):
        out[d] = Graph()
    for n in graph.nodes:
        d = place[n.name]
        g = out[d]
        inputs = []
        for i in n.inputs:
            if place[i] == d:
                inputs.append(i)
                continue
            src = place[i]
            key = f"{i}/{src}to{d}"
            recv = f"recv/{key}"
            if recv not in g.by_name:
                # sender side: [Truncate16 ->] Send in the producer's subgraph
                sg = out[src]
                x = i
                if compress:
                    x = sg._add(f"chan/{key}/trunc16", "Truncate16", [x], {}, "u16", graph.by_name[i].shape)
                sg._add(f"send/{key}", "Send", [x], {"tensor_name": i, "send_device": src, "recv_device": d},
                        "u16" if compress else "f32", graph.by_name[i].shape)
                # receiver side: Recv [-> Expand16], shared by every consumer on d
                r = g._add(recv, "Recv", [], {"tensor_name": i, "send_device": src, "recv_device": d},
                           "u16" if compress else "f32", graph.by_name[i].shape)
                if compress:
                    g._add(f"chan/{key}/expand16", "Expand16", [r], {}, "f32", graph.by_name[i].shape)
            inputs.append(f"chan/{key}/expand16" if compress else recv)
        g._add(n.name, n.op, inputs, n.attrs, n.dtype, n.shape)
    return out


def with_channel_codec(graph: Graph, place: Dict[str, int]) -> Graph:
    """Reading A34: the graph with every channel contracted to x -> Truncate16 -> Expand16."""
    chans = {(x, d) for x, _, d, _ in cross_edges(graph, place)}
    g = Graph()
    for n in graph.nodes:
        inputs = []
        for i in n.inputs:
            d = place[n.name]
            if (i, d) in chans:
                key = f"{i}/{place[i]}to{d}"
                if f"chan/{key}/expand16" not in g.by_name:
                    t = g._add(f"chan/{key}/trunc16", "Truncate16", [i], {}, "u16", graph.by_name[i].shape)
                    g._add(f"chan/{key}/expand16", "Expand16", [t], {}, "f32", graph.by_name[i].shape)
                inputs.append(f"chan/{key}/expand16")
            else:
                inputs.append(i)
        g._add(n.name, n.op, inputs, n.attrs, n.dtype, n.shape)
    return g


def train_step_model_parallel(mg: MLPGraph, Ws, bs, X, Y, world: int, compress: bool = True) -> dict:
    """One step of the layer-partitioned MLP (one replica, N devices): the codec graph's
    forward + gradients, each variable updated by its own device (reading A9)."""
    place = place_mlp(mg, world)
    g = with_channel_codec(mg.graph, place) if compress else mg.graph
    variables = _variables(mg, Ws, bs, "f32")
    fetch = [mg.grads[v] for v in mg.weights + mg.biases] + [mg.cost]
    out = execute(g, _feeds(mg, X, Y), fetch, dict(variables), "f32")
    new = {v: K.apply_gradient_descent(variables[v], mg.lr, out[mg.grads[v]], "f32") for v in mg.weights + mg.biases}
    return {"W": [new[v] for v in mg.weights], "b": [new[v] for v in mg.biases], "loss": float(out[mg.cost]),
            "grads": {v: out[mg.grads[v]] for v in mg.weights + mg.biases}, "graph": g, "place": place}
