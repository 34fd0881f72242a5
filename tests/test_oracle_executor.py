"""Pins for oracle.executor (PAPER.md:335-344 dependency counting, :581-598 pruning).  CPU only."""
import numpy as np

from oracle.executor import closure, execute
from oracle.mlp import build_mlp
from synth import rng


def _setup():
    mg = build_mlp((4, 3, 2), "MSE", 0.5)
    g = rng(9)
    vars_ = {"W1": g.uniform(-1, 1, (4, 3)).astype(np.float32), "b1": np.zeros(3, np.float32),
             "W2": g.uniform(-1, 1, (3, 2)).astype(np.float32), "b2": np.zeros(2, np.float32)}
    feeds = {"x": g.uniform(0, 1, (5, 4)).astype(np.float32), "y": g.uniform(0, 1, (5, 2)).astype(np.float32)}
    return mg, vars_, feeds


def test_forward_fetch_runs_no_gradient_nodes():
    # SPEC.md:367 "running the forward fetches alone executes zero gradient nodes"
    mg, vars_, feeds = _setup()
    trace = []
    execute(mg.graph, feeds, [mg.cost], dict(vars_), trace=trace)
    assert not [t for t in trace if t.startswith("grad/") or t.startswith("update/")]
    assert set(trace) == set(closure(mg.graph, [mg.cost], feeds.keys()))


def test_fed_endpoint_prunes_its_producers():
    # feeding an intermediate replaces it; its producers do not run.
    mg, vars_, feeds = _setup()
    trace = []
    z = np.ones((5, 3), np.float32)
    out = execute(mg.graph, {"layer1/Add": z, "y": feeds["y"]}, ["layer1/Relu"], dict(vars_), trace=trace)
    assert trace == ["layer1/Add", "layer1/Relu"]
    assert np.array_equal(out["layer1/Relu"], z)


def test_trace_is_topological_and_construction_tie_break():
    mg, vars_, feeds = _setup()
    trace = []
    execute(mg.graph, feeds, mg.applies, dict(vars_), trace=trace)
    pos = {n: i for i, n in enumerate(trace)}
    for name in trace:
        for i in mg.graph.by_name[name].inputs:
            assert pos[i] < pos[name]
    # every node runs exactly once
    assert len(trace) == len(set(trace))


def test_apply_nodes_mutate_variables_once():
    mg, vars_, feeds = _setup()
    v = dict(vars_)
    execute(mg.graph, feeds, mg.applies, v)
    for name in ("W1", "b1", "W2", "b2"):
        assert not np.array_equal(v[name], vars_[name]), name
