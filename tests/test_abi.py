"""The C-ABI library (CPU-side): loads, exports every symbol include/dflow.h declares,
builds graphs/gradients identical in structure to the oracle's, applies the same
compression pass, rejects graphs its planner cannot fuse.  No GPU needed."""
import ctypes as C
import json
import os
import re

import pytest

import paper_1603_04467_b200 as D
from oracle import graph as OG
from oracle.mlp import build_mlp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "dflow.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dflow_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(D.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(D.EXPORTED)


def _canon(js):
    d = json.loads(js)
    return [(n["name"], n["op"], n["inputs"], n["attrs"], n["dtype"], n["shape"]) for n in d["nodes"]]


@pytest.mark.parametrize("dims,loss,with_dx", [((784, 100), "SUM", True), ((784, 1024, 1024, 10), "MSE", False),
                                               ((8, 4, 4, 4, 2), "MSE", True)])
def test_c_graph_and_gradients_match_oracle_structurally(dims, loss, with_dx):
    mg = build_mlp(dims, loss, 0.25, with_dx=with_dx)
    m = D.mlp_graph(dims, loss, 0.25, with_dx=with_dx)
    try:
        assert _canon(D.graph_json(m.graph)) == _canon(mg.graph.to_json())
    finally:
        D.dflow_graph_destroy(m.graph)


def _status(fn, *args):
    return fn(*args)


def test_error_codes_match_spec_and_leave_graph_unchanged():
    g = C.c_void_p()
    D.check(D.dflow_graph_create(C.byref(g)))
    out = C.c_int32()
    W = C.c_int32()
    D.check(D.dflow_variable(g, b"W", D.DFLOW_F32, 2, D.i64_array([3, 2]), C.byref(W)))
    x = C.c_int32()
    D.check(D.dflow_placeholder(g, b"x", D.DFLOW_F32, 2, D.i64_array([-1, 3]), C.byref(x)))
    before = D.graph_json(g)
    assert D.dflow_variable(g, b"W", D.DFLOW_F32, 2, D.i64_array([3, 2]), C.byref(out)) == D.DFLOW_DUPLICATE_NAME
    assert D.dflow_relu(g, b"r", 99, C.byref(out)) == D.DFLOW_DANGLING_INPUT
    assert D.dflow_matmul(g, b"m", W.value, W.value, 0, 0, C.byref(out)) == D.DFLOW_SHAPE_MISMATCH
    assert D.dflow_gradients(g, x.value, 1, D.node_array([W.value]), (C.c_int32 * 1)()) == D.DFLOW_NON_SCALAR_TARGET
    assert D.dflow_relu(g, b"bad name!", x.value, C.byref(out)) == D.DFLOW_INVALID_ARGUMENT
    assert D.graph_json(g) == before
    # the last failing call's message names what was wrong
    assert D.dflow_relu(g, b"bad name!", x.value, C.byref(out)) == D.DFLOW_INVALID_ARGUMENT
    assert b"name" in D.dflow_last_error().lower()
    D.dflow_graph_destroy(g)


def test_status_names():
    for code, name in D.STATUS.items():
        assert D.dflow_status_name(code).decode() == name


def _session_graph_json_or_status(m, world, exchange):
    """Session creation runs the pass + planner before touching the GPU; on a CPU box
    it then fails with DFLOW_CUDA.  The planner verdict is what we check here."""
    s = C.c_void_p()
    opts = D.make_options(world=world, rank=0, exchange=exchange, max_local_rows=8)
    fake_id = (C.c_uint8 * 128)()
    return D.dflow_session_create(m.graph, C.byref(opts), fake_id, C.byref(s)), s


@pytest.mark.parametrize("world,exchange", [(1, "TRUNC16"), (2, "TRUNC16"), (4, "FP32"), (2, "FP32_NCCL"),
                                            (2, "SR16")])
def test_planner_accepts_mlp_graphs(world, exchange):
    m = D.mlp_graph((16, 8, 4), "MSE", 0.5)
    st, s = _session_graph_json_or_status(m, world, exchange)
    try:
        # OK on a GPU box, DFLOW_CUDA (no device) on CPU — never UNIMPLEMENTED
        assert st in (D.DFLOW_OK, D.DFLOW_CUDA), D.dflow_last_error()
    finally:
        if st == D.DFLOW_OK:
            D.dflow_session_destroy(s)
        D.dflow_graph_destroy(m.graph)


def test_planner_rejects_graph_without_relu_grad():
    # A hand-built "backward" that skips ReluGrad must be rejected (planner contract).
    g = C.c_void_p()
    D.check(D.dflow_graph_create(C.byref(g)))
    o = C.c_int32()

    def mk(fn, *a):
        D.check(fn(g, *a, C.byref(o)))
        return o.value
    x = mk(D.dflow_placeholder, b"x", D.DFLOW_F32, 2, D.i64_array([-1, 8]))
    y = mk(D.dflow_placeholder, b"y", D.DFLOW_F32, 2, D.i64_array([-1, 4]))
    W = mk(D.dflow_variable, b"W", D.DFLOW_F32, 2, D.i64_array([8, 4]))
    b = mk(D.dflow_variable, b"b", D.DFLOW_F32, 1, D.i64_array([4]))
    r = mk(D.dflow_relu, b"r", mk(D.dflow_add, b"a", mk(D.dflow_matmul, b"m", x, W, 0, 0), b))
    Cn = mk(D.dflow_loss, b"C", D.DFLOW_LOSS_MSE, r, y)
    # wrong: dW = x^T * lossgrad without the ReluGrad
    grads = (C.c_int32 * 1)()
    D.check(D.dflow_gradients(g, Cn, 1, D.node_array([r]), grads))  # dC/dr = LossGrad only
    dW = mk(D.dflow_matmul, b"bad_dW", x, grads[0], 1, 0)
    mk(D.dflow_apply_gradient_descent, b"uW", W, C.c_float(0.5), dW)
    s = C.c_void_p()
    opts = D.make_options(max_local_rows=8)
    st = D.dflow_session_create(g, C.byref(opts), None, C.byref(s))
    assert st == D.DFLOW_UNIMPLEMENTED, (st, D.dflow_last_error())
    D.dflow_graph_destroy(g)


@pytest.mark.parametrize("world,exchange", [(1, "TRUNC16"), (2, "TRUNC16"), (4, "TRUNC16"), (2, "FP32"),
                                            (8, "FP32_NCCL"), (2, "NONE"), (4, "SR16"), (1, "SR16")])
def test_compression_pass_matches_oracle_pass(world, exchange):
    # The C pass (insert_exchange) and the oracle's produce the same rewritten graph.
    dims = (16, 8, 4)
    mg = build_mlp(dims, "MSE", 0.5)
    m = D.mlp_graph(dims, "MSE", 0.5)
    out = C.c_void_p()
    try:
        D.check(D.dflow_graph_insert_exchange(m.graph, world, D.EXCHANGES[exchange], C.byref(out)))
        ref = OG.insert_exchange(mg.graph, world, exchange)
        assert _canon(D.graph_json(out)) == _canon(ref.to_json())
        names = [n.name for n in ref.nodes]
        if world > 1 and exchange in ("TRUNC16", "SR16"):
            code = "trunc16" if exchange == "TRUNC16" else "sround16"
            for v in ("W1", "b1", "W2", "b2"):
                i = names.index(f"update/{v}")
                assert names[i - 3:i] == [f"xchg/{v}/{code}", f"xchg/{v}/mean", f"xchg/{v}/expand16"]
        if world == 1 or exchange == "NONE":
            assert ref.to_json() == mg.graph.to_json()
    finally:
        D.dflow_graph_destroy(out)
        D.dflow_graph_destroy(m.graph)


@pytest.mark.parametrize("world,exchange", [(2, "TRUNC16"), (4, "SR16"), (2, "FP32")])
def test_async_compression_pass_matches_oracle_and_plans(world, exchange):
    # f3: code -> expand -> apply per replica, no mean; the planner takes it
    dims = (16, 8, 4)
    mg = build_mlp(dims, "MSE", 0.5)
    m = D.mlp_graph(dims, "MSE", 0.5)
    out = C.c_void_p()
    try:
        D.check(D.dflow_graph_insert_exchange(m.graph, world, D.EXCHANGES[exchange] | 0x100, C.byref(out)))
        ref = OG.insert_exchange(mg.graph, world, exchange, asynchronous=True)
        assert _canon(D.graph_json(out)) == _canon(ref.to_json())
        assert not any("mean" in n.name for n in ref.nodes)
        opts = D.make_options(world=world, exchange=exchange, max_local_rows=8, async_dp=1)
        s = C.c_void_p()
        st = D.dflow_session_create(m.graph, C.byref(opts), (C.c_uint8 * 128)(), C.byref(s))
        assert st in (D.DFLOW_OK, D.DFLOW_CUDA), D.dflow_last_error()  # never UNIMPLEMENTED
        if st == D.DFLOW_OK:
            D.dflow_session_destroy(s)
    finally:
        D.dflow_graph_destroy(out)
        D.dflow_graph_destroy(m.graph)


def test_round16_key_matches_the_oracle_key_derivation():
    # host code of the product vs the oracle's independent implementation (reading A27)
    from oracle.codec import sr_key
    k = C.c_uint32()
    for seed in (0, 1, 0xDEADBEEF):
        for step in (1, 2, 77):
            for layer in (0, 3):
                for stage in (0, 1):
                    for rank in (0, 5):
                        D.check(D.dflow_round16_key(seed, step, layer, stage, rank, C.byref(k)))
                        assert k.value == sr_key(seed, step, layer, stage, rank)


@pytest.mark.parametrize("dims,world", [((16, 8, 4), 2), ((8, 6, 4, 2), 3), ((8, 8, 8, 8, 8), 2), ((8, 8, 8, 8, 8), 4)])
def test_partition_pass_matches_oracle_partition(dims, world):
    # f4: the C partition pass and the oracle's give the same per-device
    # subgraphs (Send/Recv canonicalised per endpoint and destination, channel codec)
    from oracle.partition import partition, place_mlp
    mg = build_mlp(dims, "MSE", 0.5)
    m = D.mlp_graph(dims, "MSE", 0.5)
    try:
        names = [n["name"] for n in json.loads(D.graph_json(m.graph))["nodes"]]
        place = place_mlp(mg, world)
        arr = (C.c_int32 * len(names))(*[place[nm] for nm in names])
        ref = partition(mg.graph, place)
        for d in range(world):
            out = C.c_void_p()
            D.check(D.dflow_graph_partition(m.graph, arr, len(names), d, 1, C.byref(out)))
            try:
                assert _canon(D.graph_json(out)) == _canon(ref[d].to_json()), d
            finally:
                D.dflow_graph_destroy(out)
    finally:
        D.dflow_graph_destroy(m.graph)


@pytest.mark.parametrize("dims,world", [((16, 8, 4), 2), ((8, 8, 8, 8, 8), 4)])
def test_model_parallel_session_plans(dims, world):
    # f4: the planner + partition check accept the layer-partitioned MLP (on CPU the session
    # stops at the missing device, never at UNIMPLEMENTED); more ranks than layers is refused
    m = D.mlp_graph(dims, "MSE", 0.5)
    try:
        for rank in range(world):
            opts = D.make_options(world=world, rank=rank, max_local_rows=8, model_parallel=1)
            s = C.c_void_p()
            st = D.dflow_session_create(m.graph, C.byref(opts), (C.c_uint8 * 128)(), C.byref(s))
            assert st in (D.DFLOW_OK, D.DFLOW_CUDA), D.dflow_last_error()
            if st == D.DFLOW_OK:
                D.dflow_session_destroy(s)
        opts = D.make_options(world=len(dims), rank=0, max_local_rows=8, model_parallel=1)
        s = C.c_void_p()
        assert D.dflow_session_create(m.graph, C.byref(opts), (C.c_uint8 * 128)(), C.byref(s)) == \
            D.DFLOW_INVALID_ARGUMENT
    finally:
        D.dflow_graph_destroy(m.graph)


def test_option_validation_for_the_widening_rows():
    # f3 / f4 option combinations the session refuses before touching a device
    m = D.mlp_graph((16, 8, 4), "MSE", 0.5)
    try:
        bad = [dict(world=2, async_dp=1, precision=D.DFLOW_PRECISION_3XTF32),   # async: bf16 only
               dict(world=2, async_dp=1, exchange="FP32_NCCL"),                  # async: TRUNC16/SR16/FP32
               dict(world=2, model_parallel=1, async_dp=1),                     # one or the other
               dict(world=2, model_parallel=1, precision=D.DFLOW_PRECISION_3XTF32),
               dict(world=3, model_parallel=1),                                 # more ranks than layers
               dict(world=2, exchange=9)]                                       # unknown exchange
        for kw in bad:
            opts = D.make_options(rank=0, max_local_rows=8, **kw)
            s = C.c_void_p()
            st = D.dflow_session_create(m.graph, C.byref(opts), (C.c_uint8 * 128)(), C.byref(s))
            assert st == D.DFLOW_INVALID_ARGUMENT, (kw, st, D.dflow_last_error())
    finally:
        D.dflow_graph_destroy(m.graph)
