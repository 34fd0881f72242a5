"""paper_1603_04467_b200 — Python binding of libdflow (include/dflow.h).

Argument marshalling only (ctypes): every step of the replicated MLP train
step runs in the library's sm_100a kernels.  There is no CPU fallback — if
``libdflow.so`` is missing, importing this package raises ImportError; on a box
without a B200 every compute call returns DFLOW_CUDA and raises DflowError.

The functions keep the C names (``dflow_graph_create``, ``dflow_train_step``,
...).  ``check`` turns a status into an exception; ``mlp_graph`` builds the
stacked Relu(XW+b) graph of PAPER.md Fig.1 through the C API.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdflow.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python paper_1603_04467_b200/build.py` "
                      "(dflow has no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants
DFLOW_OK = 0
STATUS = {0: "DFLOW_OK", 1: "DFLOW_INVALID_ARGUMENT", 2: "DFLOW_DUPLICATE_NAME", 3: "DFLOW_UNKNOWN_OP",
          4: "DFLOW_DANGLING_INPUT", 5: "DFLOW_SHAPE_MISMATCH", 6: "DFLOW_NON_DIFFERENTIABLE",
          7: "DFLOW_NON_SCALAR_TARGET", 8: "DFLOW_UNIMPLEMENTED", 9: "DFLOW_NOT_INITIALIZED", 10: "DFLOW_CUDA",
          11: "DFLOW_NCCL", 12: "DFLOW_OOM", 13: "DFLOW_SESSION_POISONED", 14: "DFLOW_BUFFER_TOO_SMALL"}
for _k, _v in STATUS.items():
    globals()[_v] = _k
DFLOW_F32, DFLOW_BF16, DFLOW_U16 = 1, 7, 8
DFLOW_BATCH = -1
DFLOW_LOSS_MSE, DFLOW_LOSS_SUM = 0, 1
DFLOW_PRECISION_BF16, DFLOW_PRECISION_3XTF32 = 0, 1
DFLOW_EXCHANGE_TRUNC16, DFLOW_EXCHANGE_FP32, DFLOW_EXCHANGE_FP32_NCCL, DFLOW_EXCHANGE_NONE = 0, 1, 2, 3
DFLOW_EXCHANGE_SR16 = 4
EXCHANGES = {"TRUNC16": 0, "FP32": 1, "FP32_NCCL": 2, "NONE": 3, "SR16": 4}
EPI_F32, EPI_TRUNC16, EPI_BIAS_RELU, EPI_RELUGRAD = 0, 1, 2, 3


class dflow_options(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("device", C.c_int32), ("precision", C.c_int32),
                ("exchange", C.c_int32), ("overlap", C.c_int32), ("sm_reserve", C.c_int32),
                ("max_local_rows", C.c_int64), ("p2p", C.c_int32), ("sr_seed", C.c_uint32),
                ("async_dp", C.c_int32), ("model_parallel", C.c_int32), ("graphs", C.c_int32),
                ("defer_apply", C.c_int32)]


class dflow_stats(C.Structure):
    _fields_ = [("launches_per_step", C.c_int32), ("gemm_launches_per_step", C.c_int32), ("layers", C.c_int32),
                ("nonfinite", C.c_int32), ("gemm_ms", C.c_double), ("other_ms", C.c_double),
                ("exchange_ms", C.c_double), ("timed_steps", C.c_int64), ("gemm_flops_per_step", C.c_double),
                ("multicast", C.c_int32)]


_p = C.c_void_p
_i32, _i64, _sz = C.c_int32, C.c_int64, C.c_size_t
_node = C.c_int32
_pnode = C.POINTER(C.c_int32)
_pi64 = C.POINTER(C.c_int64)

_SIGS = {
    "dflow_last_error": (C.c_char_p, []),
    "dflow_status_name": (C.c_char_p, [_i32]),
    "dflow_version": (C.c_char_p, []),
    "dflow_graph_create": (_i32, [C.POINTER(_p)]),
    "dflow_graph_destroy": (None, [_p]),
    "dflow_graph_num_nodes": (_i32, [_p, C.POINTER(_i32)]),
    "dflow_node_by_name": (_i32, [_p, C.c_char_p, _pnode]),
    "dflow_placeholder": (_i32, [_p, C.c_char_p, _i32, _i32, _pi64, _pnode]),
    "dflow_variable": (_i32, [_p, C.c_char_p, _i32, _i32, _pi64, _pnode]),
    "dflow_matmul": (_i32, [_p, C.c_char_p, _node, _node, _i32, _i32, _pnode]),
    "dflow_add": (_i32, [_p, C.c_char_p, _node, _node, _pnode]),
    "dflow_relu": (_i32, [_p, C.c_char_p, _node, _pnode]),
    "dflow_loss": (_i32, [_p, C.c_char_p, _i32, _node, _node, _pnode]),
    "dflow_gradients": (_i32, [_p, _node, _i32, _pnode, _pnode]),
    "dflow_apply_gradient_descent": (_i32, [_p, C.c_char_p, _node, C.c_float, _node, _pnode]),
    "dflow_graph_to_json": (_i32, [_p, C.c_char_p, _sz, C.POINTER(_sz)]),
    "dflow_graph_insert_exchange": (_i32, [_p, _i32, _i32, C.POINTER(_p)]),
    "dflow_nccl_unique_id": (_i32, [C.POINTER(C.c_uint8)]),
    "dflow_session_create": (_i32, [_p, C.POINTER(dflow_options), C.POINTER(C.c_uint8), C.POINTER(_p)]),
    "dflow_session_destroy": (None, [_p]),
    "dflow_session_graph_to_json": (_i32, [_p, C.c_char_p, _sz, C.POINTER(_sz)]),
    "dflow_variable_assign": (_i32, [_p, _node, _p, _i32, _p]),
    "dflow_variable_read": (_i32, [_p, _node, _p, _i32, _p]),
    "dflow_train_step": (_i32, [_p, _i32, _pnode, C.POINTER(_p), _pi64, _i64, C.POINTER(C.c_float), _p]),
    "dflow_train_step_host": (_i32, [_p, _i32, _pnode, C.POINTER(_p), _pi64, _i64, C.POINTER(C.c_float), _p]),
    "dflow_train_step_host_pipelined": (_i32, [_p, _i32, _pnode, C.POINTER(_p), _pi64, _i64, C.POINTER(C.c_float),
                                               C.POINTER(C.c_int32), _p]),
    "dflow_session_last_loss": (_i32, [_p, C.POINTER(C.c_float), C.POINTER(C.c_int32)]),
    "dflow_forward": (_i32, [_p, _i32, _pnode, C.POINTER(_p), _pi64, _i64, _node, _p, _p]),
    "dflow_fetch_gradients": (_i32, [_p, _i32, _pnode, C.POINTER(_p), _pi64, _i64, _i32, _pnode, C.POINTER(_p), _p]),
    "dflow_fetch_relu_masks": (_i32, [_p, _i32, C.POINTER(C.c_uint32)]),
    "dflow_session_set_timing": (_i32, [_p, _i32]),
    "dflow_session_sync": (_i32, [_p, _p]),
    "dflow_session_stats": (_i32, [_p, C.POINTER(dflow_stats)]),
    "dflow_truncate16": (_i32, [_p, _p, _sz, _p]),
    "dflow_round16": (_i32, [_p, _p, _sz, C.c_uint32, C.c_int, C.c_int64, _p]),
    "dflow_async_pull": (_i32, [_p, _p]),
    "dflow_graph_partition": (_i32, [_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_int32, C.POINTER(_p)]),
    "dflow_round16_key": (_i32, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.POINTER(C.c_uint32)]),
    "dflow_expand16": (_i32, [_p, _p, _sz, _p]),
    "dflow_exchange": (_i32, [_p, _p, _p, _sz, _p]),
    "dflow_gemm_bf16": (_i32, [_i64, _i64, _i64, _p, _i64, _i32, _p, _i64, _i32, _i32, _p, _i64, _p, _i64, _p, _p,
                               _i64, _i32, _p]),
    "dflow_gemm_3xtf32": (_i32, [_i64, _i64, _i64, _p, _p, _i64, _i32, _p, _p, _i64, _i32, _p, _i64, _i32, _p]),
    "dflow_split_tf32": (_i32, [_p, _p, _p, _sz, _p]),
    "dflow_device_die_map": (_i32, [_i32, C.POINTER(C.c_int32), _i32, C.POINTER(C.c_double)]),
    "dflow_sim_world_create": (_i32, [_i32, _i32, C.POINTER(_p)]),
    "dflow_sim_world_destroy": (None, [_p]),
    "dflow_sim_world_stream": (_i32, [_p, C.POINTER(_p)]),
    "dflow_sim_world_drop_rank": (_i32, [_p, _i32]),
    "dflow_sim_sessions_create": (_i32, [_p, _p, C.POINTER(dflow_options), C.POINTER(_p)]),
    "dflow_sim_train_step": (_i32, [_p, C.POINTER(_p), _i32, _pnode, C.POINTER(_p), _pi64, _i64,
                                    C.POINTER(C.c_float)]),
    "dflow_sim_exchange": (_i32, [_p, C.POINTER(_p), C.POINTER(_p), C.POINTER(_p), _sz]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f

EXPORTED = tuple(_SIGS)


class DflowError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


def check(status: int) -> None:
    if status != DFLOW_OK:
        raise DflowError(status, (dflow_last_error() or b"").decode(errors="replace"))


# ---------------------------------------------------------------- marshalling helpers
def node_array(ids):
    return (_node * len(ids))(*ids)


def ptr_array(ptrs):
    return (_p * len(ptrs))(*[_p(p) for p in ptrs])


def i64_array(vals):
    return (C.c_int64 * len(vals))(*vals)


def graph_json(g) -> str:
    need = _sz(0)
    dflow_graph_to_json(g, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    check(dflow_graph_to_json(g, buf, need.value, C.byref(need)))
    return buf.value.decode()


def session_json(s) -> str:
    need = _sz(0)
    dflow_session_graph_to_json(s, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    check(dflow_session_graph_to_json(s, buf, need.value, C.byref(need)))
    return buf.value.decode()


class MLP:
    """Node ids of a stacked Relu(XW+b) graph built through the C API."""

    def __init__(self, graph, x, y, weights, biases, relus, cost, grads, applies, dx=None):
        self.graph, self.x, self.y = graph, x, y
        self.weights, self.biases, self.relus, self.cost = weights, biases, relus, cost
        self.grads, self.applies, self.dx = grads, applies, dx


def mlp_graph(dims, loss: str = "MSE", lr: float = 0.25, with_dx: bool = False, train: bool = True,
              x_dtype: int = DFLOW_F32) -> MLP:
    """Builds Fig.1's Relu(XW+b), stacked, + its gradient graph (dflow_gradients) and
    one ApplyGradientDescent per variable, with the node names the oracle uses."""
    g = _p()
    check(dflow_graph_create(C.byref(g)))
    L = len(dims) - 1
    out = _node()

    def mk(fn, *args):
        check(fn(g, *args, C.byref(out)))
        return out.value

    kind = DFLOW_LOSS_MSE if loss == "MSE" else DFLOW_LOSS_SUM
    Ws, bs, relus = [], [], []
    if L == 1:
        bs.append(mk(dflow_variable, b"b", DFLOW_F32, 1, i64_array([dims[1]])))
        Ws.append(mk(dflow_variable, b"W", DFLOW_F32, 2, i64_array([dims[0], dims[1]])))
        x = mk(dflow_placeholder, b"x", x_dtype, 2, i64_array([DFLOW_BATCH, dims[0]]))
        y = mk(dflow_placeholder, b"y", DFLOW_F32, 2, i64_array([DFLOW_BATCH, dims[1]])) if kind == 0 else -1
        mm = mk(dflow_matmul, b"MatMul", x, Ws[0], 0, 0)
        ad = mk(dflow_add, b"Add", mm, bs[0])
        relus.append(mk(dflow_relu, b"ReLU", ad))
    else:
        x = mk(dflow_placeholder, b"x", x_dtype, 2, i64_array([DFLOW_BATCH, dims[0]]))
        y = mk(dflow_placeholder, b"y", DFLOW_F32, 2, i64_array([DFLOW_BATCH, dims[-1]])) if kind == 0 else -1
        a = x
        for l in range(1, L + 1):
            Ws.append(mk(dflow_variable, f"W{l}".encode(), DFLOW_F32, 2, i64_array([dims[l - 1], dims[l]])))
            bs.append(mk(dflow_variable, f"b{l}".encode(), DFLOW_F32, 1, i64_array([dims[l]])))
            mm = mk(dflow_matmul, f"layer{l}/MatMul".encode(), a, Ws[-1], 0, 0)
            ad = mk(dflow_add, f"layer{l}/Add".encode(), mm, bs[-1])
            a = mk(dflow_relu, f"layer{l}/Relu".encode(), ad)
            relus.append(a)
    cost = mk(dflow_loss, b"C", kind, relus[-1], y)
    xs = []
    for W, b in zip(Ws, bs):
        xs += [W, b]
    if with_dx:
        xs.append(x)
    gout = (_node * len(xs))()
    check(dflow_gradients(g, cost, len(xs), node_array(xs), gout))
    grads = dict(zip(xs, list(gout)))
    applies = []
    if train:
        for v in xs:
            if v == x:
                continue
            nm = (b"update/" + _node_name(g, v))
            applies.append(mk(dflow_apply_gradient_descent, nm, v, C.c_float(lr), grads[v]))
    return MLP(g, x, y, Ws, bs, relus, cost, grads, applies, grads.get(x) if with_dx else None)


def _node_name(g, nid) -> bytes:
    import json
    return json.loads(graph_json(g))["nodes"][nid]["name"].encode()


def make_options(world=1, rank=0, device=0, precision=DFLOW_PRECISION_BF16, exchange="TRUNC16", overlap=1,
                 sm_reserve=0, max_local_rows=1, p2p=0, sr_seed=0, graphs=0, async_dp=0,
                 model_parallel=0, defer_apply=0) -> dflow_options:
    ex = EXCHANGES[exchange] if isinstance(exchange, str) else int(exchange)
    return dflow_options(world, rank, device, precision, ex, overlap, sm_reserve, max_local_rows, p2p, sr_seed,
                         async_dp, model_parallel, graphs, defer_apply)


def session_create(mlp_or_graph, opts: dflow_options, nccl_id: bytes = None):
    g = mlp_or_graph.graph if isinstance(mlp_or_graph, MLP) else mlp_or_graph
    s = _p()
    idp = None
    if nccl_id is not None:
        idp = (C.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
    check(dflow_session_create(g, C.byref(opts), idp, C.byref(s)))
    return s


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(dflow_nccl_unique_id(buf))
    return bytes(buf)


def sim_world(world: int, device: int = 0):
    """A simulated world of `world` ranks on one GPU (include/dflow.h, test harness)."""
    w = _p()
    check(dflow_sim_world_create(world, device, C.byref(w)))
    return w


def sim_sessions(w, mlp_or_graph, opts: dflow_options, world: int):
    g = mlp_or_graph.graph if isinstance(mlp_or_graph, MLP) else mlp_or_graph
    out = (_p * world)()
    check(dflow_sim_sessions_create(w, g, C.byref(opts), out))
    return [out[r] for r in range(world)]


def sim_stream(w):
    st = _p()
    check(dflow_sim_world_stream(w, C.byref(st)))
    return st
