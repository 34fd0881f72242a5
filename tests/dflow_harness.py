"""Test-side harness: drives libdflow through its C ABI with torch CUDA tensors.

Only marshalling; no arithmetic of the method.  Used by the -m gpu tests.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

import paper_1603_04467_b200 as D


def dev_ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def stream_ptr():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Run:
    """One session on one GPU holding an MLP graph."""

    def __init__(self, dims, loss="MSE", lr=0.25, rows=256, exchange="TRUNC16", world=1, rank=0, device=0,
                 with_dx=False, nccl_id=None, overlap=1, sm_reserve=0, train=True, precision="bf16", p2p=0,
                 sr_seed=0, graphs=0, async_dp=0, model_parallel=0, defer_apply=0):
        self.mlp = D.mlp_graph(dims, loss, lr, with_dx=with_dx, train=train)
        self.dims = tuple(dims)
        self.loss = loss
        prec = D.DFLOW_PRECISION_3XTF32 if precision == "3xtf32" else D.DFLOW_PRECISION_BF16
        opts = D.make_options(world=world, rank=rank, device=device, exchange=exchange, max_local_rows=rows,
                              overlap=overlap, sm_reserve=sm_reserve, precision=prec, p2p=p2p, sr_seed=sr_seed,
                              graphs=graphs, async_dp=async_dp, model_parallel=model_parallel,
                              defer_apply=defer_apply)
        self.s = D.session_create(self.mlp, opts, nccl_id)

    def close(self):
        if self.s:
            D.dflow_session_destroy(self.s)
            self.s = None
        if self.mlp.graph:
            D.dflow_graph_destroy(self.mlp.graph)
            self.mlp.graph = None

    def assign(self, Ws, bs):
        for nid, W in zip(self.mlp.weights, Ws):
            a = np.ascontiguousarray(W, np.float32)
            D.check(D.dflow_variable_assign(self.s, nid, a.ctypes.data_as(C.c_void_p), 0, stream_ptr()))
        for nid, b in zip(self.mlp.biases, bs):
            a = np.ascontiguousarray(b, np.float32)
            D.check(D.dflow_variable_assign(self.s, nid, a.ctypes.data_as(C.c_void_p), 0, stream_ptr()))

    def read(self):
        Ws, bs = [], []
        for l, nid in enumerate(self.mlp.weights):
            a = np.empty((self.dims[l], self.dims[l + 1]), np.float32)
            D.check(D.dflow_variable_read(self.s, nid, a.ctypes.data_as(C.c_void_p), 0, stream_ptr()))
            Ws.append(a)
        for l, nid in enumerate(self.mlp.biases):
            a = np.empty((self.dims[l + 1],), np.float32)
            D.check(D.dflow_variable_read(self.s, nid, a.ctypes.data_as(C.c_void_p), 0, stream_ptr()))
            bs.append(a)
        return Ws, bs

    def _feeds(self, X: torch.Tensor, Y):
        ids, ptrs, lds = [self.mlp.x], [X.data_ptr()], [X.stride(0)]
        if Y is not None:
            ids.append(self.mlp.y)
            ptrs.append(Y.data_ptr())
            lds.append(Y.stride(0))
        return D.node_array(ids), D.ptr_array(ptrs), D.i64_array(lds), len(ids)

    def step(self, X: torch.Tensor, Y=None, want_loss=True):
        ids, ptrs, lds, n = self._feeds(X, Y)
        loss = C.c_float(0)
        D.check(D.dflow_train_step(self.s, n, ids, ptrs, lds, X.shape[0], C.byref(loss) if want_loss else None,
                                   stream_ptr()))
        return loss.value

    def gradients(self, X: torch.Tensor, Y=None, with_dx=False):
        ids, ptrs, lds, n = self._feeds(X, Y)
        outs, nodes = [], []
        for l in range(len(self.dims) - 1):
            outs.append(torch.empty((self.dims[l], self.dims[l + 1]), dtype=torch.float32, device=X.device))
            nodes.append(self.mlp.grads[self.mlp.weights[l]])
            outs.append(torch.empty((self.dims[l + 1],), dtype=torch.float32, device=X.device))
            nodes.append(self.mlp.grads[self.mlp.biases[l]])
        if with_dx:
            outs.append(torch.empty((X.shape[0], self.dims[0]), dtype=torch.float32, device=X.device))
            nodes.append(self.mlp.dx)
        D.check(D.dflow_fetch_gradients(self.s, n, ids, ptrs, lds, X.shape[0], len(nodes), D.node_array(nodes),
                                        D.ptr_array([o.data_ptr() for o in outs]), stream_ptr()))
        torch.cuda.synchronize()
        res = [o.cpu().numpy() for o in outs]
        L = len(self.dims) - 1
        gW = [res[2 * l] for l in range(L)]
        gb = [res[2 * l + 1] for l in range(L)]
        return gW, gb, (res[-1] if with_dx else None)

    def masks(self, rows):
        """GPU relu masks {relu node name (oracle naming): bool [rows, out]} of the last forward."""
        out = {}
        L = len(self.dims) - 1
        for l in range(1, L + 1):
            cols = self.dims[l]
            words = (rows * cols + 31) // 32
            buf = np.zeros(words, np.uint32)
            D.check(D.dflow_fetch_relu_masks(self.s, l, buf.ctypes.data_as(C.POINTER(C.c_uint32))))
            bits = np.unpackbits(buf.view(np.uint8), bitorder="little")[: rows * cols].reshape(rows, cols)
            name = "ReLU" if L == 1 else f"layer{l}/Relu"
            out[name] = bits.astype(bool)
        return out

    def forward(self, X: torch.Tensor, Y=None, fetch=None):
        ids, ptrs, lds, n = self._feeds(X, Y)
        if fetch is None:
            fetch = self.mlp.cost
        if fetch == self.mlp.cost:
            out = torch.empty(1, dtype=torch.float32, device=X.device)
        else:
            l = self.mlp.relus.index(fetch)
            out = torch.empty((X.shape[0], self.dims[l + 1]), dtype=torch.float32, device=X.device)
        D.check(D.dflow_forward(self.s, n, ids, ptrs, lds, X.shape[0], fetch, C.c_void_p(out.data_ptr()),
                                stream_ptr()))
        torch.cuda.synchronize()
        return out.cpu().numpy()

    def stats(self):
        st = D.dflow_stats()
        D.check(D.dflow_session_stats(self.s, C.byref(st)))
        return st


def normwise(a, ref):
    a, ref = np.asarray(a, np.float64), np.asarray(ref, np.float64)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(a - ref)) / den) if den > 0 else float(np.max(np.abs(a)))


class SimRun:
    """A simulated world of `world` ranks on one GPU (dflow_sim_*): the N-GPU step's sessions
    and kernels, driven through the C ABI.  Rank r's calls go through self.ranks[r]."""

    def __init__(self, dims, loss="MSE", lr=0.25, rows=256, world=2, exchange="TRUNC16", p2p=0, sr_seed=0,
                 precision="bf16", defer_apply=0, async_dp=0, model_parallel=0, device=0):
        self.mlp = D.mlp_graph(dims, loss, lr)
        self.dims, self.loss, self.world = tuple(dims), loss, world
        prec = D.DFLOW_PRECISION_3XTF32 if precision == "3xtf32" else D.DFLOW_PRECISION_BF16
        opts = D.make_options(world=world, rank=0, device=device, exchange=exchange, max_local_rows=rows,
                              precision=prec, p2p=p2p, sr_seed=sr_seed, defer_apply=defer_apply,
                              async_dp=async_dp, model_parallel=model_parallel)
        self.w = D.sim_world(world, device)
        self.sessions = D.sim_sessions(self.w, self.mlp, opts, world)
        self.stream = D.sim_stream(self.w)

    def close(self):
        for s in self.sessions:
            if s:
                D.dflow_session_destroy(s)
        self.sessions = []
        if self.w:
            D.dflow_sim_world_destroy(self.w)
            self.w = None
        if self.mlp.graph:
            D.dflow_graph_destroy(self.mlp.graph)
            self.mlp.graph = None

    def assign(self, Ws, bs):
        for s in self.sessions:
            for nid, a in list(zip(self.mlp.weights, Ws)) + list(zip(self.mlp.biases, bs)):
                a = np.ascontiguousarray(a, np.float32)
                D.check(D.dflow_variable_assign(s, nid, a.ctypes.data_as(C.c_void_p), 0, self.stream))

    def read(self, r):
        s = self.sessions[r]
        Ws, bs = [], []
        for l, nid in enumerate(self.mlp.weights):
            a = np.empty((self.dims[l], self.dims[l + 1]), np.float32)
            D.check(D.dflow_variable_read(s, nid, a.ctypes.data_as(C.c_void_p), 0, self.stream))
            Ws.append(a)
        for l, nid in enumerate(self.mlp.biases):
            a = np.empty((self.dims[l + 1],), np.float32)
            D.check(D.dflow_variable_read(s, nid, a.ctypes.data_as(C.c_void_p), 0, self.stream))
            bs.append(a)
        return Ws, bs

    def _ids(self, with_y):
        ids = [self.mlp.x] + ([self.mlp.y] if with_y else [])
        return ids

    def step(self, Xs, Ys=None, want_loss=True):
        """One synchronous train step on every rank: Xs[r], Ys[r] device tensors [b, *]."""
        torch.cuda.synchronize()  # the feeds were written on torch's stream
        with_y = Ys is not None
        ids = self._ids(with_y)
        ptrs, lds = [], [Xs[0].stride(0)] + ([Ys[0].stride(0)] if with_y else [])
        for r in range(self.world):
            ptrs.append(Xs[r].data_ptr())
            if with_y:
                ptrs.append(Ys[r].data_ptr())
        loss = (C.c_float * self.world)()
        D.check(D.dflow_sim_train_step(self.w, (C.c_void_p * self.world)(*self.sessions), len(ids), D.node_array(ids),
                                       D.ptr_array(ptrs), D.i64_array(lds), Xs[0].shape[0],
                                       loss if want_loss else None))
        return list(loss)

    def step_rank(self, r, X, Y=None):
        """dflow_train_step of rank r alone (async_dp sessions: no collective inside)."""
        torch.cuda.synchronize()
        ids = self._ids(Y is not None)
        ptrs = [X.data_ptr()] + ([Y.data_ptr()] if Y is not None else [])
        lds = [X.stride(0)] + ([Y.stride(0)] if Y is not None else [])
        loss = C.c_float(0)
        D.check(D.dflow_train_step(self.sessions[r], len(ids), D.node_array(ids), D.ptr_array(ptrs),
                                   D.i64_array(lds), X.shape[0], C.byref(loss), self.stream))
        return loss.value

    def gradients(self, r, X, Y=None):
        torch.cuda.synchronize()
        ids = self._ids(Y is not None)
        ptrs = [X.data_ptr()] + ([Y.data_ptr()] if Y is not None else [])
        lds = [X.stride(0)] + ([Y.stride(0)] if Y is not None else [])
        outs, nodes = [], []
        for l in range(len(self.dims) - 1):
            outs.append(torch.empty((self.dims[l], self.dims[l + 1]), dtype=torch.float32, device=X.device))
            nodes.append(self.mlp.grads[self.mlp.weights[l]])
            outs.append(torch.empty((self.dims[l + 1],), dtype=torch.float32, device=X.device))
            nodes.append(self.mlp.grads[self.mlp.biases[l]])
        torch.cuda.synchronize()
        D.check(D.dflow_fetch_gradients(self.sessions[r], len(ids), D.node_array(ids), D.ptr_array(ptrs),
                                        D.i64_array(lds), X.shape[0], len(nodes), D.node_array(nodes),
                                        D.ptr_array([o.data_ptr() for o in outs]), self.stream))
        self.sync()
        res = [o.cpu().numpy() for o in outs]
        L = len(self.dims) - 1
        return [res[2 * l] for l in range(L)], [res[2 * l + 1] for l in range(L)]

    def exchange(self, grads):
        """dflow_exchange on every rank: grads[r] device fp32 [n] -> outs[r]."""
        torch.cuda.synchronize()
        n = grads[0].numel()
        outs = [torch.empty(n, dtype=torch.float32, device=grads[0].device) for _ in range(self.world)]
        torch.cuda.synchronize()
        D.check(D.dflow_sim_exchange(self.w, (C.c_void_p * self.world)(*self.sessions),
                                     D.ptr_array([g.data_ptr() for g in grads]),
                                     D.ptr_array([o.data_ptr() for o in outs]), n))
        return [o.cpu().numpy() for o in outs]

    def sync(self):
        import ctypes
        # the world's stream is a cudaStream_t; torch can wrap it for a synchronize
        torch.cuda.ExternalStream(self.stream.value).synchronize()
