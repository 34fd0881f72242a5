"""N > 1 host logic on CPU (world_size 2, gloo): the rank sharding, the id
broadcast and max-over-ranks timing that bench.py uses, and the exchange
protocol of the CUDA path (per-layer bucket [dW || db] padded to 8N, rank j owns
elements [j*P/N, (j+1)*P/N), all-to-all -> owner fold -> all-gather of 16-bit
payloads) replayed with gloo collectives and the oracle's arithmetic on each
rank's own shard; the result must equal the single-process oracle N-replica step
bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from oracle.codec import expand16, truncate16
from oracle.exchange import owner_reduce_trunc16
from oracle.mlp import build_mlp, replica_gradients, train_step
from synth import C2, batch, init_params, with_batch


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = with_batch(C2, 64)
        row0, b = bench.shard_rows(w.batch, world, rank)
        # id broadcast (the NCCL unique id path) and max-over-ranks timing
        payload = bytes(range(128)) if rank == 0 else None
        got = bench.broadcast_bytes(payload, dist, "cpu")
        assert got == bytes(range(128))
        assert bench.max_over_ranks(float(rank + 1), dist, "cpu") == float(world)
        Ws, bs = init_params(w)
        X, Y = batch(w, rows=b, row0=row0)
        mg = build_mlp(w.dims, w.loss, w.lr)
        g = replica_gradients(mg, Ws, bs, X, Y)
        new = []
        for v, var in zip(mg.weights + mg.biases, Ws + bs):
            P = g[v].size
            ppad = -(-P // (8 * world)) * (8 * world)
            shard = ppad // world
            q = np.zeros(ppad, np.uint16)
            q[:P] = truncate16(g[v].ravel())
            # all-to-all: rank j receives everyone's shard j (in rank order)
            parts = [torch.from_numpy(q.astype(np.int32)) for _ in range(world)]
            gathered = [torch.zeros(ppad, dtype=torch.int32) for _ in range(world)]
            dist.all_gather(gathered, parts[0])
            recv = [gathered[r].numpy().astype(np.uint16)[rank * shard:(rank + 1) * shard] for r in range(world)]
            own = owner_reduce_trunc16(recv)
            allg = [torch.zeros(shard, dtype=torch.int32) for _ in range(world)]
            dist.all_gather(allg, torch.from_numpy(own.astype(np.int32)))
            full = np.concatenate([a.numpy().astype(np.uint16) for a in allg])[:P]
            ghat = expand16(full).reshape(var.shape)
            s = (np.float32(w.lr) * ghat).astype(np.float32)
            new.append((var - s).astype(np.float32))
        if rank == 0:
            X, Y = batch(w)
            ref = train_step(mg, Ws, bs, X, Y, world, "TRUNC16")
            ok = all(np.array_equal(a, r) for a, r in zip(new, ref["W"] + ref["b"]))
            out.put(ok)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_protocol_matches_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def test_shard_rows_cover_the_batch_without_overlap():
    for world in (1, 2, 4, 8):
        spans = [bench.shard_rows(32768, world, r) for r in range(world)]
        assert spans[0][0] == 0 and all(b == 32768 // world for _, b in spans)
        assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        bench.shard_rows(100, 8, 0)
