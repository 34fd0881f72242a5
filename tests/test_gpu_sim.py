"""The N-GPU step on ONE GPU: simulated worlds of N = 2, 4, 8 ranks (include/dflow.h
dflow_sim_*), bit-exact against the oracle.  PAPER.md §7 :934-941 (synchronous replicas,
"combine the gradients"), §5.5 :813-821 (the 32->16 channel codec), :948-955 (asynchronous
replicas), :958-972 (model parallelism); SURVEY §8(a) a6-a9, §8(f) f1-f4.

Each simulated rank is a full session created with the options it would have on N GPUs;
the fused NVLink exchange stores into the other ranks' buffers on the same device, so these
tests run the production kernels of the N > 1 path — the dW GEMM with EPI_TRUNC16_P2P (CTA
pair, BN = 256, at the C3 width with 2048 rows per rank; single CTA at the C2 width), the
per-layer db pass k_colsum_final_p2p, the owner fold k_owner_reduce_p2p with owner-apply
(bf16) and without it (3xTF32: u16 gather + k_apply_sgd_tf32), the NCCL-schedule kernels
k_owner_reduce_t16 / k_owner_reduce_f32 / k_apply_sgd_vec on u16 or fp32 between simulated
all-to-all / all-gather copies, the SR16 coder, EPI_ASYNC_PUSH and the f4 channel ends.

Checks (as tests/mgpu_worker.py on real GPUs):
  P4   dflow_exchange alone == oracle.exchange.combine, bit for bit (ragged n)
  P4'  W, b after one step == oracle apply(oracle combine(GPU's own fp32 gradients of every
       rank)), bit for bit, on every rank (P11)
  gate (C2 width) W after one step within 2e-2 (bf16) / 1e-4 (3xTF32 + FP32 channel) of the
       oracle's N-replica step on the same global batch
  P11  all ranks bitwise identical after 4 steps; defer_apply == eager join bit for bit
"""
import ctypes as C
import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1603_04467_b200 as D  # noqa: E402
from dflow_harness import SimRun, normwise  # noqa: E402
from oracle import kernels as OK  # noqa: E402
from oracle.async_dp import push  # noqa: E402
from oracle.exchange import combine  # noqa: E402
from oracle.mlp import build_mlp, train_step  # noqa: E402
from oracle.partition import train_step_model_parallel  # noqa: E402
import synth  # noqa: E402

SEED = 1234  # SR16 draw streams (reading A27)
C3W_ROWS = 2048  # per rank: the dW GEMM (8192 x 8192, K = 2048) runs the CTA-pair kernel


def _parse(spec):
    ex, p2p, defer, prec = spec, 0, 0, "bf16"
    if ex.endswith("_DEFER"):
        ex, defer = ex[:-6], 1
    if ex.endswith("_TF32"):
        ex, prec = ex[:-5], "3xtf32"
    if ex.endswith("_P2P"):
        ex, p2p = ex[:-4], 1
    return ex, p2p, defer, prec


def _workload(width, world):
    if width == "C2":
        return synth.with_batch(synth.C2, 256)
    # C3 width (8192 x 8192 layers, the bench's tile configuration), two layers
    return synth.Workload("C3w2", (8192, 8192, 8192), C3W_ROWS * world, "MSE", 2.0 ** -2, "he")


def _buckets(gW, gb):
    return [np.concatenate([a.ravel(), c.ravel()]).astype(np.float32) for a, c in zip(gW, gb)]


def _bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _rank_feeds(w, world, step=None):
    b = w.batch // world
    X, Y = synth.batch(w, step=step)
    return ([torch.from_numpy(X[r * b:(r + 1) * b]).cuda() for r in range(world)],
            [torch.from_numpy(Y[r * b:(r + 1) * b]).cuda() for r in range(world)], X, Y)


def _sync_case(world, spec, width):
    ex, p2p, defer, prec = _parse(spec)
    w = _workload(width, world)
    b = w.batch // world
    Ws, bs = synth.init_params(w)
    run = SimRun(w.dims, "MSE", w.lr, rows=b, world=world, exchange=ex, p2p=p2p, sr_seed=SEED, precision=prec,
                 defer_apply=defer)
    try:
        run.assign(Ws, bs)
        # P4: the exchange alone on random gradients of a ragged length
        n = 100003
        gs = [synth.rng(500 + r).standard_normal(n).astype(np.float32) for r in range(world)]
        outs = run.exchange([torch.from_numpy(g).cuda() for g in gs])
        ref = combine(gs, ex if ex != "FP32_NCCL" else "FP32", sr=(SEED, 1, 0))
        # (the simulated all-reduce sums in rank order, so FP32_NCCL is bit-exact here too)
        assert all(_bits_equal(o, ref) for o in outs), "P4: exchange differs from the oracle"

        Xs, Ys, X, Y = _rank_feeds(w, world)
        per_rank = [_buckets(*run.gradients(r, Xs[r], Ys[r])) for r in range(world)]
        losses = run.step(Xs, Ys)
        assert len(set(np.float32(v).tobytes() for v in losses)) == 1, losses  # one all-reduced loss
        got = [run.read(r) for r in range(world)]
        # P11: every rank holds the same bits
        for r in range(1, world):
            assert all(_bits_equal(a, c) for a, c in zip(got[0][0] + got[0][1], got[r][0] + got[r][1])), r
        # P4': oracle combine + ApplyGradientDescent of the GPU's own gradients, bit for bit
        Wg, bg = got[0]
        for l in range(w.layers):
            nw = Ws[l].size
            ghat = combine([p[l] for p in per_rank], ex if ex != "FP32_NCCL" else "FP32", sr=(SEED, 1, l))
            new_w = OK.apply_gradient_descent(Ws[l], w.lr, ghat[:nw].reshape(Ws[l].shape), "f32")
            new_b = OK.apply_gradient_descent(bs[l], w.lr, ghat[nw:], "f32")
            assert _bits_equal(new_w, Wg[l]), f"P4': W_{l + 1} differs from oracle exchange + apply"
            assert _bits_equal(new_b, bg[l]), f"P4': b_{l + 1} differs from oracle exchange + apply"
        del per_rank
        if width == "C2":  # the north-star gate against the oracle's N-replica step
            mg = build_mlp(w.dims, "MSE", w.lr)
            oref = train_step(mg, Ws, bs, X, Y, world, ex if ex != "FP32_NCCL" else "FP32", sr_seed=SEED, step=1)
            err = max(normwise(a, r) for a, r in zip(Wg + bg, oref["W"] + oref["b"]))
            tol = 1e-4 if (prec == "3xtf32" and ex == "FP32") else 2e-2
            assert err < tol, err
            assert abs(losses[0] - oref["loss"]) / oref["loss"] < tol
        # three more steps: the replicas stay identical (P11)
        for step in range(3):
            Xs, Ys, _, _ = _rank_feeds(w, world, step=step)
            run.step(Xs, Ys, want_loss=False)
        fin = [run.read(r) for r in range(world)]
        for r in range(1, world):
            assert all(_bits_equal(a, c) for a, c in zip(fin[0][0] + fin[0][1], fin[r][0] + fin[r][1])), r
        return fin[0]
    finally:
        run.close()


SYNC_C2 = [(n, e) for n in (2, 4, 8) for e in ("TRUNC16_P2P", "SR16_P2P", "TRUNC16", "FP32")] + [
    (2, "FP32_NCCL"), (8, "SR16"), (2, "TRUNC16_P2P_TF32"), (8, "TRUNC16_P2P_TF32"), (4, "FP32_TF32"),
    (4, "TRUNC16_P2P_DEFER"), (8, "TRUNC16_P2P_DEFER"), (8, "TRUNC16_DEFER")]


@pytest.mark.parametrize("world,spec", SYNC_C2)
def test_sim_step_c2_width(world, spec):
    """C2 widths (784-1024-1024-10, global batch 256): every GEMM on the single-CTA tile."""
    _sync_case(world, spec, "C2")


SYNC_C3W = [(2, "TRUNC16_P2P"), (4, "TRUNC16_P2P"), (8, "TRUNC16_P2P"), (8, "SR16_P2P"), (4, "TRUNC16"),
            (4, "TRUNC16_P2P_DEFER"), (4, "TRUNC16_P2P_TF32")]


@pytest.mark.parametrize("world,spec", SYNC_C3W)
def test_sim_step_c3_width(world, spec):
    """C3 width (8192 x 8192 layers), 2048 rows per rank: the dW GEMM of the exchange
    (EPI_TRUNC16_P2P) runs the CTA-pair 256 x 256 kernel the C3 bench runs at N = 2..8."""
    _sync_case(world, spec, "C3w")


@pytest.mark.parametrize("world,spec,width", [(4, "TRUNC16_P2P", "C2"), (8, "TRUNC16", "C2"),
                                              (4, "TRUNC16_P2P", "C3w")])
def test_sim_defer_equals_eager(world, spec, width):
    """options.defer_apply runs the same arithmetic: 4 steps give the eager join's bits."""
    a = _sync_case(world, spec + "_DEFER", width)
    b = _sync_case(world, spec, width)
    assert all(_bits_equal(x, y) for x, y in zip(a[0] + a[1], b[0] + b[1]))


@pytest.mark.parametrize("world,exchange,width", [(2, "TRUNC16", "C2"), (2, "SR16", "C2"), (4, "FP32", "C2"),
                                                  (8, "TRUNC16", "C2"), (4, "TRUNC16", "C3w")])
def test_sim_async_replicas(world, exchange, width):
    """f3: replicas serialised in rank order — each pull == the oracle's
    shared W after the previous pushes, and the final shared W == oracle.async_dp.push of the
    GPU's own gradients in rank order, bit for bit (EPI_ASYNC_PUSH: single CTA at the C2
    width, CTA pair at the C3 width).  Then all ranks push from one point at once: at N = 2
    every element equals one of the two application orders."""
    w = _workload(width, world)
    b = w.batch // world
    Ws, bs = synth.init_params(w)
    Xs, Ys, _, _ = _rank_feeds(w, world)
    run = SimRun(w.dims, "MSE", w.lr, rows=b, world=world, exchange=exchange, sr_seed=SEED, async_dp=2)
    try:
        run.assign(Ws, bs)
        Wref = [(a.copy(), c.copy()) for a, c in zip(Ws, bs)]
        for turn in range(world):
            D.check(D.dflow_async_pull(run.sessions[turn], run.stream))
            Wp, bp = run.read(turn)
            assert all(_bits_equal(a, r[0]) and _bits_equal(c, r[1]) for a, c, r in zip(Wp, bp, Wref)), turn
            gW, gb = run.gradients(turn, Xs[turn], Ys[turn])
            run.step_rank(turn, Xs[turn], Ys[turn])
            Wref = [push(Wl, bl, gw, gbl, w.lr, turn, world, exchange, (SEED, 1, l))
                    for l, ((Wl, bl), gw, gbl) in enumerate(zip(Wref, gW, gb))]
        run.sync()
        Wf, bf = run.read(0)
        assert all(_bits_equal(a, r[0]) and _bits_equal(c, r[1]) for a, c, r in zip(Wf, bf, Wref))
    finally:
        run.close()
    if world != 2 or width != "C2":
        return
    run = SimRun(w.dims, "MSE", w.lr, rows=b, world=world, exchange=exchange, sr_seed=SEED, async_dp=2)
    try:
        run.assign(Ws, bs)
        gs = []
        for r in range(world):
            D.check(D.dflow_async_pull(run.sessions[r], run.stream))
            gs.append(run.gradients(r, Xs[r], Ys[r]))
        run.step(Xs, Ys)  # every rank pushes (host threads enqueue concurrently)
        Wf, bf = run.read(0)

        def sequence(order):
            cur = [(a.copy(), c.copy()) for a, c in zip(Ws, bs)]
            for r in order:
                cur = [push(Wl, bl, gw, gbl, w.lr, r, world, exchange, (SEED, 1, l))
                       for l, ((Wl, bl), gw, gbl) in enumerate(zip(cur, gs[r][0], gs[r][1]))]
            return cur
        fwd, rev = sequence(range(world)), sequence(reversed(range(world)))
        for (a, c), (f1, f2), (r1, r2) in zip(zip(Wf, bf), fwd, rev):
            assert np.all((a.view(np.uint32) == f1.view(np.uint32)) | (a.view(np.uint32) == r1.view(np.uint32)))
            assert np.all((c.view(np.uint32) == f2.view(np.uint32)) | (c.view(np.uint32) == r2.view(np.uint32)))
    finally:
        run.close()


@pytest.mark.parametrize("world", [2, 3])
def test_sim_model_parallel_exact(world):
    """f4 (readings A32-A34) in the P12 exact regime: the layer-partitioned
    step over `world` simulated devices == oracle.partition.train_step_model_parallel, bit for
    bit, for every layer (read from its owner rank)."""
    X, Y, Ws, bs, lr = synth.exact_regime()
    dims = (X.shape[1],) + tuple(W.shape[1] for W in Ws)
    L = len(dims) - 1
    run = SimRun(dims, "MSE", lr, rows=X.shape[0], world=world, model_parallel=1)
    try:
        run.assign(Ws, bs)
        Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
        losses = run.step([Xd] * world, [Yd] * world)
        assert len(set(np.float32(v).tobytes() for v in losses)) == 1, losses
        mg = build_mlp(dims, "MSE", lr)
        mp = train_step_model_parallel(mg, Ws, bs, X, Y, world)
        for l in range(L):
            owner = (l * world) // L
            Wg, bg = run.read(owner)
            assert _bits_equal(Wg[l], mp["W"][l]) and _bits_equal(bg[l], mp["b"][l]), l
    finally:
        run.close()


def test_sim_model_parallel_c2(world=2):
    """f4 on C2-shaped random data: W after one step within the bf16 tolerance of the oracle's
    partitioned step; three more steps lower the loss."""
    w = synth.with_batch(synth.C2, 256)
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w)
    run = SimRun(w.dims, "MSE", w.lr, rows=w.batch, world=world, model_parallel=1)
    try:
        run.assign(Ws, bs)
        Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
        losses = [run.step([Xd] * world, [Yd] * world)[0]]
        L = w.layers
        Wg = [run.read((l * world) // L)[0][l] for l in range(L)]
        bg = [run.read((l * world) // L)[1][l] for l in range(L)]
        mp = train_step_model_parallel(build_mlp(w.dims, "MSE", w.lr), Ws, bs, X, Y, world)
        assert max(normwise(a, r) for a, r in zip(Wg + bg, mp["W"] + mp["b"])) < 2e-2
        assert abs(losses[0] - mp["loss"]) / mp["loss"] < 2e-2
        for k in range(3):
            Xs, Ys = synth.batch(w, step=1 + k)
            losses.append(run.step([torch.from_numpy(Xs).cuda()] * world, [torch.from_numpy(Ys).cuda()] * world)[0])
        assert np.mean(losses[-2:]) < losses[0], losses
    finally:
        run.close()


def test_sim_dead_peer_poisons_within_timeout(monkeypatch):
    """A rank that dies mid-step (sends no contributions) must not hang the GPU: every bounded
    flag wait gives up after DFLOW_P2P_TIMEOUT_MS and every session of the world reports
    DFLOW_SESSION_POISONED (abort and restart)."""
    monkeypatch.setenv("DFLOW_P2P_TIMEOUT_MS", "300")
    w = synth.with_batch(synth.C2, 128)
    world = 2
    Ws, bs = synth.init_params(w)
    run = SimRun(w.dims, "MSE", w.lr, rows=w.batch // world, world=world, exchange="TRUNC16", p2p=1)
    try:
        run.assign(Ws, bs)
        Xs, Ys, _, _ = _rank_feeds(w, world)
        run.step(Xs, Ys)  # a healthy step first
        D.check(D.dflow_sim_world_drop_rank(run.w, 1))
        t0 = time.time()
        try:
            run.step(Xs, Ys)
        except D.DflowError as e:
            assert e.status == D.DFLOW_SESSION_POISONED, e
        run.sync()
        elapsed = time.time() - t0
        assert elapsed < 30, elapsed  # bounded: a handful of 0.3 s waits, not a hang
        for s in run.sessions:
            a = np.empty(w.dims[1], np.float32)
            st = D.dflow_variable_read(s, run.mlp.biases[0], a.ctypes.data_as(C.c_void_p), 0, run.stream)
            assert st == D.DFLOW_SESSION_POISONED, D.STATUS.get(st)
    finally:
        run.close()


def test_rejected_step_changes_nothing():
    """A step rejected by its argument checks (here: the MSE target not fed) returns
    DFLOW_INVALID_ARGUMENT on every rank before anything is enqueued and does not advance the
    step counter that keys the flags and the SR16 draws: the next good step gives exactly the
    bits of a world that never saw the bad call (SR16 over the fused channel, N = 4)."""
    w = synth.with_batch(synth.C2, 256)
    world = 4
    b = w.batch // world
    Ws, bs = synth.init_params(w)
    Xs, Ys, _, _ = _rank_feeds(w, world)
    res = []
    for bad in (True, False):
        run = SimRun(w.dims, "MSE", w.lr, rows=b, world=world, exchange="SR16", p2p=1, sr_seed=SEED)
        try:
            run.assign(Ws, bs)
            if bad:
                with pytest.raises(D.DflowError) as e:
                    run.step(Xs, None)
                assert e.value.status == D.DFLOW_INVALID_ARGUMENT
            run.step(Xs, Ys)
            run.step(Xs, Ys)
            res.append(run.read(0))
        finally:
            run.close()
    assert all(_bits_equal(a, c) for a, c in zip(res[0][0] + res[0][1], res[1][0] + res[1][1]))
