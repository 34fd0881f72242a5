"""GPU parity of the whole train step vs the oracle (single GPU, N = 1).

Tolerances from north_star: bf16 path within 2e-2 (normwise max relative error
of W after one step, reading A15 (i)); gradients checked mask-locked at the same
tolerance (A15 (ii), A22).  P12: bitwise in the exact-arithmetic regime.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.mlp import build_mlp, forward, train_step  # noqa: E402
from synth import C1, C1_BIAS, C2, C3, batch, exact_regime, init_params, with_batch  # noqa: E402
import ctypes as C  # noqa: E402

import paper_1603_04467_b200 as D  # noqa: E402
from dflow_harness import Run, normwise, stream_ptr  # noqa: E402

BF16_TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"


def _dev(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _one_step_parity(w, rows=None):
    rows = rows or w.batch
    Ws, bs = init_params(w)
    X, Y = batch(w, rows=rows)
    run = Run(w.dims, w.loss, w.lr, rows=rows, with_dx=(w.layers == 1))
    try:
        run.assign(Ws, bs)
        Xd, Yd = _dev(X), _dev(Y)
        # gradients (no update) + the GPU's relu masks for the mask-locked oracle
        gW, gb, dx = run.gradients(Xd, Yd, with_dx=(w.layers == 1))
        masks = run.masks(rows)
        mg = build_mlp(w.dims, w.loss, w.lr, with_dx=(w.layers == 1))
        locked = train_step(mg, Ws, bs, X, Y, 1, "TRUNC16", masks=[masks])
        errs = {}
        for l in range(w.layers):
            errs[f"dW{l + 1}"] = normwise(gW[l], locked["ghat"][mg.weights[l]])
            errs[f"db{l + 1}"] = normwise(gb[l], locked["ghat"][mg.biases[l]])
        if dx is not None:
            errs["dx"] = normwise(dx, locked["per_replica"][0]["dx"])
        # one train step; W after vs the (unlocked) oracle — the gate as stated (A15 (i))
        loss = run.step(Xd, Yd)
        Wg, bg = run.read()
        ref = train_step(mg, Ws, bs, X, Y, 1, "TRUNC16")
        for l in range(w.layers):
            errs[f"W{l + 1}_after"] = normwise(Wg[l], ref["W"][l])
            errs[f"b{l + 1}_after"] = normwise(bg[l], ref["b"][l])
        errs["loss"] = abs(loss - ref["loss"]) / abs(ref["loss"])
        return errs, locked["flips"]
    finally:
        run.close()


@pytest.mark.parametrize("w", [C1, C1_BIAS], ids=["C1", "C1_bias"])
def test_config1_fig1_step_and_fig5_gradients(w):
    errs, flips = _one_step_parity(w)
    print(errs, flips)
    assert max(errs.values()) < BF16_TOL, errs


def test_config2_mnist_step():
    errs, flips = _one_step_parity(C2)
    print(errs, flips)
    assert max(errs.values()) < BF16_TOL, errs


@pytest.mark.parametrize("rows", [1, 100, 129, 300])
def test_ragged_batches(rows):
    errs, _ = _one_step_parity(with_batch(C2, rows), rows=rows)
    assert max(errs.values()) < BF16_TOL, errs


def test_config3_width_reduced_batch():
    errs, flips = _one_step_parity(with_batch(C3, 512))
    print(errs, flips)
    assert max(errs.values()) < BF16_TOL, errs


# SURVEY §8(c) P14, predicted before any GPU run (numpy emulation, C3 width): bf16 gradients
# mask-locked ~5.6e-3, W after one step 7.2e-5 - 3.6e-4, loss 3e-5 - 3e-3 relative
P14_C3_GRAD_LOCKED, P14_C3_W_AFTER = 5.6e-3, 3.6e-4


def test_config3_width_bench_tile_configuration():
    """C3 width at B = 2048: the auto rule picks the CTA-pair 256 x 256 kernels with the
    dynamic tile scheduler and raster group 8 for the forward, the loss-fused forward, the
    dgrad and the fused-SGD wgrad — the configuration bench.py times (B = 32768 only adds
    M tiles).  Gradients mask-locked and W after one step against the oracle (A15, A22),
    and inside a small factor of the P14 band."""
    rows = 2048
    errs, flips = _one_step_parity(with_batch(C3, rows))
    print(errs, flips)
    assert max(errs.values()) < BF16_TOL, errs
    grad = max(v for k, v in errs.items() if k.startswith(("dW", "db")))
    wafter = max(v for k, v in errs.items() if k.endswith("_after"))
    assert grad < 3 * P14_C3_GRAD_LOCKED, (grad, errs)
    assert wafter < 3 * P14_C3_W_AFTER, (wafter, errs)


def test_p12_exact_regime_bitwise():
    # Every stored intermediate is exact in bf16 and fp32 sums are order-free:
    # the GPU step must equal the oracle bit for bit (W, b after the step and grads).
    X, Y, Ws, bs, lr = exact_regime()
    dims = (784, 1024, 1024, 16)
    run = Run(dims, "MSE", lr, rows=X.shape[0])
    try:
        run.assign(Ws, bs)
        Xd, Yd = _dev(X), _dev(Y)
        gW, gb, _ = run.gradients(Xd, Yd)
        mg = build_mlp(dims, "MSE", lr)
        ref = train_step(mg, Ws, bs, X, Y, 1, "TRUNC16")
        for l in range(3):
            assert np.array_equal(gW[l], ref["ghat"][mg.weights[l]]), f"dW{l + 1}"
            assert np.array_equal(gb[l], ref["ghat"][mg.biases[l]]), f"db{l + 1}"
        loss = run.step(Xd, Yd)
        Wg, bg = run.read()
        for l in range(3):
            assert np.array_equal(Wg[l], ref["W"][l]), f"W{l + 1}"
            assert np.array_equal(bg[l], ref["b"][l]), f"b{l + 1}"
        assert loss == pytest.approx(ref["loss"], rel=1e-6)
    finally:
        run.close()


def test_p9_zero_lr_keeps_weights_bitwise():
    w = with_batch(C2, 128)
    Ws, bs = init_params(w)
    X, Y = batch(w)
    run = Run(w.dims, "MSE", 0.0, rows=128)
    try:
        run.assign(Ws, bs)
        loss = run.step(_dev(X), _dev(Y))
        Wg, bg = run.read()
        for a, b in zip(Wg + bg, Ws + bs):
            assert np.array_equal(a, b)
        mg = build_mlp(w.dims, "MSE", 0.0)
        ref = float(forward(mg, Ws, bs, X, Y)[mg.cost])
        assert abs(loss - ref) / ref < BF16_TOL
    finally:
        run.close()


def test_forward_fetch_matches_oracle():
    w = with_batch(C2, 256)
    Ws, bs = init_params(w)
    X, Y = batch(w)
    run = Run(w.dims, "MSE", w.lr, rows=256)
    try:
        run.assign(Ws, bs)
        Xd, Yd = _dev(X), _dev(Y)
        a3 = run.forward(Xd, Yd, fetch=run.mlp.relus[-1])
        c = run.forward(Xd, Yd)
        mg = build_mlp(w.dims, "MSE", w.lr)
        ref = forward(mg, Ws, bs, X, Y, fetch=[mg.acts[-1], mg.cost])
        assert normwise(a3, ref[mg.acts[-1]]) < BF16_TOL
        assert abs(float(c[0]) - float(ref[mg.cost])) / float(ref[mg.cost]) < BF16_TOL
    finally:
        run.close()


def test_p16_hundred_steps_config2():
    # PAPER.md:877-878 lessons 3-4; W after 100 steps within the bf16 tolerance.
    w = C2
    Ws, bs = init_params(w)
    run = Run(w.dims, "MSE", w.lr, rows=w.batch)
    mg = build_mlp(w.dims, "MSE", w.lr)
    try:
        run.assign(Ws, bs)
        Wr, br = Ws, bs
        losses_g, losses_r = [], []
        for step in range(100):
            X, Y = batch(w, step=step)
            losses_g.append(run.step(_dev(X), _dev(Y)))
            ref = train_step(mg, Wr, br, X, Y, 1, "TRUNC16")
            Wr, br = ref["W"], ref["b"]
            losses_r.append(ref["loss"])
        Wg, bg = run.read()
        errs = [normwise(a, b) for a, b in zip(Wg + bg, Wr + br)]
        print("loss gpu", losses_g[::10], "oracle", losses_r[::10], "W err", errs)
        assert max(errs) < BF16_TOL
        assert losses_g[-1] < losses_g[0]
    finally:
        run.close()


def test_host_fed_steps_match_device_fed_bitwise():
    # dflow_train_step_host: x uploads first, y under the first layers, step i+1's upload under
    # step i's backward; the result must be the device-fed step's, bit for bit, every step
    w = with_batch(C2, 512)
    Ws, bs = init_params(w)
    dev = Run(w.dims, "MSE", w.lr, rows=w.batch)
    host = Run(w.dims, "MSE", w.lr, rows=w.batch)
    try:
        dev.assign(Ws, bs)
        host.assign(Ws, bs)
        ids, lds = D.node_array([host.mlp.x, host.mlp.y]), D.i64_array([w.dims[0], w.dims[-1]])
        for step in range(4):
            X, Y = batch(w, step=step)
            ld = dev.step(_dev(X), _dev(Y))
            Xh, Yh = torch.from_numpy(X).pin_memory(), torch.from_numpy(Y).pin_memory()
            lh = C.c_float(0)
            D.check(D.dflow_train_step_host(host.s, 2, ids, D.ptr_array([Xh.data_ptr(), Yh.data_ptr()]), lds,
                                            w.batch, C.byref(lh) if step % 2 == 0 else None, stream_ptr()))
            if step % 2 == 0:
                assert np.float32(lh.value).view(np.uint32) == np.float32(ld).view(np.uint32), step
        Wd, bd = dev.read()
        Wh, bh = host.read()
        for a, b in zip(Wd + bd, Wh + bh):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    finally:
        dev.close()
        host.close()


@pytest.mark.parametrize("graphs", [0, 1])
def test_pipelined_host_steps_match_device_fed_bitwise(graphs):
    # dflow_train_step_host_pipelined: every call returns the PREVIOUS step's loss; all host
    # buffers (distinct per step, pinned) stay untouched until the next call; the losses and
    # the parameters must be the device-fed steps', bit for bit (with and without step graphs)
    w = with_batch(C2, 512)
    Ws, bs = init_params(w)
    dev = Run(w.dims, "MSE", w.lr, rows=w.batch)
    host = Run(w.dims, "MSE", w.lr, rows=w.batch, graphs=graphs)
    try:
        dev.assign(Ws, bs)
        host.assign(Ws, bs)
        ids, lds = D.node_array([host.mlp.x, host.mlp.y]), D.i64_array([w.dims[0], w.dims[-1]])
        steps = 5
        bufs = [tuple(torch.from_numpy(a).pin_memory() for a in batch(w, step=k)) for k in range(steps)]
        want = [dev.step(_dev(X.numpy()), _dev(Y.numpy())) for X, Y in bufs]
        got = []
        for k, (Xh, Yh) in enumerate(bufs):
            lh, has = C.c_float(0), C.c_int32(-1)
            D.check(D.dflow_train_step_host_pipelined(host.s, 2, ids, D.ptr_array([Xh.data_ptr(), Yh.data_ptr()]),
                                                      lds, w.batch, C.byref(lh), C.byref(has), stream_ptr()))
            assert has.value == (1 if k else 0), (k, has.value)
            if has.value:
                got.append(lh.value)
        lh, has = C.c_float(0), C.c_int32(-1)
        D.check(D.dflow_session_last_loss(host.s, C.byref(lh), C.byref(has)))
        assert has.value == 1
        got.append(lh.value)
        D.check(D.dflow_session_last_loss(host.s, C.byref(lh), C.byref(has)))
        assert has.value == 0  # nothing pending any more
        assert np.array_equal(np.float32(got).view(np.uint32), np.float32(want).view(np.uint32)), (got, want)
        Wd, bd = dev.read()
        Wh, bh = host.read()
        for a, b in zip(Wd + bd, Wh + bh):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    finally:
        dev.close()
        host.close()


def test_p15_non_finite_guard():
    # PAPER.md:879 (lesson 5, non-finite checks): a NaN / Inf reaching the step shows up in
    # the loss and the session's nonfinite flag; a clean step clears it
    w = with_batch(C2, 64)
    Ws, bs = init_params(w)
    run = Run(w.dims, "MSE", w.lr, rows=w.batch)
    try:
        run.assign(Ws, bs)
        X, Y = batch(w)
        assert np.isfinite(run.step(_dev(X), _dev(Y))) and run.stats().nonfinite == 0
        for bad in (np.nan, np.inf):
            Yb = Y.copy()
            Yb[3, 5] = bad
            loss = run.step(_dev(X), _dev(Yb))
            assert not np.isfinite(loss) and run.stats().nonfinite == 1
            run.assign(Ws, bs)  # the poisoned update is discarded by re-assigning
        assert np.isfinite(run.step(_dev(X), _dev(Y))) and run.stats().nonfinite == 0
    finally:
        run.close()


def test_step_graphs_replay_bitwise():
    # opt.graphs: the captured-and-replayed step computes exactly what the launched one does,
    # for device feeds (two feed signatures -> two graphs) and host feeds
    w = with_batch(C2, 256)
    Ws, bs = init_params(w)
    plain = Run(w.dims, "MSE", w.lr, rows=w.batch)
    graph = Run(w.dims, "MSE", w.lr, rows=w.batch, graphs=1)
    try:
        plain.assign(Ws, bs)
        graph.assign(Ws, bs)
        bufs = [(_dev(batch(w, step=k)[0]), _dev(batch(w, step=k)[1])) for k in range(2)]
        for step in range(6):
            X, Y = batch(w, step=step)
            Xd, Yd = bufs[step % 2]
            Xd.copy_(torch.from_numpy(X))
            Yd.copy_(torch.from_numpy(Y))
            lp = plain.step(Xd, Yd)
            lg = graph.step(Xd, Yd, want_loss=(step != 3))
            if step != 3:
                assert np.float32(lp).view(np.uint32) == np.float32(lg).view(np.uint32), step
        ids, lds = D.node_array([graph.mlp.x, graph.mlp.y]), D.i64_array([w.dims[0], w.dims[-1]])
        for step in range(6, 9):
            X, Y = batch(w, step=step)
            lp = plain.step(_dev(X), _dev(Y))
            Xh, Yh = torch.from_numpy(X).pin_memory(), torch.from_numpy(Y).pin_memory()
            lh = C.c_float(0)
            D.check(D.dflow_train_step_host(graph.s, 2, ids, D.ptr_array([Xh.data_ptr(), Yh.data_ptr()]), lds,
                                            w.batch, C.byref(lh), stream_ptr()))
            assert np.float32(lp).view(np.uint32) == np.float32(lh.value).view(np.uint32), step
        Wp, bp = plain.read()
        Wg, bg = graph.read()
        for a, b in zip(Wp + bp, Wg + bg):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    finally:
        plain.close()
        graph.close()


def test_raster_group_leaves_results_bitwise(monkeypatch):
    # The tile raster (DFLOW_GEMM_GROUP_{FWD,DGRAD,WGRAD}) only reorders which SM
    # computes which output tile: every tile's k-walk, and the per-tile loss / db partials that
    # are summed in tile order, are unchanged, so W, b and the loss must be bit-identical.
    w = with_batch(C3, 2048)
    Ws, bs = init_params(w)
    X, Y = batch(w)
    out = []
    for groups in [{}, {"DFLOW_GEMM_GROUP_FWD": "2", "DFLOW_GEMM_GROUP_DGRAD": "3", "DFLOW_GEMM_GROUP_WGRAD": "5"}]:
        for k in ("DFLOW_GEMM_GROUP_FWD", "DFLOW_GEMM_GROUP_DGRAD", "DFLOW_GEMM_GROUP_WGRAD"):
            monkeypatch.delenv(k, raising=False)
        for k, v in groups.items():
            monkeypatch.setenv(k, v)
        run = Run(w.dims, w.loss, w.lr, rows=2048)
        try:
            run.assign(Ws, bs)
            loss = run.step(_dev(X), _dev(Y))
            Wg, bg = run.read()
            out.append((loss, Wg, bg))
        finally:
            run.close()
    (l0, W0, b0), (l1, W1, b1) = out
    assert l0 == l1
    for a, b in zip(W0 + b0, W1 + b1):
        assert np.array_equal(a, b)


def test_wide_tile_knob_leaves_results_bitwise(monkeypatch):
    # DFLOW_GEMM_TILE512=1 (off by default) runs every GEMM of the step on the
    # 256 x 512 pair tile (fused loss seed, ReluGrad + db partials, fused SGD included): each
    # output element still accumulates its K products in the same order, so W and b after a
    # step are bit-identical; the cost's fp64 partials are summed per tile, so only the sum
    # order of the loss changes.
    w = with_batch(C3, 2048)
    Ws, bs = init_params(w)
    X, Y = batch(w)
    out = []
    for wide in ("0", "1"):
        monkeypatch.setenv("DFLOW_GEMM_TILE512", wide)
        run = Run(w.dims, w.loss, w.lr, rows=2048)
        try:
            run.assign(Ws, bs)
            loss = run.step(_dev(X), _dev(Y))
            Wg, bg = run.read()
            out.append((loss, Wg, bg))
        finally:
            run.close()
    (l0, W0, b0), (l1, W1, b1) = out
    assert abs(l0 - l1) <= 1e-6 * abs(l0)
    for a, b in zip(W0 + b0, W1 + b1):
        assert np.array_equal(a, b)


def test_loss_bitwise_reproducible_under_dynamic_scheduler():
    """The cost is summed from one fp64 partial per (tile, CTA, epilogue warp) in a fixed
    order, so repeated forwards give the same bits even though the dynamic tile scheduler
    hands tiles to different CTAs each time (C3 width, B = 2048: CTA-pair loss epilogue)."""
    w = with_batch(C3, 2048)
    Ws, bs = init_params(w)
    X, Y = batch(w)
    run = Run(w.dims, w.loss, w.lr, rows=w.batch)
    try:
        run.assign(Ws, bs)
        Xd, Yd = _dev(X), _dev(Y)
        vals = {run.forward(Xd, Yd)[0].tobytes() for _ in range(8)}
        assert len(vals) == 1
    finally:
        run.close()
