"""Pins for the oracle's replicated train step: P9, P10, P12, P14/P17.  CPU only."""
import numpy as np
import pytest

from oracle.mlp import build_mlp, forward, train_step
from synth import C2, exact_regime, init_params, batch, rng, with_batch


def _normwise(a, ref):
    a, ref = np.asarray(a, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(a - ref)) / max(np.max(np.abs(ref)), 1e-300))


def test_p9_zero_learning_rate_is_identity():
    # PAPER.md:877 (lesson 3): with lr = 0 the update leaves W bitwise unchanged and
    # the loss equals the forward-only loss.
    w = with_batch(C2, 64)
    Ws, bs = init_params(w)
    X, Y = batch(w)
    mg = build_mlp(w.dims, "MSE", 0.0)
    out = train_step(mg, Ws, bs, X, Y, n_replicas=2, exchange="TRUNC16")
    for a, b in zip(out["W"] + out["b"], Ws + bs):
        assert np.array_equal(a, b)
    fwd = float(forward(mg, Ws, bs, X[:32], Y[:32])[mg.cost])
    fwd2 = float(forward(mg, Ws, bs, X[32:], Y[32:])[mg.cost])
    assert out["loss"] == pytest.approx((fwd + fwd2) / 2, rel=1e-7)


def test_p10_replicas_equal_one_replica_on_the_concatenated_batch():
    # "behave exactly as if we were running the sequential SGD
    # algorithm with a batch size of 1000".  Pure f64: <= 1e-12; fp32 op
    # boundaries: <= 1e-5.
    dims = (20, 16, 12, 4)
    g = rng(11)
    Ws = [g.uniform(-0.5, 0.5, (dims[i], dims[i + 1])) for i in range(3)]
    bs = [g.uniform(-0.1, 0.1, dims[i + 1]) for i in range(3)]
    X = g.uniform(0, 1, (32, dims[0]))
    Y = g.uniform(0, 1, (32, dims[-1]))
    mg = build_mlp(dims, "MSE", 0.25)
    one = train_step(mg, Ws, bs, X, Y, 1, "FP32", mode="f64")
    four = train_step(mg, Ws, bs, X, Y, 4, "FP32", mode="f64")
    for a, b in zip(four["W"] + four["b"], one["W"] + one["b"]):
        assert _normwise(a, b) <= 1e-12
    one32 = train_step(mg, Ws, bs, X, Y, 1, "FP32", mode="f32")
    four32 = train_step(mg, Ws, bs, X, Y, 4, "FP32", mode="f32")
    for a, b in zip(four32["W"] + four32["b"], one32["W"] + one32["b"]):
        assert _normwise(a, b) <= 1e-5
    for v in mg.weights + mg.biases:  # gradients themselves
        assert _normwise(four["ghat"][v], one["ghat"][v]) <= 1e-12


def _bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float32 (test-side emulation of
    the GPU operand precision, reading A19)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def _grid_exponent(x):
    x = np.asarray(x, np.float64)
    for e in range(0, 80):
        s = x * 2.0 ** e
        if np.all(s == np.round(s)):
            return e
    raise AssertionError("values not on a power-of-two grid")


def test_p12_exact_regime_is_exact():
    # Every stored intermediate is exactly representable in bf16 (activations,
    # dZ) and every gradient sum fits in <= 22 significant bits on its grid, so the
    # fp32-boundary oracle equals the pure-f64 step bit for bit and any fp32
    # summation order (a GPU's) must reproduce it.
    X, Y, Ws, bs, lr = exact_regime()
    mg = build_mlp((784, 1024, 1024, 16), "MSE", lr)
    ex = train_step(mg, Ws, bs, X, Y, 1, "FP32", mode="f32",
                    masks=None)
    f64 = train_step(mg, Ws, bs, X, Y, 1, "FP32", mode="f64")
    for v in mg.weights + mg.biases:
        assert np.array_equal(ex["ghat"][v].astype(np.float64), f64["ghat"][v]), v
    # representability of stored intermediates
    from oracle.mlp import replica_gradients
    extra = mg.acts + [mg.graph.by_name[a].name for a in mg.acts]
    r = replica_gradients(mg, Ws, bs, X, Y, "f64", extra=list(dict.fromkeys(mg.acts + [
        "grad/C/pred", "grad/layer3/Relu/x", "grad/layer2/Relu/x", "grad/layer1/Relu/x"])))
    for name in mg.acts + ["grad/layer3/Relu/x", "grad/layer2/Relu/x", "grad/layer1/Relu/x"]:
        v = r[name].astype(np.float32)
        assert np.array_equal(_bf16(v), v), name
    # partial sums of dW = A^T dZ fit in 22 bits on the common grid
    acts = [X] + [r[a] for a in mg.acts[:-1]]
    dzs = [r[f"grad/layer{l}/Relu/x"] for l in (1, 2, 3)]
    nonzero = 0
    for A, dZ in zip(acts, dzs):
        e = _grid_exponent(A) + _grid_exponent(dZ)
        bound = np.abs(A).T @ np.abs(dZ)
        assert np.max(bound) * 2.0 ** e < 2 ** 22
        nonzero += int(np.count_nonzero(A.T @ dZ))
    assert nonzero > 1000  # enough nonzero dW entries to expose a misplaced tile


def _emulated_bf16_step(w, Ws, bs, X, Y):
    """bf16-operand / f64-accumulate emulation of the GPU step (P14 prediction)."""
    acts, pre = [_bf16(X)], []
    for W, b in zip(Ws, bs):
        z = acts[-1].astype(np.float64) @ _bf16(W).astype(np.float64) + b
        pre.append(z)
        acts.append(_bf16(np.maximum(z, 0).astype(np.float32)))
    a = np.maximum(pre[-1], 0).astype(np.float32)
    rows, cols = a.shape
    dA = (a.astype(np.float64) - Y) / (rows * cols)
    dZ = _bf16((dA * (pre[-1] > 0)).astype(np.float32)).astype(np.float64)
    gW, gb = [None] * len(Ws), [None] * len(Ws)
    masks = {}
    for l in reversed(range(len(Ws))):
        gW[l] = acts[l].astype(np.float64).T @ dZ
        gb[l] = dZ.sum(0)
        if l > 0:
            dX = dZ @ _bf16(Ws[l]).astype(np.float64).T
            dZ = _bf16((dX * (pre[l - 1] > 0)).astype(np.float32)).astype(np.float64)
    for l in range(len(Ws)):
        masks[f"layer{l + 1}/Relu"] = pre[l] > 0
    return gW, gb, masks


def test_p14_p17_error_magnitude_bands_and_mask_locking():
    # PAPER.md:880-888 (lesson 6): predict the error magnitude before any GPU run.
    # bf16 emulation vs the oracle: weights-after-one-step far inside 2e-2; gradients
    # mask-locked (A22) tighter than unlocked; the oracle's flip count is small.
    w = with_batch(C2, 256)
    Ws, bs = init_params(w)
    X, Y = batch(w)
    mg = build_mlp(w.dims, "MSE", w.lr)
    gW, gb, masks = _emulated_bf16_step(w, Ws, bs, X, Y)
    ref = train_step(mg, Ws, bs, X, Y, 1, "FP32")
    locked = train_step(mg, Ws, bs, X, Y, 1, "FP32", masks=[masks])
    assert sum(locked["flips"]) < 0.01 * 256 * (1024 + 1024 + 10)
    errs_locked = [_normwise(gW[l], locked["ghat"][mg.weights[l]]) for l in range(3)]
    assert max(errs_locked) < 2e-2 and max(errs_locked) > 1e-5
    W_after = [(Ws[l] - np.float32(w.lr) * gW[l].astype(np.float32)).astype(np.float32) for l in range(3)]
    errs_w = [_normwise(W_after[l], ref["W"][l]) for l in range(3)]
    assert max(errs_w) < 1e-3
