"""f2 on one GPU ("mathematically correct probabilistic
rounding" vs the paper's truncation): a simulated world of N = 4 ranks.

  A. The signature of the two codecs on real gradients (P18): every rank's fp32 dW of the
     C2-shaped MLP, exchanged through the TRUNC16 and SR16 channels and through the FP32
     channel (the exact mean up to one fp32 rounding).  Truncation's two stages bias the mean
     by about -2 x 2^-8 E[1/m] ~ -5e-3 relative; stochastic rounding is unbiased, so its mean
     signed relative error sits at ~0 (within the noise of N = 4 draws per element).
  B. Training: 60 synchronous C2 steps from the same initialisation and batches with each
     channel: the loss falls under all three, and the TRUNC16 and SR16 curves stay within a
     few per mille of FP32's (the paper's observation that the lossy channel trains).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from dflow_harness import SimRun  # noqa: E402

N = 4
SEED = 77


def _per_rank_grads(w, Ws, bs):
    b = w.batch // N
    X, Y = synth.batch(w)
    run = SimRun(w.dims, "MSE", w.lr, rows=b, world=N, exchange="FP32")
    try:
        run.assign(Ws, bs)
        out = []
        for r in range(N):
            gW, _ = run.gradients(r, torch.from_numpy(X[r * b:(r + 1) * b]).cuda(),
                                  torch.from_numpy(Y[r * b:(r + 1) * b]).cuda())
            out.append(gW[1].ravel())  # the second layer (2048 x 2048)
        return out
    finally:
        run.close()


def _exchange(w, grads, exchange):
    run = SimRun(w.dims, "MSE", w.lr, rows=8, world=N, exchange=exchange, sr_seed=SEED)
    try:
        return run.exchange([torch.from_numpy(g).cuda() for g in grads])[0]
    finally:
        run.close()


def test_sr16_unbiased_truncation_biased_on_real_gradients():
    # 8192 rows per rank (the C3 bench's per-GPU batch at N = 4): every rank's gradient is a
    # long sum with the same sign as the mean, the regime of P18 (with a few dozen rows per
    # rank the ranks' signs disagree and the first stage's biases cancel in the mean)
    w = synth.Workload("sig_2048", (2048, 2048, 2048), 4 * 8192, "MSE", 2.0 ** -2, "he")
    Ws, bs = synth.init_params(w)
    grads = _per_rank_grads(w, Ws, bs)
    ref = _exchange(w, grads, "FP32").astype(np.float64)
    sel = np.abs(ref) > 1e-3 * np.max(np.abs(ref))  # away from exact cancellation
    t16 = _exchange(w, grads, "TRUNC16").astype(np.float64)
    sr16 = _exchange(w, grads, "SR16").astype(np.float64)
    # signed relative error (g_hat - g) / g: < 0 when the magnitude shrinks, whatever the sign
    bias_t = float(np.mean((t16[sel] - ref[sel]) / ref[sel]))
    bias_s = float(np.mean((sr16[sel] - ref[sel]) / ref[sel]))
    print({"trunc16_mean_rel": bias_t, "sr16_mean_rel": bias_s, "elements": int(sel.sum())})
    assert -8e-3 < bias_t < -2e-3, bias_t                 # two truncations toward zero (P18)
    assert abs(bias_s) < 0.1 * abs(bias_t), (bias_s, bias_t)  # unbiased (reading A26)
    # both within the two-stage bound, element by element: stage 1 moves each g_r by < 2^-7 |g_r|,
    # stage 2 the mean by < 2^-7 of itself: |g_hat - mean| < 2^-7 (A + |mean| + 2^-7 A),
    # A = sum_r |g_r| / N (SR16's draws move a value by less than one bf16 ulp as well)
    A = np.mean([np.abs(g.astype(np.float64)) for g in grads], axis=0)
    bound = 2.0 ** -7 * (A + np.abs(ref) + 2.0 ** -7 * A) + 1e-30
    assert np.all(np.abs(t16 - ref) <= bound)
    assert np.all(np.abs(sr16 - ref) <= bound)


def test_three_channels_train_alike():
    w = synth.with_batch(synth.C2, 256)
    Ws, bs = synth.init_params(w)
    b = w.batch // N
    curves = {}
    for ex in ("FP32", "TRUNC16", "SR16"):
        run = SimRun(w.dims, "MSE", w.lr, rows=b, world=N, exchange=ex, p2p=1 if ex != "FP32" else 0, sr_seed=SEED)
        try:
            run.assign(Ws, bs)
            losses = []
            for step in range(60):
                X, Y = synth.batch(w, step=step)
                losses.append(run.step([torch.from_numpy(X[r * b:(r + 1) * b]).cuda() for r in range(N)],
                                       [torch.from_numpy(Y[r * b:(r + 1) * b]).cuda() for r in range(N)])[0])
            curves[ex] = np.array(losses)
        finally:
            run.close()
    print({k: (float(v[0]), float(v[-1])) for k, v in curves.items()})
    for ex, c in curves.items():
        assert np.mean(c[-10:]) < 0.8 * np.mean(c[:5]), (ex, c[:5], c[-10:])
    for ex in ("TRUNC16", "SR16"):
        dev = np.max(np.abs(curves[ex] - curves["FP32"]) / curves["FP32"])
        assert dev < 1e-2, (ex, dev)
