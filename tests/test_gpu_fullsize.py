"""Parity at BASELINE.json's full size, in the launch configuration bench.py times
(C3: 4 x 8192^2, B = 32768, one GPU): sampled outputs the oracle's definitions can
compute one by one.

* forward: rows of A_1 = relu(X W_1 + b_1), recomputed in f64 from the same bf16
  operands the GPU multiplies (reading A13), within bf16 output rounding;
* forward of every layer and the loss seed on sampled rows, by the oracle's own chain from
  X (its activations rounded to bf16 as the path stores them, reading A13), against the
  GPU's A_1 .. A_L and dZ_L rows — this ties the stored operands of the next check to the
  oracle;
* dW_L entries = sum over all 32768 rows of A_{L-1}[r, i] dZ_L[r, j], with
  dZ_L = 1[a > 0] (a - y) / (rows * cols) from the stored A_L and y and rounded to bf16
  as stored, recomputed in f64: the GPU's K = 32768 accumulation must agree to fp32
  accumulation accuracy;
* the train step's update equals W - lr * dW element by element (reading A9).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from dflow_harness import Run  # noqa: E402
from oracle import kernels as OK  # noqa: E402


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def test_c3_full_batch_sampled_parity():
    assert torch.cuda.is_available()
    w = synth.C3
    rows = w.batch
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w)
    run = Run(w.dims, "MSE", w.lr, rows=rows)
    try:
        run.assign(Ws, bs)
        Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
        g = np.random.default_rng(5)
        # ---- forward, layer 1, sampled rows
        A1 = run.forward(Xd, Yd, fetch=run.mlp.relus[0])
        rs = g.choice(rows, 8, replace=False)
        z = OK.matmul(_bf16(X[rs]), _bf16(Ws[0]), 0, 0, "f64") + bs[0].astype(np.float64)
        ref = np.maximum(z, 0)
        err = np.abs(A1[rs] - ref) / (np.abs(ref) + 1e-3)
        assert np.max(err) < 2 ** -7, float(np.max(err))  # bf16 rounding of the stored activation
        # ---- the oracle's own forward chain on sampled rows, every layer, and the loss seed
        A_gpu = [A1] + [run.forward(Xd, Yd, fetch=run.mlp.relus[l]) for l in range(1, w.layers)]
        rs = g.choice(rows, 16, replace=False)
        a = X[rs].astype(np.float64)
        for l in range(w.layers):
            z = OK.matmul(_bf16(a), _bf16(Ws[l]), 0, 0, "f64") + bs[l].astype(np.float64)
            a = np.maximum(z, 0)
            err = np.max(np.abs(A_gpu[l][rs] - a)) / np.max(np.abs(a))
            assert err < 2e-2, (l, float(err))  # bf16 storage of every activation, propagated
            if l + 1 < w.layers:
                a = _bf16(a).astype(np.float64)  # stored as bf16 for the next layer (A13)
        # loss seed where both sides take the same Relu branch (a pre-activation within
        # rounding of 0 may flip: reading A22 — counted, and required to be rare)
        agree = (a > 0) == (A_gpu[-1][rs] > 0)
        assert np.mean(~agree) < 1e-3, float(np.mean(~agree))
        seed_ref = np.where(a > 0, (a - Y[rs]) / (rows * w.dims[-1]), 0.0)
        seed_gpu = np.where(A_gpu[-1][rs] > 0, (A_gpu[-1][rs].astype(np.float64) - Y[rs]) / (rows * w.dims[-1]), 0.0)
        # |seed error| <= |A_L error| / (rows * cols), the A_L error bounded just above
        assert np.max(np.abs(seed_gpu - seed_ref)[agree]) <= 2e-2 * np.max(np.abs(a)) / (rows * w.dims[-1])
        A3, AL = A_gpu[2], A_gpu[3]                             # bf16 values as stored (A_{L-1}), fp32 A_L
        del A1, A_gpu
        # ---- dW_L sampled entries over the full batch (K = 32768)
        gW, gb, _ = run.gradients(Xd, Yd)
        d = (AL.astype(np.float32) - Y) / np.float32(rows * w.dims[-1])
        dZ = _bf16(np.where(AL > 0, d, 0.0).astype(np.float32)).astype(np.float64)
        ii = g.choice(w.dims[3], 16, replace=False)
        jj = g.choice(w.dims[4], 16, replace=False)
        ref = A3[:, ii].astype(np.float64).T @ dZ[:, jj]
        bound = np.abs(A3[:, ii]).astype(np.float64).T @ np.abs(dZ[:, jj])
        got = gW[3][np.ix_(ii, jj)]
        # fp32 accumulation over K = 32768 in 2048 tensor-core MMAs, each truncating to the
        # accumulator's ulp (reading A25): |err| <~ 2048 * 2^-24 * sum|terms| = 1.2e-4 * bound
        assert np.all(np.abs(got - ref) <= 2.5e-4 * bound + 1e-30), float(np.max(np.abs(got - ref) / bound))
        # db_L = column sums of the stored dZ_L
        refb = dZ[:, jj].sum(0)
        assert np.allclose(gb[3][jj], refb, rtol=1e-5, atol=1e-5 * np.abs(dZ[:, jj]).sum(0).max())
        del A3, AL
        # ---- the update: W_after == fl(W - fl(lr * dW)) for every element (N = 1: no codec)
        run.step(Xd, Yd)
        Wa, ba = run.read()
        for l in range(w.layers):
            exp = OK.apply_gradient_descent(Ws[l], w.lr, gW[l], "f32")
            assert np.array_equal(Wa[l], exp), l
            expb = OK.apply_gradient_descent(bs[l], w.lr, gb[l], "f32")
            assert np.array_equal(ba[l], expb), l
    finally:
        run.close()


def test_c5_full_batch_sampled_parity():
    """C5 (16 x 4096^2, B = 65536, the fp32-faithful 3xTF32 path) at full size on one GPU:
    sampled forward rows and dW_L entries against f64 recomputations from the exact fp32
    values the GPU stores (tf32 pairs join exactly, reading A14), gated at the north star's
    1e-4 relative to the |terms| bound; the update element by element (reading A9)."""
    assert torch.cuda.is_available()
    w = synth.C5
    rows = w.batch
    L = w.layers
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w)
    run = Run(w.dims, "MSE", w.lr, rows=rows, precision="3xtf32")
    try:
        run.assign(Ws, bs)
        Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
        g = np.random.default_rng(6)
        # ---- forward, layer 1, sampled rows: fp32-faithful, so f64 of the fp32 inputs
        A1 = run.forward(Xd, Yd, fetch=run.mlp.relus[0])
        rs = g.choice(rows, 8, replace=False)
        x64, w64 = X[rs].astype(np.float64), Ws[0].astype(np.float64)
        z = x64 @ w64 + bs[0].astype(np.float64)
        bound = np.abs(x64) @ np.abs(w64) + np.abs(bs[0]).astype(np.float64)
        err = np.abs(A1[rs] - np.maximum(z, 0)) / bound
        assert np.max(err) < 1e-5, float(np.max(err))
        del A1
        # ---- dW_L sampled entries over the full batch (K = 65536)
        Aprev = run.forward(Xd, Yd, fetch=run.mlp.relus[L - 2])   # fp32 A_{L-1} (hi + lo)
        AL = run.forward(Xd, Yd, fetch=run.mlp.relus[L - 1])      # fp32 A_L
        gW, gb, _ = run.gradients(Xd, Yd)
        d = (AL - Y) / np.float32(rows * w.dims[-1])               # (a - y) / 2^28: exact scaling
        dZ = np.where(AL > 0, d, np.float32(0)).astype(np.float64)
        ii = g.choice(w.dims[L - 1], 16, replace=False)
        jj = g.choice(w.dims[L], 16, replace=False)
        ref = Aprev[:, ii].astype(np.float64).T @ dZ[:, jj]
        bound = np.abs(Aprev[:, ii]).astype(np.float64).T @ np.abs(dZ[:, jj])
        got = gW[L - 1][np.ix_(ii, jj)]
        rel = np.abs(got - ref) / (bound + 1e-300)
        assert np.max(rel) < 1e-4, float(np.max(rel))
        refb = dZ[:, jj].sum(0)
        assert np.allclose(gb[L - 1][jj], refb, rtol=1e-5, atol=1e-5 * np.abs(dZ[:, jj]).sum(0).max())
        del Aprev, AL
        # ---- the update: W_after == fl(W - fl(lr * dW)) for every element (N = 1: no codec)
        run.step(Xd, Yd)
        Wa, ba = run.read()
        for l in range(L):
            exp = OK.apply_gradient_descent(Ws[l], w.lr, gW[l], "f32")
            assert np.array_equal(Wa[l], exp), l
            expb = OK.apply_gradient_descent(bs[l], w.lr, gb[l], "f32")
            assert np.array_equal(ba[l], expb), l
    finally:
        run.close()
