"""GPU parity of the fp32-faithful 3xTF32 path (NK4-NK6) vs the oracle.

north_star: the fp32-faithful path agrees within max relative error 1e-4 on
weights after one step (reading A15 (i)); gradients are gated mask-locked at the
same tolerance (A15 (ii), A22).  P12: bitwise in the exact-arithmetic regime.
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1603_04467_b200 as D  # noqa: E402
from dflow_harness import Run, normwise, stream_ptr  # noqa: E402
from oracle import kernels as OK  # noqa: E402
from oracle.mlp import build_mlp, train_step  # noqa: E402
from synth import C1, C1_BIAS, C2, C5, batch, exact_regime, init_params, rng, with_batch  # noqa: E402

TF32_TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"


def _vp(t):
    return C.c_void_p(t.data_ptr())


def _tf32_rna_reference(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest, ties away from zero, to 10 mantissa bits: add half of
    2^13 to the magnitude bits and clear the low 13 (finite inputs)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return r.view(np.float32)


def test_split_tf32_bit_exact():
    g = rng(41)
    x = (g.standard_normal(100003) * np.exp(g.uniform(-20, 20, 100003))).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    hi, lo = torch.empty_like(xd), torch.empty_like(xd)
    D.check(D.dflow_split_tf32(_vp(xd), _vp(hi), _vp(lo), x.size, stream_ptr()))
    torch.cuda.synchronize()
    h, l = hi.cpu().numpy(), lo.cpu().numpy()
    assert np.array_equal(h.view(np.uint32), _tf32_rna_reference(x).view(np.uint32))
    assert np.array_equal((h + l).view(np.uint32), x.view(np.uint32))  # hi + lo == x exactly


def _split_dev(a):
    t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    hi, lo = torch.empty_like(t), torch.empty_like(t)
    D.check(D.dflow_split_tf32(_vp(t), _vp(hi), _vp(lo), t.numel(), stream_ptr()))
    return hi, lo


@pytest.mark.parametrize("tile", [1, 2])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (0, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (100, 100, 784), (257, 300, 200), (512, 512, 1024)])
def test_3xtf32_gemm_layouts(M, N, K, a_mn, b_mn, tile):
    # fp32 operands with full 24-bit mantissas: a 1xTF32 GEMM errs ~2^-11 relative,
    # 3xTF32 ~2^-21; the gate (4e-6 of |A||B|) only passes with all three products
    g = rng(2000 + M + N + K + 7 * a_mn + 3 * b_mn)
    A = g.uniform(-1, 1, (M, K)).astype(np.float32)
    B = g.uniform(-1, 1, (K, N)).astype(np.float32)
    a_store = np.ascontiguousarray(A.T if a_mn else A)
    b_store = np.ascontiguousarray(B if b_mn else B.T)
    pad = lambda x: np.ascontiguousarray(np.pad(x, ((0, 0), (0, (-x.shape[1]) % 8))))
    ahi, alo = _split_dev(pad(a_store))
    bhi, blo = _split_dev(pad(b_store))
    out = torch.empty((M, N + (-N) % 4), dtype=torch.float32, device="cuda")
    D.check(D.dflow_gemm_3xtf32(M, N, K, _vp(ahi), _vp(alo), ahi.shape[1], a_mn, _vp(bhi), _vp(blo), bhi.shape[1],
                                b_mn, _vp(out), out.stride(0), tile, stream_ptr()))
    torch.cuda.synchronize()
    ref = OK.matmul(A, B, 0, 0, "f64")
    bound = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)
    err = np.abs(out.cpu().numpy()[:, :N] - ref)
    assert np.all(err <= 4e-6 * bound), float(np.max(err / bound))


def _one_step(w, rows=None):
    rows = rows or w.batch
    Ws, bs = init_params(w)
    X, Y = batch(w, rows=rows)
    run = Run(w.dims, w.loss, w.lr, rows=rows, with_dx=(w.layers == 1), precision="3xtf32")
    try:
        run.assign(Ws, bs)
        Xd = torch.from_numpy(X).cuda()
        Yd = None if Y is None else torch.from_numpy(Y).cuda()
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
def test_config1_fp32_faithful(w):
    errs, flips = _one_step(w)
    print(errs, flips)
    assert max(errs.values()) < TF32_TOL, errs


def test_config2_fp32_faithful():
    errs, flips = _one_step(C2)
    print(errs, flips)
    assert max(errs.values()) < TF32_TOL, errs


def test_config5_deep_reduced():
    # C5 widths and depth (16 x 4096^2) at a reduced batch the oracle finishes quickly
    errs, flips = _one_step(with_batch(C5, 256))
    print({k: v for k, v in errs.items() if v > 1e-6}, flips)
    assert max(errs.values()) < TF32_TOL, errs


def test_p12_exact_regime_bitwise_3xtf32():
    X, Y, Ws, bs, lr = exact_regime()
    dims = (784, 1024, 1024, 16)
    run = Run(dims, "MSE", lr, rows=X.shape[0], precision="3xtf32")
    try:
        run.assign(Ws, bs)
        Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
        gW, gb, _ = run.gradients(Xd, Yd)
        mg = build_mlp(dims, "MSE", lr)
        ref = train_step(mg, Ws, bs, X, Y, 1, "TRUNC16")
        for l in range(3):
            assert np.array_equal(gW[l], ref["ghat"][mg.weights[l]]), f"dW{l + 1}"
            assert np.array_equal(gb[l], ref["ghat"][mg.biases[l]]), f"db{l + 1}"
        run.step(Xd, Yd)
        Wg, bg = run.read()
        for l in range(3):
            assert np.array_equal(Wg[l], ref["W"][l]), f"W{l + 1}"
            assert np.array_equal(bg[l], ref["b"][l]), f"b{l + 1}"
    finally:
        run.close()
