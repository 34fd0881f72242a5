"""GPU unit parity: codec (P2 exhaustive), tcgen05 GEMM layouts/epilogues vs the oracle.

Run with -m gpu on a B200.  Everything goes through the C ABI (libdflow.so).
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1603_04467_b200 as D  # noqa: E402
from oracle import kernels as OK  # noqa: E402
from oracle.codec import expand16, sr16, sr_key, sr_random, truncate16  # noqa: E402
from synth import random_f32_bits  # noqa: E402
from synth import rng  # noqa: E402
from dflow_harness import stream_ptr  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    torch.cuda.init()


def _vp(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def test_p2_truncate16_exhaustive_all_2_32_patterns():
    # every fp32 bit pattern -> its high half-word, bit-exact vs the oracle.
    chunk = 1 << 28
    dst = torch.empty(chunk, dtype=torch.int16, device="cuda")
    for c in range(1 << 32 >> 28):
        bits = np.arange(c * chunk, (c + 1) * chunk, dtype=np.uint64).astype(np.uint32)
        src = torch.from_numpy(bits.view(np.int32)).cuda()
        D.check(D.dflow_truncate16(_vp(src), _vp(dst), chunk, stream_ptr()))
        got = dst.cpu().numpy().view(np.uint16)
        exp = truncate16(bits.view(np.float32))
        assert np.array_equal(got, exp), f"chunk {c}"


def test_p2_expand16_exhaustive():
    q = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    src = torch.from_numpy(q.view(np.int16)).cuda()
    dst = torch.empty(1 << 16, dtype=torch.float32, device="cuda")
    D.check(D.dflow_expand16(_vp(src), _vp(dst), 1 << 16, stream_ptr()))
    assert np.array_equal(dst.cpu().numpy().view(np.uint32), expand16(q).view(np.uint32))


@pytest.mark.parametrize("n", [0, 1, 7, 9, 1000, 12345])
def test_codec_ragged_lengths(n):
    x = (rng(5).standard_normal(max(n, 1)).astype(np.float32))[:n]
    src = torch.from_numpy(x).cuda() if n else torch.empty(0, device="cuda")
    q = torch.empty(max(n, 1), dtype=torch.int16, device="cuda")
    D.check(D.dflow_truncate16(_vp(src), _vp(q), n, stream_ptr()))
    if n:
        assert np.array_equal(q.cpu().numpy()[:n].view(np.uint16), truncate16(x))


@pytest.mark.parametrize("n,idx_base", [(1, 0), (9, 0), (4099, 0), (1 << 20, 0), (1000, 123456789)])
def test_sr16_kernel_bit_exact_vs_oracle(n, idx_base):
    # f2: the SR16 coding (readings A26-A27) on random bit patterns (incl. specials): GPU
    # codes == the oracle's (bits + r) >> 16 with its own generator's draws
    x = random_f32_bits(n)
    key = sr_key(77, 3, 2, 0, 1)
    src = torch.from_numpy(x.view(np.int32)).cuda()
    q = torch.empty(n, dtype=torch.int16, device="cuda")
    D.check(D.dflow_round16(_vp(src), _vp(q), n, key, 1, idx_base, stream_ptr()))
    exp = sr16(x, sr_random(key, np.arange(idx_base, idx_base + n)))
    assert np.array_equal(q.cpu().numpy().view(np.uint16), exp)
    # stochastic = 0 is plain truncation
    D.check(D.dflow_round16(_vp(src), _vp(q), n, key, 0, idx_base, stream_ptr()))
    assert np.array_equal(q.cpu().numpy().view(np.uint16), truncate16(x))


# ---------------------------------------------------------------- GEMM
def _bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def _layout(M, N, K, a_mn, b_mn, g, ints):
    """Logical A [M,K], B [K,N] (bf16-exact values) and their device storage."""
    if ints:
        A = g.integers(-4, 5, (M, K)).astype(np.float32)
        B = g.integers(-4, 5, (K, N)).astype(np.float32)
    else:
        A = _bf16_round(g.uniform(-1, 1, (M, K)))
        B = _bf16_round(g.uniform(-1, 1, (K, N)))
    a_store = A.T if a_mn else A          # a_mn: stored [K, M]
    b_store = B if b_mn else B.T          # b_mn: stored [K, N]; else [N, K]
    pad = lambda x: np.pad(x, ((0, 0), (0, (-x.shape[1]) % 8)))
    a_dev = torch.from_numpy(np.ascontiguousarray(pad(a_store))).to(torch.bfloat16).cuda()
    b_dev = torch.from_numpy(np.ascontiguousarray(pad(b_store))).to(torch.bfloat16).cuda()
    return A, B, a_dev, b_dev


def _gemm(M, N, K, a_dev, a_mn, b_dev, b_mn, epi, tile, out=None, out32=None, bias=None, mask=None):
    D.check(D.dflow_gemm_bf16(M, N, K, _vp(a_dev), a_dev.stride(0), a_mn, _vp(b_dev), b_dev.stride(0), b_mn, epi,
                              _vp(out), out.stride(0) if out is not None else 0, _vp(out32),
                              out32.stride(0) if out32 is not None else 0, _vp(bias), _vp(mask),
                              mask.stride(0) if mask is not None else 0, tile, stream_ptr()))
    torch.cuda.synchronize()


SHAPES = [(128, 128, 64), (100, 100, 784), (257, 300, 200), (256, 1024, 784), (512, 512, 1024),
          (1000, 520, 130), (33, 10, 1024), (784, 100, 100)]
LAYOUTS = [(0, 1, D.EPI_F32), (0, 0, D.EPI_F32), (1, 1, D.EPI_F32)]


@pytest.mark.parametrize("tile", [1, 2, 3])
@pytest.mark.parametrize("a_mn,b_mn,epi", LAYOUTS)
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_layouts_exact_integers(M, N, K, a_mn, b_mn, epi, tile):
    # Small integers: every fp32 partial sum is exact, so any misplaced tile,
    # transposed operand or wrong descriptor shows as a bit difference.
    g = rng(1000 + M + N + K)
    A, B, a_dev, b_dev = _layout(M, N, K, a_mn, b_mn, g, ints=True)
    out32 = torch.full((M, N + (-N) % 4), float("nan"), dtype=torch.float32, device="cuda")
    _gemm(M, N, K, a_dev, a_mn, b_dev, b_mn, epi, tile, out32=out32)
    ref = OK.matmul(A, B, 0, 0, "f64")
    assert np.array_equal(out32.cpu().numpy()[:, :N], ref.astype(np.float32))


@pytest.mark.parametrize("tile", [1, 2, 3])
@pytest.mark.parametrize("M,N,K", [(300, 260, 520), (1024, 1024, 4096)])
def test_gemm_random_floats_tolerance(M, N, K, tile):
    g = rng(7)
    for a_mn, b_mn, _ in LAYOUTS:
        A, B, a_dev, b_dev = _layout(M, N, K, a_mn, b_mn, g, ints=False)
        out32 = torch.empty((M, N), dtype=torch.float32, device="cuda")
        _gemm(M, N, K, a_dev, a_mn, b_dev, b_mn, D.EPI_F32, tile, out32=out32)
        ref = OK.matmul(A, B, 0, 0, "f64")
        bound = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)
        err = np.abs(out32.cpu().numpy() - ref)
        assert np.all(err <= 2e-6 * bound + 1e-30), (a_mn, b_mn, float(np.max(err / (bound + 1e-30))))


@pytest.mark.parametrize("tile", [1, 2, 3])
@pytest.mark.parametrize("M,N,K", [(300, 260, 520), (100, 100, 784), (512, 512, 512)])
def test_gemm_epilogue_trunc16(M, N, K, tile):
    g = rng(8)
    A, B, a_dev, b_dev = _layout(M, N, K, 1, 1, g, ints=True)
    out = torch.zeros((M, N + (-N) % 8), dtype=torch.int16, device="cuda")
    _gemm(M, N, K, a_dev, 1, b_dev, 1, D.EPI_TRUNC16, tile, out=out)
    ref = OK.matmul(A, B, 0, 0, "f64").astype(np.float32)
    assert np.array_equal(out.cpu().numpy()[:, :N].view(np.uint16), truncate16(ref))


@pytest.mark.parametrize("tile", [1, 2, 3])
@pytest.mark.parametrize("M,N,K", [(300, 260, 520), (100, 100, 784), (512, 1024, 256)])
def test_gemm_epilogue_bias_relu(M, N, K, tile):
    g = rng(9)
    A, B, a_dev, b_dev = _layout(M, N, K, 0, 1, g, ints=True)
    bias = g.integers(-8, 9, N).astype(np.float32)
    ldo = N + (-N) % 8
    out = torch.zeros((M, ldo), dtype=torch.bfloat16, device="cuda")
    out32 = torch.zeros((M, N + (-N) % 4), dtype=torch.float32, device="cuda")
    _gemm(M, N, K, a_dev, 0, b_dev, 1, D.EPI_BIAS_RELU, tile, out=out, out32=out32,
          bias=torch.from_numpy(bias).cuda())
    z = OK.add(OK.matmul(A, B, 0, 0, "f64"), bias, "f32")
    a = OK.relu(z, "f32")
    assert np.array_equal(out32.cpu().numpy()[:, :N], a)
    assert np.array_equal(out.float().cpu().numpy()[:, :N], _bf16_round(a))


@pytest.mark.parametrize("tile", [1, 2, 3])
@pytest.mark.parametrize("M,N,K", [(300, 260, 520), (256, 784, 1024), (512, 512, 512)])
def test_gemm_epilogue_relugrad(M, N, K, tile):
    g = rng(10)
    A, B, a_dev, b_dev = _layout(M, N, K, 0, 0, g, ints=True)
    mask_vals = _bf16_round(g.uniform(-1, 1, (M, N)) * (g.random((M, N)) < 0.7))
    ldm = N + (-N) % 8
    mask = torch.from_numpy(np.pad(mask_vals, ((0, 0), (0, ldm - N)))).to(torch.bfloat16).cuda()
    out = torch.zeros((M, ldm), dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, K, a_dev, 0, b_dev, 0, D.EPI_RELUGRAD, tile, out=out, mask=mask)
    ref = OK.relu_grad(OK.matmul(A, B, 0, 0, "f32"), mask_vals, "f32")
    assert np.array_equal(out.float().cpu().numpy()[:, :N], _bf16_round(ref))
