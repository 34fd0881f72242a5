"""Diagnose the 3xTF32 GEMM on tiny shapes: per layout, error of the result vs
candidate products (A B, with lo parts zero / real)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04467_b200 as D  # noqa: E402


def vp(t):
    return C.c_void_p(t.data_ptr())


def run(M, N, K, a_mn, b_mn, tile, zero_lo, seed=0):
    g = np.random.default_rng(seed)
    A = g.integers(-3, 4, (M, K)).astype(np.float32)
    B = g.integers(-3, 4, (K, N)).astype(np.float32)
    a_store = np.ascontiguousarray(A.T if a_mn else A)
    b_store = np.ascontiguousarray(B if b_mn else B.T)
    ah = torch.from_numpy(a_store).cuda()
    bh = torch.from_numpy(b_store).cuda()
    al = torch.zeros_like(ah) if zero_lo else ah.clone() * 0 + 2.0 ** -12
    bl = torch.zeros_like(bh) if zero_lo else bh.clone() * 0 + 2.0 ** -12
    out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    D.check(D.dflow_gemm_3xtf32(M, N, K, vp(ah), vp(al), ah.shape[1], a_mn, vp(bh), vp(bl), bh.shape[1], b_mn,
                                vp(out), N, tile, sp))
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    ref = A.astype(np.float64) @ B.astype(np.float64)
    if not zero_lo:
        e = 2.0 ** -12
        ref = ref + e * (A.sum(1, keepdims=True) + B.sum(0, keepdims=True))
    err = np.abs(o - ref).max()
    print(f"M{M} N{N} K{K} a_mn{a_mn} b_mn{b_mn} tile{tile} zero_lo{zero_lo}: max err {err:.4g}  "
          f"o[0,:4]={o[0, :4]} ref[0,:4]={ref[0, :4]}")
    return err


if __name__ == "__main__":
    for (a_mn, b_mn) in [(0, 0), (0, 1), (1, 1)]:
        for tile in (1, 2):
            for K in (8, 32, 64):
                run(256 if tile == 2 else 128, 256 if tile == 2 else 128, K, a_mn, b_mn, tile, True)
            run(128, 128, 64, a_mn, b_mn, tile, False)
