"""Standalone timing of the C3 GEMM shapes (forward / dgrad / wgrad) through
dflow_gemm_bf16, beside torch.matmul (cuBLAS) on the same shapes, for a few
tile-raster group sizes (DFLOW_GEMM_GROUP is read at plan time).

    python scripts/gemm_sweep.py [--b 32768] [--width 8192] [--groups 4,8,16,32]
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04467_b200 as D  # noqa: E402


def time_fn(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=32768)
    ap.add_argument("--width", type=int, default=8192)
    ap.add_argument("--groups", default="8")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    b, w = args.b, args.width
    dev = "cuda"
    A = torch.rand(b, w, device=dev).to(torch.bfloat16)       # activations [b, in]
    W = (torch.rand(w, w, device=dev) - 0.5).to(torch.bfloat16)  # [in, out]
    dZ = (torch.rand(b, w, device=dev) - 0.5).to(torch.bfloat16)
    bias = torch.zeros(w, device=dev)
    out_bf = torch.empty(b, w, dtype=torch.bfloat16, device=dev)
    out32 = torch.empty(w, w, dtype=torch.float32, device=dev)
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    flops = 2.0 * b * w * w
    res = {"shape": [b, w], "flops_per_gemm": flops}

    def ours(M, N, K, Ad, am, Bd, bm, epi, out=None, o32=None, mask=None, bias_=None):
        def f():
            D.check(D.dflow_gemm_bf16(M, N, K, vp(Ad), Ad.stride(0), am, vp(Bd), Bd.stride(0), bm, epi, vp(out),
                                      out.stride(0) if out is not None else 0, vp(o32),
                                      o32.stride(0) if o32 is not None else 0, vp(bias_), vp(mask),
                                      mask.stride(0) if mask is not None else 0, 0, sp))
        return f

    for g in [int(x) for x in args.groups.split(",")]:
        os.environ["DFLOW_GEMM_GROUP"] = str(g)
        fwd = ours(b, w, w, A, 0, W, 1, D.EPI_BIAS_RELU, out=out_bf, bias_=bias)
        dgr = ours(b, w, w, dZ, 0, W, 0, D.EPI_RELUGRAD, out=out_bf, mask=A)
        wgr = ours(w, w, b, A, 1, dZ, 1, D.EPI_F32, o32=out32)
        for name, fn in (("fwd", fwd), ("dgrad", dgr), ("wgrad", wgr)):
            ms = time_fn(fn, args.reps)
            res[f"ours_g{g}_{name}_ms"] = ms
            res[f"ours_g{g}_{name}_tflops"] = flops / ms / 1e9
    res["cublas_fwd_ms"] = time_fn(lambda: torch.matmul(A, W, out=out_bf), args.reps)
    res["cublas_dgrad_ms"] = time_fn(lambda: torch.matmul(dZ, W.t(), out=out_bf), args.reps)
    res["cublas_wgrad_ms"] = time_fn(lambda: torch.matmul(A.t(), dZ), args.reps)
    for k in ("fwd", "dgrad", "wgrad"):
        res[f"cublas_{k}_tflops"] = flops / res[f"cublas_{k}_ms"] / 1e9
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
