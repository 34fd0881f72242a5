"""Standalone timing of the C3 GEMM shapes (forward / dgrad / wgrad) through
dflow_gemm_bf16, beside torch.matmul (cuBLAS) on the same shapes, for a few
tile-raster group sizes and L2 prefetch distances (DFLOW_GEMM_GROUP,
DFLOW_GEMM_PREFETCH are read at plan time).

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
    ap.add_argument("--prefetch", default="8", help="L2 prefetch distances (DFLOW_GEMM_PREFETCH)")
    ap.add_argument("--debug", default="0", help="profiling variants (DFLOW_GEMM_DEBUG bit flags)")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--ab", type=int, default=0, help="rounds of interleaved ours / cuBLAS timing per shape")
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

    for g, pf, dbg in [(int(x), int(y), int(z)) for x in args.groups.split(",") for y in args.prefetch.split(",")
                       for z in args.debug.split(",")]:
        os.environ["DFLOW_GEMM_GROUP"] = str(g)
        os.environ["DFLOW_GEMM_PREFETCH"] = str(pf)
        os.environ["DFLOW_GEMM_DEBUG"] = str(dbg)
        fwd = ours(b, w, w, A, 0, W, 1, D.EPI_BIAS_RELU, out=out_bf, bias_=bias)
        dgr = ours(b, w, w, dZ, 0, W, 0, D.EPI_RELUGRAD, out=out_bf, mask=A)
        wgr = ours(w, w, b, A, 1, dZ, 1, D.EPI_F32, o32=out32)
        for name, fn in (("fwd", fwd), ("dgrad", dgr), ("wgrad", wgr)):
            ms = time_fn(fn, args.reps)
            tag = f"g{g}_p{pf}" + (f"_d{dbg}" if dbg else "")
            res[f"ours_{tag}_{name}_ms"] = ms
            res[f"ours_{tag}_{name}_tflops"] = flops / ms / 1e9
    os.environ["DFLOW_GEMM_DEBUG"] = "0"
    if args.ab:
        # same shapes back to back, alternating, so both see the same power / thermal state
        os.environ["DFLOW_GEMM_PREFETCH"] = "0"
        pairs = {"fwd": (ours(b, w, w, A, 0, W, 1, D.EPI_BIAS_RELU, out=out_bf, bias_=bias),
                         lambda: torch.matmul(A, W, out=out_bf)),
                 "dgrad": (ours(b, w, w, dZ, 0, W, 0, D.EPI_RELUGRAD, out=out_bf, mask=A),
                           lambda: torch.matmul(dZ, W.t(), out=out_bf)),
                 "wgrad": (ours(w, w, b, A, 1, dZ, 1, D.EPI_F32, o32=out32), lambda: torch.matmul(A.t(), dZ))}
        for name, (fo, fc) in pairs.items():
            to, tc = [], []
            for _ in range(args.ab):
                to.append(time_fn(fo, args.reps))
                tc.append(time_fn(fc, args.reps))
            res[f"ab_{name}_ours_ms"] = sorted(to)[len(to) // 2]
            res[f"ab_{name}_cublas_ms"] = sorted(tc)[len(tc) // 2]
            res[f"ab_{name}_ratio"] = res[f"ab_{name}_cublas_ms"] / res[f"ab_{name}_ours_ms"]
    if args.no_cublas:
        print(json.dumps(res, indent=1))
        return
    res["cublas_fwd_ms"] = time_fn(lambda: torch.matmul(A, W, out=out_bf), args.reps)
    res["cublas_dgrad_ms"] = time_fn(lambda: torch.matmul(dZ, W.t(), out=out_bf), args.reps)
    res["cublas_wgrad_ms"] = time_fn(lambda: torch.matmul(A.t(), dZ), args.reps)
    for k in ("fwd", "dgrad", "wgrad"):
        res[f"cublas_{k}_tflops"] = flops / res[f"cublas_{k}_ms"] / 1e9
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
