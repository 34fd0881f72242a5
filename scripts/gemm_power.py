"""Sustained (power-capped) GEMM rate and SM clock per variant: each variant runs back to back
for --seconds with nvidia-smi sampling clocks and power, so variants are compared in the
steady state the step runs in (the 1 kW cap sets the clock; energy per FLOP decides speed).

    python scripts/gemm_power.py [--seconds 3] [--variants fwd,fwd_d2,fwd_cublas,wgrad,wgrad_cublas]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1603_04467_b200 as D  # noqa: E402
from bench import Clocks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=32768)
    ap.add_argument("--width", type=int, default=8192)
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--variants", default="fwd,fwd_d2,fwd_cublas,dgrad,dgrad_cublas,wgrad,wgrad_d2,wgrad_cublas")
    args = ap.parse_args()
    b, w = args.b, args.width
    dev = "cuda"
    A = torch.rand(b, w, device=dev).to(torch.bfloat16)
    W = (torch.rand(w, w, device=dev) - 0.5).to(torch.bfloat16)
    dZ = (torch.rand(b, w, device=dev) - 0.5).to(torch.bfloat16)
    bias = torch.zeros(w, device=dev)
    out_bf = torch.empty(b, w, dtype=torch.bfloat16, device=dev)
    out32 = torch.empty(w, w, dtype=torch.float32, device=dev)
    out_w16 = torch.empty(w, w, dtype=torch.bfloat16, device=dev)
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    flops = 2.0 * b * w * w

    tile = [0]

    def ours(M, N, K, Ad, am, Bd, bm, epi, out=None, o32=None, mask=None, bias_=None):
        t = tile[0]

        def f():
            D.check(D.dflow_gemm_bf16(M, N, K, vp(Ad), Ad.stride(0), am, vp(Bd), Bd.stride(0), bm, epi, vp(out),
                                      out.stride(0) if out is not None else 0, vp(o32),
                                      o32.stride(0) if o32 is not None else 0, vp(bias_), vp(mask),
                                      mask.stride(0) if mask is not None else 0, t, sp))
        return f

    def split_wgrad(P):
        kc = b // P
        fns = [ours(w, w, kc, A[p * kc:], 1, dZ[p * kc:], 1, D.EPI_F32, o32=out32) for p in range(P)]

        def f():
            for fn in fns:
                fn()
        return f

    table = {
        "fwd": lambda: ours(b, w, w, A, 0, W, 1, D.EPI_BIAS_RELU, out=out_bf, bias_=bias),
        "dgrad": lambda: ours(b, w, w, dZ, 0, W, 0, D.EPI_RELUGRAD, out=out_bf, mask=A),
        "wgrad": lambda: ours(w, w, b, A, 1, dZ, 1, D.EPI_F32, o32=out32),
        # the wgrad as P passes over K / P rows each (fp32 out rewritten per pass): does an
        # L2-sized K chunk cut DRAM traffic enough to pay for the extra passes?
        "wgrad_split4": lambda: split_wgrad(4),
        "wgrad_split2": lambda: split_wgrad(2),
        "fwd_cublas": lambda: (lambda: torch.matmul(A, W, out=out_bf)),
        "dgrad_cublas": lambda: (lambda: torch.matmul(dZ, W.t(), out=out_bf)),
        "wgrad_cublas": lambda: (lambda: torch.matmul(A.t(), dZ, out=out_w16)),
    }
    res = {"shape": [b, w]}
    for v in args.variants.split(","):
        # suffix _t<k>: force tile config k (3 = the 256 x 512 pair tile); _d<k>: debug bits
        vv, _, tsel = v.partition("_t")
        tile[0] = int(tsel) if tsel.isdigit() else 0
        if not tsel.isdigit():
            vv = v
        base, _, dbg = vv.partition("_d")
        if base.endswith("_cublas") or v.endswith("_cublas"):
            base, dbg = v, ""
        os.environ["DFLOW_GEMM_DEBUG"] = dbg or "0"
        fn = table[base]()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        clk = Clocks(torch.cuda.current_device())
        clk.start()
        time.sleep(0.2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        t_end = time.time() + args.seconds
        e0.record()
        while time.time() < t_end:
            for _ in range(20):
                fn()
            n += 20
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        c = clk.stop()
        ms = e0.elapsed_time(e1) / n
        res[v] = {"ms": ms, "tflops": flops / ms / 1e9, "sm_mhz": c.get("sm_mhz"), "power_w_max": c.get("power_w_max"),
                  "reasons": c.get("reasons"), "launches": n}
        print(v, json.dumps(res[v]), flush=True)
        time.sleep(1.0)
    os.environ["DFLOW_GEMM_DEBUG"] = "0"
    print(json.dumps(res))


if __name__ == "__main__":
    main()
