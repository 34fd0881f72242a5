"""Latency of small GEMMs (the C2 shapes) through dflow_gemm_bf16 vs torch.matmul (cuBLAS):
per-launch time from CUDA events over many back-to-back launches, and a single launch
bracketed by synchronisation (the latency seen when kernels do not overlap)."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04467_b200 as D  # noqa: E402


def per_launch(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    back = e0.elapsed_time(e1) / reps * 1000
    single = []
    for _ in range(20):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        single.append(e0.elapsed_time(e1) * 1000)
    return back, sorted(single)[len(single) // 2]


def main():
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    res = {}
    for (M, N, K) in [(256, 1024, 64), (256, 1024, 784), (256, 1024, 1024), (256, 16, 1024), (784, 1024, 256),
                      (1024, 1024, 256), (2048, 2048, 2048)]:
        A = torch.rand(M, K, device="cuda").to(torch.bfloat16)
        B = torch.rand(K, N, device="cuda").to(torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)

        def ours():
            D.check(D.dflow_gemm_bf16(M, N, K, C.c_void_p(A.data_ptr()), K, 0, C.c_void_p(B.data_ptr()), N, 1,
                                      D.EPI_F32, None, 0, C.c_void_p(out.data_ptr()), N, None, None, 0, 0, sp))
        o2 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ob, os_ = per_launch(ours)
        cb, cs = per_launch(lambda: torch.matmul(A, B, out=o2))
        res[f"{M}x{N}x{K}"] = {"ours_us": ob, "ours_single_us": os_, "cublas_us": cb, "cublas_single_us": cs}
        print(f"{M}x{N}x{K}: ours {ob:.1f} us (single {os_:.1f})  cublas {cb:.1f} us (single {cs:.1f})", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
