"""Per-launch time of the C3 GEMM variants at the N = 8 local batch (b = 4096) through
dflow_gemm_bf16 (EPI_F32 and the fused epilogues where the standalone entry supports them):
forward A[b,in] K-major x W[in,out] MN-major; dgrad dZ[b,out] K-major x W as K-major;
wgrad A[b,in] MN-major x dZ[b,out] MN-major.  CUDA events over 20 back-to-back launches."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04467_b200 as D  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
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
    b, w = int(sys.argv[1]) if len(sys.argv) > 1 else 4096, 8192
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    A = (torch.rand(b, w, device="cuda") - 0.5).to(torch.bfloat16)
    Wt = (torch.rand(w, w, device="cuda") - 0.5).to(torch.bfloat16)
    dZ = (torch.rand(b, w, device="cuda") - 0.5).to(torch.bfloat16)
    o_bw = torch.empty(b, w, device="cuda", dtype=torch.float32)
    o_ww = torch.empty(w, w, device="cuda", dtype=torch.float32)
    p = lambda t: C.c_void_p(t.data_ptr())
    cases = {
        "fwd  M=b N=w K=w (A K-major, B MN-major)": lambda: D.dflow_gemm_bf16(
            b, w, w, p(A), w, 0, p(Wt), w, 1, D.EPI_F32, None, 0, p(o_bw), w, None, None, 0, 0, sp),
        "dgrad M=b N=w K=w (both K-major)": lambda: D.dflow_gemm_bf16(
            b, w, w, p(dZ), w, 0, p(Wt), w, 0, D.EPI_F32, None, 0, p(o_bw), w, None, None, 0, 0, sp),
        "wgrad M=w N=w K=b (both MN-major)": lambda: D.dflow_gemm_bf16(
            w, w, b, p(A), w, 1, p(dZ), w, 1, D.EPI_F32, None, 0, p(o_ww), w, None, None, 0, 0, sp),
    }
    flops = 2.0 * b * w * w
    for name, fn in cases.items():
        ms = timed(lambda: D.check(fn()))
        print(f"{name}: {ms * 1000:.1f} us  {flops / ms / 1e9:.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
