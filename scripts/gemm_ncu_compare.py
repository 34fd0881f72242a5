"""ours vs cuBLAS on the C3 forward and weight-gradient shapes, one launch each after warm-up,
for an `ncu --set full` side-by-side (power-relevant counters: instructions, L2 and DRAM
traffic, shared-memory wavefronts at the same work)."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1603_04467_b200 as D  # noqa: E402

b, w = 32768, 8192
A = torch.rand(b, w, device="cuda").to(torch.bfloat16)
W = (torch.rand(w, w, device="cuda") - 0.5).to(torch.bfloat16)
dZ = (torch.rand(b, w, device="cuda") - 0.5).to(torch.bfloat16)
bias = torch.zeros(w, device="cuda")
out_bf = torch.empty(b, w, dtype=torch.bfloat16, device="cuda")
out32 = torch.empty(w, w, dtype=torch.float32, device="cuda")
out_w16 = torch.empty(w, w, dtype=torch.bfloat16, device="cuda")
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None


def ours_fwd():
    D.check(D.dflow_gemm_bf16(b, w, w, vp(A), w, 0, vp(W), w, 1, D.EPI_BIAS_RELU, vp(out_bf), w, None, 0, vp(bias),
                              None, 0, 0, sp))


def ours_wgrad():
    D.check(D.dflow_gemm_bf16(w, w, b, vp(A), w, 1, vp(dZ), w, 1, D.EPI_F32, None, 0, vp(out32), w, None, None, 0, 0,
                              sp))


fns = [ours_fwd, lambda: torch.matmul(A, W, out=out_bf), ours_wgrad, lambda: torch.matmul(A.t(), dZ, out=out_w16)]
for f in fns:  # warm-up (outside the capture: ncu --launch-skip)
    f()
torch.cuda.synchronize()
for f in fns:
    f()
torch.cuda.synchronize()
print("ok")
