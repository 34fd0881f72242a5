"""One C3-width train step of a simulated world per exchange schedule (run under ncu): the
N > 1 HBM kernels — owner fold (+ owner-apply), db pass, u16 / fp32 owner reduce, u16 apply,
asynchronous pull / push — on one GPU.  In the simulated world the peers' buffers live on the
same device, so every "NVLink" store is an HBM store here: the captures measure each kernel's
DRAM efficiency, not the link.

    python scripts/profile_exchange_kernels.py [world] [rows_per_rank]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from dflow_harness import SimRun  # noqa: E402
import synth  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
w = synth.Workload("C3w2", (8192, 8192, 8192), rows * world, "MSE", 2.0 ** -2, "he")
Ws, bs = synth.init_params(w)
X, Y = synth.batch(w)
Xs = [torch.from_numpy(X[r * rows:(r + 1) * rows]).cuda() for r in range(world)]
Ys = [torch.from_numpy(Y[r * rows:(r + 1) * rows]).cuda() for r in range(world)]
for name, kw in (("p2p_owner_apply", dict(exchange="TRUNC16", p2p=1)),
                 ("nccl_schedule_trunc16", dict(exchange="TRUNC16", p2p=0)),
                 ("nccl_schedule_fp32", dict(exchange="FP32", p2p=0)),
                 ("async_trunc16", dict(exchange="TRUNC16", async_dp=1))):
    run = SimRun(w.dims, "MSE", w.lr, rows=rows, world=world, **kw)
    run.assign(Ws, bs)
    for _ in range(2):
        run.step(Xs, Ys)
    run.close()
    print(name, "ok", flush=True)
