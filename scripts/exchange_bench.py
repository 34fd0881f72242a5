"""Exchange microbenchmark: time of the gradient combine alone
(a6-a8 through dflow_exchange) per bucket size, for TRUNC16 (alltoall u16 + owner
fold + allgather u16), FP32 (same schedule, fp32 payloads) and ncclAllReduce fp32.

    python -m torch.distributed.run --nproc-per-node N scripts/exchange_bench.py
"""
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1603_04467_b200 as D  # noqa: E402


def main():
    rank, world, local = bench.env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rows = []
    for mode in ("TRUNC16", "FP32", "FP32_NCCL"):
        # an NCCL unique id bootstraps exactly one communicator: fresh id per session
        nid = bench.broadcast_bytes(D.nccl_unique_id() if rank == 0 else None, dist, "cuda")
        mlp = D.mlp_graph((8, 8), "MSE", 0.5)
        s = D.session_create(mlp, D.make_options(world=world, rank=rank, device=local, exchange=mode,
                                                 max_local_rows=8), nid)
        for lg in range(18, 27, 2):
            n = 1 << lg
            g = torch.randn(n, device="cuda")
            o = torch.empty_like(g)
            for _ in range(3):
                D.check(D.dflow_exchange(s, C.c_void_p(g.data_ptr()), C.c_void_p(o.data_ptr()), n, sp))
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record()
            for _ in range(reps):
                D.check(D.dflow_exchange(s, C.c_void_p(g.data_ptr()), C.c_void_p(o.data_ptr()), n, sp))
            e1.record()
            torch.cuda.synchronize()
            ms = bench.max_over_ranks(e0.elapsed_time(e1) / reps, dist, "cuda")
            pay = 2 if mode == "TRUNC16" else 4
            wire = 2 * (world - 1) / world * n * pay  # alltoall + allgather (or ring allreduce) per GPU
            rows.append({"mode": mode, "n_params": n, "fp32_MiB": n * 4 / 2 ** 20, "ms": ms,
                         "algbw_GBps": n * 4 / ms / 1e6, "wire_bytes_per_gpu": wire,
                         "busbw_GBps": wire / ms / 1e6})
        D.dflow_session_destroy(s)
        D.dflow_graph_destroy(mlp.graph)
    if rank == 0:
        print(json.dumps({"world": world, "rows": rows}, indent=1))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
