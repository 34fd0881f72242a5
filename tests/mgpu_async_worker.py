"""One rank of the asynchronous data-parallel checks (f3), launched by tests/test_gpu_async.py
via torchrun.  PAPER.md:948-955; readings A29-A31.

  A1 serialised replicas, bit-exact: rank 0 pulls, computes g_0 (fetched, same kernels) and
     pushes; then rank 1 pulls (== the oracle's W after rank 0's push, bit for bit), computes
     g_1 and pushes; ...; the shared W after all pushes == oracle.async_dp.push applied in
     rank order to the GPU's own fp32 gradients, bit for bit.
  A2 concurrent replicas from one point: every rank pulls W0 (barrier), computes g_r, and all
     push at once: every element == the sequential result in SOME order — exactly one of the
     two orders at N = 2; within the reassociation bound at N > 2.
  A3 free-running: every rank trains 30 steps on its own batches with no barrier; the loss
     falls and the shared parameters stay finite.
Rank 0 writes a JSON verdict to argv[1].
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1603_04467_b200 as D  # noqa: E402
from dflow_harness import Run  # noqa: E402
from oracle.async_dp import push  # noqa: E402
import synth  # noqa: E402


def barrier():
    torch.cuda.synchronize()
    dist.barrier()


def main(out_path, exchange):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def nid():
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(D.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        return bytes(t.cpu().numpy().tobytes())

    seed = 4321
    w = synth.with_batch(synth.C2, 64 * world)
    b = 64
    Ws, bs = synth.init_params(w)
    verdict = {"world": world, "exchange": exchange}

    def session(mode):
        r = Run(w.dims, "MSE", w.lr, rows=b, exchange=exchange, world=world, rank=rank, device=local, nccl_id=nid(),
                sr_seed=seed, async_dp=mode)
        r.assign(Ws, bs)
        barrier()
        return r

    def my_batch(step):
        X, Y = synth.batch(w, step=step)
        return (torch.from_numpy(X[rank * b:(rank + 1) * b]).cuda(), torch.from_numpy(Y[rank * b:(rank + 1) * b]).cuda())

    def flat(gW, gb):
        return [(np.asarray(a, np.float32), np.asarray(c, np.float32)) for a, c in zip(gW, gb)]

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    # ---------------- A1: serialised replicas
    run = session(2)  # explicit pulls
    ok_pull, ok_final = True, True
    Wref = [(np.asarray(a, np.float32).copy(), np.asarray(c, np.float32).copy()) for a, c in zip(Ws, bs)]
    for turn in range(world):
        if turn == rank:
            D.check(D.dflow_async_pull(run.s, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
            Wp, bp = run.read()
            ok_pull &= all(np.array_equal(a.view(np.uint32), r[0].view(np.uint32)) and
                           np.array_equal(c.view(np.uint32), r[1].view(np.uint32)) for a, c, r in zip(Wp, bp, Wref))
            X, Y = my_batch(0)
            gW, gb, _ = run.gradients(X, Y)
            run.step(X, Y)
            mine = flat(gW, gb)
        else:
            mine = None
        barrier()
        g = gather(mine)[turn]
        Wref = [push(Wl, bl, gw, gbl, w.lr, turn, world, exchange, (seed, 1, l))
                for l, ((Wl, bl), (gw, gbl)) in enumerate(zip(Wref, g))]
    Wf, bf = run.read()
    ok_final = all(np.array_equal(a.view(np.uint32), r[0].view(np.uint32)) and
                   np.array_equal(c.view(np.uint32), r[1].view(np.uint32)) for a, c, r in zip(Wf, bf, Wref))
    verdict["a1_pulls_bitexact"] = bool(all(gather(ok_pull)))
    verdict["a1_final_bitexact"] = bool(ok_final)
    run.close()
    barrier()

    # ---------------- A2: concurrent pushes from one point
    run = session(2)
    D.check(D.dflow_async_pull(run.s, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    X, Y = my_batch(1)
    gW, gb, _ = run.gradients(X, Y)
    barrier()
    run.step(X, Y)  # all ranks push at once
    barrier()
    Wf, bf = run.read()
    gs = gather(flat(gW, gb))
    W0 = [(np.asarray(a, np.float32), np.asarray(c, np.float32)) for a, c in zip(Ws, bs)]

    def sequence(order):
        cur = [(a.copy(), c.copy()) for a, c in W0]
        for r in order:
            cur = [push(Wl, bl, gw, gbl, w.lr, r, world, exchange, (seed, 1, l))
                   for l, ((Wl, bl), (gw, gbl)) in enumerate(zip(cur, gs[r]))]
        return cur
    fwd, rev = sequence(range(world)), sequence(reversed(range(world)))
    if world == 2:
        ok = True
        for (a, c), (f1, f2), (r1, r2) in zip(zip(Wf, bf), fwd, rev):
            ok &= bool(np.all((a.view(np.uint32) == f1.view(np.uint32)) | (a.view(np.uint32) == r1.view(np.uint32))))
            ok &= bool(np.all((c.view(np.uint32) == f2.view(np.uint32)) | (c.view(np.uint32) == r2.view(np.uint32))))
        verdict["a2_one_of_the_orders"] = ok
    worst = 0.0
    for l, ((a, c), (f1, f2)) in enumerate(zip(zip(Wf, bf), fwd)):
        for k, (got, ref) in enumerate(((a, f1), (c, f2))):
            # any order differs from the rank order by re-rounding: two orders of N sequential
            # roundings (<= 1/2 ulp each) differ by <= N ulps; use 2 (N - 1) of the largest
            # intermediate |W0| + lr * sum_r |g_r| (N = 2: two roundings per order)
            mag = np.abs(W0[l][k]).astype(np.float64) + w.lr * sum(np.abs(gs[r][l][k]).astype(np.float64)
                                                                    for r in range(world))
            bound = np.spacing(mag.astype(np.float32)).astype(np.float64) * 2 * (world - 1)
            worst = max(worst, float(np.max(np.abs(got.astype(np.float64) - ref) / bound)))
    verdict["a2_reassociation_ratio"] = worst  # <= 1: within the re-rounding bound of the rank order
    run.close()
    barrier()

    # ---------------- A3: free-running replicas
    # (every replica applies a full step, so N replicas move N times as far per unit of
    # wall time as one; the usual async-SGD scaling lr / N keeps the run in the stable range)
    run = Run(w.dims, "MSE", w.lr / world, rows=b, exchange=exchange, world=world, rank=rank, device=local,
              nccl_id=nid(), sr_seed=seed, async_dp=1)
    run.assign(Ws, bs)
    barrier()
    losses = []
    for step in range(40):
        X, Y = my_batch(2 + step)
        losses.append(run.step(X, Y))
    barrier()
    Wf, bf = run.read()
    finite = all(np.all(np.isfinite(a)) for a in Wf + bf)
    first, last = gather(float(np.mean(losses[:3]))), gather(float(np.mean(losses[-10:])))
    verdict["a3_loss_first_last"] = [float(np.mean(first)), float(np.mean(last))]
    verdict["a3_ok"] = bool(finite)
    verdict["a3_ok_all"] = bool(all(gather(verdict["a3_ok"])) and np.mean(last) < np.mean(first))
    run.close()
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(verdict, f)
    barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "TRUNC16")
