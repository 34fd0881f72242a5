"""f2 comparison: the three gradient channels side by side on N GPUs.

  A. C2 (784-1024-1024-10, B = 256 global) trained for --steps synchronous steps with the
     FP32, TRUNC16 and SR16 exchanges from the same initialisation and batches: loss curves.
  B. C4's signature (C3 gradients at N ranks, local batch 32768 / N): the exchanged mean
     gradient of every layer under TRUNC16 and SR16 against the FP32 exchange of the same
     gradients — mean signed relative error (truncation's bias vs ~0) and max |error|.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        scripts/sr_convergence.py --out gpurun_out/sr_convergence.json
"""
import argparse
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
import synth  # noqa: E402
from dflow_harness import Run, stream_ptr  # noqa: E402

EXCHANGES = ("FP32", "TRUNC16", "SR16")


def nccl_id(rank):
    t = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(D.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def curves(rank, world, local, steps, seed):
    w = synth.C2
    b = w.batch // world
    Ws, bs = synth.init_params(w)
    out = {}
    for ex in EXCHANGES:
        run = Run(w.dims, "MSE", w.lr, rows=b, exchange=ex, world=world, rank=rank, device=local,
                  nccl_id=nccl_id(rank), sr_seed=seed)
        run.assign(Ws, bs)
        losses = []
        for step in range(steps):
            X, Y = synth.batch(w, step=step)
            losses.append(run.step(torch.from_numpy(X[rank * b:(rank + 1) * b]).cuda(),
                                   torch.from_numpy(Y[rank * b:(rank + 1) * b]).cuda()))
        out[ex] = losses
        run.close()
    return out


def signature(rank, world, local, seed):
    w = synth.C3
    b = w.batch // world
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w)
    run = Run(w.dims, "MSE", w.lr, rows=b, exchange="FP32", world=world, rank=rank, device=local,
              nccl_id=nccl_id(rank))
    run.assign(Ws, bs)
    Xd = torch.from_numpy(X[rank * b:(rank + 1) * b]).cuda()
    Yd = torch.from_numpy(Y[rank * b:(rank + 1) * b]).cuda()
    del X, Y
    grads = [torch.empty((w.dims[l], w.dims[l + 1]), dtype=torch.float32, device="cuda") for l in range(w.layers)]
    nodes = [run.mlp.grads[run.mlp.weights[l]] for l in range(w.layers)]
    ids = D.node_array([run.mlp.x, run.mlp.y])
    D.check(D.dflow_fetch_gradients(run.s, 2, ids, D.ptr_array([Xd.data_ptr(), Yd.data_ptr()]),
                                    D.i64_array([Xd.stride(0), Yd.stride(0)]), b, len(nodes), D.node_array(nodes),
                                    D.ptr_array([g.data_ptr() for g in grads]), stream_ptr()))
    torch.cuda.synchronize()
    sessions = {ex: Run((16, 16), "MSE", 0.5, rows=16, exchange=ex, world=world, rank=rank, device=local,
                        nccl_id=nccl_id(rank), sr_seed=seed) for ex in EXCHANGES}
    res = {}
    for l, g in enumerate(grads):
        outs = {}
        for ex, r in sessions.items():
            o = torch.empty_like(g)
            D.check(D.dflow_exchange(r.s, C.c_void_p(g.data_ptr()), C.c_void_p(o.data_ptr()), g.numel(),
                                     stream_ptr()))
            outs[ex] = o
        torch.cuda.synchronize()
        ref = outs["FP32"].double()
        big = ref.abs() > 1e-30
        for ex in ("TRUNC16", "SR16"):
            rel = ((outs[ex].double() - ref) / ref)[big]
            res[f"layer{l + 1}_{ex}"] = {"mean_rel_err": float(rel.mean()), "max_abs_rel_err": float(rel.abs().max()),
                                         "elements": int(big.sum())}
    for r in sessions.values():
        r.close()
    run.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--out", default="gpurun_out/sr_convergence.json")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = {"world": world, "steps": args.steps, "sr_seed": args.seed}
    res["c2_loss"] = curves(rank, world, local, args.steps, args.seed)
    res["c4_signature"] = signature(rank, world, local, args.seed)
    if rank == 0:
        c = res["c2_loss"]
        res["c2_summary"] = {ex: {"first": c[ex][0], "step10": c[ex][min(10, len(c[ex]) - 1)],
                                  "last": c[ex][-1],
                                  "mean_last50": float(np.mean(c[ex][-50:]))} for ex in EXCHANGES}
        res["c2_summary"]["max_rel_dev_vs_FP32"] = {
            ex: float(np.max(np.abs(np.array(c[ex]) - np.array(c["FP32"])) / np.array(c["FP32"])))
            for ex in ("TRUNC16", "SR16")}
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps({k: v for k, v in res.items() if k != "c2_loss"}, indent=1))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
