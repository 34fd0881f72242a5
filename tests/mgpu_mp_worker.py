"""One rank of the model-parallel checks (f4), launched by tests/test_gpu_mp.py via torchrun.
PAPER.md:399-430 (Send/Recv partitioning), 813-821 (channel codec), 958-972 (Fig. 8);
readings A32-A34.

  M1 exact regime (P12 inputs: every stored value and every channel tensor exact in 16 bits):
     the N-rank layer-partitioned step == oracle.partition.train_step_model_parallel == the
     single-device oracle step, bit for bit, for every layer (read from its owner rank).
  M2 C2-shaped random data: W, b after one step within the bf16 tolerance of the oracle's
     partitioned step (codec on both channels); the loss every rank reports is the last
     rank's, within tolerance of the oracle's.
  M3 three further steps: the loss falls.
Rank 0 writes a JSON verdict to argv[1].
"""
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
from dflow_harness import Run, normwise  # noqa: E402
from oracle.mlp import build_mlp, train_step  # noqa: E402
from oracle.partition import train_step_model_parallel  # noqa: E402
import synth  # noqa: E402


def main(out_path):
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

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def owned(L):  # reading A32
        return [l for l in range(L) if (l * world) // L == rank]

    def run_case(dims, lr, X, Y, Ws, bs, steps):
        L = len(dims) - 1
        run = Run(dims, "MSE", lr, rows=X.shape[0], world=world, rank=rank, device=local, nccl_id=nid(),
                  model_parallel=1)
        run.assign(Ws, bs)
        Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
        losses = [run.step(Xd, Yd)]
        Wg, bg = run.read()
        mine = {l: (Wg[l], bg[l]) for l in owned(L)}
        for k in range(steps):
            Xs, Ys = batches[k]
            losses.append(run.step(torch.from_numpy(Xs).cuda(), torch.from_numpy(Ys).cuda()))
        run.close()
        allmine = {}
        for d in gather(mine):
            allmine.update(d)
        return [allmine[l][0] for l in range(L)], [allmine[l][1] for l in range(L)], losses

    verdict = {"world": world}
    # ---------------- M1 exact regime, bit for bit
    X, Y, Ws, bs, lr = synth.exact_regime()
    dims = (X.shape[1],) + tuple(W.shape[1] for W in Ws)
    batches = []
    if len(dims) - 1 >= world:
        Wg, bg, losses = run_case(dims, lr, X, Y, Ws, bs, 0)
        mg = build_mlp(dims, "MSE", lr)
        mp = train_step_model_parallel(mg, Ws, bs, X, Y, world)
        sd = train_step(mg, Ws, bs, X, Y, 1, "FP32")
        verdict["m1_bitexact_vs_partitioned_oracle"] = all(
            np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(Wg + bg, mp["W"] + mp["b"]))
        verdict["m1_equals_single_device"] = all(
            np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(mp["W"] + mp["b"], sd["W"] + sd["b"]))
        verdict["m1_loss"] = [losses[0], mp["loss"]]
    # ---------------- M2 / M3 random data, tolerance
    w = synth.with_batch(synth.C2, 256) if world <= 3 else synth.Workload("mp4", (512, 512, 512, 512, 16), 256, "MSE",
                                                                           2.0 ** -5, "he")
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w)
    batches = [synth.batch(w, step=1 + k) for k in range(3)]
    Wg, bg, losses = run_case(w.dims, w.lr, X, Y, Ws, bs, 3)
    mg = build_mlp(w.dims, "MSE", w.lr)
    mp = train_step_model_parallel(mg, Ws, bs, X, Y, world)
    errs = [normwise(a, b) for a, b in zip(Wg + bg, mp["W"] + mp["b"])]
    verdict["m2_w_after_max_err"] = max(errs)
    verdict["m2_loss_rel_err"] = abs(losses[0] - mp["loss"]) / mp["loss"]
    verdict["m2_losses_agree_across_ranks"] = len(set(np.float32(v).tobytes() for v in gather(losses[0]))) == 1
    verdict["m3_losses"] = losses
    verdict["m3_falls"] = bool(np.mean(losses[-2:]) < losses[0])
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(verdict, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
