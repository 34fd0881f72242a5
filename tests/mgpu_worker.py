"""One rank of the N-GPU parity checks (launched by tests/test_gpu_multi.py via torchrun).

Checks, for world = N GPUs over NCCL (§7 :934-941, §5.5 :813-821):
  P4  exchange bit-exact: dflow_exchange(g_r) == oracle combine of the same g_r
  P4' step bit-exact: W after dflow_train_step == oracle apply(oracle combine(trunc(g_r)))
      where g_r are the GPU's own fp32 gradients of rank r (fetched, same kernels)
  P11 every rank holds bitwise identical W, b after each step
  gate W after one step vs the oracle's N-replica step within 2e-2 (bf16)
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
from dflow_harness import Run, normwise, stream_ptr  # noqa: E402
from oracle import kernels as OK  # noqa: E402
from oracle.exchange import combine  # noqa: E402
from oracle.mlp import build_mlp, train_step  # noqa: E402
import synth  # noqa: E402


def main(out_path, exchange):
    p2p = 0
    defer = 0
    host = 0
    precision = "bf16"
    if exchange.endswith("_HOST"):  # + pipelined host-fed steps == device-fed steps, bitwise
        exchange, host = exchange[:-5], 1
    if exchange.endswith("_DEFER"):  # options.defer_apply: the same bits as the eager join
        exchange, defer = exchange[:-6], 1
    if exchange.endswith("_TF32"):  # the fp32-faithful 3xTF32 path over the same channel
        exchange, precision = exchange[:-5], "3xtf32"
    if exchange.endswith("_P2P"):  # the fused NVLink exchange (f1): same bits as the NCCL path
        exchange, p2p = exchange[:-4], 1
    seed = 1234  # SR16 draw streams (reading A27)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(D.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    nid = bytes(idt.cpu().numpy().tobytes())
    verdict = {"world": world, "exchange": exchange, "p2p": p2p, "defer_apply": defer}

    w = synth.with_batch(synth.C2, 256)
    b = w.batch // world
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w)
    Xr, Yr = X[rank * b:(rank + 1) * b], Y[rank * b:(rank + 1) * b]
    run = Run(w.dims, "MSE", w.lr, rows=b, exchange=exchange, world=world, rank=rank, device=local, nccl_id=nid,
              p2p=p2p, sr_seed=seed, precision=precision, defer_apply=defer)
    verdict["precision"] = precision
    run.assign(Ws, bs)
    Xd, Yd = torch.from_numpy(Xr).cuda(), torch.from_numpy(Yr).cuda()

    # --- P4: exchange alone on random gradients (ragged length)
    n = 100003
    g_local = synth.rng(500 + rank).standard_normal(n).astype(np.float32)
    gd = torch.from_numpy(g_local).cuda()
    outd = torch.empty(n, dtype=torch.float32, device="cuda")
    D.check(D.dflow_exchange(run.s, C.c_void_p(gd.data_ptr()), C.c_void_p(outd.data_ptr()), n, stream_ptr()))
    torch.cuda.synchronize()
    all_g = [synth.rng(500 + r).standard_normal(n).astype(np.float32) for r in range(world)]
    # (the first standalone exchange of the session: SR16 step 1, layer 0)
    ref = combine(all_g, exchange if exchange != "FP32_NCCL" else "FP32", sr=(seed, 1, 0))
    got = outd.cpu().numpy()
    if exchange == "FP32_NCCL":
        verdict["p4_exchange_max_rel"] = normwise(got, ref)
        verdict["p4_exchange_ok"] = verdict["p4_exchange_max_rel"] < 1e-6
    else:
        verdict["p4_exchange_ok"] = bool(np.array_equal(got.view(np.uint32), ref.view(np.uint32)))

    # --- per-rank GPU gradients, gathered on every rank
    gW, gb, _ = run.gradients(Xd, Yd)
    flat = np.concatenate([np.concatenate([a.ravel(), c.ravel()]) for a, c in zip(gW, gb)]).astype(np.float32)
    t = torch.from_numpy(flat).cuda()
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    per_rank = [x.cpu().numpy() for x in gathered]

    # --- one train step
    loss = run.step(Xd, Yd)
    Wg, bg = run.read()
    mine = np.concatenate([np.concatenate([a.ravel(), c.ravel()]) for a, c in zip(Wg, bg)])
    mt = torch.from_numpy(mine).cuda()
    allW = [torch.empty_like(mt) for _ in range(world)]
    dist.all_gather(allW, mt)
    verdict["p11_replicas_identical"] = all(bool(torch.equal(allW[0], x)) for x in allW)

    # P4': oracle exchange + apply of the GPU's own gradients == the GPU step, bit for bit
    if exchange == "SR16":
        # per layer bucket [dW_l ; db_l], the session's first train step (epoch 1)
        ok = True
        off = 0
        for l in range(w.layers):
            nw, nb = Ws[l].size, bs[l].size
            ghat = combine([p[off:off + nw + nb] for p in per_rank], "SR16", sr=(seed, 1, l))
            new_w = OK.apply_gradient_descent(Ws[l], w.lr, ghat[:nw].reshape(Ws[l].shape), "f32")
            new_b = OK.apply_gradient_descent(bs[l], w.lr, ghat[nw:], "f32")
            ok &= bool(np.array_equal(new_w.view(np.uint32), Wg[l].view(np.uint32)))
            ok &= bool(np.array_equal(new_b.view(np.uint32), bg[l].view(np.uint32)))
            off += nw + nb
        verdict["p4_step_bitexact"] = ok
    if exchange in ("TRUNC16", "FP32"):
        ok = True
        off = 0
        for l in range(w.layers):
            for arr, var, lr in ((Ws[l], "W", w.lr), (bs[l], "b", w.lr)):
                sz = arr.size
                ghat = combine([p[off:off + sz] for p in per_rank], exchange).reshape(arr.shape)
                new = OK.apply_gradient_descent(arr, lr, ghat, "f32")
                gpu = Wg[l] if var == "W" else bg[l]
                ok &= bool(np.array_equal(new.view(np.uint32), gpu.view(np.uint32)))
                off += sz
        verdict["p4_step_bitexact"] = ok

    # gate: vs the oracle's N-replica step on the same global batch
    mg = build_mlp(w.dims, "MSE", w.lr)
    ref = train_step(mg, Ws, bs, X, Y, world, exchange if exchange != "FP32_NCCL" else "FP32", sr_seed=seed, step=1)
    errs = [normwise(a, r) for a, r in zip(Wg + bg, ref["W"] + ref["b"])]
    verdict["w_after_max_err"] = max(errs)
    verdict["loss_rel_err"] = abs(loss - ref["loss"]) / ref["loss"]

    # a few more steps: replicas stay identical (P11); in the last one only rank 0 fetches the
    # loss (the fused channel's loss exchange is one-sided: no collective for the others to miss)
    for step in range(3):
        Xs, Ys = synth.batch(w, step=step)
        run.step(torch.from_numpy(Xs[rank * b:(rank + 1) * b]).cuda(),
                 torch.from_numpy(Ys[rank * b:(rank + 1) * b]).cuda(), want_loss=(step < 2 or rank == 0))
    Wg, bg = run.read()
    mine = np.concatenate([np.concatenate([a.ravel(), c.ravel()]) for a, c in zip(Wg, bg)])
    mt = torch.from_numpy(mine).cuda()
    dist.all_gather(allW, mt)
    verdict["p11_after_4_steps"] = all(bool(torch.equal(allW[0], x)) for x in allW)
    run.close()
    if defer:
        # the same 4 steps with the eager join (defer_apply = 0): bit-identical parameters
        # (a second communicator needs its own NCCL id)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(D.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nid2 = bytes(idt.cpu().numpy().tobytes())
        eager = Run(w.dims, "MSE", w.lr, rows=b, exchange=exchange, world=world, rank=rank, device=local,
                    nccl_id=nid2, p2p=p2p, sr_seed=seed, precision=precision, defer_apply=0)
        eager.assign(Ws, bs)
        gW, gb, _ = eager.gradients(Xd, Yd)  # the same call sequence (SR16 draws are keyed by step)
        eager.step(Xd, Yd)
        for step in range(3):
            Xs, Ys = synth.batch(w, step=step)
            eager.step(torch.from_numpy(Xs[rank * b:(rank + 1) * b]).cuda(),
                       torch.from_numpy(Ys[rank * b:(rank + 1) * b]).cuda())
        We, be = eager.read()
        verdict["defer_equals_eager"] = all(bool(np.array_equal(a.view(np.uint32), c.view(np.uint32)))
                                            for a, c in zip(We + be, Wg + bg))
        eager.close()
    if host:
        # dflow_train_step_host_pipelined (each call returns the previous step's loss, loss
        # all-reduced on the exchange stream into alternating slots) against device-fed steps
        # of a twin session: every loss and the final parameters bit for bit
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(D.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nid3 = bytes(idt.cpu().numpy().tobytes())
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(D.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nid4 = bytes(idt.cpu().numpy().tobytes())
        dev = Run(w.dims, "MSE", w.lr, rows=b, exchange=exchange, world=world, rank=rank, device=local,
                  nccl_id=nid3, p2p=p2p, sr_seed=seed, precision=precision, defer_apply=defer)
        hst = Run(w.dims, "MSE", w.lr, rows=b, exchange=exchange, world=world, rank=rank, device=local,
                  nccl_id=nid4, p2p=p2p, sr_seed=seed, precision=precision, defer_apply=defer)
        dev.assign(Ws, bs)
        hst.assign(Ws, bs)
        bufs = []
        for step in range(4):
            Xs, Ys = synth.batch(w, step=10 + step)
            bufs.append((torch.from_numpy(np.ascontiguousarray(Xs[rank * b:(rank + 1) * b])).pin_memory(),
                         torch.from_numpy(np.ascontiguousarray(Ys[rank * b:(rank + 1) * b])).pin_memory()))
        want = [dev.step(Xh.cuda(), Yh.cuda()) for Xh, Yh in bufs]
        ids, lds = D.node_array([hst.mlp.x, hst.mlp.y]), D.i64_array([w.dims[0], w.dims[-1]])
        got = []
        for Xh, Yh in bufs:
            lh, has = C.c_float(0), C.c_int32(0)
            D.check(D.dflow_train_step_host_pipelined(hst.s, 2, ids, D.ptr_array([Xh.data_ptr(), Yh.data_ptr()]),
                                                      lds, b, C.byref(lh), C.byref(has), stream_ptr()))
            if has.value:
                got.append(lh.value)
        lh, has = C.c_float(0), C.c_int32(0)
        D.check(D.dflow_session_last_loss(hst.s, C.byref(lh), C.byref(has)))
        got.append(lh.value)
        Wd, bd = dev.read()
        Wh, bh = hst.read()
        verdict["host_pipelined_losses_equal"] = bool(
            len(got) == len(want) and np.array_equal(np.float32(got).view(np.uint32), np.float32(want).view(np.uint32)))
        verdict["host_pipelined_params_equal"] = all(bool(np.array_equal(a.view(np.uint32), c.view(np.uint32)))
                                                     for a, c in zip(Wd + bd, Wh + bh))
        dev.close()
        hst.close()
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(verdict, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "TRUNC16")
