#!/usr/bin/env python3
"""bench.py — replicated Relu(XW+b) MLP train step on B200 (arXiv 1603.04467 §7 sync data parallelism).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--exchange TRUNC16] [--impl reference]

One JSON line on rank 0 (the driver's contract).  Workload: BASELINE.json
configs[2] = "Wide MLP 4 layers of 8192x8192 bf16, global batch 32768, sync
data-parallel at 1/2/4/8 B200" (the metric's own config; it fits one GPU).
N > 1: launched by torchrun, one rank per GPU; the global batch is fixed
(strong scaling), each rank trains on rows [r*b, (r+1)*b), b = 32768/N, and
the gradients cross NVLink through NCCL alltoall/allgather of 16-bit truncated
payloads (§5.5).

`--impl reference` times the oracle (the plain CPU implementation written from
the paper, oracle/) on this box's host cores on a bounded sample of the same
workload — the reference arm for this tier.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "MLP train-step examples/sec at 1/2/4/8 B200; % tensor-core peak"
UNIT = "examples/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"bf16_burst": d.get("bf16_tflops", 1590.0), "bf16_sustained": d.get("bf16_tflops_sustained", 1400.0),
                "hbm": d.get("hbm_gbs", 6650.0), "source": "measured (MEASURED_PEAKS.json)"}
    return {"bf16_burst": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0,
            "source": "fallback (B200_PROFILING.md)"}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------- distributed plumbing (host logic)
def shard_rows(global_batch: int, world: int, rank: int):
    """Rows [row0, row0 + b) of the global batch for this rank (reading A4); B % N must be 0."""
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} must divide by the number of GPUs {world}")
    b = global_batch // world
    return rank * b, b


def broadcast_bytes(payload, dist, device, n: int = 128) -> bytes:
    """Rank 0's n-byte payload (the NCCL unique id) to every rank through torch.distributed."""
    import torch
    t = torch.zeros(n, dtype=torch.uint8, device=device)
    if dist.get_rank() == 0:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def max_over_ranks(v: float, dist, device) -> float:
    """Job time = the slowest rank's device time."""
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.device = device
        self.p = None

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        maxmhz = max(r[1] for r in rows)
        load = [r for r in rows if r[2] > 300] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": maxmhz, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(r[2] for r in rows)}


# ---------------------------------------------------------------- oracle (CPU) legs
def oracle_sample(w: synth.Workload, target_s: float, n_steps: int = 1):
    """Times the oracle (as it stands) on a bounded row sample of workload w."""
    from oracle.mlp import build_mlp, train_step
    Ws, bs = synth.init_params(w)
    mg = build_mlp(w.dims, w.loss, w.lr)
    # a step costs fixed + per_row * rows, and the fixed part (the f64 update of every
    # parameter, the graph walk) dominates small samples: double the rows until one step
    # takes at least half the target, then size the sample from the last two probes
    rows, probe = 32, []
    while True:
        X, Y = synth.batch(w, rows=rows)
        t0 = time.perf_counter()
        train_step(mg, Ws, bs, X, Y, 1, "TRUNC16")
        probe.append((rows, time.perf_counter() - t0))
        if probe[-1][1] >= 0.5 * target_s or rows >= w.batch:
            break
        rows = min(w.batch, rows * 2)
    if len(probe) >= 2:
        (r0, t0_), (r1, t1_) = probe[-2], probe[-1]
        per_row = max((t1_ - t0_) / (r1 - r0), t1_ / r1 * 0.25, 1e-9)
        rows = int(min(w.batch, r1 + max(0.0, target_s - t1_) / per_row))
    rows = max(16, rows // 16 * 16)
    X, Y = synth.batch(w, rows=rows)
    times = []
    for _ in range(n_steps):
        t0 = time.perf_counter()
        train_step(mg, Ws, bs, X, Y, 1, "TRUNC16")
        times.append(time.perf_counter() - t0)
    return rows, times


def numpy_f32_sample(w: synth.Workload, rows: int):
    """The best plain-CPU line: the same step in numpy float32 (multithreaded
    BLAS), no graph, no codec — forward, MSE seed, backward, SGD — on a row sample."""
    import numpy as np
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w, rows=rows)
    t0 = time.perf_counter()
    acts = [X]
    for W, b in zip(Ws, bs):
        acts.append(np.maximum(acts[-1] @ W + b, np.float32(0)))
    g = (acts[-1] - Y) / np.float32(rows * w.dims[-1])
    for l in range(len(Ws) - 1, -1, -1):
        g = g * (acts[l + 1] > 0)
        dW, db = acts[l].T @ g, g.sum(0)
        if l:
            g = g @ Ws[l].T
        Ws[l] -= np.float32(w.lr) * dW
        bs[l] -= np.float32(w.lr) * db
    return time.perf_counter() - t0


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args, w):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    # each step: one oracle step on a row sample, sized so W + K steps finish in a few minutes
    per_step_budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    rows, _ = oracle_sample(w, per_step_budget, n_steps=0)
    from oracle.mlp import build_mlp, train_step
    Ws, bs = synth.init_params(w)
    mg = build_mlp(w.dims, w.loss, w.lr)
    X, Y = synth.batch(w, rows=rows)
    for _ in range(args.warmup):
        train_step(mg, Ws, bs, X, Y, 1, "TRUNC16")
    t0 = time.perf_counter()
    for _ in range(args.steps):
        train_step(mg, Ws, bs, X, Y, 1, "TRUNC16")
    dt = time.perf_counter() - t0
    value = rows * args.steps / dt
    sample = f"one oracle (f64 numpy graph executor) step of {w.name} on {rows} rows per step"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1000 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, synth/)",
            "config": config_dict(w, args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(w, args, world):
    return {"workload": w.name, "global_batch": w.batch, "layers": w.layers, "width": w.dims[1],
            "dims": list(w.dims), "loss": w.loss, "lr": w.lr,
            "exchange": ("SENDRECV_TRUNC16_CHANNELS" if (world > 1 and getattr(args, "model_parallel", 0)) else
                         ("ASYNC_" if (world > 1 and getattr(args, "async_dp", 0)) else "") + args.exchange +
                         ("_P2P" if (args.exchange in ("TRUNC16", "SR16") and world > 1 and getattr(args, "p2p", 0)
                                     and not getattr(args, "async_dp", 0)) else "")),
            "parallelism": (f"mp{world}" if (world > 1 and getattr(args, "model_parallel", 0)) else f"dp{world}"),
            "defer_apply": int(bool(world > 1 and getattr(args, "defer_apply", 0) and
                                    not getattr(args, "model_parallel", 0) and not getattr(args, "async_dp", 0))),
            "precision": ("3xTF32 split fp32 operands (big, small), fp32 accumulate + master weights"
                          if w.precision == "3xtf32" else "bf16 operands, fp32 accumulate + master weights"),
            "l2": ("no flush: every step streams inputs and activations far larger than the 126 MB L2 "
                   f"(X fp32 {w.batch // world * w.dims[0] * 4 / 2**20:.0f} MiB per rank)")
            if w.batch // world * w.dims[0] * 4 > 126 * 2**20 else
            "inputs fit in L2 and are not flushed between steps (latency-bound configuration)"}


# ---------------------------------------------------------------- GPU leg
def run_gpu(args, w):
    import torch
    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1603_04467_b200 as D

    mp = world > 1 and getattr(args, "model_parallel", 0)
    # model parallelism (f4): one replica, every rank steps the whole batch through its layers
    row0, b = (0, w.batch) if mp else shard_rows(w.batch, world, rank)
    # NCCL id from rank 0, broadcast through torch.distributed (plumbing only)
    nid = None
    if world > 1:
        nid = broadcast_bytes(D.nccl_unique_id() if rank == 0 else None, dist, "cuda")
    tf32 = w.precision == "3xtf32"
    mlp = D.mlp_graph(w.dims, w.loss, w.lr)
    opts = D.make_options(world=world, rank=rank, device=local, exchange=args.exchange, max_local_rows=b,
                          overlap=1, sm_reserve=args.sm_reserve, p2p=args.p2p, sr_seed=1234,
                          graphs=1 if world == 1 else 0, async_dp=args.async_dp if world > 1 else 0,
                          model_parallel=1 if mp else 0,
                          defer_apply=args.defer_apply if (world > 1 and not mp and not args.async_dp) else 0,
                          precision=D.DFLOW_PRECISION_3XTF32 if tf32 else D.DFLOW_PRECISION_BF16)
    s = D.session_create(mlp, opts, nid)
    Ws, bs = synth.init_params(w)
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    for nid_, W in zip(mlp.weights, Ws):
        D.check(D.dflow_variable_assign(s, nid_, W.ctypes.data_as(C.c_void_p), 0, sp))
    for nid_, bb in zip(mlp.biases, bs):
        D.check(D.dflow_variable_assign(s, nid_, bb.ctypes.data_as(C.c_void_p), 0, sp))
    del Ws, bs
    X, Y = synth.batch(w, rows=b, row0=row0)
    Xd = torch.from_numpy(X).cuda()
    Yd = torch.from_numpy(Y).cuda()
    feeds = D.node_array([mlp.x, mlp.y])
    ptrs = D.ptr_array([Xd.data_ptr(), Yd.data_ptr()])
    lds = D.i64_array([Xd.stride(0), Yd.stride(0)])

    def step(loss=None):
        D.check(D.dflow_train_step(s, 2, feeds, ptrs, lds, b, loss, sp))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    first_loss = C.c_float(0)
    step(C.byref(first_loss))
    for _ in range(max(0, args.warmup - 1)):
        step()
    clocks = Clocks(local)
    clocks.start()
    # the median of `repeats` timed regions of exactly K steps each, every one
    # bracketed by barrier + synchronize, max over ranks
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms_list = []
    step_loss = C.c_float(0)
    for _ in range(max(1, args.repeats)):
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step(C.byref(step_loss) if args.step_loss else None)  # the loss read back every step
        # defer_apply: the last step's pending updates belong to the region
        D.check(D.dflow_session_sync(s, sp))
        e1.record(stream)
        barrier()
        ms_list.append(max_over_ranks(e0.elapsed_time(e1), dist, "cuda"))
    clk = clocks.stop()
    ms = sorted(ms_list)[len(ms_list) // 2]
    st = D.dflow_stats()
    D.check(D.dflow_session_stats(s, C.byref(st)))
    launches = st.launches_per_step
    # per-kernel timing pass (CUDA events around every launch on its own stream)
    D.check(D.dflow_session_set_timing(s, 1))
    tsteps = max(3, min(args.steps, 10))
    for _ in range(tsteps):
        step()
    D.check(D.dflow_session_stats(s, C.byref(st)))
    D.check(D.dflow_session_set_timing(s, 0))
    gemm_avg_ms = st.gemm_ms / max(1, st.timed_steps * st.gemm_launches_per_step)
    flops_per_launch = st.gemm_flops_per_step / max(1, st.gemm_launches_per_step)
    last_loss = C.c_float(0)
    step(C.byref(last_loss))

    # end-to-end through the public API with HOST buffers (pinned), copies inside the timed region
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.from_numpy(Y).pin_memory()
    hptrs = D.ptr_array([Xh.data_ptr(), Yh.data_ptr()])
    hl, has = C.c_float(0), C.c_int32(0)
    # as many steps as the timed region (the pipelined call's fill and drain are one step each)
    e2e_steps = max(3, args.steps)

    def e2e_time(pipelined):
        # every step: H2D of x, y from pinned memory and the D2H read of its loss, in the region
        call = ((lambda: D.dflow_train_step_host_pipelined(s, 2, feeds, hptrs, lds, b, C.byref(hl), C.byref(has), sp))
                if pipelined else (lambda: D.dflow_train_step_host(s, 2, feeds, hptrs, lds, b, C.byref(hl), sp)))
        D.check(call())
        if pipelined:
            D.check(D.dflow_session_last_loss(s, C.byref(hl), C.byref(has)))
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            D.check(call())
        if pipelined:  # the last step's loss
            D.check(D.dflow_session_last_loss(s, C.byref(hl), C.byref(has)))
        barrier()
        return max_over_ranks(time.perf_counter() - t0, dist, "cuda")

    # pipelining pays when the per-step upload is long (C3: 2 GiB, PCIe-bound); for tiny steps
    # (C2: 0.8 MB) the blocking call measured faster (2.54 vs 2.17 M ex/s), so the headline uses
    # the pipelined call only above 64 MiB of H2D per step; both are reported
    e2e_blocking_s = e2e_time(False)
    e2e_pipelined_s = e2e_time(True)
    pipelined = (X.nbytes + Y.nbytes) >= 64 * 2 ** 20
    e2e_s = e2e_pipelined_s if pipelined else e2e_blocking_s

    D.dflow_session_destroy(s)
    s = None
    del Xd, Yd, Xh, Yh
    sub = None
    if world == 1 and args.c5_sub and not tf32:
        sub = c5_submeasure(D, local, args)

    pk = peaks()
    step_flops = w.flops_per_example() * w.batch
    value = w.batch * args.steps / (ms / 1000.0)
    if tf32:
        # the tensor pipe runs 3 TF32 products per fp32-equivalent FLOP; TF32 dense peak =
        # 1/2 of bf16 (B200_PROFILING.md nominal ratio 1.1 / 2.25 PF) x the measured bf16 peak
        mma_mult, peak_t, peak_b, kname = 3.0, 0.5 * pk["bf16_sustained"], 0.5 * pk["bf16_burst"], \
            "gemm_kernel<3xTF32> (tcgen05 kind::tf32, NK4-NK6)"
        peak_note = ", TF32 = 0.5 x measured sustained bf16 (nominal ratio); achieved counts the 3 TF32 products"
    else:
        mma_mult, peak_t, peak_b, kname = 1.0, pk["bf16_sustained"], pk["bf16_burst"], \
            "gemm_kernel<bf16> (tcgen05 kind::f16, NK1-NK3)"
        peak_note = ", sustained bf16 (kernel timed inside a long step)"
    achieved = mma_mult * flops_per_launch / (gemm_avg_ms / 1000.0) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tp) and world == 1 and not args.batch:  # profiled at N = 1, the full batch
        try:
            traffic = json.load(open(tp)).get(w.name)
        except Exception:
            traffic = None
    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            rows, times = oracle_sample(w, args.cpu_seconds)
            cpu = {"value": rows / times[0], "unit": UNIT, "cores": cores(), "kind": "oracle",
                   "sample": f"one oracle (f64 numpy graph executor) train step of {w.name} on a {rows}-row "
                             f"sample of the global batch ({times[0]:.1f} s)"}
            f32_rows = max(256, min(w.batch, rows * 8))
            t32 = numpy_f32_sample(w, f32_rows)
            cpu32 = {"value": f32_rows / t32, "unit": UNIT, "cores": cores(), "kind": "numpy_f32",
                     "sample": f"one plain numpy float32 step (BLAS) of {w.name} on {f32_rows} rows ({t32:.1f} s)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "repeats": len(ms_list), "ms_per_step_repeats": [m / args.steps for m in ms_list],
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (3xTF32)" if tf32 else "bf16",
            "data": "synthetic (seeded, synth/; X,Y ~ U[0,1), He-uniform W)",
            "config": config_dict(w, args, world),
            "pct_tensor_peak": {"step_tflops": mma_mult * step_flops / (ms / args.steps / 1000.0) / 1e12 / world,
                                "per_gpu_frac_of_sustained": mma_mult * step_flops / (ms / args.steps / 1000.0)
                                / 1e12 / world / peak_t,
                                "per_gpu_frac_of_burst": mma_mult * step_flops / (ms / args.steps / 1000.0)
                                / 1e12 / world / peak_b},
            "roofline": {"kernel": kname, "bound": "tensor", "achieved": achieved,
                         "peak": peak_t, "unit": "TFLOP/s", "frac": achieved / peak_t,
                         # the sustained peak is cuBLAS's own power-capped rate on 8192^3; a kernel
                         # that draws less power per FLOP can sit above it, so the burst figure is
                         # reported beside it
                         "frac_of_burst": achieved / peak_b, "peak_burst": peak_b,
                         "traffic": traffic, "peak_source": pk["source"] + peak_note,
                         "avg_launch_ms": gemm_avg_ms, "flops_per_launch": flops_per_launch,
                         "gemm_share_of_step": st.gemm_ms / max(1e-9, st.gemm_ms + st.other_ms + st.exchange_ms),
                         # the per-launch events run in a pass after the timed region (events around
                         # every launch, no step graph), whose clocks can differ from the timed
                         # region's; this is the GEMM rate if the timed step split its time in the
                         # same shares (a lower bound: it charges inter-kernel gaps to the kernels)
                         "achieved_at_timed_step": flops_per_launch * st.gemm_launches_per_step
                         / max(1e-12, ms / args.steps / 1000.0 * st.gemm_ms
                               / max(1e-9, st.gemm_ms + st.other_ms)) / 1e12 * mma_mult,
                         "timing_pass_kernel_ms_per_step": (st.gemm_ms + st.other_ms) / max(1, st.timed_steps),
                         # device time per step by kind (CUDA events around every launch, rank 0;
                         # exchange kernels run on the comm stream, overlapping the backward)
                         "kernel_ms_per_step": {"gemm": st.gemm_ms / max(1, st.timed_steps),
                                                "other": st.other_ms / max(1, st.timed_steps),
                                                "exchange": st.exchange_ms / max(1, st.timed_steps)}},
            "cpu_baseline": cpu,
            "cpu_f32": cpu32 if (world == 1 and not args.no_cpu_baseline) else None,
            "e2e": {"value": w.batch * e2e_steps / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": int(X.nbytes + Y.nbytes) * world, "d2h_bytes_per_step": 4 * world,
                    "api": ("dflow_train_step_host_pipelined (returns the previous step's loss)" if pipelined
                            else "dflow_train_step_host"),
                    "steps": e2e_steps,
                    "blocking_value": w.batch * e2e_steps / e2e_blocking_s,
                    "pipelined_value": w.batch * e2e_steps / e2e_pipelined_s},
            "gpu_launches": launches * args.steps,
            "loss_read_every_step": bool(args.step_loss),
            "gather": ("nvlink_multicast" if st.multicast else "unicast") if world > 1 else None,
            "clocks": clk,
            "loss": {"first": first_loss.value, "last": last_loss.value},
        }
        if sub is not None:
            line["c5_3xtf32_n1"] = sub
        print(json.dumps(line), flush=True)
    D.dflow_graph_destroy(mlp.graph)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def c5_submeasure(D, device, args):
    """The fp32-faithful path at paper precision (BASELINE configs[4]: 16 x 4096^2, 3xTF32,
    B = 65536) on one GPU: W >= 3 warm-up + K timed steps (CUDA events, clocks sampled), and
    one per-launch timing step for the GEMM's rate against the TF32 peak."""
    import torch
    w = synth.C5
    K = max(3, min(args.steps, 5))
    mlp = D.mlp_graph(w.dims, w.loss, w.lr)
    opts = D.make_options(world=1, rank=0, device=device, exchange="TRUNC16", max_local_rows=w.batch,
                          precision=D.DFLOW_PRECISION_3XTF32, graphs=1)
    s = D.session_create(mlp, opts, None)
    try:
        Ws, bs = synth.init_params(w)
        stream = torch.cuda.current_stream()
        sp = C.c_void_p(stream.cuda_stream)
        for nid_, W in zip(mlp.weights, Ws):
            D.check(D.dflow_variable_assign(s, nid_, W.ctypes.data_as(C.c_void_p), 0, sp))
        for nid_, bb in zip(mlp.biases, bs):
            D.check(D.dflow_variable_assign(s, nid_, bb.ctypes.data_as(C.c_void_p), 0, sp))
        X, Y = synth.batch(w)
        Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
        del X, Y
        feeds = D.node_array([mlp.x, mlp.y])
        ptrs = D.ptr_array([Xd.data_ptr(), Yd.data_ptr()])
        lds = D.i64_array([Xd.stride(0), Yd.stride(0)])
        loss = C.c_float(0)

        def step():
            D.check(D.dflow_train_step(s, 2, feeds, ptrs, lds, w.batch, C.byref(loss), sp))
        for _ in range(3):
            step()
        clocks = Clocks(device)
        clocks.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(K):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        clk = clocks.stop()
        ms = e0.elapsed_time(e1) / K
        st = D.dflow_stats()
        D.check(D.dflow_session_set_timing(s, 1))
        step()
        D.check(D.dflow_session_stats(s, C.byref(st)))
        gemm_ms = st.gemm_ms / max(1, st.timed_steps * st.gemm_launches_per_step)
        tf32_flops = 3.0 * st.gemm_flops_per_step / max(1, st.gemm_launches_per_step)
        pk = peaks()
        achieved = tf32_flops / (gemm_ms / 1000.0) / 1e12
        return {"workload": w.name, "precision": "3xTF32 (fp32-faithful, reading A14)", "steps": K, "warmup": 3,
                "ms_per_step": ms, "value": w.batch / (ms / 1000.0), "unit": UNIT, "loss": loss.value,
                "gemm": {"achieved_tf32_tflops": achieved, "peak_tf32_sustained": 0.5 * pk["bf16_sustained"],
                         "frac_of_tf32_sustained": achieved / (0.5 * pk["bf16_sustained"]),
                         "frac_of_tf32_burst": achieved / (0.5 * pk["bf16_burst"]), "avg_launch_ms": gemm_ms,
                         "peak_source": pk["source"] + ", TF32 = 0.5 x bf16 (B200_PROFILING.md nominal ratio)"},
                "clocks": clk}
    finally:
        D.dflow_session_destroy(s)
        D.dflow_graph_destroy(mlp.graph)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dflow", choices=["dflow", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="override the global batch (parity/debug only)")
    ap.add_argument("--exchange", default="TRUNC16", choices=["TRUNC16", "FP32", "FP32_NCCL", "NONE", "SR16"])
    ap.add_argument("--repeats", type=int, default=3,
                    help="timed regions of K steps each; value = the median (SURVEY §8(d))")
    ap.add_argument("--model-parallel", type=int, default=0,
                    help="N > 1: 1 = layer-wise model parallelism (f4): rank r holds layers "
                         "[r L / N, (r+1) L / N), activations / their gradients cross through Send/Recv "
                         "with the 16-bit channel codec")
    ap.add_argument("--async-dp", type=int, default=0,
                    help="N > 1: 1 = asynchronous replicas (f3): each rank pulls the shared parameters, steps "
                         "and pushes its own coded update with no barrier (the exchange names the coding)")
    ap.add_argument("--defer-apply", type=int, default=1,
                    help="N > 1 synchronous: last two dW swapped, layer l's update joined only by the next "
                         "forward of layer l (options.defer_apply; same bits)")
    ap.add_argument("--sm-reserve", type=int, default=0)
    ap.add_argument("--p2p", type=int, default=1,
                    help="TRUNC16 at N > 1: 1 = fused NVLink exchange (dW epilogue stores into the owners' "
                         "buffers), 0 = NCCL alltoall/allgather")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--step-loss", type=int, default=1,
                    help="1: every timed step reads its loss back to the host (part of the region); 0: none")
    ap.add_argument("--c5-sub", type=int, default=1,
                    help="N = 1: also measure C5 (16 x 4096^2, 3xTF32, B = 65536) and report it as c5_3xtf32_n1")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("timing rules: --warmup must be >= 3")
    w = synth.CONFIGS[args.config]
    if args.batch:
        w = synth.with_batch(w, args.batch)
    if args.impl == "reference":
        return run_reference(args, w)
    return run_gpu(args, w)


if __name__ == "__main__":
    sys.exit(main())
