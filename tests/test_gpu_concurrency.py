"""Sessions sharing a process (SURVEY §8(b) "Threading": one host thread per session; works
under torchrun or one process with a thread per GPU).  Each session owns its tile-scheduler
counters, streams and buffers, so sessions stepping concurrently — on two streams of one
GPU, or from two host threads — give exactly the bits of the same steps run one after the
other (a replica's step is a pure function of W and its batch)."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from dflow_harness import Run  # noqa: E402


def _bits(a, b):
    return all(np.array_equal(x.view(np.uint32), y.view(np.uint32)) for x, y in zip(a, b))


def _case(width):
    if width == "C2":  # small GEMMs: single-CTA tiles, dW on side streams beside the dgrads
        return synth.with_batch(synth.C2, 4096)
    return synth.Workload("C3w2", (8192, 8192, 8192), 2048, "MSE", 2.0 ** -2, "he")  # CTA-pair tiles


def _reference(w, batches):
    Ws, bs = synth.init_params(w)
    run = Run(w.dims, "MSE", w.lr, rows=w.batch)
    try:
        run.assign(Ws, bs)
        for X, Y in batches:
            run.step(X, Y, want_loss=False)
        torch.cuda.synchronize()
        W, b = run.read()
        return W + b
    finally:
        run.close()


def _batches(w, steps, dev=0):
    out = []
    for k in range(steps):
        X, Y = synth.batch(w, step=k)
        out.append((torch.from_numpy(X).cuda(dev), torch.from_numpy(Y).cuda(dev)))
    return out


@pytest.mark.parametrize("width", ["C2", "C3w"])
def test_two_sessions_two_streams_one_gpu(width):
    w = _case(width)
    batches = _batches(w, 3)
    ref = _reference(w, batches)
    Ws, bs = synth.init_params(w)
    runs = [Run(w.dims, "MSE", w.lr, rows=w.batch) for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    try:
        for r in runs:
            r.assign(Ws, bs)
        torch.cuda.synchronize()
        for X, Y in batches:  # enqueue both sessions' steps back to back, no host sync between
            for r, st in zip(runs, streams):
                with torch.cuda.stream(st):
                    r.step(X, Y, want_loss=False)
        torch.cuda.synchronize()
        for r in runs:
            W, b = r.read()
            assert _bits(W + b, ref)
    finally:
        for r in runs:
            r.close()


def _threaded(w, devices):
    """One host thread per session (each on its own stream and device), stepping at once."""
    Ws, bs = synth.init_params(w)
    per = {d: _batches(w, 3, d) for d in set(devices)}
    runs = [Run(w.dims, "MSE", w.lr, rows=w.batch, device=d) for d in devices]
    out, err = [None] * len(runs), []
    try:
        for r in runs:
            r.assign(Ws, bs)
        torch.cuda.synchronize()
        go = threading.Barrier(len(runs))

        def body(i):
            try:
                torch.cuda.set_device(devices[i])
                st = torch.cuda.Stream(devices[i])
                go.wait()
                with torch.cuda.stream(st):
                    for X, Y in per[devices[i]]:
                        runs[i].step(X, Y, want_loss=(i % 2 == 0))
                st.synchronize()
                W, b = runs[i].read()
                out[i] = W + b
            except Exception as e:  # surfaced below
                err.append(e)
        ts = [threading.Thread(target=body, args=(i,)) for i in range(len(runs))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not err, err
        return out
    finally:
        for r in runs:
            r.close()


@pytest.mark.parametrize("width", ["C2", "C3w"])
def test_two_threads_one_gpu(width):
    w = _case(width)
    ref = _reference(w, _batches(w, 3))
    for res in _threaded(w, [0, 0]):
        assert _bits(res, ref)


def test_two_threads_two_gpus():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    w = _case("C3w")
    ref = _reference(w, _batches(w, 3))
    for res in _threaded(w, [0, 1]):
        assert _bits(res, ref)
