import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from dflow_harness import SimRun, Run, normwise
import synth

def same(a, b):
    return bool(np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32)))

w = synth.with_batch(synth.C2, 256)
Ws, bs = synth.init_params(w)
Ws0 = [a.copy() for a in Ws]
X, Y = synth.batch(w)
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
Xs = [Xd[:128].clone(), Xd[128:].clone()]; Ys = [Yd[:128].clone(), Yd[128:].clone()]
chk = lambda: [float(t.double().sum()) for t in Xs + Ys]
c0 = chk()
plain = []
for r in range(2):
    p = Run(w.dims, "MSE", w.lr, rows=128); p.assign(Ws, bs)
    plain.append((p.gradients(Xs[r], Ys[r]), p.forward(Xs[r], Ys[r])))
    p.close()
print("plain losses", [float(pl[1][0]) for pl in plain], "inputs unchanged", chk() == c0, flush=True)
for ex, p2p in (("FP32", 0), ("TRUNC16", 1), ("TRUNC16", 0)):
    s = SimRun(w.dims, "MSE", w.lr, rows=128, world=2, exchange=ex, p2p=p2p)
    s.assign(Ws, bs)
    for r in range(2):
        Wr, br = s.read(r)
        print(ex, p2p, "rank", r, "assigned W ok", all(same(a, b) for a, b in zip(Wr, Ws)), "b ok", all(same(a, b) for a, b in zip(br, bs)), flush=True)
    for r in range(2):
        g = s.gradients(r, Xs[r], Ys[r])
        print(ex, p2p, "rank", r, "grads == plain", [same(a, b) for a, b in zip(g[0] + g[1], plain[r][0][0] + plain[r][0][1])], flush=True)
    g0b = s.gradients(0, Xs[0], Ys[0])
    print(ex, p2p, "rank0 again == plain", [same(a, b) for a, b in zip(g0b[0] + g0b[1], plain[0][0][0] + plain[0][0][1])], "inputs unchanged", chk() == c0, flush=True)
    losses = s.step(Xs, Ys)
    print(ex, p2p, "step losses", losses, "expected", (float(plain[0][1][0]) + float(plain[1][1][0])) / 2, "inputs unchanged", chk() == c0, flush=True)
    s.close()
print("Ws unchanged", all(same(a, b) for a, b in zip(Ws, Ws0)))
