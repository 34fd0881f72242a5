"""Debug: where do simulated-world results leave the oracle (C2 width, MP exact)?"""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from dflow_harness import SimRun, Run, normwise
from oracle.mlp import build_mlp, train_step
from oracle.partition import train_step_model_parallel
import synth

def cmp(tag, a, b):
    a = np.asarray(a); b = np.asarray(b)
    neq = np.sum(a.view(np.uint32) != b.view(np.uint32))
    print(f"{tag}: shape {a.shape} mismatches {neq} normwise {normwise(a, b):.3e}", flush=True)

# 1. sim world of 1 vs plain session, C2
w = synth.with_batch(synth.C2, 256)
Ws, bs = synth.init_params(w)
X, Y = synth.batch(w)
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
r = Run(w.dims, "MSE", w.lr, rows=256); r.assign(Ws, bs)
gW, gb, _ = r.gradients(Xd, Yd); l1 = r.step(Xd, Yd); W1, b1 = r.read(); r.close()
s = SimRun(w.dims, "MSE", w.lr, rows=256, world=1); s.assign(Ws, bs)
sgW, sgb = s.gradients(0, Xd, Yd); l2 = s.step([Xd], [Yd]); W2, b2 = s.read(0); s.close()
print("loss plain", l1, "sim1", l2)
for l in range(3):
    cmp(f"dW{l+1} plain vs sim1", gW[l], sgW[l]); cmp(f"W{l+1} plain vs sim1", W1[l], W2[l])
mg = build_mlp(w.dims, "MSE", w.lr)
ref = train_step(mg, Ws, bs, X, Y, 1, "TRUNC16")
print("oracle loss", ref["loss"])
for l in range(3):
    cmp(f"W{l+1} plain vs oracle", W1[l], ref["W"][l])

# 2. sim world 2, TRUNC16 p2p, C2
for ex, p2p in (("TRUNC16", 1), ("FP32", 0)):
    s = SimRun(w.dims, "MSE", w.lr, rows=128, world=2, exchange=ex, p2p=p2p); s.assign(Ws, bs)
    Xs = [Xd[:128].contiguous(), Xd[128:].contiguous()]; Ys = [Yd[:128].contiguous(), Yd[128:].contiguous()]
    g0 = s.gradients(0, Xs[0], Ys[0]); g1 = s.gradients(1, Xs[1], Ys[1])
    r0 = Run(w.dims, "MSE", w.lr, rows=128); r0.assign(Ws, bs); p0 = r0.gradients(Xs[0], Ys[0]); r0.close()
    for l in range(3):
        cmp(f"[{ex}] rank0 dW{l+1} sim vs plain", g0[0][l], p0[0][l]); cmp(f"[{ex}] rank0 db{l+1}", g0[1][l], p0[1][l])
    losses = s.step(Xs, Ys)
    ref = train_step(mg, Ws, bs, X, Y, 2, ex)
    print(ex, "losses", losses, "oracle", ref["loss"])
    Wg, bg = s.read(0)
    for l in range(3):
        cmp(f"[{ex}] W{l+1} vs oracle", Wg[l], ref["W"][l]); cmp(f"[{ex}] b{l+1} vs oracle", bg[l], ref["b"][l])
    s.close()

# 3. MP exact world 2
X, Y, Ws, bs, lr = synth.exact_regime()
dims = (X.shape[1],) + tuple(W.shape[1] for W in Ws)
s = SimRun(dims, "MSE", lr, rows=X.shape[0], world=2, model_parallel=1); s.assign(Ws, bs)
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
losses = s.step([Xd, Xd], [Yd, Yd])
mp = train_step_model_parallel(build_mlp(dims, "MSE", lr), Ws, bs, X, Y, 2)
print("mp losses", losses, "oracle", mp["loss"])
for l in range(3):
    owner = (l * 2) // 3
    Wg, bg = s.read(owner)
    cmp(f"MP W{l+1} (owner {owner})", Wg[l], mp["W"][l]); cmp(f"MP b{l+1}", bg[l], mp["b"][l])
    d = np.argwhere(Wg[l].view(np.uint32) != mp["W"][l].view(np.uint32))[:5]
    for i, j in d:
        print("   ", i, j, Wg[l][i, j], mp["W"][l][i, j], Ws[l][i, j])
s.close()
# the same through real single-session N=1 to compare
r = Run(dims, "MSE", lr, rows=X.shape[0]); r.assign(Ws, bs); r.step(Xd, Yd); Wn, bn = r.read(); r.close()
for l in range(3):
    cmp(f"N1 W{l+1} vs MP oracle", Wn[l], mp["W"][l])
