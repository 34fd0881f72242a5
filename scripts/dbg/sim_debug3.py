import os, sys, ctypes as C
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1603_04467_b200 as D
from dflow_harness import SimRun, Run, normwise
import synth

def same(a, b):
    return bool(np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32)))

w = synth.with_batch(synth.C2, 256)
Ws, bs = synth.init_params(w)
X, Y = synth.batch(w)
Xs = [torch.from_numpy(X[:128]).cuda(), torch.from_numpy(X[128:]).cuda()]
Ys = [torch.from_numpy(Y[:128]).cuda(), torch.from_numpy(Y[128:]).cuda()]
p = Run(w.dims, "MSE", w.lr, rows=128); p.assign(Ws, bs)
pf = [p.forward(Xs[0], Ys[0], fetch=p.mlp.relus[l]) for l in range(3)]
pl = p.forward(Xs[0], Ys[0])
p.close()

def sim_forward(s, r, X, Y, fetch):
    torch.cuda.synchronize()
    ids = [s.mlp.x, s.mlp.y]
    if fetch == s.mlp.cost:
        out = torch.empty(1, dtype=torch.float32, device="cuda")
    else:
        l = s.mlp.relus.index(fetch)
        out = torch.empty((X.shape[0], s.dims[l + 1]), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    D.check(D.dflow_forward(s.sessions[r], 2, D.node_array(ids), D.ptr_array([X.data_ptr(), Y.data_ptr()]),
                            D.i64_array([X.stride(0), Y.stride(0)]), X.shape[0], fetch, C.c_void_p(out.data_ptr()), s.stream))
    s.sync()
    return out.cpu().numpy()

for world, ex in ((1, "FP32"), (2, "FP32"), (2, "TRUNC16"), (4, "FP32")):
    rows = 256 // world if world > 1 else 128
    s = SimRun(w.dims, "MSE", w.lr, rows=128, world=world, exchange=ex)
    s.assign(Ws, bs)
    for rep in range(3):
        sf = [sim_forward(s, 0, Xs[0], Ys[0], s.mlp.relus[l]) for l in range(3)]
        sl = sim_forward(s, 0, Xs[0], Ys[0], s.mlp.cost)
        print(world, ex, rep, "A_l == plain", [same(a, b) for a, b in zip(sf, pf)],
              ["%.2e" % normwise(a, b) for a, b in zip(sf, pf)], "loss", sl, pl, flush=True)
    s.close()
