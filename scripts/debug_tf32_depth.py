"""Where does 3xTF32 error grow?  Forward activations per layer vs the oracle,
for a few depths/widths (diagnostic only)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from dflow_harness import Run, normwise  # noqa: E402
from oracle.mlp import build_mlp, forward  # noqa: E402
import synth  # noqa: E402


def probe(dims, rows=256, precision="3xtf32"):
    w = synth.Workload("probe", tuple(dims), rows, "MSE", 0.25, "he", precision)
    Ws, bs = synth.init_params(w)
    X, Y = synth.batch(w)
    run = Run(dims, "MSE", 0.25, rows=rows, precision=precision)
    run.assign(Ws, bs)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    mg = build_mlp(dims, "MSE", 0.25)
    ref = forward(mg, Ws, bs, X, Y, fetch=mg.acts + [mg.cost])
    out = []
    for l, rid in enumerate(run.mlp.relus):
        a = run.forward(Xd, Yd, fetch=rid)
        r = ref[mg.acts[l]]
        out.append((l + 1, normwise(a, r), float(np.abs(r).max()), float((r > 0).mean())))
    c = run.forward(Xd, Yd)
    print(precision, dims[:3], "... L =", len(dims) - 1, "loss gpu", float(c[0]), "oracle", float(ref[mg.cost]))
    for t in out:
        print("   layer %2d  act err %.3e  max|a| %.3e  frac>0 %.3f" % t)
    run.close()


if __name__ == "__main__":
    probe((4096,) * 5)
    probe((4096,) * 17)
    probe((1024,) * 17)
    probe((4096,) * 5, precision="bf16")
