"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no matmul, no relu, no loss, no
codec, no update).  It only draws random numbers and describes workload shapes,
so that the oracle (``oracle/``) and the CUDA path (``paper_1603_04467_b200``)
can be fed identical inputs without sharing any code of the method.

Recipe (SURVEY.md §8(d) "Concrete synthetic inputs"):
every array comes from ``np.random.default_rng(SeedSequence([1603, stream]))``
with stream ids 0 = X, 1 = Y, 10+l = W_l, 100+l = b_l, 1000+step = per-step
batch.  X ~ U[0,1) (non-negative, MNIST-pixel-like, reading A11), Y ~ U[0,1)
dense targets (reading A2), W_l He-uniform U(+-sqrt(6/in)), b_l ~ U(+-0.1);
config 1 follows PAPER.md:102-103 (Fig. 1): W ~ U[-1,1), b = 0.
"""
from .inputs import *  # noqa: F401,F403
