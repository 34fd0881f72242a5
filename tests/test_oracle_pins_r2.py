"""More pins of the oracle (CPU only): the transposed-operand MatMul gradient rules and the
AddN summation EXECUTED through the executor (finite differences, P7), AddN against exact
rational sums, and reading A9's two roundings against hand-checked values.

PAPER.md §4.1 :494-518 (gradient functions per op, partials of a fan-out summed),
SPEC.md:369 (MatMul gradients), :380 (AddN), PAPER.md:262-268 (ApplyGradientDescent)."""
import itertools
from fractions import Fraction
import os

import numpy as np
import pytest

from oracle import graph as G
from oracle import kernels as K
from oracle.executor import execute
from synth import rng

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
H = 1e-5


def _fd_pin(g, cost, wrt, variables, feeds, relu_inputs):
    """Central differences in pure f64 of every entry of every `wrt` endpoint (Variables and
    fed Placeholders) against the executed gradient graph; max relative error."""
    grads = g.gradients(cost, wrt)
    ana = execute(g, feeds, grads, dict(variables), mode="f64")
    # the function is piecewise smooth: every Relu input must be away from the kink
    z = execute(g, feeds, relu_inputs, dict(variables), mode="f64")
    assert all(np.min(np.abs(v)) > 100 * H for v in z.values()), "inputs near the Relu kink"

    def cost_at():
        return float(execute(g, feeds, [cost], dict(variables), mode="f64")[cost])
    worst = 0.0
    for name, gname in zip(wrt, grads):
        arr = variables[name] if name in variables else feeds[name]
        for idx in np.ndindex(arr.shape):
            saved = arr[idx]
            arr[idx] = saved + H
            up = cost_at()
            arr[idx] = saved - H
            dn = cost_at()
            arr[idx] = saved
            fd = (up - dn) / (2 * H)
            an = float(ana[gname][idx])
            worst = max(worst, abs(fd - an) if abs(an) < 1e-8 else abs(fd - an) / abs(an))
    return worst


def _transpose_case(ta, tb, seed):
    """x (or its transpose) and W (or its transpose) through MatMul(ta, tb) -> BiasAdd -> Relu
    -> MatMul -> Relu -> MSE: both gradient rules of the transposed MatMul are on the path."""
    B, n_in, n_hid, n_out = 3, 4, 5, 2
    r = rng(80000 + seed)
    g = G.Graph()
    A = g.placeholder("A", "f32", (n_in, B) if ta else (B, n_in))
    W = g.variable("W", "f32", (n_hid, n_in) if tb else (n_in, n_hid))
    b = g.variable("b", "f32", (n_hid,))
    W2 = g.variable("W2", "f32", (n_hid, n_out))
    y = g.placeholder("y", "f32", (B, n_out))
    z1 = g.add("z1", g.matmul("m1", A, W, ta, tb), b)
    z2 = g.matmul("m2", g.relu("r1", z1), W2)
    C = g.loss("C", "MSE", g.relu("r2", z2), y)
    variables = {"W": r.uniform(-1, 1, g.by_name[W].shape), "b": r.uniform(-0.5, 0.5, n_hid),
                 "W2": r.uniform(-1, 1, (n_hid, n_out))}
    feeds = {"A": r.uniform(0, 1, g.by_name[A].shape), "y": r.uniform(0, 1, (B, n_out))}
    return g, C, [W, b, W2, A], variables, feeds, [z1, z2]


@pytest.mark.parametrize("ta,tb", list(itertools.product((0, 1), (0, 1))))
def test_p7_transposed_matmul_gradient_rules(ta, tb):
    # resample until every pre-activation is away from the kink and both layers carry signal
    for seed in range(200):
        g, C, wrt, variables, feeds, zs = _transpose_case(ta, tb, seed)
        z = execute(g, feeds, zs, dict(variables), mode="f64")
        if all(np.min(np.abs(v)) > 100 * H for v in z.values()) and all(np.any(v > 0) for v in z.values()):
            break
    names = {n.name: n for n in g.nodes}
    assert names["m1"].attrs == {"transpose_a": ta, "transpose_b": tb}
    assert _fd_pin(g, C, wrt, variables, feeds, zs) < 1e-6


def test_p7_fanout_addn_executed():
    # h and W fan out, so dW and dh are AddN nodes — executed here, and
    # finite differences catch a dropped or doubled partial
    for seed in range(200):
        r = rng(81000 + seed)
        g = G.Graph()
        W = g.variable("W", "f32", (3, 3))
        x = g.placeholder("x", "f32", (-1, 3))
        y = g.placeholder("y", "f32", (-1, 3))
        z1 = g.matmul("m1", x, W)
        h = g.relu("h", z1)
        s = g.add("s", g.matmul("m2", h, W), h)
        C = g.loss("C", "MSE", g.relu("r", s), y)
        variables = {"W": r.uniform(-1, 1, (3, 3))}
        feeds = {"x": r.uniform(0, 1, (4, 3)), "y": r.uniform(0, 1, (4, 3))}
        z = execute(g, feeds, [z1, s], dict(variables), mode="f64")
        if all(np.min(np.abs(v)) > 100 * H for v in z.values()) and all(np.mean(v > 0) > 0.3 for v in z.values()):
            break
    assert _fd_pin(g, C, [W, x], variables, feeds, [z1, s]) < 1e-6
    ops = {n.name: n.op for n in g.nodes}
    assert ops["grad/W/sum"] == "AddN" and ops["grad/h/sum"] == "AddN"


def test_add_n_exact_rational_sum():
    # AddN of three partials equals the exact sum (fractions), and in f32 mode
    # the exact sum rounded once to float32
    r = rng(82000)
    parts = [r.uniform(-1, 1, (5, 4)) for _ in range(3)]
    out64 = K.add_n(parts, "f64")
    out32 = K.add_n(parts, "f32")
    for idx in np.ndindex(5, 4):
        exact = sum(Fraction(float(p[idx])) for p in parts)
        assert abs(Fraction(float(out64[idx])) - exact) <= abs(exact) * Fraction(1, 2 ** 50)
        assert out32[idx] == np.float32(float(exact))
    # a dropped partial is caught
    assert not np.allclose(K.add_n(parts[:2], "f64"), out64)


def _rne32(q: Fraction) -> float:
    """Round an exact rational to the nearest binary32 (ties to even), normal range."""
    if q == 0:
        return 0.0
    s = -1 if q < 0 else 1
    q = abs(q)
    e = 0
    while q >= 2:
        q /= 2
        e += 1
    while q < 1:
        q *= 2
        e -= 1
    m = q * 2 ** 23
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return s * float(Fraction(fl) * Fraction(2) ** (e - 23))


def _f(h):
    return np.array([int(h, 16)], np.uint32).view(np.float32)[0]


def test_a9_two_roundings_golden():
    rows = [ln.split() for ln in open(os.path.join(GOLDEN, "sgd_two_roundings.txt")) if ln.strip() and ln[0] != "#"]
    assert len(rows) >= 3
    for w_h, lr_h, g_h, two_h, fma_h in rows:
        W, lr, g, two, fma = map(_f, (w_h, lr_h, g_h, two_h, fma_h))
        # the fixture itself, from exact rational arithmetic
        assert two == np.float32(_rne32(Fraction(float(W)) - Fraction(_rne32(Fraction(float(lr)) * Fraction(float(g))))))
        assert fma == np.float32(_rne32(Fraction(float(W)) - Fraction(float(lr)) * Fraction(float(g))))
        assert two != fma
        # the oracle's ApplyGradientDescent follows reading A9 (two roundings), not a fused op
        got = K.apply_gradient_descent(np.array([W], np.float32), float(lr), np.array([g], np.float32), "f32")[0]
        assert got.view(np.uint32) == two.view(np.uint32)
