"""Pins for the oracle kernels and gradient builder: P5, P6, P7, P8.  CPU only."""
import itertools

import numpy as np

from oracle import kernels as K
from oracle.mlp import build_mlp, replica_gradients
from synth import finite_difference_mlp, rng


def _triple_loop(A, B):
    m, k = len(A), len(A[0])
    n = len(B[0])
    return [[sum(A[i][p] * B[p][j] for p in range(k)) for j in range(n)] for i in range(m)]


def test_p5_matmul_worked_example():
    # [[1,2],[3,4]] . [[1],[1]] -> [[3],[7]]
    out = K.matmul(np.array([[1., 2.], [3., 4.]]), np.array([[1.], [1.]]), 0, 0, "f64")
    assert out.tolist() == [[3.0], [7.0]]


def test_p5_matmul_brute_force_all_transposes():
    g = rng(123)
    for (m, k, n), ta, tb in itertools.product([(1, 1, 1), (3, 5, 2), (7, 4, 9)], (0, 1), (0, 1)):
        A = g.uniform(-1, 1, (k, m) if ta else (m, k))
        B = g.uniform(-1, 1, (n, k) if tb else (k, n))
        ref = _triple_loop((A.T if ta else A).tolist(), (B.T if tb else B).tolist())
        assert np.allclose(K.matmul(A, B, ta, tb, "f64"), ref, rtol=0, atol=1e-14)


def test_p6_relu_and_relu_grad():
    # SPEC.md:233 and :368
    assert K.relu(np.array([-1., 0., 2.]), "f64").tolist() == [0., 0., 2.]
    assert K.relu_grad(np.array([5., 7.]), K.relu(np.array([-1., 2.]), "f64"), "f64").tolist() == [0., 7.]


def _loss_of(mg, Ws, bs, X, Y):
    from oracle.mlp import forward
    return float(forward(mg, Ws, bs, X, Y, mode="f64")[mg.cost])


def _fd_check(loss_kind):
    X, Y, Ws, bs = finite_difference_mlp()
    dims = (3, 5, 4, 2)
    h = 1e-5
    # resample until every pre-activation is away from the kink (|z| > 10h)
    s = 0
    while True:
        X, Y, Ws, bs = finite_difference_mlp(seed_stream=3 + s)
        a, ok = X, True
        for W, b in zip(Ws, bs):
            z = a @ W + b
            ok &= bool(np.all(np.abs(z) > 10 * h))
            a = np.maximum(z, 0)
        if ok and np.any(a > 0):
            break
        s += 1
    mg = build_mlp(dims, loss_kind, 0.1, with_dx=True)
    Yf = Y if loss_kind == "MSE" else None
    ana = replica_gradients(mg, Ws, bs, X, Yf, mode="f64")
    worst = 0.0
    params = [("W", l) for l in range(3)] + [("b", l) for l in range(3)]
    for kind, l in params:
        arr = (Ws if kind == "W" else bs)[l]
        name = (mg.weights if kind == "W" else mg.biases)[l]
        for idx in np.ndindex(arr.shape):
            saved = arr[idx]
            arr[idx] = saved + h
            up = _loss_of(mg, Ws, bs, X, Yf)
            arr[idx] = saved - h
            dn = _loss_of(mg, Ws, bs, X, Yf)
            arr[idx] = saved
            fd = (up - dn) / (2 * h)
            an = float(ana[name][idx])
            err = abs(fd - an) if abs(an) < 1e-8 else abs(fd - an) / abs(an)
            worst = max(worst, err)
    for idx in np.ndindex(X.shape):  # dx (Fig.5 returns dx)
        saved = X[idx]
        X[idx] = saved + h
        up = _loss_of(mg, Ws, bs, X, Yf)
        X[idx] = saved - h
        dn = _loss_of(mg, Ws, bs, X, Yf)
        X[idx] = saved
        fd = (up - dn) / (2 * h)
        an = float(ana["dx"][idx])
        err = abs(fd - an) if abs(an) < 1e-8 else abs(fd - an) / abs(an)
        worst = max(worst, err)
    return worst


def test_p7_finite_differences_mse():
    # central differences in f64, h = 1e-5, max rel err < 1e-6
    assert _fd_check("MSE") < 1e-6


def test_p7_finite_differences_sum():
    assert _fd_check("SUM") < 1e-6


def test_p8_closed_form_sum_one_layer():
    # SUM loss, one layer: db_j = (1/B) sum_b 1[z_bj > 0];  dW = (1/B) X^T 1[Z > 0]
    g = rng(5)
    X = g.uniform(0, 1, (6, 4))
    W = g.uniform(-1, 1, (4, 3))
    b = g.uniform(-0.5, 0.5, 3)
    mg = build_mlp((4, 3), "SUM", 0.1)
    out = replica_gradients(mg, [W], [b], X, None, mode="f64")
    M = (X @ W + b > 0).astype(np.float64)
    assert np.allclose(out["b"], M.sum(0) / 6, atol=1e-15)
    assert np.allclose(out["W"], X.T @ M / 6, atol=1e-15)


def test_p8_closed_form_least_squares_linear_regime():
    # All z > 0: MSE gradient is the textbook least-squares one, here scaled by
    # 1/(B*out): dW = X^T (XW + b - Y) / (B*out),  db = sum_rows(XW + b - Y) / (B*out)
    g = rng(6)
    X = g.uniform(0, 1, (5, 3))
    W = g.uniform(0.1, 1, (3, 2))
    b = g.uniform(0.1, 0.5, 2)
    Y = g.uniform(0, 1, (5, 2))
    mg = build_mlp((3, 2), "MSE", 0.1)
    out = replica_gradients(mg, [W], [b], X, Y, mode="f64")
    R = X @ W + b - Y
    assert np.allclose(out["W"], X.T @ R / 10, atol=1e-15)
    assert np.allclose(out["b"], R.sum(0) / 10, atol=1e-15)
    assert np.isclose(float(out["C"]), np.sum(R * R) / 20, rtol=1e-14)
