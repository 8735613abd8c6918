"""Pins for oracle/gcn.py: dense brute force, torch autograd, finite differences."""
import math

import numpy as np
import torch

from oracle import gcn
from oracle.graph import normalized_adjacency
from synth import small_random_graph


def _dense_loops(A, H, W):
    n, k = H.shape
    f = W.shape[1]
    T = np.zeros((n, f))
    for i in range(n):
        for j in range(f):
            T[i, j] = sum(H[i, t] * W[t, j] for t in range(k))
    Z = np.zeros((n, f))
    for i in range(n):
        for j in range(f):
            Z[i, j] = sum(A[i, t] * T[t, j] for t in range(n))
    return Z


def test_forward_dense_brute_force():
    d = small_random_graph(24, 50, (5, 4, 3), seed=4)
    A = normalized_adjacency(d.n, d.eu, d.ev)
    X = d.X.astype(np.float64)
    W = [w.astype(np.float64) for w in d.W]
    Z, H = gcn.forward(A, X, W)
    Ad = A.toarray()
    Z1 = _dense_loops(Ad, X, W[0])
    np.testing.assert_allclose(Z[0], Z1, rtol=1e-12, atol=1e-12)
    Z2 = _dense_loops(Ad, np.maximum(Z1, 0), W[1])
    np.testing.assert_allclose(Z[1], Z2, rtol=1e-12, atol=1e-12)


def test_rows_forward_dense_brute_force():
    """oracle.gcn.rows_forward (sampled rows of eq. 1) vs explicit loops on the dense Â."""
    d = small_random_graph(30, 70, (6, 5, 3), seed=8)
    A = normalized_adjacency(d.n, d.eu, d.ev)
    X = d.X.astype(np.float64)
    W = d.W[0].astype(np.float64)
    rows = [0, 7, 29, 13, 7]
    got = gcn.rows_forward(A, X, W, rows)
    ref = _dense_loops(A.toarray(), X, W)[rows]
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def _torch_ref(A, X, W, y, train):
    At = torch.tensor(A.toarray(), dtype=torch.float64)
    Wt = [torch.tensor(w, dtype=torch.float64, requires_grad=True) for w in W]
    h = torch.tensor(X, dtype=torch.float64)
    for l, w in enumerate(Wt):
        z = At @ (h @ w)
        h = torch.relu(z) if l < len(Wt) - 1 else z
    rows = torch.tensor(np.flatnonzero(train))
    loss = torch.nn.functional.cross_entropy(h[rows], torch.tensor(y, dtype=torch.long)[rows])
    loss.backward()
    return loss.item(), [w.grad.numpy() for w in Wt]


def test_loss_and_grads_vs_torch_autograd():
    for seed, dims in [(1, (6, 5, 3)), (2, (7, 6, 5, 4))]:
        d = small_random_graph(60, 200, dims, seed=seed)
        A = normalized_adjacency(d.n, d.eu, d.ev)
        W = [w.astype(np.float64) for w in d.W]
        loss, correct, dW = gcn.train_step(A, d.X.astype(np.float64), W, d.y, d.train)
        tl, tg = _torch_ref(A, d.X.astype(np.float64), W, d.y, d.train)
        assert abs(loss - tl) <= 1e-12 * max(1, abs(tl))
        for a, b in zip(dW, tg):
            np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-13)


def test_central_finite_differences():
    d = small_random_graph(50, 140, (4, 5, 3), seed=12)
    A = normalized_adjacency(d.n, d.eu, d.ev)
    X = d.X.astype(np.float64)
    W = [w.astype(np.float64) for w in d.W]

    def L(Ws):
        Z, _ = gcn.forward(A, X, Ws)
        return gcn.loss_grad(Z[-1], d.y, d.train)[0]

    _, _, dW = gcn.train_step(A, X, W, d.y, d.train)
    h = 1e-6
    worst = 0.0
    for l in range(len(W)):
        for (i, j) in [(0, 0), (1, 2), (W[l].shape[0] - 1, W[l].shape[1] - 1)]:
            Wp = [w.copy() for w in W]; Wm = [w.copy() for w in W]
            Wp[l][i, j] += h; Wm[l][i, j] -= h
            fd = (L(Wp) - L(Wm)) / (2 * h)
            worst = max(worst, abs(fd - dW[l][i, j]) / max(abs(fd), 1e-8))
    assert worst <= 1e-4


def test_uniform_logits_give_ln_C(spec_examples):
    C = spec_examples["uniform_logits_loss"]["classes"]
    logits = np.zeros((10, C))
    y = np.arange(10) % C
    loss, delta, _ = gcn.loss_grad(logits, y, np.ones(10, bool))
    assert abs(loss - math.log(C)) < 1e-15
    np.testing.assert_allclose(delta.sum(axis=1), 0, atol=1e-16)


def test_argmax_ties_lowest_class():
    logits = np.array([[1.0, 1.0, 0.0], [0.0, 2.0, 2.0]])
    _, _, c = gcn.loss_grad(logits, np.array([0, 1]), np.ones(2, bool))
    assert c == 2
