"""Unpartitioned full-batch GCN — the plain definition (oracle step O3).

P:L236-240 (eqs. 1-2): Z^(l) = Â H^(l-1) W^(l-1),  H^(l) = σ(Z^(l)).
P:L692: cross-entropy loss.  Readings: R3 σ = ReLU on hidden
layers, relu'(0) = 0, identity at layer L with the softmax inside the loss;
R4 no bias / dropout; R5 evaluated as Â(HW); R6 the backward is the standard
adjoint with Â symmetric: S = Â δ, ∇W = Hᵀ S, δ^(l-1) = (S Wᵀ) ⊙ 𝟙[Z^(l-1) > 0];
R7 the loss is the MEAN over the global train set; R16 argmax ties go to the
lowest class.
Pins: tests/test_oracle_gcn.py (dense brute force on tiny graphs, torch CPU
autograd in fp64, central finite differences, uniform logits ⇒ ln C).
"""
import numpy as np


def relu(x):
    return np.maximum(x, 0)


def forward(A, X, W):
    """Returns (Z list [Z^(1)..Z^(L)], H list [H^(0)..H^(L)]); H^(L) = Z^(L) (logits)."""
    L = len(W)
    H = [X]
    Z = []
    for l in range(1, L + 1):
        T = H[l - 1] @ W[l - 1]          # R5: Â (H W)
        Zl = A @ T                       # eq. (1)
        Z.append(Zl)
        H.append(relu(Zl) if l < L else Zl)   # eq. (2)
    return Z, H


def rows_forward(A, H, W, rows):
    """Z[v] = Σ_u Â[v,u] (H[u] W) for the listed rows only, one row at a time (eq. 1,
    P:L237) — the plain definition evaluated for sampled outputs of a full-size graph."""
    A = A.tocsr()
    out = np.zeros((len(rows), W.shape[1]))
    for i, v in enumerate(rows):
        lo, hi = A.indptr[v], A.indptr[v + 1]
        nb = A.indices[lo:hi]
        out[i] = A.data[lo:hi] @ (H[nb] @ W)
    return out


def log_softmax(z):
    mx = z.max(axis=1, keepdims=True)
    sh = z - mx
    return sh - np.log(np.exp(sh).sum(axis=1, keepdims=True))


def loss_grad(logits, y, train, n_train=None):
    """Mean cross-entropy over train rows (R7); δ^(L) = (softmax − onehot)/N_train on
    train rows, 0 elsewhere; correct = #(argmax == y) over train rows (R16)."""
    n_train = int(train.sum()) if n_train is None else n_train
    rows = np.flatnonzero(train)
    lsm = log_softmax(logits[rows])
    loss = -lsm[np.arange(len(rows)), y[rows]].sum() / n_train
    g = np.exp(lsm)
    g[np.arange(len(rows)), y[rows]] -= 1.0
    delta = np.zeros_like(logits)
    delta[rows] = g / n_train
    correct = int((np.argmax(logits[rows], axis=1) == y[rows]).sum())
    return loss, delta, correct


def backward(A, W, Z, H, delta_L):
    """Adjoint of forward (R6).  Returns dW list aligned with W."""
    L = len(W)
    dW = [None] * L
    delta = delta_L
    for l in range(L, 0, -1):
        S = A.T @ delta                  # Â symmetric: Âᵀ δ = Â δ
        dW[l - 1] = H[l - 1].T @ S
        if l > 1:
            delta = (S @ W[l - 1].T) * (Z[l - 2] > 0)
    return dW


def train_step(A, X, W, y, train):
    """One full-batch iteration on the whole graph: (loss, correct, dW)."""
    Z, H = forward(A, X, W)
    loss, dL, correct = loss_grad(Z[-1], y, train)
    return loss, correct, backward(A, W, Z, H, dL)
