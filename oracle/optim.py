"""Parameter update (oracle step O7).

P:L222 / P:L282: W ← W − η Σ_i ∇W L_i  (SGD, the parity default).
P:L692: "the Adam optimizer ... initial learning rate 0.01" — implemented with
PyTorch's update formula (β = (0.9, 0.999), eps = 1e-8, bias-corrected).
Pins: tests/test_oracle_optim.py (S:L329 SGD example; torch.optim.Adam in fp64).
"""
import numpy as np


def sgd(W, g, lr):
    return W - lr * g


class Adam:
    def __init__(self, shapes, lr=0.01, betas=(0.9, 0.999), eps=1e-8, dtype=np.float64):
        self.lr, self.b1, self.b2, self.eps = lr, betas[0], betas[1], eps
        self.m = [np.zeros(s, dtype=dtype) for s in shapes]
        self.v = [np.zeros(s, dtype=dtype) for s in shapes]
        self.t = 0

    def step(self, W, G):
        self.t += 1
        bc1 = 1.0 - self.b1 ** self.t
        bc2 = 1.0 - self.b2 ** self.t
        out = []
        for k, (w, g) in enumerate(zip(W, G)):
            self.m[k] = self.b1 * self.m[k] + (1.0 - self.b1) * g
            self.v[k] = self.b2 * self.v[k] + (1.0 - self.b2) * g * g
            denom = np.sqrt(self.v[k]) / np.sqrt(bc2) + self.eps
            out.append(w - (self.lr / bc1) * self.m[k] / denom)
        return out
