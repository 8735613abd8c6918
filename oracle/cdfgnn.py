"""Alg. 1 — one CDFGNN training iteration over all partitions (oracle steps O4-O8).

P:L200-225 (Alg. 1), simulated sequentially over the p parts (BSP):
  forward  l = 1..L:  Z̈_i = Â_i H_i W (eq. 1) → sync → H_i = σ(Z_i)
  loss     on master vertices only → δ̈_i^(L)
  backward l = L..1:  sync δ̈ → δ_i; S_i = Â_i δ_i;
                      ∇W_i = H_iᵀ S_i (eq. 5, reading R6);
                      δ̈_i^(l-1) = (S_i Wᵀ) ⊙ σ'(Z_i^(l-1))
  update   W ← W − η Σ_i ∇W_i or Adam; ε controller

Â_i is the part's local CSR with global-degree weights (R2); the
sum over parts is taken in ascending part order.  Reading R8: updating W after
the whole backward pass equals Alg. 1's in-loop update (δ̈^(l-1) is computed
with the old W^(l-1) and lower layers never read it).
Pins: tests/test_oracle_cdfgnn.py (p ∈ {1,2,4} with ε = 0 and no quantisation ≡
the unpartitioned gcn.train_step; dyadic fixtures bitwise).
"""
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.sparse as sp

from . import gcn
from .cache import SyncMode, SyncState, sync
from .eps import EpsController, EpsParams
from .optim import Adam, sgd


@dataclass
class TrainCfg:
    cache: bool = True
    quant_bits: int = 8
    eps0: float = 0.01
    adaptive: bool = True
    eps_params: EpsParams = field(default_factory=EpsParams)
    optimizer: str = "sgd"        # "sgd" (parity default) | "adam"
    lr: float = 0.01
    dtype: type = np.float64
    snapshot_literal: bool = False
    scatter_full: bool = False


class PartitionedGCN:
    def __init__(self, plan, X, y, train, W, cfg: TrainCfg):
        self.plan = plan
        self.cfg = cfg
        dt = cfg.dtype
        self.dt = dt
        self.L = len(W)
        self.dims = [W[0].shape[0]] + [w.shape[1] for w in W]
        self.W = [np.asarray(w, dtype=dt).copy() for w in W]
        self.n_train = int(np.asarray(train).sum())
        self.parts = []
        for pp in plan.parts:
            val = pp.val64 if dt == np.float64 else pp.val32
            A = sp.csr_matrix((val.astype(dt), pp.colidx, pp.rowptr),
                              shape=(pp.n_local, pp.n_local))
            l2g = pp.local2global
            self.parts.append(dict(
                A=A, X=np.asarray(X, dtype=dt)[l2g], y=np.asarray(y)[l2g],
                # the loss is computed on master vertices only
                train=np.asarray(train)[l2g] & pp.is_master_row()))
        mode = SyncMode(cache=cfg.cache, quant_bits=cfg.quant_bits, dtype=dt,
                        snapshot_literal=cfg.snapshot_literal, scatter_full=cfg.scatter_full)
        self.mode = mode
        self.fwd_state = [SyncState(plan, self.dims[l], dt) for l in range(1, self.L + 1)]
        self.bwd_state = [SyncState(plan, self.dims[l], dt) for l in range(1, self.L + 1)]
        self.eps_ctl = EpsController(cfg.eps0, cfg.eps_params, cfg.adaptive)
        self.adam = Adam([w.shape for w in self.W], lr=cfg.lr, dtype=dt) \
            if cfg.optimizer == "adam" else None
        self.epoch_no = 0

    def forward(self, eps, counters, follow=None):
        p = self.plan.p
        H = [[prt["X"]] for prt in self.parts]
        Z = [[] for _ in range(p)]
        for l in range(1, self.L + 1):
            Zdd = [prt["A"] @ (H[i][l - 1] @ self.W[l - 1]) for i, prt in enumerate(self.parts)]
            Zs, c = sync(self.plan, self.fwd_state[l - 1], Zdd, eps, self.mode,
                         follow=None if follow is None else follow.get(("fwd", l)))
            counters.append(("fwd", l, c))
            for i in range(p):
                Z[i].append(Zs[i])
                H[i].append(gcn.relu(Zs[i]) if l < self.L else Zs[i])
        return Z, H

    def epoch(self, follow=None):
        """One iteration of Alg. 1.  Returns a dict of loss, acc, ε used and sync counters.

        ``follow`` (trajectory follow mode): {("fwd" | "bwd", l): {"gather":
        {i: bool[M_i]}, "master": {j: bool[B_j]}}} — the cache-test decisions of those syncs
        are replaced by recorded ones (e.g. the GPU's), so a near-threshold flip caused by
        rounding cannot make the two trajectories diverge; a missing key runs the test."""
        p = self.plan.p
        eps = self.eps_ctl.eps if self.cfg.cache else 0.0
        counters = []
        Z, H = self.forward(eps, counters, follow)
        # loss on masters ∩ train, mean over the global train count (R7)
        loss = 0.0
        correct = 0
        ddot = []
        for i, prt in enumerate(self.parts):
            li, di, ci = gcn.loss_grad(Z[i][-1], prt["y"], prt["train"], self.n_train)
            loss += li
            correct += ci
            ddot.append(di)
        dW = [np.zeros_like(w) for w in self.W]
        for l in range(self.L, 0, -1):
            delta, c = sync(self.plan, self.bwd_state[l - 1], ddot, eps, self.mode,
                            follow=None if follow is None else follow.get(("bwd", l)))
            counters.append(("bwd", l, c))
            nxt = []
            for i, prt in enumerate(self.parts):
                S = prt["A"] @ delta[i]
                dW[l - 1] = dW[l - 1] + H[i][l - 1].T @ S       # ascending part order
                if l > 1:
                    nxt.append((S @ self.W[l - 1].T) * (Z[i][l - 2] > 0))
            ddot = nxt
        if self.adam is not None:
            self.W = self.adam.step(self.W, dW)
        else:
            self.W = [sgd(w, g, self.cfg.lr) for w, g in zip(self.W, dW)]
        acc = correct / self.n_train
        self.eps_ctl.step(acc)
        self.epoch_no += 1
        return dict(loss=loss, acc=acc, correct=correct, eps=eps, dW=dW, counters=counters,
                    logits=[z[-1] for z in Z])
