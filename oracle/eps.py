"""Adaptive cache threshold ε (oracle step O8).

P:L387-393 (eq. ε):
    ε = min(λ1 ε, ε + ξ)   if acc < mean_acc − μ1 and ε < ν1
        max(λ2 ε, ε − ξ)   if acc > mean_acc + μ2 and ε > ν2
        ε                  otherwise
P:L395-397: applied after each iteration; mean_acc = 0.8 mean_acc + 0.2 acc.
P:L399: μ1 = .001, μ2 = .02, ν1 = .3, ν2 = .001, ξ = .01, λ1 = 1.05, λ2 = .9.
Readings: R17 the equation is implemented literally with the
defaults list (ξ = 0.01, not the prose's 0.02 at P:L406) and then clamped to
[ν2, ν1] ("limit the value range of ε to [ν2, ν1]"); ``clamp=False``
gives the bare equation.  R18 ε₀ = 0.01, mean_acc₀ = the first epoch's acc with
no ε change at epoch 1, ε updated before mean_acc, one ε for all layers/dirs.
Pins: tests/test_oracle_eps.py (SPEC S:L412-413 values, range invariant).
"""
from dataclasses import dataclass


@dataclass
class EpsParams:
    mu1: float = 0.001
    mu2: float = 0.02
    nu1: float = 0.3
    nu2: float = 0.001
    xi: float = 0.01
    lam1: float = 1.05
    lam2: float = 0.9
    clamp: bool = True


def update_eps(eps: float, acc: float, mean_acc: float, prm: EpsParams = EpsParams()) -> float:
    if acc < mean_acc - prm.mu1 and eps < prm.nu1:
        eps = min(prm.lam1 * eps, eps + prm.xi)
    elif acc > mean_acc + prm.mu2 and eps > prm.nu2:
        eps = max(prm.lam2 * eps, eps - prm.xi)
    if prm.clamp:
        eps = min(max(eps, prm.nu2), prm.nu1)
    return eps


def update_mean(mean_acc: float, acc: float) -> float:
    return 0.8 * mean_acc + 0.2 * acc


class EpsController:
    def __init__(self, eps0: float = 0.01, prm: EpsParams = EpsParams(), adaptive: bool = True):
        self.eps = eps0
        self.mean_acc = None
        self.prm = prm
        self.adaptive = adaptive

    def step(self, acc: float) -> float:
        """Call after an epoch with that epoch's train accuracy; returns the next ε."""
        if self.mean_acc is None:
            self.mean_acc = acc
            return self.eps
        if self.adaptive:
            self.eps = update_eps(self.eps, acc, self.mean_acc, self.prm)
        self.mean_acc = update_mean(self.mean_acc, acc)
        return self.eps
