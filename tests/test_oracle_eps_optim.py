"""Pins for oracle/eps.py and oracle/optim.py."""
import numpy as np
import pytest
import torch

from oracle.eps import EpsController, EpsParams, update_eps, update_mean
from oracle.optim import Adam, sgd
from tests.conftest import golden


def test_defaults_match_paper():
    g = golden("eps_defaults.json")
    p = EpsParams()
    for k in ("mu1", "mu2", "nu1", "nu2", "xi", "lam1", "lam2"):
        assert getattr(p, k) == g[k]
    assert update_mean(1.0, 0.0) == g["ema_old"] and update_mean(0.0, 1.0) == g["ema_new"]


def test_spec_examples(spec_examples):
    for ex in spec_examples["update_epsilon"]:
        assert abs(update_eps(ex["eps"], ex["acc"], ex["mean_acc"]) - ex["new_eps"]) < 1e-15


def test_band_leaves_eps_unchanged():
    assert update_eps(0.05, 0.6, 0.6) == 0.05
    assert update_eps(0.05, 0.6 + 0.019, 0.6) == 0.05
    assert update_eps(0.05, 0.6 - 0.0009, 0.6) == 0.05


def test_clamp_reading_R17():
    bare = EpsParams(clamp=False)
    # without the clamp the equation leaves [ν2, ν1] (boundary examples of reading R17)
    assert abs(update_eps(0.299, 0.0, 1.0, bare) - 0.309) < 1e-15
    assert abs(update_eps(0.0011, 1.0, 0.0, bare) - 0.00099) < 1e-15
    assert update_eps(0.299, 0.0, 1.0) == 0.3
    assert update_eps(0.0011, 1.0, 0.0) == 0.001


def test_range_invariant_random_sequences():
    rng = np.random.default_rng(0)
    for _ in range(200):
        c = EpsController(0.01)
        for acc in rng.random(60):
            e = c.step(float(acc))
            assert 0.001 <= e <= 0.3


def test_first_epoch_sets_mean_without_change():
    c = EpsController(0.02)
    assert c.step(0.3) == 0.02 and c.mean_acc == 0.3


def test_sgd_example(spec_examples):
    ex = spec_examples["sgd"]
    np.testing.assert_allclose(sgd(np.array(ex["W"]), np.array(ex["g"]), ex["lr"]), ex["result"],
                               rtol=0, atol=1e-15)


def test_adam_vs_torch():
    rng = np.random.default_rng(1)
    W0 = [rng.standard_normal((5, 4)), rng.standard_normal((4, 3))]
    opt = Adam([w.shape for w in W0], lr=0.01)
    tw = [torch.tensor(w, dtype=torch.float64, requires_grad=True) for w in W0]
    topt = torch.optim.Adam(tw, lr=0.01, betas=(0.9, 0.999), eps=1e-8)
    W = [w.copy() for w in W0]
    for step in range(5):
        G = [rng.standard_normal(w.shape) for w in W0]
        W = opt.step(W, G)
        for t, g in zip(tw, G):
            t.grad = torch.tensor(g, dtype=torch.float64)
        topt.step()
        for a, t in zip(W, tw):
            np.testing.assert_allclose(a, t.detach().numpy(), rtol=1e-13, atol=1e-15)
