"""Pins for oracle/cdfgnn.py (Alg. 1): partitioned ≡ unpartitioned in exact mode."""
import numpy as np
import pytest

from oracle import gcn
from oracle.cdfgnn import PartitionedGCN, TrainCfg
from oracle.graph import normalized_adjacency
from oracle.optim import sgd
from oracle.partition import PartitionCfg, partition
from synth import dyadic_fixture, small_random_graph


@pytest.mark.parametrize("p", [1, 2, 4])
@pytest.mark.parametrize("cache", [True, False])
def test_exact_mode_matches_full_batch(p, cache):
    d = small_random_graph(250, 900, (6, 8, 4), seed=40 + p)
    plan = partition(d.n, d.eu, d.ev, PartitionCfg(p=p))
    cfg = TrainCfg(cache=cache, quant_bits=0, eps0=0.0, adaptive=False, lr=0.5)
    model = PartitionedGCN(plan, d.X, d.y, d.train, d.W, cfg)
    A = normalized_adjacency(d.n, d.eu, d.ev)
    W = [w.astype(np.float64) for w in d.W]
    for ep in range(3):
        loss, correct, dW = gcn.train_step(A, d.X.astype(np.float64), W, d.y, d.train)
        r = model.epoch()
        assert abs(r["loss"] - loss) <= 1e-12 * max(1.0, abs(loss))
        assert r["correct"] == correct
        for a, b in zip(r["dW"], dW):
            assert np.abs(a - b).max() <= 1e-10 * max(1e-30, np.abs(b).max())
        W = [sgd(w, g, 0.5) for w, g in zip(W, dW)]
        if p == 1:
            assert all(c.remote == 0 for _, _, c in r["counters"])


@pytest.mark.parametrize("p", [2, 3])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_dyadic_fixture_bitwise(p, dtype):
    """P-C1: on a dyadic fixture every partial sum is exact, so any summation order and the
    delta-accumulated cache aggregate give identical bits."""
    d = dyadic_fixture(n=64, r=4, dims=(16, 8, 4))
    plan = partition(d.n, d.eu, d.ev, PartitionCfg(p=p))
    A = normalized_adjacency(d.n, d.eu, d.ev)
    Zref, _ = gcn.forward(A, d.X.astype(np.float64), [w.astype(np.float64) for w in d.W])
    for cache in (True, False):
        cfg = TrainCfg(cache=cache, quant_bits=0, eps0=0.0, adaptive=False, dtype=dtype)
        model = PartitionedGCN(plan, d.X, d.y, d.train, d.W, cfg)
        cnt = []
        Z, H = model.forward(0.0, cnt)
        for pp in plan.parts:
            for l in range(len(d.W)):
                assert np.array_equal(Z[pp.part][l].astype(np.float64),
                                      Zref[l][pp.local2global])


def test_cached_int8_training_tracks_exact():
    d = small_random_graph(400, 2000, (16, 16, 5), seed=77)
    plan = partition(d.n, d.eu, d.ev, PartitionCfg(p=3))
    exact = PartitionedGCN(plan, d.X, d.y, d.train, d.W,
                           TrainCfg(cache=False, quant_bits=0, optimizer="adam"))
    cached = PartitionedGCN(plan, d.X, d.y, d.train, d.W,
                            TrainCfg(cache=True, quant_bits=8, eps0=0.01, adaptive=True,
                                     optimizer="adam"))
    le, lc, sent = [], [], 0
    for ep in range(25):
        le.append(exact.epoch()["loss"])
        r = cached.epoch()
        lc.append(r["loss"])
        sent += sum(c.remote for _, _, c in r["counters"])
    base = sum(c.baseline for _, _, c in r["counters"]) * 25
    assert lc[-1] < 0.5 * lc[0]
    assert abs(lc[-1] - le[-1]) < 0.05 * max(1.0, le[-1])
    assert sent < base
