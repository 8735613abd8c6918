"""Pins for oracle/cache.py (Alg. 2; §3.2)."""
import copy

import numpy as np
import pytest

from oracle.cache import SyncMode, SyncState, _test, pack_ref, sync
from oracle.partition import PartitionCfg, partition
from synth import small_random_graph


def _plan(p, seed=5, n=300, m=1100):
    d = small_random_graph(n, m, (4, 3), seed=seed)
    return partition(d.n, d.eu, d.ev, PartitionCfg(p=p))


def _exact(plan, X):
    """Σ over replicas of each vertex's local partial (global id space)."""
    tot = np.zeros((plan.n, X[0].shape[1]))
    for pp, x in zip(plan.parts, X):
        np.add.at(tot, pp.local2global, x)
    return tot


def test_spec_should_send(spec_examples):
    ex = spec_examples["should_send"]
    s = np.array([ex["snapshot"]])
    z = np.array([ex["current"]])
    assert bool(_test(z - s, s, ex["eps"], np.float64)[0]) == ex["send"]
    # zero snapshot: threshold 0 -> any change is sent; no change -> not sent
    assert bool(_test(z, np.zeros_like(z), 0.3, np.float64)[0])
    assert not bool(_test(z - z, z, 0.0, np.float64)[0])


def test_spec_gather_scatter_three_replicas(spec_examples):
    ex = spec_examples["gather_scatter"]
    plan = _plan(3)
    # a vertex replicated on all three parts
    u = next(x for x in range(plan.n) if bin(int(plan.replicas[x])).count("1") == 3)
    X = [np.zeros((pp.n_local, 1)) for pp in plan.parts]
    for pp, val in zip(plan.parts, ex["locals"]):
        X[pp.part][list(pp.local2global).index(u), 0] = val
    for mode in (SyncMode(cache=False), SyncMode(cache=True)):
        st = SyncState(plan, 1)
        out, _ = sync(plan, st, X, 0.0, mode)
        for pp in plan.parts:
            assert out[pp.part][list(pp.local2global).index(u), 0] == ex["result"]


def test_spec_master_pass_single_add(spec_examples):
    ex = spec_examples["master_pass"]
    plan = _plan(2)
    st = SyncState(plan, 1)
    j = 0
    pp = plan.parts[j]
    r = int(pp.halo_master[1][0])                 # a boundary master of part 0 with a mirror on 1
    st.a[j][r, 0] = ex["aggregate"][0]
    st.s_mas[j][:] = 0
    st.b_mas[j][r, 0] = ex["aggregate"][0]
    X = [np.zeros((q.n_local, 1)) for q in plan.parts]
    # mirror on part 1 sends Δ = [1] (snapshot 0 -> value 1)
    q1 = plan.parts[1]
    pos = 0
    X[1][q1.n_bmaster + q1.mirror_off[0] + pos, 0] = ex["delta"][0]
    out, c = sync(plan, st, X, 0.0, SyncMode(cache=True))
    assert st.a[j][r, 0] == ex["result"][0]
    assert c.active_mask[j][r]


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("cache", [True, False])
def test_exact_mode_equals_replica_sum(p, cache):
    plan = _plan(p, seed=p)
    rng = np.random.default_rng(p)
    st = SyncState(plan, 5)
    for it in range(4):
        X = [rng.standard_normal((pp.n_local, 5)) for pp in plan.parts]
        out, c = sync(plan, st, X, 0.0, SyncMode(cache=cache, quant_bits=0))
        tot = _exact(plan, X)
        for pp, o in zip(plan.parts, out):
            np.testing.assert_allclose(o, tot[pp.local2global], rtol=1e-12, atol=1e-12)
        assert c.baseline == 2 * sum(pp.n_mirror for pp in plan.parts)


def _drift_run(plan, eps, B, dtype, iters=12, seed=0, frac=0.3):
    rng = np.random.default_rng(seed)
    F = 6
    st = SyncState(plan, F, dtype)
    X = [rng.standard_normal((pp.n_local, F)).astype(dtype) for pp in plan.parts]
    hist = []
    for it in range(iters):
        pre = copy.deepcopy(st)
        out, c = sync(plan, st, X, eps, SyncMode(cache=True, quant_bits=B, dtype=dtype))
        hist.append((pre, copy.deepcopy(st), [x.copy() for x in X], out, c))
        X = [x + (rng.random((x.shape[0], 1)) < frac) * 0.1 * rng.standard_normal(x.shape)
             for x in X]
        X = [x.astype(dtype) for x in X]
    return hist


@pytest.mark.parametrize("eps", [0.0, 0.05, 0.3])
@pytest.mark.parametrize("B,dtype", [(8, np.float64), (8, np.float32), (0, np.float64),
                                     (4, np.float32)])
def test_coherence_and_staleness_invariants(eps, B, dtype):
    plan = _plan(3, seed=8)
    for pre, post, X, out, c in _drift_run(plan, eps, B, dtype):
        # P-C3 replica coherence: every replica of u holds the same bits
        val = {}
        for pp, o in zip(plan.parts, out):
            g = pp.local2global
            rows = np.arange(pp.n_bmaster + pp.n_mirror)
            for r in rows:
                key = int(g[r])
                if key in val:
                    assert np.array_equal(val[key], o[r])
                else:
                    val[key] = o[r].copy()
        for pp in plan.parts:
            i = pp.part
            Bi, Mi = pp.n_bmaster, pp.n_mirror
            z_m = X[i][Bi:Bi + Mi].astype(np.float64)
            s_post = post.s_mir[i].astype(np.float64)
            s_pre = pre.s_mir[i].astype(np.float64)
            sent = c.gather_mask[i]
            # predicate negation: skipped replicas are within ε of their snapshot
            dd = np.abs(z_m - s_pre).max(axis=1)
            thr = eps * np.abs(s_pre).max(axis=1)
            assert np.all(dd[~sent] <= thr[~sent] * (1 + 1e-6) + 1e-30)
            assert np.all(dd[sent] > thr[sent] * (1 - 1e-6))
            # quantised senders: residual after the snapshot update ≤ (hi − lo)/2^B (+ rounding)
            if B and sent.any():
                d = (z_m - s_pre)[sent]
                rngw = d.max(axis=1) - d.min(axis=1)
                res = np.abs(z_m[sent] - s_post[sent]).max(axis=1)
                tol = 4 * np.spacing(np.abs(z_m[sent]).max(axis=1).astype(dtype)).astype(np.float64)
                assert np.all(res <= rngw / 2 ** B + tol)
        # a = Σ_i s_i over the vertex's replicas (aggregate bookkeeping, reading R11)
        agg, snaps = {}, {}
        for pp in plan.parts:
            i = pp.part
            g = pp.local2global
            for r in range(pp.n_bmaster):
                agg[int(g[r])] = post.a[i][r].astype(np.float64)
                snaps.setdefault(int(g[r]), []).append(post.s_mas[i][r].astype(np.float64))
            for r in range(pp.n_mirror):
                snaps.setdefault(int(g[pp.n_bmaster + r]), []).append(
                    post.s_mir[i][r].astype(np.float64))
        for key, a in agg.items():
            scale = max(1.0, np.abs(a).max())
            assert np.abs(a - sum(snaps[key])).max() <= \
                (1e-10 if dtype == np.float64 else 5e-5) * scale


def test_send_set_monotone_in_eps():
    plan = _plan(3, seed=9)
    hist = _drift_run(plan, 0.05, 8, np.float64, iters=5)
    pre, _, X, _, _ = hist[-1]
    prev = None
    for eps in [0.0, 0.01, 0.05, 0.1, 0.3, 1.0]:
        st = copy.deepcopy(pre)
        _, c = sync(plan, st, X, eps, SyncMode(cache=True, quant_bits=8))
        cur = np.concatenate([c.gather_mask[i] for i in range(plan.p)])
        if prev is not None:
            assert np.all(cur <= prev)
        prev = cur


def test_first_sync_sends_every_nonzero_row():
    plan = _plan(2, seed=10)
    rng = np.random.default_rng(0)
    X = [rng.standard_normal((pp.n_local, 4)) for pp in plan.parts]
    zero_rows = 0
    for pp in plan.parts:
        rows = pp.n_bmaster + np.arange(0, pp.n_mirror, 3)
        X[pp.part][rows] = 0
        zero_rows += len(rows)
    st = SyncState(plan, 4)
    _, c = sync(plan, st, X, 0.3, SyncMode(cache=True, quant_bits=8))
    assert c.gather_sent == sum(pp.n_mirror for pp in plan.parts) - zero_rows


def test_counts_brute_force():
    plan = _plan(4, seed=12)
    for pre, post, X, out, c in _drift_run(plan, 0.05, 8, np.float64, iters=6, seed=3):
        assert c.gather_sent == sum(int(c.gather_mask[i].sum()) for i in range(plan.p))
        # every active master sends one message per mirror replica
        nmir = {}
        for (i, j), lst in plan.halo.items():
            for g in lst.tolist():
                nmir[(j, g)] = nmir.get((j, g), 0) + 1
        sc = 0
        for j in range(plan.p):
            g = plan.parts[j].local2global
            for r in np.flatnonzero(c.active_mask[j]):
                sc += nmir[(j, int(g[r]))]
        assert c.scatter_msgs == sc
        assert c.remote == c.gather_sent + c.scatter_msgs
        assert c.bytes == (c.gather_sent + c.scatter_msgs) * (6 + 12)


def test_pack_ref_matches_sync_fp32():
    plan = _plan(2, seed=13)
    hist = _drift_run(plan, 0.05, 8, np.float32, iters=4, seed=4)
    pre, post, X, out, c = hist[-1]
    for pp in plan.parts:
        i = pp.part
        z = X[i][pp.n_bmaster:pp.n_bmaster + pp.n_mirror]
        send, q, lo, hi, s_new = pack_ref(z, pre.s_mir[i], 0.05, 8)
        assert np.array_equal(send, c.gather_mask[i])
        assert np.array_equal(s_new, post.s_mir[i])
