"""Independent pins for two oracle/cache.py branches that round 1 left unpinned, and for
the message record the GPU's byte-exact message test compares against.

* follow mode (the oracle takes recorded send decisions): the override
  must replace the Alg. 2 L4/L15 predicate and nothing else —
  pinned by (a) the recorded masks and counts equal the supplied ones, (b) all-true
  masks make every replica send, so a cache without quantisation holds the exact
  replica sum Σ_i z_{i,u} (the plain definition of the gather), (c) all-false
  masks leave every boundary row at its previous synced value.
* quantise-only (reading R14 with B > 0; "Quantify only"): every replica sends
  its full value, quantised (§5).  Pinned against the exact replica sum by
  the quantiser's error bound (clamped top codes err ≤ (hi−lo)/2^B, R15):
  |b_u − Σ_i z_{i,u}| ≤ Σ_mirrors (hi−lo)/2^B + (scatter hi−lo)/2^B, plus fp32 rounding.
* message record (O10): dequantising the recorded gather codes and adding the
  master's own value reproduces the aggregate a (Alg. 2 L11-L19).
"""
import numpy as np
import pytest

from oracle.cache import SyncMode, SyncState, sync
from oracle.partition import PartitionCfg, partition
from oracle.quant import dequantize, dequantize_f32
from synth import small_random_graph


def _plan(p, seed=5, n=300, m=1100):
    d = small_random_graph(n, m, (4, 3), seed=seed)
    return partition(d.n, d.eu, d.ev, PartitionCfg(p=p))


def _exact(plan, X):
    tot = np.zeros((plan.n, X[0].shape[1]))
    for pp, x in zip(plan.parts, X):
        np.add.at(tot, pp.local2global, np.asarray(x, np.float64))
    return tot


def _boundary_rows(pp):
    return np.arange(pp.n_bmaster + pp.n_mirror)


def _drift(rng, X, frac=0.4):
    out = []
    for x in X:
        y = x.copy()
        rows = rng.random(x.shape[0]) < frac
        y[rows] += rng.standard_normal((int(rows.sum()), x.shape[1])) * 0.3
        out.append(y)
    return out


@pytest.mark.parametrize("p", [2, 4])
def test_follow_overrides_the_predicate_only(p):
    plan = _plan(p, seed=11 + p)
    rng = np.random.default_rng(p)
    F = 6
    st = SyncState(plan, F)
    X = [rng.standard_normal((pp.n_local, F)) for pp in plan.parts]
    for it in range(4):
        gm = {i: rng.random(pp.n_mirror) < 0.5 for i, pp in enumerate(plan.parts)}
        fm = {j: rng.random(pp.n_bmaster) < 0.5 for j, pp in enumerate(plan.parts)}
        s_before = [s.copy() for s in st.s_mir]
        sm_before = [s.copy() for s in st.s_mas]
        out, c = sync(plan, st, [x.copy() for x in X], 0.05, SyncMode(cache=True, quant_bits=0),
                      follow={"gather": gm, "master": fm})
        assert c.gather_sent == sum(int(m.sum()) for m in gm.values())
        assert c.master_fired == sum(int(m.sum()) for m in fm.values())
        for i, pp in enumerate(plan.parts):
            assert np.array_equal(c.gather_mask[i], gm[i])
            assert np.array_equal(c.master_fired_mask[i], fm[i])
            z_m = X[i][pp.n_bmaster:pp.n_bmaster + pp.n_mirror]
            # Alg. 2 L6 for senders, untouched snapshot otherwise
            assert np.array_equal(st.s_mir[i][gm[i]], z_m[gm[i]])
            assert np.array_equal(st.s_mir[i][~gm[i]], s_before[i][~gm[i]])
            assert np.array_equal(st.s_mas[i][fm[i]], X[i][:pp.n_bmaster][fm[i]])
            assert np.array_equal(st.s_mas[i][~fm[i]], sm_before[i][~fm[i]])
            # a master is active iff it fired or received a message (Alg. 2 L12, L18)
            recv = np.zeros(pp.n_bmaster, bool)
            for s_, q in enumerate(plan.parts):
                if s_ == i:
                    continue
                lo_r, hi_r = q.mirror_off[i], q.mirror_off[i + 1]
                recv[pp.halo_master[s_][gm[s_][lo_r:hi_r]]] = True
            assert np.array_equal(c.active_mask[i], recv | fm[i])
        X = _drift(rng, X)


@pytest.mark.parametrize("p", [2, 3])
def test_follow_all_true_holds_the_exact_replica_sum(p):
    """ε = 0.5 would skip most rows; forcing every send must give Σ_i z_{i,u} (fp64)."""
    plan = _plan(p, seed=21 + p)
    rng = np.random.default_rng(7)
    F = 5
    st = SyncState(plan, F)
    X = [rng.standard_normal((pp.n_local, F)) for pp in plan.parts]
    allt = {"gather": {i: np.ones(pp.n_mirror, bool) for i, pp in enumerate(plan.parts)},
            "master": {j: np.ones(pp.n_bmaster, bool) for j, pp in enumerate(plan.parts)}}
    for it in range(5):
        out, c = sync(plan, st, [x.copy() for x in X], 0.5, SyncMode(cache=True, quant_bits=0),
                      follow=allt)
        tot = _exact(plan, X)
        for pp, o in zip(plan.parts, out):
            rows = _boundary_rows(pp)
            ref = tot[pp.local2global[rows]]
            assert np.abs(o[rows] - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
        X = _drift(rng, X)


def test_follow_all_false_keeps_every_boundary_row():
    plan = _plan(3, seed=31)
    rng = np.random.default_rng(8)
    F = 4
    st = SyncState(plan, F)
    X = [rng.standard_normal((pp.n_local, F)) for pp in plan.parts]
    first, _ = sync(plan, st, [x.copy() for x in X], 0.0, SyncMode(cache=True, quant_bits=8))
    allf = {"gather": {i: np.zeros(pp.n_mirror, bool) for i, pp in enumerate(plan.parts)},
            "master": {j: np.zeros(pp.n_bmaster, bool) for j, pp in enumerate(plan.parts)}}
    X2 = _drift(rng, X, frac=1.0)
    out, c = sync(plan, st, [x.copy() for x in X2], 0.0, SyncMode(cache=True, quant_bits=8),
                  follow=allf)
    assert c.gather_sent == 0 and c.master_fired == 0 and c.scatter_msgs == 0 and c.active == 0
    for pp, o, f in zip(plan.parts, out, first):
        rows = _boundary_rows(pp)
        assert np.array_equal(o[rows], f[rows])


def _vertex_of_gather(plan, i, j, pos):
    pp = plan.parts[i]
    return pp.local2global[pp.n_bmaster + pp.mirror_off[j] + pos]


def _vertex_of_scatter(plan, j, i, pos):
    pp = plan.parts[j]
    return pp.local2global[pp.halo_master[i][pos]]


@pytest.mark.parametrize("B", [4, 8, 16])
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_quantise_only_error_bound_against_the_exact_sum(B, dt):
    plan = _plan(4, seed=41)
    rng = np.random.default_rng(B)
    F = 7
    st = SyncState(plan, F, dt)
    M = sum(pp.n_mirror for pp in plan.parts)
    for it in range(3):
        X = [rng.standard_normal((pp.n_local, F)).astype(dt) for pp in plan.parts]
        out, c = sync(plan, st, [x.copy() for x in X], 0.0, SyncMode(cache=False, quant_bits=B, dtype=dt))
        assert c.gather_sent == M and c.scatter_msgs == M      # R14: every replica sends
        tot = _exact(plan, X)
        bound = np.zeros(plan.n)
        mag = np.zeros(plan.n)
        for (i, j), (pos, q, lo, hi) in c.gather_msgs.items():
            assert q.min() >= 0 and q.max() <= 2 ** B - 1
            v = _vertex_of_gather(plan, i, j, pos)
            np.add.at(bound, v, (hi.astype(np.float64) - lo) / 2.0 ** B)
            np.maximum.at(mag, v, np.maximum(np.abs(lo), np.abs(hi)))
        seen = set()
        for (j, i), (pos, q, lo, hi) in c.scatter_msgs_rec.items():
            v = _vertex_of_scatter(plan, j, i, pos)
            for vv, lo_, hi_ in zip(v, lo, hi):
                if vv not in seen:             # one scatter quantisation per vertex (R12)
                    seen.add(vv)
                    bound[vv] += (float(hi_) - float(lo_)) / 2.0 ** B
                    mag[vv] = max(mag[vv], abs(float(lo_)), abs(float(hi_)))
        slack = 0.0 if dt == np.float64 else 16 * np.finfo(np.float32).eps
        views = {}
        for pp, o in zip(plan.parts, out):
            rows = _boundary_rows(pp)
            g = pp.local2global[rows]
            err = np.abs(o[rows].astype(np.float64) - tot[g]).max(axis=1)
            lim = bound[g] * (1 + 1e-9) + slack * (mag[g] + np.abs(tot[g]).max(axis=1)) * 8 + 1e-12
            assert (err <= lim).all(), float((err - lim).max())
            for gg, row in zip(g, o[rows]):
                if gg in views:                # replica coherence (P-C3)
                    assert np.array_equal(views[gg], row)
                views[gg] = row


@pytest.mark.parametrize("B", [0, 8])
def test_recorded_gather_messages_rebuild_the_aggregate(B):
    plan = _plan(3, seed=51)
    rng = np.random.default_rng(3)
    F = 5
    st = SyncState(plan, F)
    X = [rng.standard_normal((pp.n_local, F)) for pp in plan.parts]
    out, c = sync(plan, st, [x.copy() for x in X], 0.0, SyncMode(cache=True, quant_bits=B))
    for j, pp in enumerate(plan.parts):
        a = np.zeros((pp.n_bmaster, F))
        for s_ in range(plan.p):
            if s_ == j:
                continue
            pos, q, lo, hi = c.gather_msgs[(s_, j)]
            assert np.all(np.diff(pos) > 0)
            assert len(pos) == 0 or pos[-1] < plan.parts[s_].mirror_off[j + 1] - plan.parts[s_].mirror_off[j]
            pay = dequantize(q, lo, hi, B) if B else q
            a[pp.halo_master[s_][pos]] += pay
        a += X[j][:pp.n_bmaster]               # first sync: every master fires with s = 0
        assert np.abs(a - st.a[j]).max() <= 1e-12


def test_recorded_scatter_codes_rebuild_the_views_fp32():
    """fp32 replay: after the first sync (b = 0) the view of every mirror is deq(its scatter
    codes) bitwise (R12), and the scatter positions index the halo list of that mirror part."""
    plan = _plan(3, seed=61)
    rng = np.random.default_rng(4)
    F = 9
    st = SyncState(plan, F, np.float32)
    X = [rng.standard_normal((pp.n_local, F)).astype(np.float32) for pp in plan.parts]
    _, c = sync(plan, st, [x.copy() for x in X], 0.0, SyncMode(cache=True, quant_bits=8, dtype=np.float32))
    nrec = 0
    for (j, i), (pos, q, lo, hi) in c.scatter_msgs_rec.items():
        mirror = plan.parts[i]
        rows = mirror.mirror_off[j] + pos
        assert np.array_equal(st.b_mir[i][rows], dequantize_f32(q, lo, hi, 8))
        # the mirror row at that slab position is the same vertex as the master's halo entry
        assert np.array_equal(mirror.local2global[mirror.n_bmaster + rows],
                              _vertex_of_scatter(plan, j, i, pos))
        nrec += len(pos)
    assert nrec == c.scatter_msgs


@pytest.mark.parametrize("eps", [0.0, 0.05, 0.3])
@pytest.mark.parametrize("B,dt", [(8, np.float64), (0, np.float64), (8, np.float32), (16, np.float64)])
def test_full_staleness_bound_every_sync(eps, B, dt):
    """P-C4 in full (Lemma-2 style), vertex by vertex after every sync of a drifting
    run: ‖b_u − Σ_i z_{i,u}‖∞ ≤ Σ_mirrors e_i + e_master + e_scat, with e = ε‖s‖∞ for a replica
    that did not send / fire, (hi − lo)/2^B for a quantised mirror sender, 0 for an fp32 sender
    or a fired master (its own Δ never travels, R13), and e_scat = (hi − lo)/2^B of u's most
    recent scatter delta (0 without quantisation, R12)."""
    import copy
    plan = _plan(3, seed=91)
    rng = np.random.default_rng(int(eps * 100) + B)
    F = 6
    st = SyncState(plan, F, dt)
    X = [rng.standard_normal((pp.n_local, F)).astype(dt) for pp in plan.parts]
    e_scat = np.zeros(plan.n)
    for it in range(10):
        pre = copy.deepcopy(st)
        out, c = sync(plan, st, [x.copy() for x in X], eps, SyncMode(cache=True, quant_bits=B, dtype=dt))
        tot = _exact(plan, X)
        bound = np.zeros(plan.n)
        mag = np.zeros(plan.n)
        for i, pp in enumerate(plan.parts):
            Bi, Mi = pp.n_bmaster, pp.n_mirror
            g_m = pp.local2global[Bi:Bi + Mi]
            s_pre = pre.s_mir[i].astype(np.float64)
            sent = c.gather_mask[i]
            e = eps * np.abs(s_pre).max(axis=1) if Mi else np.zeros(0)
            if B:
                for (src, dst), (pos, q, lo, hi) in c.gather_msgs.items():
                    if src == i:
                        rows = pp.mirror_off[dst] + pos
                        e[rows] = (hi.astype(np.float64) - lo) / 2.0 ** B
            else:
                e[sent] = 0.0
            np.add.at(bound, g_m, e)
            g_b = pp.local2global[:Bi]
            em = eps * np.abs(pre.s_mas[i].astype(np.float64)).max(axis=1) if Bi else np.zeros(0)
            em[c.master_fired_mask[i]] = 0.0
            np.add.at(bound, g_b, em)
            np.maximum.at(mag, pp.local2global, np.abs(X[i].astype(np.float64)).max(axis=1))
        if B:
            for (j, i), (pos, q, lo, hi) in c.scatter_msgs_rec.items():
                e_scat[_vertex_of_scatter(plan, j, i, pos)] = (hi.astype(np.float64) - lo) / 2.0 ** B
        slack = 1e-12 if dt == np.float64 else 64 * np.finfo(np.float32).eps
        for pp, o in zip(plan.parts, out):
            rows = _boundary_rows(pp)
            g = pp.local2global[rows]
            err = np.abs(o[rows].astype(np.float64) - tot[g]).max(axis=1)
            lim = bound[g] + e_scat[g] + slack * (1 + mag[g] * 4)
            assert (err <= lim * (1 + 1e-9)).all(), (it, float((err - lim).max()))
        X = _drift(rng, X)
        X = [x.astype(dt) for x in X]
