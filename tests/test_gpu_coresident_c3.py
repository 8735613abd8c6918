"""The bench's partitioned single-GPU configuration at FULL size: C3 (Reddit-shaped,
configs[2]) as 4 co-resident parts on one GPU — the `coresident_p4` key of bench.py, which
times the whole method (cache test, quantise + pack, exchange, apply) on the driver's
1-GPU box.

* exact mode (ε = 0, fp32 messages, cache on): one cdfgnn_epoch; H^(1) = ReLU(Â X W^(0))
  on sampled vertices against the plain definition evaluated row by row (oracle
  gcn.rows_forward, eq. 1; P-C1: partitioned ≡ unpartitioned), every replica of a
  sampled vertex bit-identical (P-C3), the masters' logits Â H^(1) W^(1) from the GPU's own
  assembled H^(1), and loss / correct count from the masters' logits (R7, R16).
  Tolerance 1e-4 row-normwise (SURVEY §8(c4), 3xTF32 GEMMs).
* cache + int8 at full size: the first layer-1 synchronisation of seeded 256-wide
  partials — replica coherence and the quantiser's error bound against the exact replica
  sum (the oracle's Python partitioner does not reach C3's size, so the bit-exact replay of
  the same kernels runs on C1/C2 and small graphs in test_gpu_halo.py).
"""
import numpy as np
import pytest

import paper_2408_00232_b200 as cg
from oracle import gcn
from oracle.graph import normalized_adjacency
from paper_2408_00232_b200.runtime import Run
from synth import get_config
from synth.cache import cached_dataset
from tests.gpu_util import require_gpu, rownorm_err, ws_view

pytestmark = pytest.mark.gpu


def test_C3_coresident_p4_exact_epoch_sampled_parity():
    torch = require_gpu()
    ds = cached_dataset(get_config("C3"))
    F0, F1, C = ds.dims
    run = Run(ds, 4, cache=True, quant_bits=0, eps0=0.0, adaptive=False, optimizer="adam", lr=0.01,
              static_inputs=True)
    W_old = [w.astype(np.float64) for w in run.weights()]
    st = run.epoch()
    # the GPU's H^(1) and logits per part, by global id
    H1 = np.zeros((ds.n, F1))
    owner = np.full(ds.n, -1)
    logits = np.zeros((ds.n, C))
    reps = {}
    rng = np.random.default_rng(2408)
    A = normalized_adjacency(ds.n, ds.eu, ds.ev)
    deg = np.diff(A.indptr)
    sample = np.unique(np.concatenate([[int(np.argmax(deg)), int(np.argmin(deg))],
                                       rng.choice(ds.n, 40, replace=False)]))
    for t, v in enumerate(run.views):
        ptr, rows, ld = cg.act_view(run.ctx, t, 1)
        h = ws_view(run.workspace, ptr, rows, ld)[:, :F1]
        ptr, rows, ldc = cg.act_view(run.ctx, t, 2)
        z = ws_view(run.workspace, ptr, rows, ldc)[:, :C]
        g = v["local2global"]
        B, M = v["n_bmaster"], v["n_mirror"]
        own = np.r_[np.arange(B), np.arange(B + M, v["n_local"])]        # masters (R21)
        H1[g[own]] = h[own]
        logits[g[own]] = z[own]
        owner[g[own]] = t
        pos = {int(x): i for i, x in enumerate(g)}
        for u in sample:
            if int(u) in pos:
                reps.setdefault(int(u), []).append(h[pos[int(u)]])
    assert (owner >= 0).all(), "every vertex has exactly one master"
    for u, rs in reps.items():                        # replica coherence (P-C3)
        for r in rs[1:]:
            assert np.array_equal(r.view(np.uint32), rs[0].view(np.uint32)), u
    X = ds.X.astype(np.float64)
    ref_h1 = np.maximum(gcn.rows_forward(A, X, W_old[0], sample), 0)
    assert rownorm_err(H1[sample], ref_h1) <= 1e-4
    ref_lg = gcn.rows_forward(A, H1, W_old[1], sample)
    assert rownorm_err(logits[sample], ref_lg) <= 1e-4
    loss, _, correct = gcn.loss_grad(logits, ds.y, ds.train)
    assert abs(st["loss"] - loss) <= 1e-5 * max(1.0, abs(loss))
    assert st["correct"] == correct and st["total"] == int(ds.train.sum())
    # exact mode, first epoch: every boundary replica sends (snapshots start at 0)
    assert st["fwd"][0]["gather_sent"] > 0 and st["fwd"][0]["scatter_msgs"] > 0
    run.close()


def test_C3_coresident_p4_int8_first_sync_invariants():
    """Full size, cache + int8, first layer-1 synchronisation (snapshots 0, ε = 0): every
    replica of every boundary vertex holds bit-identical rows (P-C3), and each differs from
    the exact replica sum Σ_i z_{i,u} by at most the quantiser's bound (P:L602-604 with the
    clamped top code, R15): Σ_mirrors rng(z_i)/2^8 for the gather plus rng(a)/2^8 for the
    scatter, rng(a) ≤ Σ_i rng(z_i) + the gather error (P-C4 at the first sync)."""
    torch = require_gpu()
    ds = cached_dataset(get_config("C3"))
    p = 4
    plan = cg.partition(ds.n, ds.eu, ds.ev, p)
    views = [cg.plan_part(plan, i) for i in range(p)]
    dims = ds.dims
    cfg = cg.cfg_default(dims, cache_on=1, quant_bits=8)
    ws = torch.empty(cg.workspace_size(plan, list(range(p)), cfg), dtype=torch.uint8, device="cuda")
    ctx = cg.init(plan, list(range(p)), 0, 1, cfg, 0, ws)
    F = dims[1]
    rng = np.random.default_rng(5)
    Xs = [rng.standard_normal((v["n_local"], F), dtype=np.float32) for v in views]
    dev = [torch.from_numpy(x).cuda() for x in Xs]               # F = 256 = ld
    gst = cg.halo_exchange(ctx, 1, 0, dev, F, np.float32(0.0), stats=True)
    M = sum(v["n_mirror"] for v in views)
    assert gst["gather_sent"] == M                               # s = 0: every non-zero row sends
    exact = np.zeros((ds.n, F))
    rsum = np.zeros(ds.n)
    gerr = np.zeros(ds.n)
    for v, x in zip(views, Xs):
        g = v["local2global"][:v["n_bmaster"] + v["n_mirror"]]
        xb = x[:len(g)].astype(np.float64)
        np.add.at(exact, g, xb)
        rng_row = xb.max(axis=1) - xb.min(axis=1)
        np.add.at(rsum, g, rng_row)
        mir = np.zeros(len(g), bool)
        mir[v["n_bmaster"]:] = True
        np.add.at(gerr, g[mir], rng_row[mir] / 256.0)
    bound = gerr + (rsum + 2 * gerr) / 256.0
    probe = set(rng.choice(ds.n, 20000, replace=False).tolist())
    seen = {}
    worst = 0.0
    ncoh = 0
    for v, d in zip(views, dev):
        nb = v["n_bmaster"] + v["n_mirror"]
        out = d[:nb].cpu().numpy()
        g = v["local2global"][:nb]
        err = np.abs(out.astype(np.float64) - exact[g]).max(axis=1)
        slack = 64 * np.finfo(np.float32).eps * (np.abs(exact[g]).max(axis=1) + rsum[g])
        worst = max(worst, float((err / (bound[g] + slack)).max()))
        for k in np.flatnonzero(np.isin(g, list(probe))):
            gg = int(g[k])
            if gg in seen:                                       # replica coherence (P-C3)
                assert np.array_equal(seen[gg].view(np.uint32), out[k].view(np.uint32)), gg
                ncoh += 1
            seen[gg] = out[k]
    assert worst <= 1.0, worst
    assert ncoh > 1000
    ctx.close()
