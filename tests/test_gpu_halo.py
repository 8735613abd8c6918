"""GPU halo exchange (cdfgnn_halo_exchange) vs the oracle's fp32 replay — bit-exact.

Given identical fp32 inputs the cache-test masks, quantised codes (through the
snapshots / aggregates / views they produce), counters and synced rows must be
bit-identical (BASELINE.json north_star; readings R11-R15)."""
import numpy as np
import pytest

import paper_2408_00232_b200 as cg
from oracle.cache import SyncMode, SyncState, sync
from oracle.partition import PartitionCfg, partition as opartition
from synth import get_config, make_dataset, small_random_graph
from tests.gpu_util import require_gpu, ws_view

pytestmark = pytest.mark.gpu


def _setup(torch, d, p, dims, cache, quant):
    plan = cg.partition(d.n, d.eu, d.ev, p)
    oplan = opartition(d.n, d.eu, d.ev, PartitionCfg(p=p))
    cfg = cg.cfg_default(dims, cache_on=int(cache), quant_bits=quant)
    parts = list(range(p))
    ws = torch.empty(cg.workspace_size(plan, parts, cfg), dtype=torch.uint8, device="cuda")
    ctx = cg.init(plan, parts, 0, 1, cfg, 0, ws)
    return plan, oplan, ctx, ws


def _run(torch, d, p, dims, l, cache, quant, eps, steps=5, seed=0):
    plan, oplan, ctx, ws = _setup(torch, d, p, dims, cache, quant)
    F = dims[l]
    ld = cg.ld_of(F)
    st = SyncState(oplan, F, np.float32)
    mode = SyncMode(cache=bool(cache), quant_bits=quant, dtype=np.float32)
    rng = np.random.default_rng(seed)
    Xs = [rng.standard_normal((pp.n_local, F)).astype(np.float32) for pp in oplan.parts]
    for step in range(steps):
        dev = []
        for x in Xs:
            xp = np.zeros((x.shape[0], ld), np.float32)
            xp[:, :F] = x
            dev.append(torch.from_numpy(xp).cuda())
        gst = cg.halo_exchange(ctx, l, 0, dev, ld, np.float32(eps), stats=True)
        out, cnt = sync(oplan, st, [x.copy() for x in Xs], eps, mode)
        for i, pp in enumerate(oplan.parts):
            g = dev[i].cpu().numpy()
            assert np.array_equal(g[:, :F].view(np.uint32), out[i].view(np.uint32)), \
                f"step {step} part {i}: synced rows differ"
            assert not g[:, F:].any()
            if cache:
                for which, ref in ((0, st.s_mir[i]), (1, st.b_mir[i]), (2, st.s_mas[i]),
                                   (3, st.a[i]), (4, st.b_mas[i])):
                    ptr, rows, ldc = cg.cache_view(ctx, i, l, 0, which)
                    v = ws_view(ws, ptr, rows, ldc)
                    assert np.array_equal(v[:, :F].view(np.uint32), ref.view(np.uint32)), \
                        f"step {step} part {i} cache table {which} differs"
                    assert not v[:, F:].any()
                pg, rg = cg.sync_flags(ctx, i, 0)
                gf = ws_view(ws, pg, rg, 1, np.uint8)[:, 0].astype(bool)
                assert np.array_equal(gf, cnt.gather_mask[i])
                pf, rf_ = cg.sync_flags(ctx, i, 1)
                assert np.array_equal(ws_view(ws, pf, rf_, 1, np.uint8)[:, 0].astype(bool),
                                      cnt.master_fired_mask[i])
            pa, ra = cg.sync_flags(ctx, i, 2)
            assert np.array_equal(ws_view(ws, pa, ra, 1, np.uint8)[:, 0].astype(bool),
                                  cnt.active_mask[i])
        assert gst["gather_sent"] == cnt.gather_sent
        assert gst["scatter_msgs"] == cnt.scatter_msgs
        assert gst["active"] == cnt.active
        if cache:
            assert gst["master_fired"] == cnt.master_fired
        assert gst["baseline"] == cnt.baseline
        # drift: a random 40% of rows change by a small amount
        Xs = [(x + (rng.random((x.shape[0], 1)) < 0.4) * 0.05 *
               rng.standard_normal(x.shape)).astype(np.float32) for x in Xs]
    ctx.close()


@pytest.mark.parametrize("cache,quant", [(1, 8), (1, 0), (0, 8), (0, 0)])
@pytest.mark.parametrize("eps", [0.0, 0.05])
@pytest.mark.parametrize("l", [1, 2])
def test_replay_bitexact_small(cache, quant, eps, l):
    torch = require_gpu()
    d = small_random_graph(900, 4000, (8, 20, 5), seed=31)
    _run(torch, d, 3, (8, 20, 5), l, cache, quant, eps)


@pytest.mark.parametrize("F", [7, 16, 41, 256, 300])
def test_replay_widths(F):
    torch = require_gpu()
    d = small_random_graph(1500, 9000, (4, F, 3), seed=5)
    _run(torch, d, 4, (4, F, 3), 1, 1, 8, 0.02, steps=4)


def test_replay_C1_two_parts():
    """configs[0]: Cora-shaped, 2 parts on 1 GPU, ε = 0, int8."""
    torch = require_gpu()
    d = make_dataset(get_config("C1"))
    _run(torch, d, 2, (1433, 16, 7), 1, 1, 8, 0.0, steps=6)
    _run(torch, d, 2, (1433, 16, 7), 2, 1, 8, 0.0, steps=6)


def test_replay_C2_two_parts():
    """configs[1] at full size, 2 parts on 1 GPU, hidden 256, cache + int8."""
    torch = require_gpu()
    d = make_dataset(get_config("C2"))
    _run(torch, d, 2, (128, 256, 256, 40), 1, 1, 8, 0.01, steps=3)
