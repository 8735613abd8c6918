"""GPU halo exchange (cdfgnn_halo_exchange) vs the oracle's fp32 replay — bit-exact.

Given identical fp32 inputs the cache-test masks, the messages themselves (positions,
lo/hi headers and B-bit codes, read from the message regions through cdfgnn_msg_view and
compared with the oracle's recorded messages), snapshots / aggregates / views, counters
and synced rows must be bit-identical (BASELINE.json north_star; readings R11-R15), for
both message layouts and B ∈ {0, 4, 8, 16}."""
import numpy as np
import pytest

import paper_2408_00232_b200 as cg
from oracle.cache import SyncMode, SyncState, sync
from oracle.partition import PartitionCfg, partition as opartition
from synth import get_config, make_dataset, small_random_graph
from tests.gpu_util import require_gpu, ws_view

pytestmark = pytest.mark.gpu


def _setup(torch, d, p, dims, cache, quant, layout=0):
    plan = cg.partition(d.n, d.eu, d.ev, p)
    oplan = opartition(d.n, d.eu, d.ev, PartitionCfg(p=p))
    cfg = cg.cfg_default(dims, cache_on=int(cache), quant_bits=quant, msg_layout=layout)
    parts = list(range(p))
    ws = torch.empty(cg.workspace_size(plan, parts, cfg), dtype=torch.uint8, device="cuda")
    ctx = cg.init(plan, parts, 0, 1, cfg, 0, ws)
    return plan, oplan, ctx, ws


def decode_rows(raw, F, B):
    """Code rows (uint8 [k, row_bytes]) -> int64 codes [k, F] and the padding part, per the
    layout include/cdfgnn.h documents for cfg.quant_bits; B = 0: fp32 payload rows."""
    raw = np.ascontiguousarray(raw)
    if B == 8:
        full = raw.astype(np.int64)
    elif B == 4:
        full = np.empty((raw.shape[0], 2 * raw.shape[1]), np.int64)
        full[:, 0::2] = raw & 0xF
        full[:, 1::2] = raw >> 4
    elif B == 16:
        full = raw.view(np.uint16).astype(np.int64)
    else:
        full = raw.view(np.float32)
    return full[:, :F], full[:, F:]


def read_messages(ws, view, F, B):
    """Messages of one (source, receiver) pair from cdfgnn_msg_view, sorted by halo-list
    position: (pos, codes or fp32 rows, lo, hi)."""
    cap, rb = view["capacity"], view["row_bytes"]
    if view["layout"] == 1:
        sb = view["slot_bytes"]
        raw = ws_view(ws, view["base"], cap, sb, np.uint8) if cap else np.zeros((0, sb), np.uint8)
        hdr = raw[:, :16].copy().view(np.uint32)
        pos = np.flatnonzero(hdr[:, 0] == view["stamp"])
        rows = raw[pos, 16:16 + rb]
        lo, hi = hdr[pos, 1].view(np.float32), hdr[pos, 2].view(np.float32)
    else:
        cnt = int(ws_view(ws, view["count"], 1, 1, np.int32)[0, 0]) if cap else 0
        assert 0 <= cnt <= cap
        hb = view["hdr_bytes"]
        hdr = ws_view(ws, view["base"], cnt, hb // 4, np.uint32) if cnt else np.zeros((0, hb // 4), np.uint32)
        raw = ws_view(ws, view["pay"], cnt, rb, np.uint8) if cnt else np.zeros((0, rb), np.uint8)
        order = np.argsort(hdr[:, 0], kind="stable")
        pos = hdr[order, 0].astype(np.int64)
        assert np.all(np.diff(pos) > 0), "a position was sent twice"
        rows = raw[order]
        lo = hdr[order, 1].view(np.float32) if B else None
        hi = hdr[order, 2].view(np.float32) if B else None
    codes, pad = decode_rows(rows, F, B)
    assert not np.any(pad), "padding codes / columns must be zero"
    return pos, codes, lo, hi


def check_messages(ctx, ws, plan_p, cnt, F, B):
    """Every message of the last sync, byte for byte against the oracle's record (O10):
    positions, lo/hi headers (bitwise) and codes (exact) for the gather (at each master)
    and the scatter (at each mirror) phase (Alg. 2 L5-L8, L20-L22; §5)."""
    nmsg = 0
    for (src, dst), ref in cnt.gather_msgs.items():
        got = read_messages(ws, cg.msg_view(ctx, dst, 0, src), F, B)
        _same(got, ref, B, f"gather {src}->{dst}")
        nmsg += len(ref[0])
    assert nmsg == cnt.gather_sent
    nmsg = 0
    for (src, dst), ref in cnt.scatter_msgs_rec.items():
        got = read_messages(ws, cg.msg_view(ctx, dst, 1, src), F, B)
        _same(got, ref, B, f"scatter {src}->{dst}")
        nmsg += len(ref[0])
    assert nmsg == cnt.scatter_msgs


def _same(got, ref, B, what):
    gpos, gcodes, glo, ghi = got
    rpos, rcodes, rlo, rhi = ref
    assert np.array_equal(gpos, np.asarray(rpos, np.int64)), f"{what}: positions differ"
    if B:
        assert np.array_equal(gcodes, np.asarray(rcodes, np.int64)), f"{what}: codes differ"
        assert np.array_equal(glo.view(np.uint32), np.asarray(rlo, np.float32).view(np.uint32)), f"{what}: lo"
        assert np.array_equal(ghi.view(np.uint32), np.asarray(rhi, np.float32).view(np.uint32)), f"{what}: hi"
    else:
        assert np.array_equal(gcodes.view(np.uint32), np.asarray(rcodes, np.float32).view(np.uint32)), \
            f"{what}: fp32 payload differs"


def _run(torch, d, p, dims, l, cache, quant, eps, steps=5, seed=0, layout=0, msgs=True):
    plan, oplan, ctx, ws = _setup(torch, d, p, dims, cache, quant, layout)
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
        if msgs:
            check_messages(ctx, ws, p, cnt, F, quant)
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
                pg, rg = cg.sync_flags(ctx, i, l, 0, 0)
                gf = ws_view(ws, pg, rg, 1, np.uint8)[:, 0].astype(bool)
                assert np.array_equal(gf, cnt.gather_mask[i])
                pf, rf_ = cg.sync_flags(ctx, i, l, 0, 1)
                assert np.array_equal(ws_view(ws, pf, rf_, 1, np.uint8)[:, 0].astype(bool),
                                      cnt.master_fired_mask[i])
            pa, ra = cg.sync_flags(ctx, i, l, 0, 2)
            assert np.array_equal(ws_view(ws, pa, ra, 1, np.uint8)[:, 0].astype(bool),
                                  cnt.active_mask[i])
        assert gst["gather_sent"] == cnt.gather_sent
        assert gst["scatter_msgs"] == cnt.scatter_msgs
        assert gst["active"] == cnt.active
        if cache:
            assert gst["master_fired"] == cnt.master_fired
        assert gst["baseline"] == cnt.baseline
        assert gst["bytes_alg"] == cnt.bytes
        # drift: a random 40% of rows change by a small amount
        Xs = [(x + (rng.random((x.shape[0], 1)) < 0.4) * 0.05 *
               rng.standard_normal(x.shape)).astype(np.float32) for x in Xs]
    ctx.close()


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("cache,quant", [(1, 8), (1, 0), (0, 8), (0, 0), (1, 4), (1, 16), (0, 4)])
@pytest.mark.parametrize("eps", [0.0, 0.05])
@pytest.mark.parametrize("l", [1, 2])
def test_replay_bitexact_small(cache, quant, eps, l, layout):
    """Synced rows, cache tables, masks, counters and every message byte (slot-addressed and
    compacted layouts; B ∈ {0, 4, 8, 16}) vs the oracle's fp32 replay."""
    torch = require_gpu()
    d = small_random_graph(900, 4000, (8, 20, 5), seed=31)
    _run(torch, d, 3, (8, 20, 5), l, cache, quant, eps, layout=layout)


@pytest.mark.parametrize("F", [7, 16, 41, 256, 300])
@pytest.mark.parametrize("quant", [8, 4, 16])
def test_replay_widths(F, quant):
    torch = require_gpu()
    d = small_random_graph(1500, 9000, (4, F, 3), seed=5)
    _run(torch, d, 4, (4, F, 3), 1, 1, quant, 0.02, steps=4)


def test_replay_many_parts_narrow_rows():
    """p = 6 parts with 2- and 4-lane row groups (p > lanes per row: the kernels read the
    slot table per source instead of holding it in lanes)."""
    torch = require_gpu()
    d = small_random_graph(1200, 7000, (4, 5, 3), seed=9)
    _run(torch, d, 6, (4, 5, 3), 1, 1, 8, 0.01, steps=4)
    _run(torch, d, 6, (4, 5, 3), 2, 1, 8, 0.01, steps=4)
    _run(torch, d, 6, (4, 5, 3), 2, 1, 0, 0.0, steps=3)



def test_replay_C1_two_parts():
    """configs[0]: Cora-shaped, 2 parts on 1 GPU, ε = 0, int8."""
    torch = require_gpu()
    d = make_dataset(get_config("C1"))
    for layout in (0, 1):
        _run(torch, d, 2, (1433, 16, 7), 1, 1, 8, 0.0, steps=6, layout=layout)
        _run(torch, d, 2, (1433, 16, 7), 2, 1, 8, 0.0, steps=6, layout=layout)


def test_replay_C2_two_parts():
    """configs[1] at full size, 2 parts on 1 GPU, hidden 256, cache + int8."""
    torch = require_gpu()
    d = make_dataset(get_config("C2"))
    _run(torch, d, 2, (128, 256, 256, 40), 1, 1, 8, 0.01, steps=3)
    _run(torch, d, 2, (128, 256, 256, 40), 3, 1, 8, 0.0, steps=2, layout=1)
