"""Edge cases of the halo exchange and the epoch, bit-exact against the oracle's fp32 replay
(Alg. 2, §5, readings R14/R15/R24):

* ragged and minimal widths (F = 1, 5: ld = 4, 8 with zero padding) and the widest rows
  (F = 1024, B = 16);
* degenerate message rows: constant rows (hi = lo: every code 0), all-zero partials (no
  sender on the first sync: 0 > 0 is false), a single changed column;
* many parts on a small graph (p = 16, 48: parts without boundary masters or mirrors, and
  row groups with fewer lanes than parts, where the kernels read the slot table per source);
* an epoch on a graph whose parts have empty boundary sets.
"""
import numpy as np
import pytest

import paper_2408_00232_b200 as cg
from paper_2408_00232_b200.runtime import Run
from oracle.cdfgnn import PartitionedGCN, TrainCfg
from oracle.partition import PartitionCfg, partition as opartition
from synth import small_random_graph
from tests.gpu_util import require_gpu
from tests.test_gpu_halo import _run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("F,quant", [(1, 8), (1, 0), (5, 4), (5, 16), (1024, 16), (1024, 8)])
def test_ragged_and_extreme_widths(F, quant):
    torch = require_gpu()
    d = small_random_graph(600, 2500, (4, F, 3), seed=81)
    _run(torch, d, 3, (4, F, 3), 1, 1, quant, 0.02, steps=3)


def test_constant_zero_and_single_column_rows():
    """Synthetic partials with constant rows, all-zero rows and rows that change in one column
    only, through the same replay (every message byte and synced row vs the oracle)."""
    torch = require_gpu()
    from oracle.cache import SyncMode, SyncState, sync
    from tests.test_gpu_halo import _setup, check_messages
    from tests.gpu_util import ws_view
    d = small_random_graph(800, 3500, (4, 12, 3), seed=82)
    p, F = 3, 12
    plan, oplan, ctx, ws = _setup(torch, d, p, (4, F, 3), 1, 8)
    st = SyncState(oplan, F, np.float32)
    mode = SyncMode(cache=True, quant_bits=8, dtype=np.float32)
    rng = np.random.default_rng(3)
    Xs = []
    for pp in oplan.parts:
        x = rng.standard_normal((pp.n_local, F)).astype(np.float32)
        kind = rng.integers(0, 3, pp.n_local)
        x[kind == 0] = 0.0                                   # all-zero rows
        x[kind == 1] = x[kind == 1][:, :1]                   # constant rows
        Xs.append(x)
    for step in range(4):
        dev = [torch.from_numpy(x.copy()).cuda() for x in Xs]
        cg.halo_exchange(ctx, 1, 0, dev, F, np.float32(0.0), stats=True)
        out, cnt = sync(oplan, st, [x.copy() for x in Xs], 0.0, mode)
        check_messages(ctx, ws, p, cnt, F, 8)
        for i in range(p):
            assert np.array_equal(dev[i].cpu().numpy().view(np.uint32), out[i].view(np.uint32)), (step, i)
        # next step: one column of a third of the rows changes
        for x in Xs:
            rows = rng.random(x.shape[0]) < 0.33
            x[rows, int(rng.integers(0, F))] += np.float32(0.5)
    ctx.close()


@pytest.mark.parametrize("p", [16, 48])
def test_many_parts_small_graph(p):
    torch = require_gpu()
    d = small_random_graph(400, 1500, (4, 9, 3), seed=83)
    _run(torch, d, p, (4, 9, 3), 1, 1, 8, 0.01, steps=3)
    _run(torch, d, p, (4, 9, 3), 1, 0, 0, 0.0, steps=2, layout=1)


def test_epoch_with_parts_without_boundary():
    """Two disconnected halves partitioned into 2 parts: with the default EBV order each part
    may hold a whole component (no boundary vertices, no messages); the epoch still equals the
    oracle's and the unpartitioned model's trajectory (ε = 0, fp32 messages)."""
    require_gpu()
    a = small_random_graph(300, 1200, (8, 16, 4), seed=84)
    n = 2 * a.n
    eu = np.concatenate([a.eu, a.eu + a.n]).astype(np.int32)
    ev = np.concatenate([a.ev, a.ev + a.n]).astype(np.int32)
    o = np.lexsort((ev, eu))
    from synth.graphs import Dataset
    d = Dataset(n=n, eu=eu[o], ev=ev[o], X=np.concatenate([a.X, a.X[::-1]]), y=np.concatenate([a.y, a.y]),
                train=np.concatenate([a.train, a.train]), val=np.concatenate([a.val, a.val]),
                test=np.concatenate([a.test, a.test]), W=a.W, dims=a.dims)
    kw = dict(cache=True, quant_bits=0, eps0=0.0, adaptive=False, optimizer="sgd", lr=0.5)
    run = Run(d, 2, **kw)
    orc = PartitionedGCN(opartition(d.n, d.eu, d.ev, PartitionCfg(p=2)), d.X, d.y, d.train, d.W, TrainCfg(**kw))
    for ep in range(4):
        g = run.epoch()
        o_ = orc.epoch()
        assert abs(g["loss"] - o_["loss"]) <= 1e-5 * max(1.0, abs(o_["loss"]))
    run.close()


def test_maximum_classes_epoch():
    """256 classes (the loss kernel's maximum, 8 per lane): 3 exact-mode epochs, 2 parts,
    against the oracle (loss 1e-5, W row-normwise 1e-4)."""
    require_gpu()
    from tests.gpu_util import rownorm_err
    d = small_random_graph(1500, 7000, (12, 32, 256), seed=85)
    kw = dict(cache=True, quant_bits=0, eps0=0.0, adaptive=False, optimizer="sgd", lr=0.5)
    run = Run(d, 2, **kw)
    orc = PartitionedGCN(opartition(d.n, d.eu, d.ev, PartitionCfg(p=2)), d.X, d.y, d.train, d.W, TrainCfg(**kw))
    for ep in range(3):
        g = run.epoch()
        o = orc.epoch()
        assert abs(g["loss"] - o["loss"]) <= 1e-5 * max(1.0, abs(o["loss"]))
        assert g["correct"] == o["correct"]
        for wg, wo in zip(run.weights(), orc.W):
            assert rownorm_err(wg, wo) <= 1e-4
    run.close()
