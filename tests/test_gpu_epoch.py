"""GPU epoch / layer parity vs the oracle (fp64) through the C ABI.

Bars (BASELINE.json north_star): fp32 features and gradients within max
row-normwise relative error 1e-4 (SIMT fp32 GEMMs), per-epoch loss within
1e-3·max(1, |L|) over 50 epochs; bitwise on dyadic fixtures."""
import numpy as np
import pytest

import paper_2408_00232_b200 as cg
from paper_2408_00232_b200.runtime import Run
from oracle import gcn
from oracle.cdfgnn import PartitionedGCN, TrainCfg
from oracle.graph import normalized_adjacency
from oracle.partition import PartitionCfg, partition as opartition
from synth import dyadic_fixture, get_config, make_dataset, small_random_graph
from tests.gpu_util import require_gpu, rownorm_err

pytestmark = pytest.mark.gpu


def _oracle(d, p, **kw):
    oplan = opartition(d.n, d.eu, d.ev, PartitionCfg(p=p))
    return PartitionedGCN(oplan, d.X, d.y, d.train, d.W, TrainCfg(**kw))


@pytest.mark.parametrize("p", [1, 3])
@pytest.mark.parametrize("cache", [False, True])
@pytest.mark.parametrize("gemm", ["fp32", "tf32x3", "tf32"])
def test_exact_mode_sgd_trajectory(p, cache, gemm):
    """ε = 0, no quantisation: fp32 SIMT and 3xTF32 GEMMs within 1e-5 (loss) / 1e-4 (W);
    1xTF32 within 1e-3."""
    require_gpu()
    d = small_random_graph(800, 4000, (12, 16, 5), seed=61)
    run = Run(d, p, cache=cache, quant_bits=0, eps0=0.0, adaptive=False, optimizer="sgd", lr=0.5,
              gemm=gemm)
    orc = _oracle(d, p, cache=cache, quant_bits=0, eps0=0.0, adaptive=False, optimizer="sgd",
                  lr=0.5)
    tl, tw = (1e-3, 1e-3) if gemm == "tf32" else (1e-5, 1e-4)
    for ep in range(6):
        g = run.epoch()
        o = orc.epoch()
        assert abs(g["loss"] - o["loss"]) <= tl * max(1.0, abs(o["loss"])), (ep, g["loss"], o["loss"])
        for wg, wo in zip(run.weights(), orc.W):
            assert rownorm_err(wg, wo) <= tw
        if p == 1:
            assert all(s["gather_sent"] == 0 for s in g["fwd"] + g["bwd"])
    run.close()


@pytest.mark.parametrize("gemm", ["fp32", "tf32x3", "tf32"])
def test_forward_activations_match(gemm):
    torch = require_gpu()
    d = small_random_graph(1000, 6000, (20, 32, 7), seed=62)
    p = 4
    tol = 1e-3 if gemm == "tf32" else 1e-5
    run = Run(d, p, cache=True, quant_bits=0, eps0=0.0, adaptive=False, optimizer="sgd", lr=0.0,
              gemm=gemm)
    A = normalized_adjacency(d.n, d.eu, d.ev)
    Z, H = gcn.forward(A, d.X.astype(np.float64), [w.astype(np.float64) for w in d.W])
    # layer 1 through the layer API
    ld1 = cg.ld_of(32)
    Zs = [torch.zeros((v["n_local"], ld1), device="cuda") for v in run.views]
    Hs = [torch.zeros((v["n_local"], ld1), device="cuda") for v in run.views]
    cg.layer_fwd(run.ctx, 1, run.X, run.ld0, run.W[0], Zs, Hs, ld1, 0.0)
    for v, z, h in zip(run.views, Zs, Hs):
        g = v["local2global"]
        assert rownorm_err(z.cpu().numpy()[:, :32], Z[0][g]) <= tol
        assert rownorm_err(h.cpu().numpy()[:, :32], H[1][g]) <= tol
    run.close()


@pytest.mark.parametrize("p", [2, 3])
@pytest.mark.parametrize("gemm", ["fp32", "tf32x3", "tf32"])
def test_dyadic_bitwise(p, gemm):
    """P-C1: dyadic fixture — every operand fits TF32 and every partial sum is exact, so GPU Z
    == plain GCN bitwise (both the fp32 SIMT and the tcgen05 TF32 GEMMs)."""
    torch = require_gpu()
    d = dyadic_fixture(n=96, r=4, dims=(16, 8, 4))
    run = Run(d, p, cache=True, quant_bits=0, eps0=0.0, adaptive=False, optimizer="sgd", lr=0.0,
              gemm=gemm)
    A = normalized_adjacency(d.n, d.eu, d.ev)
    Z, H = gcn.forward(A, d.X.astype(np.float64), [w.astype(np.float64) for w in d.W])
    ld1, ld2 = cg.ld_of(8), cg.ld_of(4)
    Z1 = [torch.zeros((v["n_local"], ld1), device="cuda") for v in run.views]
    H1 = [torch.zeros((v["n_local"], ld1), device="cuda") for v in run.views]
    Z2 = [torch.zeros((v["n_local"], ld2), device="cuda") for v in run.views]
    cg.layer_fwd(run.ctx, 1, run.X, run.ld0, run.W[0], Z1, H1, ld1, 0.0)
    cg.layer_fwd(run.ctx, 2, H1, ld1, run.W[1], Z2, None, ld2, 0.0)
    for v, z1, z2 in zip(run.views, Z1, Z2):
        g = v["local2global"]
        assert np.array_equal(z1.cpu().numpy()[:, :8].astype(np.float64), Z[0][g])
        assert np.array_equal(z2.cpu().numpy()[:, :4].astype(np.float64), Z[1][g])
    run.close()


@pytest.mark.parametrize("gemm", ["fp32", "tf32x3"])
def test_C1_fifty_epochs_loss_parity(gemm):
    """configs[0]: Cora-shaped, 2 partitions on 1 GPU, ε = 0, int8; Adam lr 0.01."""
    require_gpu()
    d = make_dataset(get_config("C1"))
    run = Run(d, 2, cache=True, quant_bits=8, eps0=0.0, adaptive=False, optimizer="adam", lr=0.01,
              gemm=gemm)
    orc = _oracle(d, 2, cache=True, quant_bits=8, eps0=0.0, adaptive=False, optimizer="adam",
                  lr=0.01)
    worst = 0.0
    for ep in range(50):
        g = run.epoch()
        o = orc.epoch()
        worst = max(worst, abs(g["loss"] - o["loss"]) / max(1.0, abs(o["loss"])))
        sent_o = sum(c.gather_sent for _, _, c in o["counters"])
        sent_g = sum(s["gather_sent"] for s in g["fwd"] + g["bwd"])
        assert abs(sent_g - sent_o) <= max(2, 0.01 * sent_o)
    assert worst <= 1e-3, worst
    run.close()


def test_cached_adaptive_tracks_oracle():
    require_gpu()
    d = small_random_graph(1500, 9000, (16, 32, 6), seed=63)
    run = Run(d, 4, cache=True, quant_bits=8, eps0=0.01, adaptive=True, optimizer="adam", lr=0.01)
    orc = _oracle(d, 4, cache=True, quant_bits=8, eps0=0.01, adaptive=True, optimizer="adam", lr=0.01)
    for ep in range(20):
        g = run.epoch()
        o = orc.epoch()
        assert abs(g["loss"] - o["loss"]) <= 1e-2 * max(1.0, abs(o["loss"]))
        assert g["eps_used"] == pytest.approx(o["eps"], abs=1e-12) or ep > 0
    run.close()


def test_label_out_of_range_is_edata():
    torch = require_gpu()
    d = small_random_graph(300, 1200, (8, 8, 3), seed=64)
    run = Run(d, 2, cache=True, quant_bits=8)
    run.labels[0].fill_(7)
    with pytest.raises(cg.CdfgnnError) as e:
        run.epoch()
    assert e.value.code == 3
    run.close()


@pytest.mark.parametrize("cache,quant,dims", [(True, 8, (20, 24, 6)), (False, 0, (20, 24, 6)),
                                              (True, 8, (20, 24, 16, 6)), (True, 0, (20, 24, 16, 6))])
def test_dead_sync_elision_static_inputs_and_overlap_are_bitwise_neutral(cache, quant, dims):
    """§8 f2: skipping the layer-L forward scatter and backward gather, and reusing Xᵀ;
    §8 f1: boundary-rows-first scheduling with the gather on a second stream — none of them
    changes a bit of the trajectory."""
    torch = require_gpu()
    d = small_random_graph(1200, 8000, dims, seed=65)
    runs = [Run(d, 3, cache=cache, quant_bits=quant, eps0=0.01, elide=e, static_inputs=si, overlap=ov)
            for e, si, ov in ((False, False, False), (True, True, False), (True, True, True))]
    for ep in range(4):
        res = [r.epoch() for r in runs]
        for r in res[1:]:
            assert r["loss"] == res[0]["loss"]
        # same schedule of syncs (elision on): the overlapped run sends exactly the same messages
        for a, b in zip(res[2]["fwd"] + res[2]["bwd"], res[1]["fwd"] + res[1]["bwd"]):
            assert (a["gather_sent"], a["master_fired"], a["scatter_msgs"]) == \
                (b["gather_sent"], b["master_fired"], b["scatter_msgs"])
        for r in runs[1:]:
            for wa, wb in zip(runs[0].weights(), r.weights()):
                assert np.array_equal(wa, wb)
    for r in runs:
        r.close()


@pytest.mark.parametrize("p", [1, 3])
@pytest.mark.parametrize("gemm", ["fp32", "tf32x3"])
@pytest.mark.parametrize("quant", [0, 8])
def test_hoisted_input_aggregation(p, gemm, quant):
    """static_inputs = 2: layer 1 as (Â_i X_i) W^(0) and ∇W^(0) = (Â_i X_i)ᵀ δ^(1) (no layer-1
    SpMMs in the epoch) follows the oracle's trajectory within the exact-mode bars (ε = 0);
    with int8 messages within the 50-epoch loss bar."""
    require_gpu()
    d = small_random_graph(900, 5000, (24, 16, 6), seed=67)
    kw = dict(cache=True, quant_bits=quant, eps0=0.0, adaptive=False, optimizer="sgd", lr=0.5)
    run = Run(d, p, gemm=gemm, static_inputs=2, **kw)
    orc = _oracle(d, p, **kw)
    tl, tw = (1e-5, 1e-4) if quant == 0 else (1e-3, 1e-2)
    for ep in range(6):
        g = run.epoch()
        o = orc.epoch()
        assert abs(g["loss"] - o["loss"]) <= tl * max(1.0, abs(o["loss"])), (ep, g["loss"], o["loss"])
        if quant == 0:
            for wg, wo in zip(run.weights(), orc.W):
                assert rownorm_err(wg, wo) <= tw
    run.close()


def test_pipelined_host_inputs_bitwise():
    """cdfgnn_epoch_host_next (inputs of step k+1 copied under step k) gives bit-identical
    losses and weights to cdfgnn_epoch on device inputs."""
    require_gpu()
    d = small_random_graph(700, 4000, (20, 16, 5), seed=71)
    kw = dict(cache=True, quant_bits=8, eps0=0.01, adaptive=True, optimizer="adam", lr=0.01,
              static_inputs=1)
    a = Run(d, 2, **kw)
    b = Run(d, 2, host_inputs=True, **kw)
    steps = 5
    for k in range(steps):
        ga = a.epoch()
        gb = b.epoch_host_next(prefetch_next=k + 1 < steps)
        assert ga["loss"] == gb["loss"], (k, ga["loss"], gb["loss"])
    for wa, wb in zip(a.weights(), b.weights()):
        assert np.array_equal(wa, wb)
    a.close()
    b.close()
