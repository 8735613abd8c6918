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


def gpu_follow_masks(run):
    """The GPU's cache-test decisions of its latest epoch (cdfgnn_sync_flags: gather-sent per
    mirror, fired per master, for every (layer, direction)) in the oracle's follow format."""
    from tests.gpu_util import ws_view
    fol = {}
    for l in range(1, run.cfg.L + 1):
        for dr, key in ((0, "fwd"), (1, "bwd")):
            g, m = {}, {}
            for t, part in enumerate(run.parts):
                pg, rg = cg.sync_flags(run.ctx, t, l, dr, 0)
                g[part] = ws_view(run.workspace, pg, rg, 1, np.uint8)[:, 0].astype(bool)
                pf, rf = cg.sync_flags(run.ctx, t, l, dr, 1)
                m[part] = ws_view(run.workspace, pf, rf, 1, np.uint8)[:, 0].astype(bool)
            fol[(key, l)] = {"gather": g, "master": m}
    return fol


@pytest.mark.parametrize("name,p,scale,snr,quant,opt,lr", [
    ("C1", 2, None, 0.05, 8, "adam", 0.01), ("C2", 2, 0.1, 0.3, 8, "sgd", 1.0),
    ("C2", 3, 0.1, 0.3, 8, "sgd", 1.0), ("C1", 3, None, 0.05, 4, "adam", 0.01),
    ("C1", 2, None, 0.05, 16, "adam", 0.01)])
def test_follow_mode_adaptive_trajectory_50_epochs(name, p, scale, snr, quant, opt, lr):
    """Adaptive ε > 0 with the cache and B-bit messages: the oracle runs in
    follow mode on the GPU's recorded send / fire decisions (their correctness is proven
    separately by the bit-exact replay in test_gpu_halo.py), so a near-threshold flip from
    fp32 rounding cannot split the trajectories.  Per-epoch loss within 1e-3·max(1, |L|) over
    50 epochs; every sync's gather / fired / scatter counts equal the oracle's; the C++ ε
    controller's ε equals oracle/eps.py's EpsController on the GPU's accuracy sequence at
    every epoch (R17, R18), and the oracle's own ε equals the GPU's whenever the
    two accuracy counts agree.  The feature SNR knob (synth) makes accuracy climb over tens of
    epochs, so ε actually moves.  C2 (3 layers, 256 wide) trains with SGD (Alg. 1 L13):
    Adam's per-parameter normalisation turns rounding-level differences of near-zero
    gradients (fp32 GPU vs fp64 oracle) into ±lr steps and leaves the 1e-3 band within ~12
    epochs even on identical decisions, SGD keeps W linear in ∇W."""
    from oracle.eps import EpsController
    require_gpu()
    d = make_dataset(get_config(name), scale, snr=snr)
    kw = dict(cache=True, quant_bits=quant, eps0=0.01, adaptive=True, optimizer=opt, lr=lr)
    run = Run(d, p, **kw)
    orc = _oracle(d, p, **kw)
    ctl = EpsController(0.01)
    eps_seen = set()
    worst = 0.0
    for ep in range(50):
        g = run.epoch()
        o = orc.epoch(follow=gpu_follow_masks(run))
        worst = max(worst, abs(g["loss"] - o["loss"]) / max(1.0, abs(o["loss"])))
        assert worst <= 1e-3, (ep, g["loss"], o["loss"])
        # controller: the C++ update equals the oracle's on the same accuracy, bit for bit
        assert g["eps_used"] == ctl.eps
        assert g["eps_next"] == ctl.step(g["acc"]), ep
        assert abs(g["correct"] - o["correct"]) <= max(1, 0.002 * g["total"]), (ep, g["correct"], o["correct"])
        if g["correct"] == o["correct"]:
            assert g["eps_used"] == o["eps"]
        eps_seen.add(g["eps_used"])
        # same decisions => same message counts, sync by sync (elided syncs are empty on both)
        oc = {(dr, l): c for dr, l, c in o["counters"]}
        for l in range(1, run.cfg.L + 1):
            for dr, key in ((g["fwd"], "fwd"), (g["bwd"], "bwd")):
                c = oc[(key, l)]
                assert dr[l - 1]["gather_sent"] == c.gather_sent
                assert dr[l - 1]["master_fired"] == c.master_fired
                if not (key == "fwd" and l == run.cfg.L):       # elided on the GPU (§8 f2)
                    assert dr[l - 1]["scatter_msgs"] == c.scatter_msgs
    assert len(eps_seen) >= 5, sorted(eps_seen)          # ε moved: the run exercised the controller
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
    §8 f1: boundary-rows-first scheduling with the gather on a second stream, and the gather
    fused into the forward SpMM epilogue; the compacted vs slot-addressed message layout — none
    of them changes a bit of the trajectory."""
    torch = require_gpu()
    d = small_random_graph(1200, 8000, dims, seed=65)
    runs = [Run(d, 3, cache=cache, quant_bits=quant, eps0=0.01, elide=e, static_inputs=si, overlap=ov,
                msg_layout=ml, fuse_gather=fg)
            for e, si, ov, ml, fg in ((False, False, False, 0, False), (True, True, False, 0, True),
                                      (True, True, True, 0, True), (True, True, False, 1, True),
                                      (False, False, False, 1, True), (True, False, False, 0, False))]
    for ep in range(4):
        res = [r.epoch() for r in runs]
        for r in res[1:]:
            assert r["loss"] == res[0]["loss"]
        # same schedule of syncs (elision on): the overlapped run and the compacted message
        # layout send exactly the same messages as the slot-addressed one
        for other in (res[2], res[3]):
            for a, b in zip(other["fwd"] + other["bwd"], res[1]["fwd"] + res[1]["bwd"]):
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
@pytest.mark.parametrize("F0", [24, 1100])
def test_hoisted_input_aggregation(p, gemm, quant, F0):
    """static_inputs = 2: layer 1 as (Â_i X_i) W^(0) and ∇W^(0) = (Â_i X_i)ᵀ δ^(1) (no layer-1
    SpMMs in the epoch) follows the oracle's trajectory within the exact-mode bars (ε = 0);
    with int8 messages within the 50-epoch loss bar."""
    require_gpu()
    # F0 = 1100 > 1024: Â_i X_i is aggregated in 1024-column slices
    d = small_random_graph(900, 5000, (F0, 16, 6), seed=67)
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


def test_static_inputs_follow_new_host_inputs():
    """the static_inputs caches (Â_i X_i, Xᵀ) are keyed on the X buffer; host-input
    entry points rewrite a library-owned staging buffer, so new host values must invalidate
    them.  A static_inputs = 2 run fed changing host inputs tracks a per-epoch run on device
    inputs (rounding-order differences only)."""
    torch = require_gpu()
    d = small_random_graph(700, 4000, (20, 16, 5), seed=73)
    kw = dict(cache=True, quant_bits=0, eps0=0.0, adaptive=False, optimizer="sgd", lr=0.5)
    a = Run(d, 2, **kw)
    b = Run(d, 2, host_inputs=True, static_inputs=2, **kw)
    for k in range(4):
        scale = 1.0 + 0.5 * k
        for xa, xb in zip(a.X, b.X_host):
            xb.copy_(xa.cpu() * scale)
        xs = [x.clone() for x in a.X]
        for x in a.X:
            x.mul_(scale)
        ga = a.epoch()
        gb = b.epoch_host() if k % 2 == 0 else b.epoch_host_next(prefetch_next=False)
        assert abs(ga["loss"] - gb["loss"]) <= 1e-5 * max(1.0, abs(ga["loss"])), (k, ga["loss"], gb["loss"])
        for x, x0 in zip(a.X, xs):
            x.copy_(x0)
    a.close()
    b.close()


@pytest.mark.parametrize("name,scale,p", [("C4", 0.01, 4), ("C5", 0.005, 4)])
def test_C4_C5_shapes_exact_mode(name, scale, p):
    """The 3-layer C4 (100-256-256-47) and C5 (200-256-256-172) architectures on scaled-down
    graphs of their degree laws: ε = 0 and fp32 messages (P-C1) — per-epoch loss within 1e-5
    and W row-normwise within 1e-4 of the oracle (SGD, 4 epochs)."""
    require_gpu()
    d = make_dataset(get_config(name), scale)
    kw = dict(cache=True, quant_bits=0, eps0=0.0, adaptive=False, optimizer="sgd", lr=0.5)
    run = Run(d, p, **kw)
    orc = _oracle(d, p, **kw)
    for ep in range(4):
        g = run.epoch()
        o = orc.epoch()
        assert abs(g["loss"] - o["loss"]) <= 1e-5 * max(1.0, abs(o["loss"])), (ep, g["loss"], o["loss"])
        for wg, wo in zip(run.weights(), orc.W):
            assert rownorm_err(wg, wo) <= 1e-4
    run.close()


@pytest.mark.parametrize("name,scale,eps", [("C4", 0.01, 0.03), ("C4", 0.01, 0.1), ("C5", 0.005, 0.1),
                                            ("C3", 0.02, 0.3)])
def test_fixed_eps_sweep_follow_mode(name, scale, eps):
    """Points of the ε sweep (BASELINE configs[3]; §8 f3) with the cache and int8 messages: the
    oracle follows the GPU's send / fire decisions; per-epoch loss within 1e-3·max(1, |L|) and
    every sync's counts equal over 15 epochs (SGD), and the cache really skips replicas."""
    require_gpu()
    d = make_dataset(get_config(name), scale)
    kw = dict(cache=True, quant_bits=8, eps0=eps, adaptive=False, optimizer="sgd", lr=0.5)
    run = Run(d, 4, **kw)
    orc = _oracle(d, 4, **kw)
    skipped = 0
    for ep in range(15):
        g = run.epoch()
        o = orc.epoch(follow=gpu_follow_masks(run))
        assert abs(g["loss"] - o["loss"]) <= 1e-3 * max(1.0, abs(o["loss"])), (ep, g["loss"], o["loss"])
        oc = {(dr, l): c for dr, l, c in o["counters"]}
        for l in range(1, run.cfg.L + 1):
            for dr, key in ((g["fwd"], "fwd"), (g["bwd"], "bwd")):
                c = oc[(key, l)]
                assert dr[l - 1]["gather_sent"] == c.gather_sent
                assert dr[l - 1]["master_fired"] == c.master_fired
                if not (key == "fwd" and l == run.cfg.L):
                    assert dr[l - 1]["scatter_msgs"] == c.scatter_msgs
        M = sum(v["n_mirror"] for v in run.views)
        skipped += sum(M - s["gather_sent"] for s in g["fwd"] + g["bwd"][:-1])
    assert skipped > 0
    run.close()


@pytest.mark.parametrize("p,quant", [(1, 8), (3, 8), (3, 0)])
def test_fused_relu_is_bitwise_neutral(p, quant, monkeypatch):
    """σ applied in the SpMM epilogue (interior rows) and the slot master / mirror kernels
    (boundary rows) instead of a separate ReLU pass (R3): bit-identical losses and weights."""
    require_gpu()
    d = small_random_graph(1000, 7000, (16, 24, 20, 5), seed=86)
    kw = dict(cache=True, quant_bits=quant, eps0=0.01, adaptive=True, optimizer="adam", lr=0.01)
    a = Run(d, p, **kw)
    b = Run(d, p, **kw)
    for ep in range(4):
        monkeypatch.setenv("CDFGNN_FUSE_RELU", "1")
        ga = a.epoch()
        monkeypatch.setenv("CDFGNN_FUSE_RELU", "0")
        gb = b.epoch()
        assert ga["loss"] == gb["loss"], (ep, ga["loss"], gb["loss"])
        for wa, wb in zip(a.weights(), b.weights()):
            assert np.array_equal(wa, wb)
    a.close()
    b.close()
