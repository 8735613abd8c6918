"""Parity at the bench workload's FULL size, in the launch configuration bench.py times.

BASELINE.json's metric is quoted on configs[2] (C3, Reddit-shaped: 232,965 vertices,
114,615,892 CSR entries, 602-256-41); bench.py runs it as one `cdfgnn_epoch` per step
(p = 1, cache + int8, adaptive ε, Adam, 3xTF32 GEMMs, static inputs).  After one such
epoch, the activations and parameter gradients it produced are checked against the
oracle (oracle/gcn.py, fp64):
  * H^(1) = ReLU(Â X W^(0)) and the logits Â H^(1) W^(1) on sampled rows, computed one
    row at a time (`rows_forward`, eq. 1) — the first from the inputs, the second
    from the GPU's own H^(1) (itself checked on its sample);
  * loss and correct count from the GPU's logits (`loss_grad`, R7, R16);
  * ∇W^(1) = H^(1)ᵀ Â δ^(2) in full, and sampled columns of ∇W^(0) = Xᵀ Â δ^(1) with
    δ^(1) = (Â δ^(2) W^(1)ᵀ) ⊙ 𝟙[H^(1) > 0] (the adjoint, R6).
Tolerance: 1e-4 row-normwise (SURVEY §8(c4), fp32 path; 3xTF32 GEMMs).
"""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2408_00232_b200 as cg
from oracle import gcn
from paper_2408_00232_b200.runtime import Run
from synth import get_config
from synth.cache import cached_dataset
from tests.gpu_util import require_gpu, rownorm_err

pytestmark = pytest.mark.gpu


def _view(torch, ptr, rows, ld, cols, like):
    """numpy copy of a [rows x ld] fp32 buffer inside the workspace (first `cols` columns)."""
    ws = like.workspace
    off = ptr - ws.data_ptr()
    n = rows * ld * 4
    assert 0 <= off and off + n <= ws.numel()
    torch.cuda.synchronize()
    a = ws[off:off + n].cpu().numpy().view(np.float32).reshape(rows, ld)
    return a[:, :cols].astype(np.float64)


def test_C3_bench_epoch_sampled_parity():
    torch = require_gpu()
    ds = cached_dataset(get_config("C3"))
    F0, F1, C = ds.dims
    # the arguments bench.py passes for its default (cache_int8) line at N = 1
    run = Run(ds, 1, cache=True, quant_bits=8, eps0=0.01, adaptive=True, optimizer="adam", lr=0.01,
              static_inputs=True)
    W_old = [w.astype(np.float64) for w in run.weights()]
    st = run.epoch()
    v = run.views[0]
    n = v["n_local"]
    A = sp.csr_matrix((v["val"].astype(np.float64), v["colidx"], v["rowptr"]), shape=(n, n))
    X = run.X[0].cpu().numpy()[:, :F0].astype(np.float64)
    y = run.labels[0].cpu().numpy()
    train = run.masks[0].cpu().numpy().astype(bool)
    H1 = _view(torch, *cg.act_view(run.ctx, 0, 1), F1, run)
    logits = _view(torch, *cg.act_view(run.ctx, 0, 2), C, run)
    rng = np.random.default_rng(2408)
    deg = np.diff(v["rowptr"])
    rows = np.unique(np.concatenate([[int(np.argmax(deg)), int(np.argmin(deg))],
                                     rng.choice(n, 40, replace=False)]))
    # forward, sampled rows
    ref_h1 = np.maximum(gcn.rows_forward(A, X, W_old[0], rows), 0)
    assert rownorm_err(H1[rows], ref_h1) <= 1e-4
    ref_lg = gcn.rows_forward(A, H1, W_old[1], rows)
    assert rownorm_err(logits[rows], ref_lg) <= 1e-4
    # loss head on the GPU's logits
    loss, d2, correct = gcn.loss_grad(logits, y, train)
    assert abs(st["loss"] - loss) <= 1e-5 * max(1.0, abs(loss))
    assert st["correct"] == correct and st["total"] == int(train.sum())
    # ∇W^(1) in full
    S2 = A @ d2
    g1 = _view(torch, *cg.grad_view(run.ctx, 2), C, run)
    assert rownorm_err(g1, H1.T @ S2) <= 1e-4
    # ∇W^(0) on sampled columns
    d1 = (S2 @ W_old[1].T) * (H1 > 0)
    cols = np.sort(rng.choice(F1, 6, replace=False))
    ref_g0 = X.T @ (A @ d1[:, cols])
    g0 = _view(torch, *cg.grad_view(run.ctx, 1), F1, run)
    assert rownorm_err(g0[:, cols], ref_g0) <= 1e-4
    run.close()
