"""Layer forward / backward through the C ABI at configs[1] size (p = 1), checked
against oracle arithmetic in fp64 (scipy CSR for Â, numpy for the dense products).

Exercises the tcgen05 GEMMs — 3xTF32 (the default; tolerance 1e-4 row-normwise like
fp32) and 1xTF32 (checked against its rounding bound |Δ| ≤ 2^-10·Σ|a||b| propagated
through Â) — and the fp32 SIMT GEMMs (1e-4): T = H W, ∇W = Hᵀ Â δ
with K = n ≈ 169k (split-K), δ̈ = (Â δ Wᵀ) ⊙ 𝟙[H > 0]."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2408_00232_b200 as cg
from paper_2408_00232_b200.runtime import Run
from synth import get_config, make_dataset
from tests.gpu_util import require_gpu, rownorm_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    return make_dataset(get_config("C2"))


def _A(run):
    v = run.views[0]
    n = v["n_local"]
    return sp.csr_matrix((v["val"].astype(np.float64), v["colidx"], v["rowptr"]), shape=(n, n)), v


def _check(got, ref, gemm, bound=None):
    if gemm == "tf32":
        # 1xTF32: each product a·b carries ≤ 2^-10 relative error (RN inputs), fp32 sums add
        # ≤ 1e-6 of the magnitude; checked elementwise against the propagated bound
        err = np.abs(np.asarray(got, np.float64) - ref)
        assert np.all(err <= 1.05 * bound + 1e-6 * (np.abs(ref) + bound) + 1e-12)
    else:
        assert rownorm_err(got, ref) <= 1e-4


@pytest.mark.parametrize("gemm", ["tf32x3", "fp32", "tf32"])
def test_layer_fwd_bwd_full_C2(c2, gemm):
    torch = require_gpu()
    run = Run(c2, 1, cache=True, quant_bits=8, eps0=0.0, adaptive=False, gemm=gemm)
    A, v = _A(run)
    n = v["n_local"]
    u = 2.0 ** -10
    rng = np.random.default_rng(3)
    F0, F1, F2 = 128, 256, 256
    X = run.X[0]
    Xn = X.cpu().numpy().astype(np.float64)
    W0 = run.W[0]
    # ---- forward layer 1: Z = Â (X W0)
    Z = torch.zeros((n, F1), device="cuda")
    H = torch.zeros((n, F1), device="cuda")
    cg.layer_fwd(run.ctx, 1, [X], cg.ld_of(F0), W0, [Z], [H], F1, 0.0)
    W0n = W0.cpu().numpy().astype(np.float64)
    Zr = A @ (Xn[:, :F0] @ W0n)
    bZ = u * (A @ (np.abs(Xn[:, :F0]) @ np.abs(W0n)))
    _check(Z.cpu().numpy(), Zr, gemm, bZ)
    _check(H.cpu().numpy(), np.maximum(Zr, 0), gemm, bZ)
    # ---- backward layer 2 with a random δ̈: S = Â δ, ∇W1 = Hᵀ S, δ̈1 = (S W1ᵀ) ⊙ 𝟙[H > 0]
    W1 = run.W[1]
    d2 = rng.standard_normal((n, F2)).astype(np.float32) * 1e-3
    dZ = torch.from_numpy(d2).cuda()
    dW = torch.zeros((F1, F2), device="cuda")
    dprev = torch.zeros((n, F1), device="cuda")
    cg.layer_bwd(run.ctx, 2, [dZ], F2, [H], F1, W1, [dprev], dW, 0.0)
    Hn = H.cpu().numpy().astype(np.float64)
    S = A @ d2.astype(np.float64)
    dWr = Hn.T @ S
    _check(dW.cpu().numpy(), dWr, gemm, u * (np.abs(Hn).T @ np.abs(S)))
    W1n = W1.cpu().numpy().astype(np.float64)
    dpr = (S @ W1n.T) * (Hn > 0)
    _check(dprev.cpu().numpy(), dpr, gemm, u * (np.abs(S) @ np.abs(W1n).T) * (Hn > 0))
    # ---- backward layer 1 (no δ̈^(0)): ∇W0 = Xᵀ Â δ with F0 = 128, K = n
    d1 = rng.standard_normal((n, F1)).astype(np.float32) * 1e-3
    dZ1 = torch.from_numpy(d1).cuda()
    dW0 = torch.zeros((F0, F1), device="cuda")
    cg.layer_bwd(run.ctx, 1, [dZ1], F1, [X], cg.ld_of(F0), W0, None, dW0, 0.0)
    S1 = A @ d1.astype(np.float64)
    dW0r = Xn[:, :F0].T @ S1
    _check(dW0.cpu().numpy(), dW0r, gemm, u * (np.abs(Xn[:, :F0]).T @ np.abs(S1)))
    run.close()


@pytest.mark.parametrize("dims", [(40, 41, 7), (602, 256, 41), (100, 47, 16), (33, 300, 5)])
@pytest.mark.parametrize("gemm", ["tf32x3", "tf32"])
def test_odd_widths(dims, gemm):
    """Ragged M/N/K tails and narrow N (zero-filled TMA boxes, padded W rows)."""
    torch = require_gpu()
    from synth import small_random_graph
    d = small_random_graph(3000, 15000, dims, seed=17)
    run = Run(d, 1, cache=True, quant_bits=8, eps0=0.0, adaptive=False, gemm=gemm)
    u = 2.0 ** -10
    A, v = _A(run)
    n = v["n_local"]
    F0, F1, F2 = dims
    ld0, ld1, ld2 = (cg.ld_of(f) for f in dims)
    Z = torch.zeros((n, ld1), device="cuda")
    H = torch.zeros((n, ld1), device="cuda")
    cg.layer_fwd(run.ctx, 1, [run.X[0]], ld0, run.W[0], [Z], [H], ld1, 0.0)
    Xn = run.X[0].cpu().numpy().astype(np.float64)[:, :F0]
    W0 = d.W[0].astype(np.float64)
    Zr = A @ (Xn @ W0)
    _check(Z.cpu().numpy()[:, :F1], Zr, gemm, u * (A @ (np.abs(Xn) @ np.abs(W0))))
    assert not Z.cpu().numpy()[:, F1:].any()
    rng = np.random.default_rng(5)
    d2 = np.zeros((n, ld2), np.float32)
    d2[:, :F2] = rng.standard_normal((n, F2)) * 1e-2
    dW = torch.zeros((F1, F2), device="cuda")
    dprev = torch.zeros((n, ld1), device="cuda")
    cg.layer_bwd(run.ctx, 2, [torch.from_numpy(d2).cuda()], ld2, [H], ld1, run.W[1], [dprev], dW, 0.0)
    Hn = H.cpu().numpy().astype(np.float64)[:, :F1]
    S = A @ d2[:, :F2].astype(np.float64)
    _check(dW.cpu().numpy(), Hn.T @ S, gemm, u * (np.abs(Hn).T @ np.abs(S)))
    W1 = d.W[1].astype(np.float64)
    dpr = (S @ W1.T) * (Hn > 0)
    _check(dprev.cpu().numpy()[:, :F1], dpr, gemm, u * (np.abs(S) @ np.abs(W1).T) * (Hn > 0))
    assert not dprev.cpu().numpy()[:, F1:].any()
    run.close()
