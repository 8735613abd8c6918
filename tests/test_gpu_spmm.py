"""SpMM Y = Â_i T through cdfgnn_spmm, with hub rows split into
chunks summed in a fixed order (kernels_spmm.cu): values vs the plain sparse product in
fp64, bitwise run-to-run determinism, and agreement of split and unsplit schedules."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2408_00232_b200 as cg
from synth import small_random_graph
from tests.gpu_util import require_gpu, rownorm_err

pytestmark = pytest.mark.gpu


def _ctx(d, p, chunk, phases=1):
    torch = require_gpu()
    env = {"CDFGNN_SPMM_CHUNK": str(chunk), "CDFGNN_SPMM_CHUNK_WIDE": str(chunk),
           "CDFGNN_SPMM_PHASES": str(phases), "CDFGNN_SPMM_PHASE_MIN": "16"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        plan = cg.partition(d.n, d.eu, d.ev, p)
        cfg = cg.cfg_default(d.dims)
        parts = list(range(p))
        ws = torch.empty(cg.workspace_size(plan, parts, cfg), dtype=torch.uint8, device="cuda")
        ctx = cg.init(plan, parts, 0, 1, cfg, 0, ws)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return plan, ctx, ws


@pytest.mark.parametrize("chunk,phases", [(0, 1), (7, 1), (64, 1), (0, 3), (0, 8)])
@pytest.mark.parametrize("ld", [4, 44, 256])
def test_spmm_matches_sparse_product_and_is_deterministic(chunk, phases, ld):
    torch = require_gpu()
    # power-law graph: hub rows of a few hundred neighbours next to degree-1 rows
    d = small_random_graph(2500, 40000, (8, ld, 4), seed=77, tau=2.1, v0=1.0)
    plan, ctx, ws = _ctx(d, 2, chunk, phases)
    g = torch.Generator().manual_seed(5)
    for part in range(2):
        v = cg.plan_part(plan, part)
        n = v["n_local"]
        A = sp.csr_matrix((v["val"].astype(np.float64), v["colidx"], v["rowptr"]), shape=(n, n))
        T = torch.randn((n, ld), generator=g)
        ref = A @ T.numpy().astype(np.float64)
        Td = T.cuda()
        Y1 = torch.full((n, ld), float("nan"), device="cuda")
        Y2 = torch.full((n, ld), float("nan"), device="cuda")
        cg.spmm(ctx, part, Td, Y1, ld, ld)
        cg.spmm(ctx, part, Td, Y2, ld, ld)
        y1 = Y1.cpu().numpy()
        assert np.isfinite(y1).all()
        assert np.array_equal(y1, Y2.cpu().numpy())          # fixed summation order
        assert rownorm_err(y1, ref) <= 1e-5
        deg = np.diff(v["rowptr"])
        if chunk:
            assert deg.max() > 3 * chunk                      # the schedule really splits rows
    ctx.close()


def test_split_and_unsplit_schedules_agree():
    torch = require_gpu()
    d = small_random_graph(3000, 60000, (8, 64, 4), seed=78, tau=2.0, v0=1.0)
    outs = []
    for chunk, phases in ((0, 1), (16, 1), (0, 4)):
        plan, ctx, ws = _ctx(d, 1, chunk, phases)
        v = cg.plan_part(plan, 0)
        n = v["n_local"]
        T = torch.randn((n, 64), generator=torch.Generator().manual_seed(9)).cuda()
        Y = torch.empty((n, 64), device="cuda")
        cg.spmm(ctx, 0, T, Y, 64, 64)
        outs.append(Y.cpu().numpy())
        ctx.close()
    for o in outs[1:]:
        assert rownorm_err(o, outs[0]) <= 1e-5
