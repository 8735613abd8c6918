"""SpMM microbenchmark on a config's partition (cdfgnn_spmm through the C ABI).
    python tools/spmm_bench.py --config C3 --p 1 --variants "chunk:0;chunk:1024" --widths 256,44
Variant keys set the library's tuning knobs before the context is built:
chunk=CDFGNN_SPMM_CHUNK, unr=CDFGNN_SPMM_UNR, tail=CDFGNN_SPMM_TAIL, stream=CDFGNN_SPMM_STREAM."""
import argparse, os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KNOBS = {"chunk": "CDFGNN_SPMM_CHUNK", "wchunk": "CDFGNN_SPMM_CHUNK_WIDE", "phases": "CDFGNN_SPMM_PHASES", "pmin": "CDFGNN_SPMM_PHASE_MIN", "unr": "CDFGNN_SPMM_UNR", "tail": "CDFGNN_SPMM_TAIL",
         "stream": "CDFGNN_SPMM_STREAM", "shape": "CDFGNN_SPMM_SHAPE", "wshape": "CDFGNN_SPMM_WSHAPE",
         "order": "CDFGNN_SPMM_ORDER", "heavy": "CDFGNN_SPMM_HEAVY", "cslice": "CDFGNN_SPMM_CSLICE"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--p", type=int, default=1)
    ap.add_argument("--part", type=int, default=0)
    ap.add_argument("--widths", default="256,44")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="chunk:0;chunk:1024")
    ap.add_argument("--relabel", default="none", help="none | class | classdeg (vertex renumbering experiment)")
    a = ap.parse_args()
    import torch
    import paper_2408_00232_b200 as cg
    from synth import get_config
    from synth.cache import cached_dataset
    ds = cached_dataset(get_config(a.config))
    eu, ev = ds.eu, ds.ev
    if a.relabel != "none":
        import numpy as np
        deg = np.bincount(eu, minlength=ds.n) + np.bincount(ev, minlength=ds.n)
        key2 = -deg if a.relabel == "classdeg" else np.arange(ds.n)
        old_of_new = np.lexsort((key2, ds.y))
        new_of_old = np.empty(ds.n, dtype=np.int64)
        new_of_old[old_of_new] = np.arange(ds.n)
        u, w = new_of_old[eu], new_of_old[ev]
        lo, hi = np.minimum(u, w), np.maximum(u, w)
        o = np.lexsort((hi, lo))
        eu, ev = lo[o].astype(np.int32), hi[o].astype(np.int32)
    t = time.time()
    plan = cg.partition(ds.n, eu, ev, a.p)
    print("partition s", round(time.time() - t, 1), flush=True)
    v = cg.plan_part(plan, a.part, copy=False)
    n, nnz = v["n_local"], v["nnz"]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for var in a.variants.split(";"):
        kv = dict(x.split(":") for x in var.split(",")) if var else {}
        for k, env in KNOBS.items():
            if k in kv:
                os.environ[env] = kv[k]
            else:
                os.environ.pop(env, None)
        cfg = cg.cfg_default(ds.dims, timing=0)
        parts = list(range(a.p))      # world = 1 hosts every part; part `--part` is timed
        ctx_plan = plan
        ws = torch.empty(cg.workspace_size(ctx_plan, parts, cfg), dtype=torch.uint8, device="cuda")
        ctx = cg.init(ctx_plan, parts, 0, 1, cfg, 0, ws)
        for ld in [int(x) for x in a.widths.split(",")]:
            T = torch.randn((n, ld), device="cuda")
            Y = torch.empty((n, ld), device="cuda")
            ts = []
            for r in range(a.reps + 1):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                cg.spmm(ctx, a.part, T, Y, ld, ld)
                e1.record()
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            gb = (4 * (n + 1) + 8 * nnz + 4 * ld * nnz + 4 * ld * n) / 1e9
            print(json.dumps({"config": a.config, "relabel": a.relabel, "p": a.p, "part": a.part, "ld": ld, "var": var,
                              "ms": round(ms, 4), "gather_GBps": round(gb / ms * 1e3, 1)}), flush=True)
            del T, Y
        ctx.close()
        del ws


if __name__ == "__main__":
    main()
