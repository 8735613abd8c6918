"""SpMM microbenchmark on a config's partition (cdfgnn_spmm through the C ABI).
    python tools/spmm_bench.py --config C3 --p 1 --panels 64,128,256"""
import argparse, os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--p", type=int, default=1)
    ap.add_argument("--panels", default="64,128,256")
    ap.add_argument("--widths", default="256,44")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="id:0,unr:0;id:1,unr:0",
                    help="';'-separated env settings: id=CDFGNN_SPMM_IDENTITY, unr=CDFGNN_SPMM_UNR")
    a = ap.parse_args()
    import torch
    import paper_2408_00232_b200 as cg
    from synth import get_config
    from synth.cache import cached_dataset
    ds = cached_dataset(get_config(a.config))
    t = time.time()
    plan = cg.partition(ds.n, ds.eu, ds.ev, a.p)
    print("partition s", round(time.time() - t, 1), flush=True)
    cfg = cg.cfg_default(ds.dims, timing=0)
    parts = list(range(a.p))
    ws = torch.empty(cg.workspace_size(plan, parts, cfg), dtype=torch.uint8, device="cuda")
    ctx = cg.init(plan, parts, 0, 1, cfg, 0, ws)
    v = cg.plan_part(plan, 0, copy=False)
    n, nnz = v["n_local"], v["nnz"]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for ld in [int(x) for x in a.widths.split(",")]:
        T = torch.randn((n, ld), device="cuda")
        Y = torch.empty((n, ld), device="cuda")
        for var in a.variants.split(";"):
          kv = dict(x.split(":") for x in var.split(","))
          os.environ["CDFGNN_SPMM_IDENTITY"] = kv.get("id", "0")
          os.environ["CDFGNN_SPMM_UNR"] = kv.get("unr", "0")
          if "tail" in kv:
              os.environ["CDFGNN_SPMM_TAIL"] = kv["tail"]
          else:
              os.environ.pop("CDFGNN_SPMM_TAIL", None)
          for pw in [int(x) for x in a.panels.split(",")]:
            os.environ["CDFGNN_SPMM_PANEL"] = str(pw)
            ts = []
            for r in range(a.reps + 1):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                cg.spmm(ctx, 0, T, Y, ld, ld)
                e1.record()
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            gb = (4 * (n + 1) + 8 * nnz + 4 * ld * nnz + 4 * ld * n) / 1e9
            print(json.dumps({"config": a.config, "p": a.p, "ld": ld, "panel": pw, "var": var, "ms": round(ms, 4),
                              "gather_GBps": round(gb / ms * 1e3, 1)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
