"""Co-resident halo benchmark: p partitions of a config on ONE GPU (world = 1), full
epochs through cdfgnn_epoch with phase timing; used for single-GPU ncu captures of the
halo kernels (ncu must never wrap a multi-rank command).
    python tools/halo_bench.py --config C3 --p 4 --epochs 3"""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--mode", default="cache_int8")
    ap.add_argument("--overlap", type=int, default=0)
    ap.add_argument("--fuse", type=int, default=1, help="cfg.fuse_gather (gather in the SpMM epilogue)")
    a = ap.parse_args()
    import torch
    from paper_2408_00232_b200.runtime import Run
    from synth import get_config
    from synth.cache import cached_dataset
    ds = cached_dataset(get_config(a.config))
    cache, quant = {"cache_int8": (True, 8), "cache_fp32": (True, 0), "quant_only": (False, 8),
                    "nocache": (False, 0)}[a.mode]
    run = Run(ds, a.p, cache=cache, quant_bits=quant, timing=True, overlap=bool(a.overlap),
              static_inputs=True, fuse_gather=bool(a.fuse))
    import torch
    tot = []
    for e in range(a.epochs):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st = run.epoch()
        e1.record(); torch.cuda.synchronize()
        tot.append(e0.elapsed_time(e1))
        print(json.dumps({"epoch": e, "loss": st["loss"], "gemm": round(st["ms_gemm"], 3),
                          "spmm": round(st["ms_spmm"], 3), "sync": round(st["ms_sync"], 3),
                          "sync_split": [round(x, 3) for x in st["ms_sync_sub"]]}), flush=True)
    print(json.dumps({"fuse": a.fuse, "median_epoch_ms": sorted(tot[2:])[len(tot[2:]) // 2] if len(tot) > 2 else None}))
    run.close()


if __name__ == "__main__":
    main()
