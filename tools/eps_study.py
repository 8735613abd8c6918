"""Adaptive-ε study (§8 f3, the analogue of PAPER.md Fig. 7) and the ε sweep
of BASELINE.json configs[3]: per-epoch send fraction per (layer, direction), ε, loss and
train accuracy, for fixed thresholds and the adaptive controller.

Runs the p partitions co-resident on one GPU (world = 1) so it needs a single B200.
    python tools/eps_study.py --config C3 --p 4 --epochs 60 --eps adaptive,0,0.01,0.1
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--epochs", type=int, default=60)
    ap.add_argument("--eps", default="adaptive,0,0.001,0.01,0.03,0.1,0.3")
    ap.add_argument("--quant", default="8", help="comma list of B (message bits; 0 = fp32)")
    ap.add_argument("--snr", type=float, default=1.0, help="synth feature SNR knob (class-mean scale)")
    ap.add_argument("--opt", default="adam")
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    from paper_2408_00232_b200.runtime import Run
    from synth import get_config
    from synth.cache import cached_dataset
    from bench import remote_split
    ds = cached_dataset(get_config(a.config), snr=a.snr)
    plan = None
    results = []
    for e, qb in [(e, int(q)) for q in a.quant.split(",") for e in a.eps.split(",")]:
        adaptive = e == "adaptive"
        eps0 = 0.01 if adaptive else float(e)
        run = Run(ds, a.p, cache=True, quant_bits=qb, eps0=eps0, adaptive=adaptive,
                  optimizer=a.opt, lr=a.lr, timing=False, plan=plan, static_inputs=True)
        plan = run.plan
        rows = []
        t0 = time.time()
        for ep in range(a.epochs):
            st = run.epoch()
            row = {"epoch": ep, "loss": st["loss"], "acc": st["acc"], "eps": st["eps_used"]}
            for d, name in ((st["fwd"], "fwd"), (st["bwd"], "bwd")):
                for l, s in enumerate(d):
                    base = max(s["baseline"], 1)
                    row[f"{name}{l + 1}_gather_frac"] = round(s["gather_sent"] / (base / 2), 4)
                    row[f"{name}{l + 1}_scatter_frac"] = round(s["scatter_msgs"] / (base / 2), 4)
            row["msgs"] = sum(s["gather_sent"] + s["scatter_msgs"] for s in st["fwd"] + st["bwd"])
            rs = remote_split(st, sum(v["n_mirror"] for v in run.views), run.cfg.L)
            row["avoided_cache"] = rs["avoided_by_cache"]
            row["avoided_elision"] = rs["avoided_by_elision"]
            row["baseline"] = sum(s["baseline"] for s in st["fwd"] + st["bwd"])
            row["bytes_alg"] = sum(s["bytes_alg"] for s in st["fwd"] + st["bwd"])
            rows.append(row)
        torch.cuda.synchronize()
        wall = time.time() - t0
        tot_m = sum(r["msgs"] for r in rows)
        tot_b = sum(r["baseline"] for r in rows)
        summary = {"config": a.config, "p": a.p, "eps": e, "quant_bits": qb, "snr": a.snr,
                   "optimizer": a.opt, "lr": a.lr, "epochs": a.epochs,
                   "final_loss": rows[-1]["loss"], "final_acc": rows[-1]["acc"],
                   "remote_accesses_avoided_frac": round(1 - tot_m / tot_b, 4),
                   "avoided_frac_cache": round(sum(r["avoided_cache"] for r in rows) / tot_b, 4),
                   "avoided_frac_elision": round(sum(r["avoided_elision"] for r in rows) / tot_b, 4),
                   "acc_epochs": [round(r["acc"], 4) for r in rows],
                   "eps_epochs": [r["eps"] for r in rows],
                   "bytes_alg_per_epoch": int(sum(r["bytes_alg"] for r in rows) / len(rows)),
                   "wall_s": round(wall, 2)}
        print(json.dumps(summary), flush=True)
        results.append({"summary": summary, "epochs": rows})
        run.close()
        run.workspace = None          # one workspace at a time (C4 p=4 co-resident needs ~96 GB)
        del run
        torch.cuda.empty_cache()
    out = a.out or os.path.join(ROOT, "profiles", f"eps_study_{a.config}_p{a.p}_snr{a.snr}.json")
    with open(out, "w") as f:
        json.dump({"source": "tools/eps_study.py", "paper": "Fig. 7 analogue (P:L843-879); "
                   "ε controller P:L386-399", "runs": results}, f)


if __name__ == "__main__":
    main()
