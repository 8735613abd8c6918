"""Table 3 analogue (§8 f4): hierarchical EBV with γ = 0 vs γ = 0.1 on the synthetic
shapes, with the paper's host x GPU layouts (claim P:L799:
"Setting γ to 0.1 can greatly reduce the number of outer connections (31.08% on
average)").  Host-only (C++ partitioner through the C ABI).

    python tools/table3.py [--configs C3:2x2,C4:2x4,C5:2x8] [--out profiles/table3_synthetic.json]
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
    ap.add_argument("--configs", default="C3:2x2,C4:2x4,C5:2x8")
    ap.add_argument("--scale", type=float, default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "table3_synthetic.json"))
    a = ap.parse_args()
    import paper_2408_00232_b200 as cg
    from synth import get_config
    from synth.cache import cached_dataset
    rows = []
    for item in a.configs.split(","):
        key, lay = item.split(":")
        hosts, gph = (int(x) for x in lay.split("x"))
        p = hosts * gph
        t0 = time.time()
        ds = cached_dataset(get_config(key), a.scale)
        res = {"config": key, "n": ds.n, "m": ds.m, "nodes": hosts, "gpus_per_node": gph}
        for gname, gamma in (("gamma0", (0, 1)), ("gamma01", (1, 10))):
            t = time.time()
            plan = cg.partition(ds.n, ds.eu, ds.ev, p, num_hosts=hosts, gamma=gamma)
            st = cg.plan_stats(plan)
            res[gname] = {"inner": st["inner_max"], "outer": st["outer_max"], "rf": round(st["rf"], 4),
                          "edge_if": round(st["edge_if"], 4), "vertex_if": round(st["vertex_if"], 4),
                          "partition_s": round(time.time() - t, 1)}
            del plan
        o0, o1 = res["gamma0"]["outer"], res["gamma01"]["outer"]
        res["outer_reduction_pct"] = round(100.0 * (1 - o1 / o0), 2) if o0 else None
        res["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps(res), flush=True)
        rows.append(res)
    red = [r["outer_reduction_pct"] for r in rows if r["outer_reduction_pct"] is not None]
    out = {"source": "tools/table3.py (C++ EBV partitioner, synthetic graphs of SURVEY §8(d2))",
           "paper_claim_pct": 31.08, "paper_cite": "P:L799, Table 3 P:L701-734",
           "mean_outer_reduction_pct": round(sum(red) / len(red), 2) if red else None, "rows": rows}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({"mean_outer_reduction_pct": out["mean_outer_reduction_pct"]}))


if __name__ == "__main__":
    main()
