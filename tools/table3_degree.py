"""Why γ = 0.1 cuts outer connections on some graphs and not others (Table 3 analogue, §8 f4).

P:L799 claims γ = 0.1 reduces the outer (cross-host) connections by 31.08 % on average on
the paper's datasets; on the synthetic C3 / C5 shapes it raised them (profiles/
table3_synthetic.json).  This sweep separates the two suspects the round-1 verdict named:
the mean degree (the C3 shape regenerated with fewer edges, same degree law and
homophily) and the streaming edge order (input order, ascending degree sum — the default,
reading R19 —, seeded shuffle).  2 hosts x 2 GPUs, host-only (C++ partitioner via the C ABI).

    python tools/table3_degree.py [--n 232965] [--degrees 16,64,256,492] [--out ...]
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
    ap.add_argument("--n", type=int, default=60000)
    ap.add_argument("--degrees", default="8,32,128,492")
    ap.add_argument("--layout", default="2x2")
    ap.add_argument("--orders", default="0,1,2")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "table3_degree_sweep.json"))
    a = ap.parse_args()
    import numpy as np
    import paper_2408_00232_b200 as cg
    from synth import chung_lu_planted, get_config
    c3 = get_config("C3")
    hosts, gph = (int(x) for x in a.layout.split("x"))
    p = hosts * gph
    rows = []
    for deg in [int(x) for x in a.degrees.split(",")]:
        m = a.n * deg // 2
        v0 = c3.v0 * a.n / c3.n
        rng = np.random.default_rng(0xCDF6 + deg)
        eu, ev, _ = chung_lu_planted(a.n, m, c3.tau, max(v0, 1.0), c3.classes, c3.homophily, rng)
        for order in [int(x) for x in a.orders.split(",")]:
            res = {"n": a.n, "mean_degree": deg, "edge_order": ["input", "degree_sum", "shuffle"][order],
                   "layout": a.layout}
            for gname, gamma in (("gamma0", (0, 1)), ("gamma01", (1, 10))):
                t = time.time()
                plan = cg.partition(a.n, eu, ev, p, num_hosts=hosts, gamma=gamma, edge_order=order, seed=7)
                st = cg.plan_stats(plan)
                res[gname] = {"inner": st["inner_max"], "outer": st["outer_max"], "rf": round(st["rf"], 4),
                              "edge_if": round(st["edge_if"], 4), "s": round(time.time() - t, 1)}
                del plan
            o0, o1 = res["gamma0"]["outer"], res["gamma01"]["outer"]
            res["outer_reduction_pct"] = round(100.0 * (1 - o1 / o0), 2) if o0 else None
            print(json.dumps(res), flush=True)
            rows.append(res)
    with open(a.out, "w") as f:
        json.dump({"source": "tools/table3_degree.py", "paper_claim_pct": 31.08, "paper_cite": "P:L799",
                   "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
