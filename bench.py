#!/usr/bin/env python
"""Benchmark: full-batch GCN epoch of the CDFGNN hot path on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--mode cache_int8]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one partition per GPU)
    python bench.py --impl reference ...                        (the CPU oracle, timed)

A step is one Alg. 1 iteration over the whole synthetic
graph: per layer GEMM + local SpMM + cached/quantised halo exchange, loss on
masters, backward with the δ exchanges, dW allreduce, Adam, ε update.
Prints ONE JSON line on rank 0 (contract in DESIGN.md §Measurement).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full-batch GCN epoch ms at 1/2/4/8 B200; comm bytes/epoch; SpMM GB/s vs HBM"
FALLBACK_HBM_GBS = 6650.0        # B200_PROFILING.md fallback (used only without MEASURED_PEAKS.json)
NVLINK_GBS = 900.0               # nominal per direction per GPU


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cdfgnn", choices=["cdfgnn", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--mode", default="cache_int8",
                    choices=["cache_int8", "cache_fp32", "quant_only", "nocache"])
    ap.add_argument("--eps0", type=float, default=0.01)
    ap.add_argument("--transport", default="push", choices=["push", "nccl"])
    ap.add_argument("--overlap", action="store_true",
                    help="boundary-rows-first scheduling (gather phase on a second stream; off by default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--hoisted", type=int, default=1,
                    help="1: also time the hoisted-input-aggregation schedule (static_inputs = 2) and "
                         "report it under 'hoisted' (the headline keeps the per-epoch schedule)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-frac", type=float, default=0.01)
    ap.add_argument("--scale", type=float, default=None, help="shrink the graph (tests only)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": FALLBACK_HBM_GBS}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle leg
class OracleSample:
    """Estimated ms of one oracle epoch (oracle/gcn.py, fp64, p = 1) on this host.

    Sample: every dense op (GEMMs, ReLU, loss) runs at full size on operands of the
    right shape; each SpMM (scipy CSR, single-threaded) runs on a random `frac` row
    sample of Â and is scaled by 1/frac.  Â is built once, outside the timing."""

    def __init__(self, ds, frac):
        import numpy as np
        from oracle.graph import normalized_adjacency
        self.ds, self.frac = ds, frac
        self.A = normalized_adjacency(ds.n, ds.eu, ds.ev)
        self.W = [w.astype(np.float64) for w in ds.W]
        self.X = ds.X.astype(np.float64)

    def epoch_ms(self, seed=0):
        import numpy as np
        from oracle import gcn
        ds, frac, W = self.ds, self.frac, self.W
        rng = np.random.default_rng(seed)
        rows = np.sort(rng.choice(ds.n, max(1, int(frac * ds.n)), replace=False))
        As = self.A[rows]
        L = len(W)
        t_dense = 0.0
        t_spmm = 0.0
        H = [self.X]
        for l in range(1, L + 1):
            t0 = time.perf_counter(); T = H[l - 1] @ W[l - 1]; t_dense += time.perf_counter() - t0
            t0 = time.perf_counter(); _ = As @ T; t_spmm += time.perf_counter() - t0
            t0 = time.perf_counter(); Hn = gcn.relu(T) if l < L else T
            t_dense += time.perf_counter() - t0
            H.append(Hn)
        t0 = time.perf_counter()
        _, delta, _ = gcn.loss_grad(H[L], ds.y, ds.train)
        t_dense += time.perf_counter() - t0
        for l in range(L, 0, -1):
            t0 = time.perf_counter(); _ = As @ delta; t_spmm += time.perf_counter() - t0
            S = delta                                   # full-size stand-in of Â δ
            t0 = time.perf_counter()
            _ = H[l - 1].T @ S
            if l > 1:
                delta = (S @ W[l - 1].T) * (H[l - 1] > 0)
            t_dense += time.perf_counter() - t0
        return 1e3 * (t_dense + t_spmm / frac)


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def workload_config(cfgc, ds, args, world):
    """The config keys both arms report (same workload, mode and partitioning)."""
    return {"workload": f"{cfgc.key} {cfgc.name}: {ds.n} V, {2 * ds.m} CSR nnz, "
                        f"dims {'-'.join(map(str, cfgc.dims))}",
            "mode": args.mode, "partitions": world, "parallelism": f"vertex-cut p{world}",
            "l2": "inputs larger than L2 (CSR %.2f GB, X %.2f GB)" % (2 * ds.m * 8 / 1e9, ds.X.nbytes / 1e9)}


def reference_main(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from synth import get_config
    from synth.cache import cached_dataset
    ds = cached_dataset(get_config(args.config), args.scale)
    orc = OracleSample(ds, args.cpu_frac)
    for _ in range(args.warmup):
        orc.epoch_ms(seed=1)
    vals = [orc.epoch_ms(seed=2 + k) for k in range(args.steps)]
    v = statistics.mean(vals)
    sample = (f"oracle epoch (oracle/gcn.py fp64, p=1) on {args.config}: dense ops full size, "
              f"each SpMM on a {args.cpu_frac:.0%} row sample scaled by {1 / args.cpu_frac:.0f}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {**workload_config(get_config(args.config), ds, args, args.gpus),
                                        "oracle": "unpartitioned p=1 epoch, fp64 (the same Alg. 1 "
                                                  "arithmetic in exact mode)"},
        "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": cpu_cores(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


# ------------------------------------------------------------------ GPU leg
def main(args):
    if args.impl == "reference":
        return reference_main(args)
    # stdout carries exactly one JSON line: native libraries (NCCL's version banner) write to
    # fd 1 during the run, so fd 1 points at stderr until the line is printed
    sys.stdout.flush()
    real_stdout = os.dup(1)
    os.dup2(2, 1)
    try:
        return _main(args, real_stdout)
    finally:
        sys.stdout.flush()
        os.dup2(real_stdout, 1)
        os.close(real_stdout)


def _main(args, real_stdout):
    import numpy as np
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2408_00232_b200.runtime import Run
    from synth import get_config
    from synth.cache import cached_dataset
    cfgc = get_config(args.config)
    t_prep = time.time()
    if rank == 0:
        ds = cached_dataset(cfgc, args.scale)
    if dist is not None:
        dist.barrier()
    if rank != 0:
        ds = cached_dataset(cfgc, args.scale, wait_for_writer=True, write=False)
    mode = {"cache_int8": (True, 8), "cache_fp32": (True, 0), "quant_only": (False, 8),
            "nocache": (False, 0)}[args.mode]
    run = Run(ds, world, rank=rank, world=world, device=local, cache=mode[0], quant_bits=mode[1],
              eps0=args.eps0, adaptive=True, optimizer="adam", lr=0.01, timing=True,
              host_inputs=not args.no_e2e, transport=args.transport, static_inputs=True,
              overlap=args.overlap)
    t_prep = time.time() - t_prep
    for _ in range(args.warmup):
        run.epoch()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0.record(stream)
    stats = [run.epoch() for _ in range(args.steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    ms = e0.elapsed_time(e1) / args.steps

    def allred(vals, op):
        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(t, op=op)
        return t.tolist()

    sumop = dist.ReduceOp.SUM if dist else None
    maxop = dist.ReduceOp.MAX if dist else None
    ms_max = allred([ms], maxop)[0]
    comm_alg = sum(sum(s["bytes_alg"] for s in st["fwd"] + st["bwd"]) for st in stats) / args.steps
    comm_wire = sum(sum(s["bytes_wire"] for s in st["fwd"] + st["bwd"]) for st in stats) / args.steps
    remote = sum(sum(s["gather_sent"] + s["scatter_msgs"] for s in st["fwd"] + st["bwd"])
                 for st in stats) / args.steps
    base = sum(sum(s["baseline"] for s in st["fwd"] + st["bwd"]) for st in stats) / args.steps
    sp_bytes = sum(st["spmm_bytes"] for st in stats)
    sp_ms = sum(st["spmm_ms_sum"] for st in stats)
    sp_n = sum(st["spmm_launches"] for st in stats)
    ms_sync = sum(st["ms_sync"] for st in stats) / args.steps
    ms_spmm = sum(st["ms_spmm"] for st in stats) / args.steps
    ms_gemm = sum(st["ms_gemm"] for st in stats) / args.steps
    sync_sub = [round(sum(st["ms_sync_sub"][i] for st in stats) / args.steps, 3) for i in range(6)]
    tot = allred([comm_alg, comm_wire, remote, base], sumop)
    max_wire = allred([comm_wire], maxop)[0]
    ms_sync_max = allred([ms_sync], maxop)[0]
    launches = sum(st["gpu_launches"] for st in stats)
    # ---- end to end through the public API with host inputs (pinned), copies inside the region
    e2e = None
    if not args.no_e2e:
        def timed_host_loop(pipelined):
            if pipelined:
                run.epoch_host_next(prefetch_next=False)
            else:
                run.epoch_host()
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            e0.record(stream)
            for k in range(args.steps):
                if pipelined:
                    # step k's inputs were copied under step k-1 (step 0 copies its own inside the
                    # region); step k starts the copy of step k+1's — all K copies are timed
                    run.epoch_host_next(prefetch_next=k + 1 < args.steps)
                else:
                    run.epoch_host()
            e1.record(stream)
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            return allred([e0.elapsed_time(e1) / args.steps], maxop)[0]
        e2e_serial_ms = timed_host_loop(False)
        e2e_ms = timed_host_loop(True)
        # bytes the pipelined host path copies per step: at N > 1 only each part's owned X rows
        # (its M mirror rows arrive from their masters over NVLink), plus labels and masks
        h2d = 0
        for pv, x, y, m in zip(run.views, run.X_host, run.labels_host, run.masks_host):
            owned = pv["n_local"] - (pv["n_mirror"] if world > 1 else 0)
            h2d += owned * x.shape[1] * x.element_size() + y.numel() * y.element_size() + m.numel() * m.element_size()
        k = len(run.parts)
        d2h = 8 * k + 8 + 8 * 4 * 2 * run.cfg.L
        h2d_all = allred([h2d, d2h], sumop)
        e2e = {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": int(h2d_all[0]),
               "d2h_bytes_per_step": int(h2d_all[1]),
               "api": "cdfgnn_epoch_host_next: next step's pinned host inputs copied on a copy "
                      "stream under the current epoch; at N > 1 each vertex's features cross PCIe "
                      "once (owned rows) and reach its mirrors over NVLink (NCCL)",
               "serial_value": round(e2e_serial_ms, 3)}
    run.close()
    plan = run.plan
    run.workspace = None
    # ---- the same workload with the layer-1 aggregation hoisted (static_inputs = 2): Â_i X_i is
    # built once per X buffer, layer 1 runs (Â_i X_i) W^(0) and ∇W^(0) = (Â_i X_i)ᵀ δ^(1)
    hoist = None
    if args.hoisted:
        run2 = Run(ds, world, rank=rank, world=world, device=local, cache=mode[0], quant_bits=mode[1],
                   eps0=args.eps0, adaptive=True, optimizer="adam", lr=0.01, timing=True,
                   host_inputs=False, transport=args.transport, static_inputs=2, overlap=args.overlap,
                   plan=plan)
        for _ in range(args.warmup):
            run2.epoch()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e0.record(stream)
        st2 = [run2.epoch() for _ in range(args.steps)]
        e1.record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        h_ms = allred([e0.elapsed_time(e1) / args.steps], maxop)[0]
        hoist = {"value": round(h_ms, 3), "unit": "ms", "loss": st2[-1]["loss"],
                 "gpu_launches": sum(x["gpu_launches"] for x in st2),
                 "phase_ms": {k: round(sum(x["ms_" + k] for x in st2) / args.steps, 3)
                              for k in ("gemm", "spmm", "sync")},
                 "schedule": "static_inputs=2: A_i X_i aggregated once per X buffer (init), layer 1 "
                             "= (A_i X_i) W0, dW0 = (A_i X_i)^T delta1; same method, both layer-1 "
                             "SpMMs leave the epoch"}
        run2.close()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0
    # L2 read bandwidth on this GPU (the gather-bound SpMM's real ceiling): 64 MB resident buffer
    from paper_2408_00232_b200.api import bandwidth_probe
    probe = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    l2_gbs = bandwidth_probe(probe, 64 << 20, 64)
    del probe
    peaks, src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    sp_ld = stats[-1]["spmm_ld"]
    sp_c = sum(st["spmm_bytes_compulsory"] for st in stats)
    achieved = (sp_bytes / (sp_ms * 1e-3) / 1e9) if sp_ms > 0 else None
    avg_launch_ms = sp_ms / sp_n if sp_n else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.config}_p{world}_{args.mode}_spmm_ld{sp_ld}")
        except Exception:
            traffic = None
    out = {
        "metric": METRIC, "value": round(ms_max, 3), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {**workload_config(cfgc, ds, args, world),
                   "transport": ["none", "nccl", "nvlink-push"][stats[-1]["transport"]],
                   "overlap": args.overlap and world > 1 and stats[-1]["transport"] != 1},
        "comm_bytes_per_epoch": int(tot[0]), "comm_wire_bytes_per_epoch": int(tot[1]),
        "remote_accesses_per_epoch": int(tot[2]), "remote_accesses_baseline": int(tot[3]),
        "remote_accesses_avoided_frac": round(1 - tot[2] / tot[3], 4) if tot[3] else None,
        "nvlink": {"max_wire_bytes_per_gpu": int(max_wire), "sync_ms": round(ms_sync_max, 3),
                   "frac_of_900": round(max_wire / (ms_sync_max * 1e-3) / 1e9 / NVLINK_GBS, 4)
                   if ms_sync_max > 0 and max_wire > 0 else None},
        "phase_ms": {"gemm": round(ms_gemm, 3), "spmm": round(ms_spmm, 3), "sync": round(ms_sync, 3),
                     "sync_split": dict(zip(["gather_pack", "gather_xfer", "master_apply",
                                             "scatter_pack", "scatter_xfer", "mirror_apply"], sync_sub))},
        "loss": stats[-1]["loss"], "train_acc": stats[-1]["acc"], "eps": stats[-1]["eps_used"],
        "roofline": {"kernel": f"spmm (ld={sp_ld}, the dominant launch group)", "bound": "hbm",
                     "achieved": round(achieved, 1) if achieved else None, "peak": hbm,
                     "unit": "GB/s", "frac": round(achieved / hbm, 4) if achieved else None,
                     "traffic": traffic, "peak_source": src,
                     "bytes_model": "gather model per launch: 4(n+1) + 8 nnz + 4 ld nnz + 4 ld n",
                     "bytes_per_launch": round(sp_bytes / sp_n) if sp_n else None,
                     "compulsory_bytes_per_launch": round(sp_c / sp_n) if sp_n else None,
                     "avg_launch_ms": round(avg_launch_ms, 4) if avg_launch_ms else None,
                     "dram_gbs": round(traffic / (avg_launch_ms * 1e-3) / 1e9, 1)
                     if (traffic and avg_launch_ms) else None,
                     "l2_read_gbs_probe": round(l2_gbs, 1),
                     "frac_of_l2": round(achieved / l2_gbs, 4) if achieved else None,
                     "launches": sp_n},
        "gpu_launches": launches,
        "prep_s": round(t_prep, 1),
    }
    if e2e:
        out["e2e"] = e2e
    if hoist:
        out["hoisted"] = hoist
    if clk:
        out["clocks"] = clk
    if world == 1 and not args.no_cpu_baseline:
        v = OracleSample(ds, args.cpu_frac).epoch_ms()
        out["cpu_baseline"] = {
            "value": round(v, 1), "unit": "ms", "cores": cpu_cores(), "kind": "oracle",
            "sample": f"oracle/gcn.py epoch (fp64, p=1): dense ops full size, each SpMM on a "
                      f"{args.cpu_frac:.0%} row sample scaled by {1 / args.cpu_frac:.0f} "
                      f"(scipy CSR single-threaded, numpy BLAS multi-threaded)"}
    sys.stdout.flush()
    os.write(real_stdout, (json.dumps(out) + "\n").encode())
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main(parse()))
