"""Multi-GPU halo replay, bitwise against the oracle (run under torchrun, one part per GPU).

Every rank draws the same seeded partials for all p = world parts, runs
cdfgnn_halo_exchange on its own part (NVLink push with slot-addressed messages, or NCCL
send/recv with compacted buffers), and replays the same sync with oracle.cache.sync in fp32
mode (reading R15).  Its synced rows, cache tables, send / fired / active flags, counters and
— slot layout — every received message (positions, lo/hi, codes) must be bit-identical to
the oracle's for its part (Alg. 2, §5).
    torchrun --nproc-per-node N tools/halo_replay_mgpu.py [--transport push|nccl]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--transport", default="push")
    ap.add_argument("--steps", type=int, default=4)
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2408_00232_b200 as cg
    from oracle.cache import SyncMode, SyncState, sync
    from oracle.partition import PartitionCfg, partition as opartition
    from synth import small_random_graph
    from tests.gpu_util import ws_view
    from tests.test_gpu_halo import read_messages, _same

    d = small_random_graph(3000, 20000, (8, 24, 6), seed=77)
    p = world
    plan = cg.partition(d.n, d.eu, d.ev, p)
    oplan = opartition(d.n, d.eu, d.ev, PartitionCfg(p=p))
    fails = []
    for cache, quant, eps, l in ((1, 8, 0.0, 1), (1, 8, 0.05, 1), (1, 0, 0.0, 2), (0, 8, 0.0, 1),
                                 (1, 4, 0.02, 1), (1, 16, 0.02, 2), (0, 0, 0.0, 2)):
        dims = (8, 24, 6)
        F = dims[l]
        ld = cg.ld_of(F)
        cfg = cg.cfg_default(dims, cache_on=cache, quant_bits=quant,
                             transport={"push": 0, "nccl": 1}[a.transport])
        ws = torch.empty(cg.workspace_size(plan, [rank], cfg), dtype=torch.uint8, device="cuda")
        uid = [cg.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = cg.init(plan, [rank], rank, world, cfg, local, ws, uid[0])
        st = SyncState(oplan, F, np.float32)
        mode = SyncMode(cache=bool(cache), quant_bits=quant, dtype=np.float32)
        rng = np.random.default_rng(1234 + quant + l)
        Xs = [rng.standard_normal((pp.n_local, F)).astype(np.float32) for pp in oplan.parts]
        tag = f"cache={cache} B={quant} eps={eps} l={l}"
        for step in range(a.steps):
            xp = np.zeros((Xs[rank].shape[0], ld), np.float32)
            xp[:, :F] = Xs[rank]
            dev = torch.from_numpy(xp).cuda()
            gst = cg.halo_exchange(ctx, l, 0, [dev], ld, np.float32(eps), stats=True)
            out, cnt = sync(oplan, st, [x.copy() for x in Xs], eps, mode)
            g = dev.cpu().numpy()
            if not np.array_equal(g[:, :F].view(np.uint32), out[rank].view(np.uint32)):
                fails.append(f"{tag} step {step}: synced rows")
            if cache:
                for which, ref in ((0, st.s_mir[rank]), (1, st.b_mir[rank]), (2, st.s_mas[rank]),
                                   (3, st.a[rank]), (4, st.b_mas[rank])):
                    ptr, rows, ldc = cg.cache_view(ctx, 0, l, 0, which)
                    if not np.array_equal(ws_view(ws, ptr, rows, ldc)[:, :F].view(np.uint32), ref.view(np.uint32)):
                        fails.append(f"{tag} step {step}: cache table {which}")
                pg, rg = cg.sync_flags(ctx, 0, l, 0, 0)
                if not np.array_equal(ws_view(ws, pg, rg, 1, np.uint8)[:, 0].astype(bool), cnt.gather_mask[rank]):
                    fails.append(f"{tag} step {step}: gather flags")
                pf, rf = cg.sync_flags(ctx, 0, l, 0, 1)
                if not np.array_equal(ws_view(ws, pf, rf, 1, np.uint8)[:, 0].astype(bool), cnt.master_fired_mask[rank]):
                    fails.append(f"{tag} step {step}: fired flags")
            # counters are global (this rank's share): compare the sums over ranks
            mine = torch.tensor([gst["gather_sent"], gst["scatter_msgs"], gst["active"]], dtype=torch.int64,
                                device="cuda")
            dist.all_reduce(mine)
            if mine.tolist() != [cnt.gather_sent, cnt.scatter_msgs, cnt.active]:
                fails.append(f"{tag} step {step}: counters {mine.tolist()} vs "
                             f"{[cnt.gather_sent, cnt.scatter_msgs, cnt.active]}")
            if a.transport == "push":
                # slot layout: the gather messages this master received and the scatter messages
                # this mirror received, byte for byte
                try:
                    for (src, dst), ref in cnt.gather_msgs.items():
                        if dst == rank:
                            _same(read_messages(ws, cg.msg_view(ctx, 0, 0, src), F, quant), ref, quant,
                                  f"gather {src}->{dst}")
                    for (src, dst), ref in cnt.scatter_msgs_rec.items():
                        if dst == rank:
                            _same(read_messages(ws, cg.msg_view(ctx, 0, 1, src), F, quant), ref, quant,
                                  f"scatter {src}->{dst}")
                except AssertionError as e:
                    fails.append(f"{tag} step {step}: {e}")
            Xs = [(x + (rng.random((x.shape[0], 1)) < 0.4) * 0.05 *
                   rng.standard_normal(x.shape)).astype(np.float32) for x in Xs]
        ctx.close()
        del ws
    bad = torch.tensor([len(fails)], dtype=torch.int64, device="cuda")
    dist.all_reduce(bad)
    for f in fails[:10]:
        print(json.dumps({"rank": rank, "fail": f}), flush=True)
    if rank == 0:
        print(json.dumps({"halo_replay": "PASS" if bad.item() == 0 else "FAIL", "world": world,
                          "transport": a.transport}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if bad.item() == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
