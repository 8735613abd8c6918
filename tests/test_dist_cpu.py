"""N > 1 host logic on CPU (gloo, world size 2): every rank derives the same
dataset and the same partition plan independently, the NCCL unique id travels
by broadcast_object_list, and bench's max-over-ranks reduction picks the slowest."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import paper_2408_00232_b200 as cg
    from synth import small_random_graph
    d = small_random_graph(1500, 8000, (8, 8, 4), seed=5)
    plan = cg.partition(d.n, d.eu, d.ev, world * 2)
    import hashlib
    h = hashlib.sha256()
    for b in [d.eu.tobytes(), d.X.tobytes(), plan.edge_part.tobytes(), plan.master.tobytes()] + \
            [cg.plan_part(plan, i)["local2global"].tobytes() for i in range(world * 2)]:
        h.update(b)
    digest = h.hexdigest()
    got = [None] * world
    dist.all_gather_object(got, digest)
    obj = [cg.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, len(set(got)), len(obj[0]), t.item()))
    dist.destroy_process_group()


def test_two_rank_host_logic():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ndigest, uid_len, mx in res:
        assert ndigest == 1          # identical plans on every rank
        assert uid_len == 128        # NCCL unique id broadcast intact
        assert mx == float(world)    # max over ranks


def _slot_worker(rank, world, port, q):
    """Each rank holds only its own part's view (as a GPU rank does) and checks, against the
    views the other ranks send over gloo, the invariant the slot-addressed exchange rests on:
    slot k of the (mirror part i -> master part j) region is the same vertex on both sides —
    i's k-th mirror of master j (its mirror slab, ascending gid, R21) and j's k-th entry of the
    halo list shared with i — and the master side's row is a boundary master of j."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2408_00232_b200 as cg
    from synth import small_random_graph
    d = small_random_graph(2500, 14000, (8, 8, 4), seed=6)
    plan = cg.partition(d.n, d.eu, d.ev, world)
    v = cg.plan_part(plan, rank)
    g = v["local2global"]
    B = v["n_bmaster"]
    mine = {"mirror": {j: g[B + v["mirror_off"][j]:B + v["mirror_off"][j + 1]].tolist() for j in range(world)},
            "halo": {s: g[v["halo_local"][v["halo_off"][s]:v["halo_off"][s + 1]]].tolist() for s in range(world)},
            "halo_rows": v["halo_local"].tolist(), "B": B}
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    ok = True
    for j in range(world):
        if j == rank:
            continue
        # my mirrors of master j, slot by slot, equal j's halo list shared with me
        ok &= allv[j]["halo"][rank] == mine["mirror"][j]
        # and j's halo rows are boundary masters of j
        ok &= all(0 <= r < allv[j]["B"] for r in allv[j]["halo_rows"])
        ok &= mine["mirror"][j] == sorted(mine["mirror"][j])
    q.put((rank, bool(ok), sum(len(x) for x in mine["mirror"].values())))
    dist.destroy_process_group()


def test_two_rank_slot_positions_agree():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_slot_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    assert sum(m for _, _, m in res) > 0        # the partition really has mirrors
