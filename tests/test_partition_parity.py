"""Host C++ partitioner (cdfgnn_partition, C ABI) vs the oracle — bit-exact.

Parity contract (BASELINE.json north_star): partition maps,
masters, local numbering, halo lists, CSR structure and fp32 Â weights identical.
Runs on CPU (host code only; no GPU call)."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2408_00232_b200 as cg
from oracle.partition import PartitionCfg, partition as opartition, stats as ostats
from synth import get_config, make_dataset, small_random_graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "cdfgnn.h")).read()
    declared = set(re.findall(r"\b(cdfgnn_[a-z0-9_]+)\s*\(", hdr))
    lib = os.path.join(ROOT, "paper_2408_00232_b200", "libcdfgnn.so")
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (cdfgnn_[a-z0-9_]+)", out))
    assert declared, "no declarations parsed"
    assert declared <= exported, f"missing: {sorted(declared - exported)}"
    undefined = subprocess.run(["nm", "-D", "--undefined-only", lib], capture_output=True, text=True).stdout
    assert "cdfgnn" not in undefined, "library references cdfgnn symbols it does not define"


def _compare(d, p, hosts=1, order=1, oorder="degsum", gamma=(1, 10), self_loops=False, seed=0):
    plan = cg.partition(d.n, d.eu, d.ev, p, num_hosts=hosts, edge_order=order, gamma=gamma,
                        self_loops=self_loops, seed=seed)
    op = opartition(d.n, d.eu, d.ev, PartitionCfg(p=p, num_hosts=hosts, edge_order=oorder,
                                                  gamma=gamma, self_loops=self_loops, seed=seed))
    assert np.array_equal(plan.edge_part, op.edge_part)
    assert np.array_equal(plan.master, op.master)
    for i in range(p):
        v = cg.plan_part(plan, i)
        o = op.parts[i]
        assert v["n_bmaster"] == o.n_bmaster and v["n_mirror"] == o.n_mirror
        assert np.array_equal(v["local2global"], o.local2global)
        assert np.array_equal(v["mirror_off"], o.mirror_off)
        assert np.array_equal(v["rowptr"], o.rowptr)
        assert np.array_equal(v["colidx"], o.colidx)
        assert np.array_equal(v["val"].view(np.uint32), o.val32.view(np.uint32))
        assert v["n_edges"] == o.n_edges
        hl = [o.halo_master[s] if s != i else np.zeros(0, np.int64) for s in range(p)]
        assert np.array_equal(v["halo_local"], np.concatenate(hl))
        assert np.array_equal(v["halo_off"], np.concatenate([[0], np.cumsum([len(x) for x in hl])]))
    s = cg.plan_stats(plan)
    os_ = ostats(op)
    assert abs(s["rf"] - os_.rf) < 1e-12 and abs(s["edge_if"] - os_.edge_if) < 1e-12
    assert abs(s["vertex_if"] - os_.vertex_if) < 1e-12
    assert s["inner_max"] == os_.inner_max and s["outer_max"] == os_.outer_max
    assert s["total_mirrors"] == os_.total_mirrors


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_random_graphs(p):
    d = small_random_graph(700, 3000, (4, 3), seed=100 + p)
    _compare(d, p)


@pytest.mark.parametrize("hosts,order,oorder", [(2, 0, "input"), (2, 2, "shuffle"), (4, 1, "degsum")])
def test_hosts_and_orders(hosts, order, oorder):
    d = small_random_graph(500, 2000, (4, 3), seed=7)
    _compare(d, 4, hosts=hosts, order=order, oorder=oorder, seed=99)


def test_self_loops_and_gamma0():
    d = small_random_graph(300, 1000, (4, 3), seed=8)
    _compare(d, 3, self_loops=True)
    _compare(d, 3, gamma=(0, 1))


@pytest.mark.parametrize("p", [2, 8])
def test_config_C1(p):
    _compare(make_dataset(get_config("C1")), p)


@pytest.mark.slow
def test_config_C2_p2():
    _compare(make_dataset(get_config("C2")), 2)


def test_input_errors():
    eu = np.array([0, 1], np.int32)
    ev = np.array([1, 1], np.int32)
    with pytest.raises(cg.CdfgnnError) as e:
        cg.partition(3, eu, ev, 2)
    assert e.value.code == 3            # self-loop -> EDATA
    with pytest.raises(cg.CdfgnnError) as e:
        cg.partition(3, np.array([0, 0], np.int32), np.array([1, 1], np.int32), 2)
    assert e.value.code == 3            # duplicate
    with pytest.raises(cg.CdfgnnError) as e:
        cg.partition(3, np.array([0], np.int32), np.array([5], np.int32), 2)
    assert e.value.code == 3            # out of range
    with pytest.raises(cg.CdfgnnError) as e:
        cg.partition(3, np.array([0], np.int32), np.array([1], np.int32), 0)
    assert e.value.code == 2            # p < 1 -> EUSAGE


def test_context_usage_errors_without_gpu():
    """Config validation happens on the host (cdfgnn_workspace_size, no device touched): layer
    widths above 1024, more than 256 classes, message widths other than 0/4/8/16 bits, an empty
    edge list, and k outside [1, p] are EUSAGE."""
    from synth import small_random_graph
    d = small_random_graph(200, 800, (8, 16, 4), seed=3)
    plan = cg.partition(d.n, d.eu, d.ev, 2)
    ok = cg.cfg_default((8, 16, 256))
    assert cg.workspace_size(plan, [0, 1], ok) > 0                 # 256 classes: the maximum
    for dims, kw in (((8, 1025, 4), {}), ((8, 16, 257), {}), ((8, 16, 4), {"quant_bits": 12}),
                     ((8, 16, 4), {"quant_bits": 2}), ((8, 16, 4), {"msg_layout": 3})):
        with pytest.raises(cg.CdfgnnError) as e:
            cg.workspace_size(plan, [0, 1], cg.cfg_default(dims, **kw))
        assert e.value.code == 2, (dims, kw)
    with pytest.raises(cg.CdfgnnError) as e:
        cg.workspace_size(plan, [0, 1, 2], cg.cfg_default((8, 16, 4)))
    assert e.value.code == 2                                         # k > p
    with pytest.raises(cg.CdfgnnError) as e:
        cg.partition(3, np.zeros(0, np.int32), np.zeros(0, np.int32), 2)
    assert e.value.code == 2                                         # m == 0
