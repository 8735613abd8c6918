"""Hierarchical EBV vertex-cut partitioner, plan construction and statistics (oracle O2).

Follows §6 of the paper step by step:
  * P:L612-618 (eq. Eva):  Eva_{(u,v)}(i) = (1-γ)(𝟙[i∉d_rep_u] + 𝟙[i∉d_rep_v])
        + γ(𝟙[host_i∉h_rep_u] + 𝟙[host_i∉h_rep_v]) + α e_count[i]/(|E|/p)
        + β v_count[i]/(|V|/p)
  * d_rep / h_rep / e_count / v_count bookkeeping.
  * "we assign it edge by edge ... select the GPU ID that minimizes the
    evaluation function".
  * replication factor, edge and vertex imbalance factors.
  * P:L196 / P:L295: one replica is chosen as master (reading R20: the first part
    the vertex is assigned to).  P:L327-329: local renumbering (reading R21).
  * Table 3 "Inner"/"Outer" = max over subgraphs of messages sent from
    that device to the same / another host.

Scores are evaluated EXACTLY: Eva is multiplied by gd*ad*bd*|E|*|V| (γ = gn/gd,
α = an/ad, β = bn/bd) so every comparison is an integer comparison and ties go
to the lowest part id (reading R20).  ``eva_exact`` keeps the paper's real-valued
form (fractions) and is what the integer form is pinned against.
Pins: tests/test_oracle_partition.py.
"""
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Dict, List, Optional, Tuple

import numpy as np

from .graph import degrees, edge_weight

MASK64 = (1 << 64) - 1


@dataclass
class PartitionCfg:
    p: int
    num_hosts: int = 1
    host_of: Optional[List[int]] = None      # part -> host; default i * num_hosts // p
    alpha: Tuple[int, int] = (1, 1)
    beta: Tuple[int, int] = (1, 1)
    gamma: Tuple[int, int] = (1, 10)
    edge_order: str = "degsum"               # "input" | "degsum" | "shuffle"   (reading R19)
    seed: int = 0
    self_loops: bool = False

    def hosts(self) -> List[int]:
        if self.host_of is not None:
            return list(self.host_of)
        return [i * self.num_hosts // self.p for i in range(self.p)]


def splitmix64(x: int) -> int:
    """Counter-based generator used for the 'shuffle' edge order (both sides implement it)."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def edge_order(n: int, eu: np.ndarray, ev: np.ndarray, cfg: PartitionCfg) -> np.ndarray:
    """Streaming order of the edges (reading R19; the paper leaves it unstated)."""
    m = len(eu)
    if cfg.edge_order == "input":
        return np.arange(m)
    if cfg.edge_order == "degsum":
        d = degrees(n, eu, ev)
        a = np.minimum(eu, ev).astype(np.int64)
        b = np.maximum(eu, ev).astype(np.int64)
        # ascending (d_u + d_v), ties by (min id, max id)
        return np.lexsort((b, a, d[eu] + d[ev]))
    if cfg.edge_order == "shuffle":
        keys = [(splitmix64((cfg.seed ^ (e * 0xD1B54A32D192ED03)) & MASK64), e) for e in range(m)]
        keys.sort()
        return np.array([e for _, e in keys], dtype=np.int64)
    raise ValueError(cfg.edge_order)


def eva_exact(u: int, v: int, i: int, d_rep: List[set], h_rep: List[set], host_of: List[int],
              e_count: List[int], v_count: List[int], E: int, V: int, p: int,
              alpha=Fraction(1), beta=Fraction(1), gamma=Fraction(1, 10)) -> Fraction:
    """Eva_{(u,v)}(i) exactly as printed, in rational arithmetic."""
    alpha, beta, gamma = Fraction(alpha), Fraction(beta), Fraction(gamma)
    rep = int(i not in d_rep[u]) + int(i not in d_rep[v])
    hst = int(host_of[i] not in h_rep[u]) + int(host_of[i] not in h_rep[v])
    return ((1 - gamma) * rep + gamma * hst
            + alpha * Fraction(e_count[i] * p, E) + beta * Fraction(v_count[i] * p, V))


def ebv_partition(n: int, eu: np.ndarray, ev: np.ndarray, cfg: PartitionCfg):
    """Assign every edge to a part and pick masters (reading R20).

    Returns (edge_part int32[m], master int32[n])."""
    p = cfg.p
    m = len(eu)
    if p < 1 or m == 0:
        raise ValueError("p >= 1 and m >= 1 required")
    host = cfg.hosts()
    gn, gd = cfg.gamma
    an, ad = cfg.alpha
    bn, bd = cfg.beta
    E, V = m, n
    # integer coefficients of Eva * (gd*ad*bd*E*V)
    c_rep = (gd - gn) * ad * bd * E * V
    c_host = gn * ad * bd * E * V
    c_e = an * gd * bd * p * V
    c_v = bn * gd * ad * p * E
    d_rep = [0] * n          # bitmask of parts holding a replica of the vertex
    h_rep = [0] * n          # bitmask of hosts holding a replica
    e_count = [0] * p
    v_count = [0] * p
    master = [-1] * n
    edge_part = np.empty(m, dtype=np.int32)
    eu_l = eu.tolist(); ev_l = ev.tolist()
    for e in edge_order(n, eu, ev, cfg).tolist():
        u, v = eu_l[e], ev_l[e]
        du, dv, hu, hv = d_rep[u], d_rep[v], h_rep[u], h_rep[v]
        best = None
        bi = 0
        for i in range(p):
            bit = 1 << i
            hb = 1 << host[i]
            rep = (0 if du & bit else 1) + (0 if dv & bit else 1)
            hst = (0 if hu & hb else 1) + (0 if hv & hb else 1)
            s = c_rep * rep + c_host * hst + c_e * e_count[i] + c_v * v_count[i]
            if best is None or s < best:     # strict: ties keep the lowest id
                best = s
                bi = i
        edge_part[e] = bi
        e_count[bi] += 1
        bit = 1 << bi
        for x in (u, v):
            if not d_rep[x] & bit:
                d_rep[x] |= bit
                v_count[bi] += 1
                if master[x] < 0:
                    master[x] = bi           # master = first-assigned part (R20)
            h_rep[x] |= 1 << host[bi]
    # isolated vertices: after all edges, to argmin v_count (ties lowest id)  (R20)
    for x in range(n):
        if master[x] < 0:
            bi = min(range(p), key=lambda i: (v_count[i], i))
            master[x] = bi
            v_count[bi] += 1
    return edge_part, np.asarray(master, dtype=np.int32)


@dataclass
class PartPlan:
    """One subgraph in local numbering (reading R21):
    [boundary masters ↑gid][mirrors grouped by master part ↑, then ↑gid][interior ↑gid]."""
    part: int
    local2global: np.ndarray      # int64 [n_local]
    n_bmaster: int                # B_i
    n_mirror: int                 # M_i
    mirror_off: np.ndarray        # int64 [p+1]: mirror slab of master part j = local rows
                                  #   [B + mirror_off[j], B + mirror_off[j+1])
    halo_master: Dict[int, np.ndarray]   # src part s -> local rows (on this master part) of
                                         #   halo list (s, this), position order
    rowptr: np.ndarray            # int64 [n_local+1]
    colidx: np.ndarray            # int64 [nnz] ascending per row
    val64: np.ndarray             # fp64 weights 1/sqrt(d_u d_v), global degrees
    n_edges: int                  # |E_i| (undirected edges assigned here)

    @property
    def n_local(self) -> int:
        return int(self.local2global.shape[0])

    @property
    def val32(self) -> np.ndarray:
        return self.val64.astype(np.float32)

    def is_master_row(self) -> np.ndarray:
        r = np.zeros(self.n_local, dtype=bool)
        r[:self.n_bmaster] = True
        r[self.n_bmaster + self.n_mirror:] = True
        return r


@dataclass
class Plan:
    n: int
    m: int
    p: int
    edge_part: np.ndarray
    master: np.ndarray
    replicas: np.ndarray          # int64 bitmask per vertex
    parts: List[PartPlan]
    halo: Dict[Tuple[int, int], np.ndarray]   # (mirror part i, master part j) -> ↑gid
    host_of: List[int]


def build_plan(n: int, eu: np.ndarray, ev: np.ndarray, edge_part: np.ndarray,
               master: np.ndarray, cfg: PartitionCfg) -> Plan:
    p = cfg.p
    if p > 62:
        raise ValueError("oracle plan supports p <= 62")
    m = len(eu)
    eu = np.asarray(eu, dtype=np.int64)
    ev = np.asarray(ev, dtype=np.int64)
    edge_part = np.asarray(edge_part, dtype=np.int64)
    master = np.asarray(master, dtype=np.int64)
    # replica sets: the parts of a vertex's incident edges, plus its master part
    rep = np.zeros(n, dtype=np.int64)
    np.bitwise_or.at(rep, eu, np.left_shift(1, edge_part))
    np.bitwise_or.at(rep, ev, np.left_shift(1, edge_part))
    rep |= np.left_shift(1, master)
    nrep = np.zeros(n, dtype=np.int64)
    for i in range(p):
        nrep += (rep >> i) & 1
    deg = degrees(n, eu, ev, cfg.self_loops)
    halo = {}
    for i in range(p):
        on_i = ((rep >> i) & 1).astype(bool)
        for j in range(p):
            if i != j:
                # vertices with master on j and a mirror on i, ascending global id
                halo[(i, j)] = np.flatnonzero((master == j) & on_i)
    parts = []
    for i in range(p):
        bmasters = np.flatnonzero((master == i) & (nrep >= 2))
        slabs = [halo[(i, j)] if j != i else np.empty(0, dtype=np.int64) for j in range(p)]
        moff = np.zeros(p + 1, dtype=np.int64)
        moff[1:] = np.cumsum([len(s) for s in slabs])
        interior = np.flatnonzero((master == i) & (nrep == 1))
        l2g = np.concatenate([bmasters] + slabs + [interior]).astype(np.int64)
        g2l = np.full(n, -1, dtype=np.int64)
        g2l[l2g] = np.arange(len(l2g))
        sel = np.flatnonzero(edge_part == i)
        r = np.concatenate([g2l[eu[sel]], g2l[ev[sel]]])
        c = np.concatenate([g2l[ev[sel]], g2l[eu[sel]]])
        w = np.concatenate([edge_weight(deg[eu[sel]], deg[ev[sel]])] * 2)
        if cfg.self_loops:
            own = np.concatenate([bmasters, interior])
            r = np.concatenate([r, g2l[own]]); c = np.concatenate([c, g2l[own]])
            w = np.concatenate([w, edge_weight(deg[own], deg[own])])
        nl = len(l2g)
        order = np.lexsort((c, r))
        rowptr = np.zeros(nl + 1, dtype=np.int64)
        rowptr[1:] = np.cumsum(np.bincount(r, minlength=nl))
        parts.append(PartPlan(part=i, local2global=l2g, n_bmaster=len(bmasters),
                              n_mirror=int(moff[-1]), mirror_off=moff, halo_master={},
                              rowptr=rowptr, colidx=c[order], val64=w[order],
                              n_edges=len(sel)))
    for j in range(p):
        g2l = np.full(n, -1, dtype=np.int64)
        g2l[parts[j].local2global] = np.arange(parts[j].n_local)
        for s in range(p):
            if s != j:
                parts[j].halo_master[s] = g2l[halo[(s, j)]]
    return Plan(n=n, m=m, p=p, edge_part=edge_part.astype(np.int32),
                master=master.astype(np.int32), replicas=rep, parts=parts,
                halo=halo, host_of=cfg.hosts())


def partition(n: int, eu: np.ndarray, ev: np.ndarray, cfg: PartitionCfg) -> Plan:
    ep, ms = ebv_partition(n, eu, ev, cfg)
    return build_plan(n, eu, ev, ep, ms, cfg)


@dataclass
class PartitionStats:
    rf: float                 # Σ|V_i| / |V|
    edge_if: float            # max|E_i| / (|E|/p)
    vertex_if: float          # max|V_i| / (Σ|V_i|/p)
    total_mirrors: int        # M = Σ_u (r_u - 1)
    inner_max: int            # Table 3 "Inner"
    outer_max: int            # Table 3 "Outer"
    sum_vi: int
    max_ei: int


def stats(plan: Plan) -> PartitionStats:
    p, n, m = plan.p, plan.n, plan.m
    vi = [pp.n_local for pp in plan.parts]
    ei = [pp.n_edges for pp in plan.parts]
    host = plan.host_of
    inner = [0] * p
    outer = [0] * p
    for (i, j), lst in plan.halo.items():
        k = len(lst)
        # gather: i (mirror) sends k messages to j; scatter: j (master) sends k to i
        if host[i] == host[j]:
            inner[i] += k; inner[j] += k
        else:
            outer[i] += k; outer[j] += k
    return PartitionStats(
        rf=sum(vi) / n,
        edge_if=max(ei) / (m / p),
        vertex_if=max(vi) / (sum(vi) / p),
        total_mirrors=sum(vi) - n,
        inner_max=max(inner), outer_max=max(outer), sum_vi=sum(vi), max_ei=max(ei))


def outer_reduction(outer_gamma0: int, outer_gamma01: int) -> float:
    """Relative reduction of outer connections by γ=0.1 vs γ=0."""
    return 1.0 - outer_gamma01 / outer_gamma0
