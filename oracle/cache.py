"""Gather/scatter synchronisation with the adaptive vertex cache (oracle steps O4, O9, O10).

Follows the paper in its own order:
  * §3.2: gather — each mirror sends its value to the master, which
    sums them with its own; scatter — the master sends the aggregate back and the
    mirrors replace their value.
  * Alg. 2, for Z and δ alike:
      L3-L9   mirror u on part i: if ‖z_{i,u} − z̃_{i,u}‖∞ > ε‖z̃_{i,u}‖∞, send
              Δ = z_{i,u} − z̃_{i,u} to the master and update z̃_{i,u}
      L10     bulk synchronise
      L11-L13 master: z̃_{·,u} += Δ for every received message; mark u active
      L14-L19 master's own replica: the same test; z̃_{·,u} += z − z̃_{i,u};
              z̃_{i,u} ← z; mark active
      L20-L22 every active u: send the cached aggregate to its mirrors
  * Z is assembled from the cached aggregate z̃_{·,j}.
  * §5: the message (a difference) is B-bit linearly quantised.

Readings:
  R10 the cache covers boundary (replicated) vertices only; interior rows use
      the fresh local value.
  R11 under quantisation the mirror snapshot follows what the master received:
      z̃_{i,u} ← z̃_{i,u} + deq(q(Δ))  (``snapshot_literal`` gives z̃ ← z).
  R12 the scatter payload is the quantised delta a − b of the aggregate a
      against the replicas' broadcast view b; every replica (master included)
      applies b += deq(q), so b is bit-identical everywhere.  Without
      quantisation b ← a (fp32 payload).  ``scatter_full`` quantises a itself.
  R13 the master adds received Δ in ascending source part, then its own Δ,
      unquantised (it never travels).
  R14 "no cache": snapshots pinned at 0, aggregate and view reset each sync,
      every replica sends its full value (the fresh fixed-order sum);
      "quantise only" is the same with B-bit payloads.
  R15 the test is  max_j |z_j − s_j| > RN(ε32 · max_j |s_j|)  (strict), over the
      F valid columns; fp32 replay follows the canonical op sequence.

Counters (O9, R25): gather_sent, master_fired, active, scatter_msgs,
remote = gather_sent + scatter_msgs, baseline = 2·M, bytes (F+12 per int8
message, 4F+4 per fp32 message: the paper's B·L + 2T plus a 32-bit position).
Pins: tests/test_oracle_cache.py (ε = 0 ∧ no quantisation ⇒ exact sum;
replica coherence; Lemma-2-style staleness bound; predicate negation; send-set
monotone in ε; first sync sends every non-zero row; brute-force counts).
"""
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from .quant import dequantize, dequantize_f32, quantize, quantize_f32


@dataclass
class SyncMode:
    cache: bool = True            # False: reading R14 "no cache" baseline
    quant_bits: int = 0           # 0: fp32/fp64 payloads; B > 0: B-bit linear quantisation
    dtype: type = np.float64      # np.float32 = R15 kernel-replay arithmetic
    snapshot_literal: bool = False
    scatter_full: bool = False


@dataclass
class SyncCounters:
    gather_sent: int = 0
    master_fired: int = 0
    active: int = 0
    scatter_msgs: int = 0
    bytes: int = 0
    baseline: int = 0             # 2·M: every mirror gathers, every master scatters to every mirror
    gather_mask: Dict[int, np.ndarray] = field(default_factory=dict)   # part -> bool[M_i]
    master_fired_mask: Dict[int, np.ndarray] = field(default_factory=dict)
    active_mask: Dict[int, np.ndarray] = field(default_factory=dict)   # part -> bool[B_i]
    # the messages themselves (O10, §5): (src, dst) -> (pos, payload, lo, hi) where
    # pos are the halo-list positions of the sent vertices (ascending), payload the B-bit codes
    # q [k, F] (int64) or, without quantisation, the fp payload rows; lo, hi the per-vertex
    # headers (None without quantisation).  gather: mirror part -> master part (position in
    # the mirror slab of that master); scatter: master part -> mirror part (position in the
    # halo list of that mirror part).
    gather_msgs: Dict[tuple, tuple] = field(default_factory=dict)
    scatter_msgs_rec: Dict[tuple, tuple] = field(default_factory=dict)

    @property
    def remote(self) -> int:
        return self.gather_sent + self.scatter_msgs


class SyncState:
    """Cache tables of one (layer, direction): z̃_{i,u} (s) and z̃_{·,u} (a, b)."""

    def __init__(self, plan, F: int, dtype=np.float64):
        self.F = F
        self.s_mir = [np.zeros((pp.n_mirror, F), dtype) for pp in plan.parts]
        self.b_mir = [np.zeros((pp.n_mirror, F), dtype) for pp in plan.parts]
        self.s_mas = [np.zeros((pp.n_bmaster, F), dtype) for pp in plan.parts]
        self.a = [np.zeros((pp.n_bmaster, F), dtype) for pp in plan.parts]
        self.b_mas = [np.zeros((pp.n_bmaster, F), dtype) for pp in plan.parts]


def _linf(x):
    return np.abs(x).max(axis=1) if x.shape[1] else np.zeros(x.shape[0], x.dtype)


def _test(d, s, eps, dt):
    """Alg. 2 L4 / L15: ‖d‖∞ > ε ‖s‖∞ (R15: threshold rounded once in the working precision)."""
    if dt == np.float32:
        thr = (np.float32(eps) * _linf(s).astype(np.float32)).astype(np.float32)
    else:
        thr = eps * _linf(s)
    return _linf(d) > thr


def _q(d, B, dt):
    if dt == np.float32:
        q, lo, hi = quantize_f32(d, B)
        return q, lo, hi, dequantize_f32(q, lo, hi, B)
    q, lo, hi = quantize(d, B)
    return q, lo, hi, dequantize(q, lo, hi, B)


def msg_bytes(F: int, B: int) -> int:
    return F + 12 if B == 8 else (4 * F + 4 if B == 0 else (B * F + 7) // 8 + 12)


def sync(plan, st: SyncState, X: List[np.ndarray], eps: float, mode: SyncMode,
         follow: Optional[dict] = None):
    """One gather + scatter round (one 'synchronisation').

    X[i]: part i's local partial values [n_i, F] (Z̈ or δ̈).  Returns (list of synced
    arrays, SyncCounters).  ``follow`` = {"gather": {i: bool[M_i]}, "master": {j: bool[B_j]}}
    replaces the cache-test decisions by recorded ones (trajectory follow mode)."""
    p = plan.p
    dt = mode.dtype
    B = mode.quant_bits
    F = st.F
    eps = float(eps)
    X = [np.asarray(x, dtype=dt) for x in X]
    out = [x.copy() for x in X]
    cnt = SyncCounters()
    cnt.baseline = 2 * sum(pp.n_mirror for pp in plan.parts)
    msgs = {}
    # ---- Alg. 2 L3-L9: every mirror tests its value and sends Δ to its master ----
    for i in range(p):
        P = plan.parts[i]
        Bi = P.n_bmaster
        z = X[i][Bi:Bi + P.n_mirror]
        s = st.s_mir[i]
        if mode.cache:
            d = (z - s).astype(dt)
            send = _test(d, s, eps, dt)
        else:
            d = z.copy()
            send = np.ones(P.n_mirror, dtype=bool)
        if follow is not None:
            send = follow["gather"][i].copy()
        cnt.gather_mask[i] = send
        for j in range(p):
            if j == i:
                continue
            lo_r, hi_r = P.mirror_off[j], P.mirror_off[j + 1]
            pos = np.flatnonzero(send[lo_r:hi_r])
            rows = lo_r + pos
            if B:
                q, qlo, qhi, deq = _q(d[rows], B, dt)
                payload = deq
                cnt.gather_msgs[(i, j)] = (pos, q, qlo, qhi)
                if mode.cache:
                    if mode.snapshot_literal:
                        s[rows] = z[rows]
                    else:
                        s[rows] = (s[rows] + deq).astype(dt)       # R11
            else:
                payload = d[rows]
                cnt.gather_msgs[(i, j)] = (pos, payload.copy(), None, None)
                if mode.cache:
                    s[rows] = z[rows]                              # Alg. 2 L6
            msgs[(i, j)] = (pos, payload)
            cnt.gather_sent += len(pos)
            cnt.bytes += len(pos) * msg_bytes(F, B)
    # ---- Alg. 2 L10: bulk synchronise (all messages delivered) ----
    scat = {}
    for j in range(p):
        P = plan.parts[j]
        Bj = P.n_bmaster
        a = st.a[j] if mode.cache else np.zeros((Bj, F), dt)
        active = np.zeros(Bj, dtype=bool)
        # L11-L13: received Δ in ascending source part (R13)
        for s_ in range(p):
            if s_ == j:
                continue
            pos, payload = msgs[(s_, j)]
            rows = P.halo_master[s_][pos]
            a[rows] = (a[rows] + payload).astype(dt)
            active[rows] = True
        # L14-L19: the master's own replica, unquantised (R13)
        z = X[j][:Bj]
        if mode.cache:
            sm = st.s_mas[j]
            d = (z - sm).astype(dt)
            fired = _test(d, sm, eps, dt)
            if follow is not None:
                fired = follow["master"][j].copy()
            a[fired] = (a[fired] + d[fired]).astype(dt)
            sm[fired] = z[fired]
        else:
            fired = np.ones(Bj, dtype=bool)
            a = (a + z).astype(dt)
        active |= fired
        cnt.master_fired_mask[j] = fired
        cnt.active_mask[j] = active
        cnt.master_fired += int(fired.sum())
        cnt.active += int(active.sum())
        # L20-L22: scatter every active master's cached aggregate (R12)
        act = np.flatnonzero(active)
        bold = st.b_mas[j] if mode.cache else np.zeros((Bj, F), dt)
        if B:
            delta = a[act] if mode.scatter_full else (a[act] - bold[act]).astype(dt)
            q, qlo, qhi, deq = _q(delta, B, dt)
            bnew = deq if mode.scatter_full else (bold[act] + deq).astype(dt)
            scat[j] = (active, deq, q, qlo, qhi)
        else:
            bnew = a[act].copy()
            scat[j] = (active, bnew, bnew, None, None)
        if mode.cache:
            st.b_mas[j][act] = bnew
            out[j][:Bj] = st.b_mas[j]
        else:
            bm = np.zeros((Bj, F), dt)
            bm[act] = bnew
            out[j][:Bj] = bm
        if mode.cache:
            st.a[j] = a
    # ---- mirrors receive the scatter and replace their value ----
    for i in range(p):
        P = plan.parts[i]
        Bi = P.n_bmaster
        bmir = st.b_mir[i] if mode.cache else np.zeros((P.n_mirror, F), dt)
        for j in range(p):
            if j == i:
                continue
            active, pay, sq, slo, shi = scat[j]
            hm = plan.parts[j].halo_master[i]            # halo list (i, j) on the master side
            act_rows_j = np.flatnonzero(active)
            # payload row index for each active master of j
            idx_of = np.full(plan.parts[j].n_bmaster, -1, dtype=np.int64)
            idx_of[act_rows_j] = np.arange(len(act_rows_j))
            sel = idx_of[hm]
            pos = np.flatnonzero(sel >= 0)
            rows = P.mirror_off[j] + pos
            if B and not mode.scatter_full:
                bmir[rows] = (bmir[rows] + pay[sel[pos]]).astype(dt)
            else:
                bmir[rows] = pay[sel[pos]]
            cnt.scatter_msgs += len(pos)
            cnt.bytes += len(pos) * msg_bytes(F, B)
            k = sel[pos]
            cnt.scatter_msgs_rec[(j, i)] = (pos, sq[k].copy(),
                                            None if slo is None else slo[k].copy(),
                                            None if shi is None else shi[k].copy())
        out[i][Bi:Bi + P.n_mirror] = bmir
    return out, cnt


def pack_ref(z, s, eps: float, B: int):
    """fp32 replay of one part's gather-side test + quantise + snapshot update (O10).

    z, s: float32 [rows, F].  Returns (send bool[rows], q uint8 [k, F], lo, hi,
    s_new float32 [rows, F]) following R11 and R15."""
    z = np.asarray(z, np.float32)
    s = np.asarray(s, np.float32)
    d = (z - s).astype(np.float32)
    send = _test(d, s, eps, np.float32)
    s_new = s.copy()
    rows = np.flatnonzero(send)
    if B:
        q, lo, hi = quantize_f32(d[rows], B)
        s_new[rows] = (s[rows] + dequantize_f32(q, lo, hi, B)).astype(np.float32)
        return send, q.astype(np.uint8), lo, hi, s_new
    s_new[rows] = z[rows]
    return send, d[rows], None, None, s_new
