"""Thin Python wrappers over include/cdfgnn.h (marshalling only; see _lib.py)."""
import ctypes
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import CdfgnnError, check

_c = L.lib()


def ld_of(F: int) -> int:
    """Row stride of an F-wide fp32 matrix: roundup(F, 4) (reading R24)."""
    return (F + 3) // 4 * 4


def last_error() -> str:
    return _c.cdfgnn_last_error().decode()


def version() -> str:
    return _c.cdfgnn_version().decode()


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return None if t is None else t.data_ptr()


# ---------------------------------------------------------------- partitioning
class Plan:
    """Owns a cdfgnn_plan*; freed with the object."""

    def __init__(self, handle, n, m, p):
        self._h = handle
        self.n, self.m, self.p = n, m, p
        self.edge_part = None
        self.master = None

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _c is not None:
                _c.cdfgnn_plan_free(self._h)
                self._h = None
        except Exception:
            pass


def partition(n: int, eu: np.ndarray, ev: np.ndarray, p: int, num_hosts: int = 1,
              host_of: Optional[Sequence[int]] = None, alpha=(1, 1), beta=(1, 1), gamma=(1, 10),
              edge_order: int = 1, seed: int = 0, self_loops: bool = False) -> Plan:
    """cdfgnn_partition: hierarchical EBV vertex-cut."""
    eu = np.ascontiguousarray(eu, dtype=np.int32)
    ev = np.ascontiguousarray(ev, dtype=np.int32)
    m = int(eu.shape[0])
    cfg = L.PartitionCfgC()
    check(_c.cdfgnn_partition_cfg_default(ctypes.byref(cfg), p))
    cfg.num_hosts = num_hosts
    hosts = None
    if host_of is not None:
        hosts = np.ascontiguousarray(host_of, dtype=np.int32)
        cfg.host_of = hosts.ctypes.data_as(L.P(L.c_i32))
    cfg.alpha_num, cfg.alpha_den = alpha
    cfg.beta_num, cfg.beta_den = beta
    cfg.gamma_num, cfg.gamma_den = gamma
    cfg.edge_order = edge_order
    cfg.seed = seed
    cfg.self_loops = 1 if self_loops else 0
    ep = np.empty(max(m, 1), dtype=np.int32)
    ms = np.empty(max(n, 1), dtype=np.int32)
    h = ctypes.c_void_p()
    check(_c.cdfgnn_partition(n, m, eu.ctypes.data_as(L.P(L.c_i32)), ev.ctypes.data_as(L.P(L.c_i32)),
                              ctypes.byref(cfg), ep.ctypes.data_as(L.P(L.c_i32)),
                              ms.ctypes.data_as(L.P(L.c_i32)), ctypes.byref(h)))
    plan = Plan(h, n, m, p)
    plan.edge_part = ep[:m]
    plan.master = ms[:n]
    return plan


def plan_part(plan: Plan, part: int, copy: bool = True) -> Dict[str, np.ndarray]:
    """cdfgnn_plan_part as numpy arrays (copies unless copy=False)."""
    v = L.PartViewC()
    check(_c.cdfgnn_plan_part(plan.handle, part, ctypes.byref(v)))
    p = plan.p
    f = (lambda a: a.copy()) if copy else (lambda a: a)
    return dict(
        part=v.part, n_local=v.n_local, n_bmaster=v.n_bmaster, n_mirror=v.n_mirror,
        n_edges=v.n_edges, nnz=v.nnz,
        local2global=f(L.as_numpy(v.local2global, v.n_local, np.int32)),
        rowptr=f(L.as_numpy(v.rowptr, v.n_local + 1, np.int32)),
        colidx=f(L.as_numpy(v.colidx, v.nnz, np.int32)),
        val=f(L.as_numpy(v.val, v.nnz, np.float32)),
        mirror_off=f(L.as_numpy(v.mirror_off, p + 1, np.int64)),
        halo_off=f(L.as_numpy(v.halo_off, p + 1, np.int64)),
        halo_local=f(L.as_numpy(v.halo_local, int(L.as_numpy(v.halo_off, p + 1, np.int64)[-1]),
                                np.int32)),
    )


def plan_stats(plan: Plan) -> Dict[str, float]:
    s = L.PartitionStatsC()
    check(_c.cdfgnn_plan_stats(plan.handle, ctypes.byref(s)))
    return {k: getattr(s, k) for k, _ in L.PartitionStatsC._fields_}


# ---------------------------------------------------------------- context
def cfg_default(dims: Sequence[int], **kw) -> L.CfgC:
    cfg = L.CfgC()
    check(_c.cdfgnn_cfg_default(ctypes.byref(cfg)))
    cfg.L = len(dims) - 1
    for i, d in enumerate(dims):
        cfg.dims[i] = d
    for k, v in kw.items():
        if not hasattr(cfg, k):
            raise AttributeError(k)
        setattr(cfg, k, v)
    return cfg


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(_c.cdfgnn_get_unique_id(buf))
    return buf.raw


def workspace_size(plan: Plan, parts: Sequence[int], cfg: L.CfgC) -> int:
    arr = (L.c_i32 * len(parts))(*parts)
    out = ctypes.c_size_t()
    check(_c.cdfgnn_workspace_size(plan.handle, arr, len(parts), ctypes.byref(cfg), ctypes.byref(out)))
    return out.value


class Ctx:
    def __init__(self, handle, plan, parts, cfg, workspace):
        self._h = handle
        self.plan = plan          # keep the plan alive (the ctx borrows nothing, but views do)
        self.parts = list(parts)
        self.cfg = cfg
        self.workspace = workspace

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            check(_c.cdfgnn_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init(plan: Plan, parts: Sequence[int], rank: int, world: int, cfg: L.CfgC, device: int,
         workspace, nccl_uid: Optional[bytes] = None) -> Ctx:
    """cdfgnn_init over a caller-owned torch uint8 CUDA workspace."""
    arr = (L.c_i32 * len(parts))(*parts)
    h = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(nccl_uid, 128) if nccl_uid is not None else None
    check(_c.cdfgnn_init(plan.handle, arr, len(parts), rank, world, uid, device,
                         ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                         ctypes.byref(cfg), ctypes.byref(h)))
    return Ctx(h, plan, parts, cfg, workspace)


def destroy(ctx: Ctx):
    ctx.close()


def _stats_dict(s: L.SyncStatsC) -> Dict[str, int]:
    return {k: getattr(s, k) for k, _ in L.SyncStatsC._fields_}


def halo_exchange(ctx: Ctx, l: int, direction: int, X: List, ld: int, eps: float,
                  stats: bool = False, stream=None):
    st = L.SyncStatsC() if stats else None
    check(_c.cdfgnn_halo_exchange(ctx.handle, l, direction, L.ptr_array([_ptr(x) for x in X]), ld,
                                  eps, ctypes.byref(st) if st else None, _stream(stream)))
    return _stats_dict(st) if st else None


def layer_fwd(ctx: Ctx, l: int, H_in: List, ld_in: int, W, Z: List, H_out: Optional[List],
              ld_out: int, eps: float, stats: bool = False, stream=None):
    st = L.SyncStatsC() if stats else None
    check(_c.cdfgnn_layer_fwd(ctx.handle, l, L.ptr_array([_ptr(x) for x in H_in]), ld_in, _ptr(W),
                              L.ptr_array([_ptr(x) for x in Z]),
                              L.ptr_array([_ptr(x) for x in H_out]) if H_out is not None else None,
                              ld_out, eps, ctypes.byref(st) if st else None, _stream(stream)))
    return _stats_dict(st) if st else None


def layer_bwd(ctx: Ctx, l: int, dZ: List, ld: int, H_in: List, ld_in: int, W, dZ_prev: Optional[List],
              dW, eps: float, stats: bool = False, stream=None):
    st = L.SyncStatsC() if stats else None
    check(_c.cdfgnn_layer_bwd(ctx.handle, l, L.ptr_array([_ptr(x) for x in dZ]), ld,
                              L.ptr_array([_ptr(x) for x in H_in]), ld_in, _ptr(W),
                              L.ptr_array([_ptr(x) for x in dZ_prev]) if dZ_prev is not None else None,
                              _ptr(dW), eps, ctypes.byref(st) if st else None, _stream(stream)))
    return _stats_dict(st) if st else None


def _epoch_dict(s: L.EpochStatsC, nl: int) -> Dict:
    d = {k: getattr(s, k) for k, _ in L.EpochStatsC._fields_ if k not in ("fwd", "bwd", "ms_sync_sub")}
    d["ms_sync_sub"] = list(s.ms_sync_sub)
    d["fwd"] = [_stats_dict(s.fwd[i]) for i in range(nl)]
    d["bwd"] = [_stats_dict(s.bwd[i]) for i in range(nl)]
    return d


def epoch(ctx: Ctx, X: List, labels: List, train_mask: List, W: List, stream=None) -> Dict:
    st = L.EpochStatsC()
    check(_c.cdfgnn_epoch(ctx.handle, L.ptr_array([_ptr(x) for x in X]),
                          L.ptr_array([_ptr(x) for x in labels]),
                          L.ptr_array([_ptr(x) for x in train_mask]),
                          L.ptr_array([_ptr(w) for w in W]), ctypes.byref(st), _stream(stream)))
    return _epoch_dict(st, ctx.cfg.L)


def epoch_host(ctx: Ctx, X_host: List, labels_host: List, train_host: List, W: List,
               stream=None) -> Dict:
    """X_host etc.: pinned (or plain) CPU tensors / numpy arrays in local row order."""
    def hp(a):
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
    st = L.EpochStatsC()
    check(_c.cdfgnn_epoch_host(ctx.handle, L.ptr_array([hp(x) for x in X_host]),
                               L.ptr_array([hp(x) for x in labels_host]),
                               L.ptr_array([hp(x) for x in train_host]),
                               L.ptr_array([_ptr(w) for w in W]), ctypes.byref(st), _stream(stream)))
    return _epoch_dict(st, ctx.cfg.L)


def epoch_host_next(ctx: Ctx, X_host: Optional[List], labels_host: Optional[List],
                    train_host: Optional[List], W: List, X_next: Optional[List] = None,
                    labels_next: Optional[List] = None, train_next: Optional[List] = None,
                    stream=None) -> Dict:
    """cdfgnn_epoch_host_next: this step on host inputs (ignored when the previous call
    prefetched them) and an overlapped copy of the next step's host inputs (*_next)."""
    def hp(a):
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

    def arr(xs):
        return L.ptr_array([hp(x) for x in xs]) if xs is not None else None
    st = L.EpochStatsC()
    check(_c.cdfgnn_epoch_host_next(ctx.handle, arr(X_host), arr(labels_host), arr(train_host),
                                    arr(X_next), arr(labels_next), arr(train_next),
                                    L.ptr_array([_ptr(w) for w in W]), ctypes.byref(st),
                                    _stream(stream)))
    return _epoch_dict(st, ctx.cfg.L)


def cache_view(ctx: Ctx, local_part: int, l: int, direction: int, which: int):
    """(device pointer, rows, ld) of a cache table (0 s_mir, 1 b_mir, 2 s_mas, 3 a, 4 b_mas)."""
    p = ctypes.c_void_p()
    rows = L.c_i64()
    ld = L.c_i64()
    check(_c.cdfgnn_cache_view(ctx.handle, local_part, l, direction, which, ctypes.byref(p),
                               ctypes.byref(rows), ctypes.byref(ld)))
    return p.value, rows.value, ld.value


def act_view(ctx: Ctx, local_part: int, l: int):
    """(device pointer, rows, ld) of H^(l) (l < L) or the logits (l = L) of the last epoch."""
    p = ctypes.c_void_p()
    rows = L.c_i64()
    ld = L.c_i64()
    check(_c.cdfgnn_act_view(ctx.handle, local_part, l, ctypes.byref(p), ctypes.byref(rows), ctypes.byref(ld)))
    return p.value, rows.value, ld.value


def grad_view(ctx: Ctx, l: int):
    """(device pointer, rows, ld) of ∇W^(l-1) of the last epoch."""
    p = ctypes.c_void_p()
    rows = L.c_i64()
    ld = L.c_i64()
    check(_c.cdfgnn_grad_view(ctx.handle, l, ctypes.byref(p), ctypes.byref(rows), ctypes.byref(ld)))
    return p.value, rows.value, ld.value


def sync_flags(ctx: Ctx, local_part: int, l: int, direction: int, which: int):
    """(device pointer, rows) of the uint8 flags of the latest sync of (l, direction):
    which 0 gather-sent per mirror, 1 master-fired, 2 active."""
    p = ctypes.c_void_p()
    rows = L.c_i64()
    check(_c.cdfgnn_sync_flags(ctx.handle, local_part, l, direction, which, ctypes.byref(p),
                               ctypes.byref(rows)))
    return p.value, rows.value


def msg_view(ctx: Ctx, local_part: int, phase: int, src: int) -> Dict:
    """cdfgnn_msg_view as a dict (device pointers as ints)."""
    v = L.MsgViewC()
    check(_c.cdfgnn_msg_view(ctx.handle, local_part, phase, src, ctypes.byref(v)))
    return {k: getattr(v, k) for k, _ in L.MsgViewC._fields_}


def reset_caches(ctx: Ctx, stream=None):
    check(_c.cdfgnn_reset_caches(ctx.handle, _stream(stream)))


def get_eps(ctx: Ctx):
    e = L.c_f64()
    m = L.c_f64()
    check(_c.cdfgnn_get_eps(ctx.handle, ctypes.byref(e), ctypes.byref(m)))
    return e.value, m.value


def set_eps(ctx: Ctx, eps: float):
    check(_c.cdfgnn_set_eps(ctx.handle, eps))


def spmm(ctx: Ctx, local_part: int, T, Y, ld: int, F: int, stream=None):
    check(_c.cdfgnn_spmm(ctx.handle, local_part, _ptr(T), _ptr(Y), ld, F, _stream(stream)))


def bandwidth_probe(buf, bytes_: int, reps: int, stream=None) -> float:
    """cdfgnn_bandwidth_probe: GB/s of streaming 16-byte reads over `bytes_` of `buf`."""
    out = L.c_f64()
    check(_c.cdfgnn_bandwidth_probe(ctypes.c_void_p(buf.data_ptr()), bytes_, reps, ctypes.byref(out),
                                    _stream(stream)))
    return out.value
