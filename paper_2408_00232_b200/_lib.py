"""ctypes binding of libcdfgnn (include/cdfgnn.h) — argument marshalling only.

Every function keeps the C name without the ``cdfgnn_`` prefix.  Device
buffers are passed as torch CUDA tensors (their ``data_ptr()``), streams as
``torch.cuda.Stream`` (default: the current stream).  The library must be built
(``python -m paper_2408_00232_b200.build``); importing this module raises if it
is missing — there is no fallback path.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcdfgnn.so")

MAX_PARTS = 64
MAX_LAYERS = 8

OK, EUSAGE, EDATA, EPROTO, ECUDA, ENCCL, EWORKSPACE = 0, 2, 3, 4, 5, 6, 7


class CdfgnnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"cdfgnn error {code}: {msg}")
        self.code = code


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2408_00232_b200.build`")

try:  # share the NCCL copy torch loads (same soname, same file)
    import torch  # noqa: F401
except Exception:  # pragma: no cover
    pass

_lib = ctypes.CDLL(LIB_PATH)

c_i32, c_i64, c_u64, c_f32, c_f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_double
P = ctypes.POINTER
c_void_p = ctypes.c_void_p


class PartitionCfgC(ctypes.Structure):
    _fields_ = [("num_parts", c_i32), ("num_hosts", c_i32), ("host_of", P(c_i32)),
                ("alpha_num", c_i64), ("alpha_den", c_i64), ("beta_num", c_i64),
                ("beta_den", c_i64), ("gamma_num", c_i64), ("gamma_den", c_i64),
                ("edge_order", c_i32), ("seed", c_u64), ("self_loops", c_i32)]


class PartViewC(ctypes.Structure):
    _fields_ = [("part", c_i32), ("n_local", c_i64), ("n_bmaster", c_i64), ("n_mirror", c_i64),
                ("n_edges", c_i64), ("nnz", c_i64), ("local2global", P(c_i32)),
                ("rowptr", P(c_i32)), ("colidx", P(c_i32)), ("val", P(c_f32)),
                ("mirror_off", P(c_i64)), ("halo_off", P(c_i64)), ("halo_local", P(c_i32))]


class PartitionStatsC(ctypes.Structure):
    _fields_ = [("rf", c_f64), ("edge_if", c_f64), ("vertex_if", c_f64),
                ("total_mirrors", c_i64), ("inner_max", c_i64), ("outer_max", c_i64),
                ("sum_vi", c_i64), ("max_ei", c_i64)]


class CfgC(ctypes.Structure):
    _fields_ = [("L", c_i32), ("dims", c_i32 * (MAX_LAYERS + 1)), ("cache_on", c_i32),
                ("eps_init", c_f64), ("adaptive", c_i32), ("mu1", c_f64), ("mu2", c_f64),
                ("nu1", c_f64), ("nu2", c_f64), ("xi", c_f64), ("lam1", c_f64), ("lam2", c_f64),
                ("eps_clamp", c_i32), ("quant_bits", c_i32), ("optimizer", c_i32), ("lr", c_f64),
                ("beta1", c_f64), ("beta2", c_f64), ("adam_eps", c_f64), ("gemm_tf32", c_i32),
                ("timing", c_i32), ("transport", c_i32), ("elide_dead_syncs", c_i32),
                ("static_inputs", c_i32), ("overlap", c_i32), ("msg_layout", c_i32),
                ("fuse_gather", c_i32)]


class MsgViewC(ctypes.Structure):
    _fields_ = [("layout", c_i32), ("base", c_void_p), ("pay", c_void_p), ("count", c_void_p),
                ("capacity", c_i64), ("hdr_bytes", c_i64), ("row_bytes", c_i64),
                ("slot_bytes", c_i64), ("stamp", ctypes.c_uint32), ("quant_bits", c_i32)]


class SyncStatsC(ctypes.Structure):
    _fields_ = [("gather_sent", c_i64), ("master_fired", c_i64), ("active", c_i64),
                ("scatter_msgs", c_i64), ("baseline", c_i64), ("bytes_alg", c_i64),
                ("bytes_wire", c_i64)]


class EpochStatsC(ctypes.Structure):
    _fields_ = [("loss", c_f64), ("correct", c_i64), ("total", c_i64), ("acc", c_f64),
                ("eps_used", c_f64), ("eps_next", c_f64), ("fwd", SyncStatsC * MAX_LAYERS),
                ("bwd", SyncStatsC * MAX_LAYERS), ("gpu_launches", c_i32), ("ms_gemm", c_f64),
                ("ms_spmm", c_f64), ("ms_sync", c_f64), ("ms_other", c_f64),
                ("spmm_ld", c_i32), ("spmm_launches", c_i32), ("spmm_bytes", c_f64),
                ("spmm_bytes_compulsory", c_f64), ("spmm_ms_sum", c_f64),
                ("ms_sync_sub", c_f64 * 6), ("transport", c_i32)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("cdfgnn_partition_cfg_default", c_i32, [P(PartitionCfgC), c_i32])
_sig("cdfgnn_partition", c_i32, [c_i64, c_i64, P(c_i32), P(c_i32), P(PartitionCfgC), P(c_i32),
                                 P(c_i32), P(c_void_p)])
_sig("cdfgnn_plan_num_parts", c_i32, [c_void_p])
_sig("cdfgnn_plan_part", c_i32, [c_void_p, c_i32, P(PartViewC)])
_sig("cdfgnn_plan_stats", c_i32, [c_void_p, P(PartitionStatsC)])
_sig("cdfgnn_plan_free", None, [c_void_p])
_sig("cdfgnn_cfg_default", c_i32, [P(CfgC)])
_sig("cdfgnn_get_unique_id", c_i32, [c_void_p])
_sig("cdfgnn_workspace_size", c_i32, [c_void_p, P(c_i32), c_i32, P(CfgC), P(ctypes.c_size_t)])
_sig("cdfgnn_init", c_i32, [c_void_p, P(c_i32), c_i32, c_i32, c_i32, c_void_p, c_i32, c_void_p,
                            ctypes.c_size_t, P(CfgC), P(c_void_p)])
_sig("cdfgnn_destroy", c_i32, [c_void_p])
_sig("cdfgnn_halo_exchange", c_i32, [c_void_p, c_i32, c_i32, P(c_void_p), c_i64, c_f32,
                                     P(SyncStatsC), c_void_p])
_sig("cdfgnn_layer_fwd", c_i32, [c_void_p, c_i32, P(c_void_p), c_i64, c_void_p, P(c_void_p),
                                 P(c_void_p), c_i64, c_f32, P(SyncStatsC), c_void_p])
_sig("cdfgnn_layer_bwd", c_i32, [c_void_p, c_i32, P(c_void_p), c_i64, P(c_void_p), c_i64, c_void_p,
                                 P(c_void_p), c_void_p, c_f32, P(SyncStatsC), c_void_p])
_sig("cdfgnn_epoch", c_i32, [c_void_p, P(c_void_p), P(c_void_p), P(c_void_p), P(c_void_p),
                             P(EpochStatsC), c_void_p])
_sig("cdfgnn_epoch_host", c_i32, [c_void_p, P(c_void_p), P(c_void_p), P(c_void_p), P(c_void_p),
                                  P(EpochStatsC), c_void_p])
_sig("cdfgnn_epoch_host_next", c_i32, [c_void_p, P(c_void_p), P(c_void_p), P(c_void_p), P(c_void_p),
                                       P(c_void_p), P(c_void_p), P(c_void_p), P(EpochStatsC), c_void_p])
_sig("cdfgnn_cache_view", c_i32, [c_void_p, c_i32, c_i32, c_i32, c_i32, P(c_void_p), P(c_i64),
                                  P(c_i64)])
_sig("cdfgnn_sync_flags", c_i32, [c_void_p, c_i32, c_i32, c_i32, c_i32, P(c_void_p), P(c_i64)])
_sig("cdfgnn_msg_view", c_i32, [c_void_p, c_i32, c_i32, c_i32, P(MsgViewC)])
_sig("cdfgnn_act_view", c_i32, [c_void_p, c_i32, c_i32, P(c_void_p), P(c_i64), P(c_i64)])
_sig("cdfgnn_grad_view", c_i32, [c_void_p, c_i32, P(c_void_p), P(c_i64), P(c_i64)])
_sig("cdfgnn_reset_caches", c_i32, [c_void_p, c_void_p])
_sig("cdfgnn_get_eps", c_i32, [c_void_p, P(c_f64), P(c_f64)])
_sig("cdfgnn_set_eps", c_i32, [c_void_p, c_f64])
_sig("cdfgnn_spmm", c_i32, [c_void_p, c_i32, c_void_p, c_void_p, c_i64, c_i32, c_void_p])
_sig("cdfgnn_bandwidth_probe", c_i32, [c_void_p, c_i64, c_i32, P(c_f64), c_void_p])
_sig("cdfgnn_last_error", ctypes.c_char_p, [])
_sig("cdfgnn_version", ctypes.c_char_p, [])



def lib():
    return _lib


def check(rc):
    if rc != OK:
        raise CdfgnnError(rc, _lib.cdfgnn_last_error().decode())
    return rc


def ptr_array(ptrs):
    arr = (c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = None if p is None else int(p)
    return arr


def as_numpy(ptr, count, dtype):
    if count == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(count,)).view(dtype)
