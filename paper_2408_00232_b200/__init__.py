"""B200-native CDFGNN hot path (arXiv 2408.00232): partitioner + per-layer
distributed full-batch GCN step behind the C ABI of include/cdfgnn.h.

The functions below carry the C names (without the ``cdfgnn_`` prefix) and only
marshal arguments; every step of the path runs in libcdfgnn.so (host C++
partitioner, sm_100a kernels, NCCL).  ``runtime.Run`` wires a synthetic
dataset, torch device memory and a process group to them.

The library is loaded on first use of any of these names (so that
``paper_2408_00232_b200.build`` can rebuild it); loading fails loudly if it has
not been built — there is no fallback path.
"""
_API = (
    "Plan", "Ctx", "CdfgnnError", "partition", "plan_part", "plan_stats", "cfg_default",
    "get_unique_id", "workspace_size", "init", "destroy", "halo_exchange", "layer_fwd",
    "layer_bwd", "epoch", "epoch_host", "epoch_host_next", "cache_view", "act_view", "grad_view", "sync_flags", "msg_view",
    "reset_caches", "get_eps",
    "set_eps", "spmm", "bandwidth_probe", "last_error", "version", "ld_of",
)

__all__ = list(_API)


def __getattr__(name):
    if name in _API:
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
