"""Driver plumbing: a synthetic dataset + torch device memory + process group -> libcdfgnn.

Everything numerical runs in libcdfgnn.so; this module only lays the inputs out
in each part's local row order (reading R21), allocates the caller-owned
workspace with torch, broadcasts the NCCL unique id over torch.distributed and
calls the C ABI (via api.py).
"""
from typing import Dict, List, Optional

import numpy as np

from . import api


def local_inputs(ds, pv: Dict, ld0: int):
    """Part-local X (n_i x ld0, zero padding), labels (int32) and train mask (uint8)."""
    l2g = pv["local2global"]
    X = np.zeros((len(l2g), ld0), dtype=np.float32)
    X[:, :ds.X.shape[1]] = ds.X[l2g]
    return X, np.ascontiguousarray(ds.y[l2g], dtype=np.int32), \
        np.ascontiguousarray(ds.train[l2g], dtype=np.uint8)


GEMM_MODES = {"fp32": 0, "tf32": 1, "tf32x3": 3}   # cfg.gemm_tf32: SIMT fp32 / tcgen05 1x / 3x TF32


class Run:
    """One process's view of a CDFGNN training run (one GPU, k local parts)."""

    def __init__(self, ds, p: int, rank: int = 0, world: int = 1, device: int = 0,
                 cache: bool = True, quant_bits: int = 8, eps0: float = 0.01,
                 adaptive: bool = True, optimizer: str = "adam", lr: float = 0.01,
                 timing: bool = False, plan: Optional[api.Plan] = None,
                 host_inputs: bool = False, partition_kw: Optional[Dict] = None,
                 gemm: str = "tf32x3", transport: str = "push", elide: bool = True,
                 static_inputs: int = 0, overlap: bool = False, msg_layout: int = 0,
                 fuse_gather: bool = True):
        import torch
        self.torch = torch
        self.ds = ds
        self.p, self.rank, self.world, self.device = p, rank, world, device
        self.dev = torch.device("cuda", device)
        self.plan = plan if plan is not None else api.partition(ds.n, ds.eu, ds.ev, p,
                                                                **(partition_kw or {}))
        self.parts = list(range(p)) if world == 1 else [rank]
        self.cfg = api.cfg_default(ds.dims, cache_on=int(cache), quant_bits=quant_bits,
                                   eps_init=eps0, adaptive=int(adaptive),
                                   optimizer=1 if optimizer == "adam" else 0, lr=lr,
                                   timing=int(timing), gemm_tf32=GEMM_MODES[gemm],
                                   transport={"push": 0, "nccl": 1}[transport],
                                   elide_dead_syncs=int(elide), static_inputs=int(static_inputs),
                                   overlap=int(overlap), msg_layout=int(msg_layout),
                                   fuse_gather=int(fuse_gather))
        nbytes = api.workspace_size(self.plan, self.parts, self.cfg)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        uid = None
        if world > 1:
            import torch.distributed as dist
            obj = [api.get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        self.ctx = api.init(self.plan, self.parts, rank, world, self.cfg, device, self.workspace, uid)
        self.ld0 = api.ld_of(ds.dims[0])
        self.views = [api.plan_part(self.plan, i, copy=True) for i in self.parts]
        self.X, self.labels, self.masks = [], [], []
        self.X_host, self.labels_host, self.masks_host = [], [], []
        for pv in self.views:
            X, y, m = local_inputs(ds, pv, self.ld0)
            if host_inputs:
                self.X_host.append(torch.from_numpy(X).pin_memory())
                self.labels_host.append(torch.from_numpy(y).pin_memory())
                self.masks_host.append(torch.from_numpy(m).pin_memory())
            self.X.append(torch.from_numpy(X).to(self.dev))
            self.labels.append(torch.from_numpy(y).to(self.dev))
            self.masks.append(torch.from_numpy(m).to(self.dev))
        self.W = [torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32)).to(self.dev)
                  for w in ds.W]

    def epoch(self, stream=None) -> Dict:
        return api.epoch(self.ctx, self.X, self.labels, self.masks, self.W, stream)

    def epoch_host(self, stream=None) -> Dict:
        return api.epoch_host(self.ctx, self.X_host, self.labels_host, self.masks_host, self.W,
                              stream)

    def epoch_host_next(self, prefetch_next: bool, stream=None) -> Dict:
        """Host-input epoch; prefetch_next copies the next step's (static) inputs under it."""
        nx = (self.X_host, self.labels_host, self.masks_host) if prefetch_next else (None, None, None)
        return api.epoch_host_next(self.ctx, self.X_host, self.labels_host, self.masks_host, self.W,
                                   *nx, stream)

    def weights(self) -> List[np.ndarray]:
        return [w.detach().cpu().numpy() for w in self.W]

    def close(self):
        self.ctx.close()
