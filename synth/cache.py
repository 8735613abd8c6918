"""On-disk cache of generated datasets (npz under $CDFGNN_DATA_CACHE or /tmp)."""
import os
import time

import numpy as np

from .configs import GraphConfig
from .graphs import Dataset, make_dataset

CACHE_DIR = os.environ.get("CDFGNN_DATA_CACHE", "/tmp/cdfgnn_data")


def _path(cfg: GraphConfig, scale, snr=1.0):
    tag = f"{cfg.key}_{cfg.seed:x}" + ("" if scale in (None, 1.0) else f"_s{scale}") + \
        ("" if snr == 1.0 else f"_snr{snr}")
    return os.path.join(CACHE_DIR, tag + ".npz")


def cached_dataset(cfg: GraphConfig, scale=None, wait_for_writer: bool = False,
                   write: bool = True, snr: float = 1.0) -> Dataset:
    path = _path(cfg, scale, snr)
    if wait_for_writer:
        t0 = time.time()
        while not os.path.exists(path) and time.time() - t0 < 1800:
            time.sleep(0.5)
    if os.path.exists(path):
        z = np.load(path)
        W = [z[f"W{i}"] for i in range(len(cfg.dims) - 1)]
        return Dataset(n=int(z["n"]), eu=z["eu"], ev=z["ev"], X=z["X"], y=z["y"], train=z["train"],
                       val=z["val"], test=z["test"], W=W, dims=tuple(cfg.dims), name=str(z["name"]))
    d = make_dataset(cfg, scale, snr)
    if write:
        os.makedirs(CACHE_DIR, exist_ok=True)
        tmp = path + f".tmp{os.getpid()}.npz"
        np.savez(tmp, n=d.n, eu=d.eu, ev=d.ev, X=d.X, y=d.y, train=d.train, val=d.val,
                 test=d.test, name=d.name, **{f"W{i}": w for i, w in enumerate(d.W)})
        os.replace(tmp, path)
    return d
