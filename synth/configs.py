"""The five workload shapes of BASELINE.json ``configs`` (SURVEY.md §8 config key).

``nnz`` counts directed CSR entries (reading R23): undirected pairs = nnz // 2.
Degree-law parameters (tau, v0) were solved so the expected maximum degree
matches the real graph's; they are generator inputs only.
"""
from dataclasses import dataclass, field
from typing import List


@dataclass(frozen=True)
class GraphConfig:
    key: str            # "C1".."C5"
    name: str
    n: int              # vertices
    nnz: int            # directed CSR entries (2 x undirected edges)
    dims: tuple         # F_0 -> ... -> F_L
    tau: float          # power-law exponent of expected degrees
    v0: float           # rank offset of the Chung-Lu weights
    homophily: float    # P(second endpoint drawn inside the first endpoint's class)
    gpus: tuple         # GPU counts BASELINE.json quotes this config at
    parts_per_gpu: int = 1
    seed: int = 0

    @property
    def m(self) -> int:
        return self.nnz // 2

    @property
    def classes(self) -> int:
        return self.dims[-1]

    @property
    def L(self) -> int:
        return len(self.dims) - 1


def _c(i, **kw):
    return GraphConfig(seed=0xCDF60000 + i, **kw)


CONFIGS = {
    # configs[0]: Cora-shaped, 2 partitions on 1 GPU, eps = 0 and int8 on.
    "C1": _c(1, key="C1", name="cora-shaped", n=2708, nnz=10556, dims=(1433, 16, 7),
             tau=2.5, v0=2.1, homophily=0.8, gpus=(1,), parts_per_gpu=2),
    # configs[1]: ogbn-arxiv-shaped; 1,166,243 is odd, so nnz = 2 * 583,121.
    "C2": _c(2, key="C2", name="ogbn-arxiv-shaped", n=169343, nnz=1166242,
             dims=(128, 256, 256, 40), tau=2.5, v0=0.4, homophily=0.65, gpus=(1, 2)),
    # configs[2]: Reddit-shaped (the bench workload).
    "C3": _c(3, key="C3", name="reddit-shaped", n=232965, nnz=114615892,
             dims=(602, 256, 41), tau=2.2, v0=492.0, homophily=0.8, gpus=(1, 2, 4, 8)),
    # configs[3]: ogbn-products-shaped, 8 GPUs with an eps sweep.
    "C4": _c(4, key="C4", name="ogbn-products-shaped", n=2449029, nnz=61859140,
             dims=(100, 256, 256, 47), tau=2.2, v0=145.0, homophily=0.8, gpus=(8,)),
    # configs[4]: large power-law, 8 GPUs, ablation no-cache / cache / cache+int8.
    "C5": _c(5, key="C5", name="large-power-law", n=1600000, nnz=264000000,
             dims=(200, 256, 256, 172), tau=2.2, v0=883.0, homophily=0.7, gpus=(8,)),
}


def get_config(key: str) -> GraphConfig:
    return CONFIGS[key.upper()]
