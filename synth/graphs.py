"""Seeded graph / feature / label / weight generators (inputs only, no method arithmetic).

Recipe:
  * graph: degree-corrected planted-partition Chung-Lu.  Vertex weights
    theta_v ~ (v + v0)^(-1/(tau-1)) scaled to sum nnz; the first endpoint of an
    edge is drawn ~theta, the second ~theta inside the first endpoint's class with
    probability h, else ~theta globally.  Self-loops dropped, duplicates removed,
    topped up to exactly m = nnz/2 undirected pairs; isolated vertices get one
    edge each, paid for by removing edges whose endpoints both keep degree >= 1.
    Vertex ids are randomly permuted.  Edges are returned once, as (min, max),
    sorted lexicographically.
  * labels: the planted class, uniform over C classes.
  * features: x_v = snr * mu_{y_v} + N(0, I), mu_c ~ N(0, I), fp32.  ``snr`` (feature
    signal-to-noise knob, default 1 = the SURVEY §8(d2) recipe) scales the class means:
    small values (e.g. 0.05 at F_0 = 128) make the classes overlap so train accuracy
    climbs over tens of epochs instead of saturating at once (used by the adaptive-ε
    study and the follow-mode trajectory tests; inputs only).
  * masks: train / val / test = 60 / 20 / 20 by a seeded shuffle.
  * weights: Glorot-uniform U(+-sqrt(6/(F_in+F_out))), fp32, [F_in x F_out].
"""
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .configs import GraphConfig


@dataclass
class Dataset:
    n: int
    eu: np.ndarray          # int32 [m], eu < ev
    ev: np.ndarray          # int32 [m]
    X: np.ndarray           # float32 [n, F0]
    y: np.ndarray           # int32 [n]
    train: np.ndarray       # bool [n]
    val: np.ndarray         # bool [n]
    test: np.ndarray        # bool [n]
    W: List[np.ndarray]     # float32 [F_{l-1}, F_l]
    dims: tuple
    name: str = ""

    @property
    def m(self) -> int:
        return int(self.eu.shape[0])


def _rngs(seed: int, k: int = 4):
    ss = np.random.SeedSequence(seed)
    return [np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(k)]


def _sorted_unique(a: np.ndarray) -> np.ndarray:
    a = np.sort(a)
    if a.size == 0:
        return a
    keep = np.empty(a.size, dtype=bool)
    keep[0] = True
    np.not_equal(a[1:], a[:-1], out=keep[1:])
    return a[keep]


class _CdfSampler:
    """Inverse-CDF sampling with a guide table (O(1) expected per draw)."""

    def __init__(self, cdf: np.ndarray, buckets: Optional[int] = None):
        self.cdf = cdf
        k = buckets or max(1024, 4 * cdf.shape[0])
        self.k = k
        # guide[b] = first index i with cdf[i] > b / k
        self.guide = np.searchsorted(cdf, np.arange(k, dtype=np.float64) / k, side="right")
        np.minimum(self.guide, cdf.shape[0] - 1, out=self.guide)

    def __call__(self, r: np.ndarray) -> np.ndarray:
        cdf = self.cdf
        b = np.minimum((r * self.k).astype(np.int64), self.k - 1)
        i = self.guide[b]
        last = cdf.shape[0] - 1
        while True:
            adv = (cdf[i] <= r) & (i < last)
            if not adv.any():
                return i
            i[adv] += 1


def chung_lu_planted(n: int, m: int, tau: float, v0: float, classes: int,
                     homophily: float, rng: np.random.Generator):
    """Return (eu, ev, y): m undirected edges (eu < ev, sorted) and planted classes."""
    if m <= 0 or n < 2:
        raise ValueError("need n >= 2 and m >= 1")
    if m > n * (n - 1) // 2:
        raise ValueError("m exceeds the number of vertex pairs")
    ranks = np.arange(n, dtype=np.float64)
    theta = (ranks + v0) ** (-1.0 / (tau - 1.0))
    theta *= (2.0 * m) / theta.sum()
    cdf = np.cumsum(theta)
    cdf /= cdf[-1]
    cls = rng.integers(0, classes, size=n).astype(np.int32)
    # per-class CDFs laid end to end: class c occupies [c, c+1)
    order = np.argsort(cls, kind="stable")
    cls_sorted = cls[order]
    w_sorted = theta[order]
    cum = np.cumsum(w_sorted)
    starts = np.searchsorted(cls_sorted, np.arange(classes), side="left")
    ends = np.searchsorted(cls_sorted, np.arange(classes), side="right")
    cdf_cat = np.empty(n, dtype=np.float64)
    for c in range(classes):
        s, e = starts[c], ends[c]
        if e == s:
            continue
        base = cum[s - 1] if s > 0 else 0.0
        seg = (cum[s:e] - base) / (cum[e - 1] - base)
        cdf_cat[s:e] = c + seg
        cdf_cat[e - 1] = c + 1.0
    glob = _CdfSampler(cdf)
    cat = _CdfSampler(cdf_cat / classes)
    keys = np.empty(0, dtype=np.int64)          # sorted, unique
    need = m
    rounds = 0
    while need > 0:
        rounds += 1
        if rounds > 200:
            raise RuntimeError("Chung-Lu top-up did not converge")
        k = int(need * 1.15) + 64
        u = glob(rng.random(k))
        inclass = rng.random(k) < homophily
        v = glob(rng.random(k))
        ni = int(inclass.sum())
        if ni:
            cu = cls[u[inclass]]
            v[inclass] = order[cat((cu + rng.random(ni)) / classes)]
        ok = u != v
        u, v = u[ok], v[ok]
        new = np.minimum(u, v).astype(np.int64) * n + np.maximum(u, v)
        new = _sorted_unique(new)
        if keys.size:
            pos = np.searchsorted(keys, new)
            pos[pos == keys.size] = 0
            new = new[keys[pos] != new]
        if new.size > need:
            # drop a uniformly random surplus (unbiased trim to exactly m)
            new = np.sort(rng.choice(new, size=need, replace=False))
        keys = np.sort(np.concatenate([keys, new])) if keys.size else new
        need = m - keys.shape[0]
    eu = (keys // n).astype(np.int64)
    ev = (keys % n).astype(np.int64)
    # connect isolated vertices, then remove the same number of surplus edges
    deg = np.bincount(eu, minlength=n) + np.bincount(ev, minlength=n)
    iso = np.flatnonzero(deg == 0)
    if iso.size:
        keyset = set()
        add_u, add_v = [], []
        for w in iso.tolist():
            while True:
                p = int(glob(rng.random(1))[0])
                if p == w:
                    continue
                kk = (min(w, p), max(w, p))
                if kk in keyset:
                    continue
                keyset.add(kk)
                add_u.append(kk[0]); add_v.append(kk[1])
                deg[w] += 1; deg[p] += 1
                break
        # remove len(iso) existing edges whose endpoints both keep degree >= 1
        keep = np.ones(eu.shape[0], dtype=bool)
        removed = 0
        for e in rng.permutation(eu.shape[0]).tolist():
            if removed == iso.size:
                break
            a, b = int(eu[e]), int(ev[e])
            if deg[a] >= 2 and deg[b] >= 2:
                keep[e] = False
                deg[a] -= 1; deg[b] -= 1
                removed += 1
        if removed != iso.size:
            raise RuntimeError("could not rebalance isolated vertices")
        eu = np.concatenate([eu[keep], np.asarray(add_u, dtype=np.int64)])
        ev = np.concatenate([ev[keep], np.asarray(add_v, dtype=np.int64)])
    # random vertex-id permutation
    perm = rng.permutation(n)
    pu, pv = perm[eu], perm[ev]
    key = np.sort(np.minimum(pu, pv).astype(np.int64) * n + np.maximum(pu, pv))
    y = np.empty(n, dtype=np.int32)
    y[perm] = cls
    return (key // n).astype(np.int32), (key % n).astype(np.int32), y


def glorot_weights(dims, rng: np.random.Generator) -> List[np.ndarray]:
    out = []
    for fi, fo in zip(dims[:-1], dims[1:]):
        lim = np.sqrt(6.0 / (fi + fo))
        out.append(rng.uniform(-lim, lim, size=(fi, fo)).astype(np.float32))
    return out


def _features_masks(n, y, f0, classes, rng_f, rng_m, snr: float = 1.0):
    mu = rng_f.standard_normal((classes, f0), dtype=np.float32)
    X = rng_f.standard_normal((n, f0), dtype=np.float32)
    if snr != 1.0:
        mu *= np.float32(snr)
    X += mu[y]
    perm = rng_m.permutation(n)
    ntr = int(round(0.6 * n))
    nva = int(round(0.2 * n))
    train = np.zeros(n, dtype=bool); train[perm[:ntr]] = True
    val = np.zeros(n, dtype=bool); val[perm[ntr:ntr + nva]] = True
    test = np.zeros(n, dtype=bool); test[perm[ntr + nva:]] = True
    return X, train, val, test


def make_dataset(cfg: GraphConfig, scale: Optional[float] = None, snr: float = 1.0) -> Dataset:
    """Generate a config's dataset.  ``scale`` < 1 shrinks n and nnz (same mean degree);
    ``snr`` scales the feature class means (see the module docstring)."""
    n, m = cfg.n, cfg.m
    v0 = cfg.v0
    if scale is not None and scale != 1.0:
        n = max(64, int(round(cfg.n * scale)))
        m = max(n, int(round(cfg.m * scale)))
        v0 = cfg.v0 * scale
        m = min(m, n * (n - 1) // 4)
    rg, rf, rm, rw = _rngs(cfg.seed)
    eu, ev, y = chung_lu_planted(n, m, cfg.tau, v0, cfg.classes, cfg.homophily, rg)
    X, train, val, test = _features_masks(n, y, cfg.dims[0], cfg.classes, rf, rm, snr)
    W = glorot_weights(cfg.dims, rw)
    name = cfg.key if scale in (None, 1.0) else f"{cfg.key}@{scale}"
    if snr != 1.0:
        name += f"/snr{snr}"
    return Dataset(n=n, eu=eu, ev=ev, X=X, y=y, train=train, val=val, test=test,
                   W=W, dims=tuple(cfg.dims), name=name)


def small_random_graph(n: int, m: int, dims, seed: int, classes: Optional[int] = None,
                       tau: float = 2.5, v0: float = 1.0, homophily: float = 0.7,
                       snr: float = 1.0) -> Dataset:
    """A small heavy-tailed dataset for unit tests."""
    classes = classes or dims[-1]
    rg, rf, rm, rw = _rngs(seed)
    eu, ev, y = chung_lu_planted(n, m, tau, v0, classes, homophily, rg)
    X, train, val, test = _features_masks(n, y, dims[0], classes, rf, rm, snr)
    W = glorot_weights(dims, rw)
    return Dataset(n=n, eu=eu, ev=ev, X=X, y=y, train=train, val=val, test=test,
                   W=W, dims=tuple(dims), name=f"rand{n}x{m}")


def circulant_edges(n: int, r: int):
    """r-regular circulant graph (r even): v ~ v+k mod n for k = 1..r/2."""
    assert r % 2 == 0 and n > r
    a, b = [], []
    for k in range(1, r // 2 + 1):
        v = np.arange(n)
        w = (v + k) % n
        a.append(np.minimum(v, w)); b.append(np.maximum(v, w))
    a = np.concatenate(a); b = np.concatenate(b)
    key = a.astype(np.int64) * n + b
    key = np.unique(key)
    return (key // n).astype(np.int32), (key % n).astype(np.int32)


def dyadic_fixture(n: int = 64, r: int = 4, dims=(16, 8, 4), seed: int = 7) -> Dataset:
    """Dyadic fixture: r-regular circulant graph (so every
    normalised weight is 1/r), integer features in [-4, 4], W in {-1, 0, 1}.
    Every product and partial sum is exactly representable in fp32/TF32."""
    rg, rf, rm, rw = _rngs(seed)
    eu, ev = circulant_edges(n, r)
    perm = rg.permutation(n)
    pu, pv = perm[eu], perm[ev]
    a = np.minimum(pu, pv); b = np.maximum(pu, pv)
    srt = np.argsort(a.astype(np.int64) * n + b, kind="stable")
    eu, ev = a[srt].astype(np.int32), b[srt].astype(np.int32)
    classes = dims[-1]
    y = rf.integers(0, classes, size=n).astype(np.int32)
    X = rf.integers(-4, 5, size=(n, dims[0])).astype(np.float32)
    W = [rw.integers(-1, 2, size=(fi, fo)).astype(np.float32)
         for fi, fo in zip(dims[:-1], dims[1:])]
    perm2 = rm.permutation(n)
    ntr = int(round(0.6 * n))
    train = np.zeros(n, dtype=bool); train[perm2[:ntr]] = True
    val = np.zeros(n, dtype=bool); val[perm2[ntr:]] = True
    test = np.zeros(n, dtype=bool)
    return Dataset(n=n, eu=eu, ev=ev, X=X, y=y, train=train, val=val, test=test,
                   W=W, dims=tuple(dims), name=f"dyadic{n}r{r}")
