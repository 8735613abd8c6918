"""Normalised adjacency of the whole graph (oracle step O1).

P:L231-232 (§3.1): "Let A_i be the adjacency matrix of subgraph i and D_i be the
corresponding submatrix in the original degree matrix.  Â_i = D_i^{-1/2} A_i
D_i^{-1/2}".  Readings: R1 no self-loops unless ``self_loops``
(then A + I); R2 the degrees are the GLOBAL degrees of the original graph.
Pins: tests/test_oracle_graph.py (triangle 0.5, star 1/sqrt(3) [S:L61-63],
sum of degrees = 2|E| [S:L84], dense brute force).
"""
import numpy as np
import scipy.sparse as sp


def degrees(n: int, eu: np.ndarray, ev: np.ndarray, self_loops: bool = False) -> np.ndarray:
    """d_v = number of edges incident to v in the original graph (+1 with a self-loop)."""
    d = np.bincount(eu, minlength=n).astype(np.int64) + np.bincount(ev, minlength=n)
    if self_loops:
        d = d + 1
    return d


def edge_weight(du, dv):
    """w_uv = 1 / sqrt(d_u d_v) in fp64 (the (u, v) entry of D^-1/2 A D^-1/2)."""
    return 1.0 / np.sqrt(np.asarray(du, dtype=np.float64) * np.asarray(dv, dtype=np.float64))


def normalized_adjacency(n: int, eu: np.ndarray, ev: np.ndarray,
                         self_loops: bool = False) -> sp.csr_matrix:
    """Â = D^-1/2 (A [+ I]) D^-1/2 as a symmetric fp64 CSR matrix."""
    d = degrees(n, eu, ev, self_loops)
    rows = [eu, ev]
    cols = [ev, eu]
    if self_loops:
        rows.append(np.arange(n)); cols.append(np.arange(n))
    r = np.concatenate(rows).astype(np.int64)
    c = np.concatenate(cols).astype(np.int64)
    w = edge_weight(d[r], d[c])
    A = sp.csr_matrix((w, (r, c)), shape=(n, n))
    A.sort_indices()
    return A
