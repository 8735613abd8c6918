"""Pins for oracle/graph.py: worked examples and a dense brute force."""
import math

import numpy as np

from oracle.graph import degrees, normalized_adjacency
from synth import small_random_graph


def test_spec_normalize_examples(spec_examples):
    for ex in spec_examples["normalize"]:
        e = np.array(ex["edges"])
        A = normalized_adjacency(ex["n"], e[:, 0], e[:, 1])
        vals = A.tocoo()
        # every listed edge, in both directions, carries the printed weight
        for u, v in ex["edges"]:
            assert math.isclose(A[u, v], ex["weight"], rel_tol=1e-15)
            assert math.isclose(A[v, u], ex["weight"], rel_tol=1e-15)
        assert vals.nnz == 2 * len(ex["edges"])


def test_degree_sum_is_twice_edges():
    d = small_random_graph(300, 900, (8, 4, 3), seed=3)
    deg = degrees(d.n, d.eu, d.ev)
    assert deg.sum() == 2 * d.m


def _brute_dense(n, eu, ev, self_loops=False):
    A = np.zeros((n, n))
    for u, v in zip(eu.tolist(), ev.tolist()):
        A[u, v] = 1.0
        A[v, u] = 1.0
    if self_loops:
        A += np.eye(n)
    deg = A.sum(axis=1)
    out = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if A[i, j]:
                out[i, j] = A[i, j] / math.sqrt(deg[i] * deg[j])
    return out


def test_dense_brute_force():
    for seed, sl in [(1, False), (2, True), (5, False)]:
        d = small_random_graph(40, 90, (4, 3), seed=seed)
        A = normalized_adjacency(d.n, d.eu, d.ev, self_loops=sl).toarray()
        np.testing.assert_allclose(A, _brute_dense(d.n, d.eu, d.ev, sl), rtol=0, atol=1e-15)
        assert np.array_equal(A, A.T)
