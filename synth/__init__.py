"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path.

This module holds NO arithmetic of the CDFGNN method (no normalisation, no
partitioning, no GCN, no cache, no quantisation).  It only draws the inputs the
method consumes — an undirected edge list, vertex features, labels, split
masks and initial weights — from fixed seeds, with the shapes of the paper's
workloads (Table 1; BASELINE.json ``configs``).  The
recipe is stated in DESIGN.md §"Input recipe".
"""
from .configs import CONFIGS, GraphConfig, get_config
from .graphs import (
    Dataset,
    chung_lu_planted,
    circulant_edges,
    dyadic_fixture,
    make_dataset,
    small_random_graph,
    glorot_weights,
)

__all__ = [
    "CONFIGS",
    "GraphConfig",
    "get_config",
    "Dataset",
    "chung_lu_planted",
    "circulant_edges",
    "dyadic_fixture",
    "make_dataset",
    "small_random_graph",
    "glorot_weights",
]
