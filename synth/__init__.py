"""Seeded synthetic heterograph + tensor generators.

This module is the ONLY code shared by the fp64 oracle tests and the CUDA
path: it draws graphs and random tensors and holds none of the layer's
arithmetic (no GEMM, softmax, aggregation or preprocessing).  Recipe: SURVEY.md
§8(d) "Synthetic inputs", restated in DESIGN.md §4.
"""
from .heterograph import (  # noqa: F401
    CONFIGS, GraphConfig, HeteroGraph, HgtTensors, LayerTensors, make_graph, make_hgt_tensors, make_tensors,
    random_graph, get_config,
)
