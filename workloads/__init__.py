"""Seeded synthetic workload generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no cell, no schedule, no
gradient): it only draws graph shapes, inputs, parameters and cotangents.
Both `oracle/` and `paper_1712_04048_b200/` consume its arrays; neither
imports the other.  See DESIGN.md "Input recipe".
"""
from .gen import (  # noqa: F401
    Batch,
    CELL_TREE_FC,
    CELL_TREE_LSTM,
    CONFIGS,
    chain,
    complete_binary_tree,
    make_batch,
    make_config_batch,
    n_params,
    remy_tree,
    sst_lengths,
    subset_csr,
    batch_from_graphs,
)
