"""CPU oracle (TEST INFRASTRUCTURE ONLY; see cavs_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports it.
"""
from .cavs_oracle import (  # noqa: F401
    OracleError,
    TREE_FC,
    TREE_LSTM,
    backward,
    bf16r,
    forward,
    global_children,
    levels_recursive,
    lm_head,
    loss,
    pack,
    run,
    schedule,
    schedule_alg1,
    unpack,
    validate,
)
