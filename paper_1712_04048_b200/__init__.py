"""B200-native (sm_100a) level-batched vertex-function engine for the hot path of
Cavs (Zhang et al., arXiv 1712.04048): F over a minibatch of input graphs G,
forward and backward, behind the C-ABI in include/cavs.h.

Importing this package loads libcavs.so and fails loudly if it is missing.
"""
from .cavs import (  # noqa: F401
    PHASES,
    BF16,
    CELLS,
    Context,
    CavsError,
    EXPORTS,
    FP32,
    LIB_PATH,
    TREE_FC,
    TREE_LSTM,
    lib,
    param_count,
)
