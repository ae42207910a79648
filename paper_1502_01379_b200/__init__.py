"""B200-native butterfly factorization hot path (arxiv/paper_1502_01379).

Drop-in for the reference package ``butterfly``'s apply/construction path:
same names, factor layout and errors; compute runs in libbfly.so (sm_100a)
through the C ABI of include/bfly.h.
"""

from ._lib import OracleError
from .factors import (BlockDiagonalFactor, ButterflyFactors, DevicePlan, MiddleFactor, NnzReport,
                      TransferFactor, factors_equal, from_arrays)
from .partition import BlockId, DyadicPartition, block_cols, block_rows, level_geometry, make_partition

__all__ = [n for n in dir() if not n.startswith("_")]
__version__ = "0.1.0"
