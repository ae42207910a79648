"""B200-native butterfly factorization hot path (arxiv/paper_1502_01379).

Drop-in for the reference package ``butterfly``'s apply/construction path:
same names, factor layout and errors; compute runs in libbfly.so (sm_100a)
through the C ABI of include/bfly.h.
"""

from ._lib import OracleError
from .factors import (BlockDiagonalFactor, ButterflyFactors, DevicePlan, MiddleFactor, NnzReport,
                      TransferFactor, factors_equal, from_arrays)
from .construct import (DEFAULT_PARAMS, OversamplingParams, block_diagonal_probe, factorize,
                        middle_factorization_matvec, middle_factorization_sampling, recursive_factor_u,
                        recursive_factor_v)
from .kernels import (ComposedOperator, DenseOracle, DftKernel, DftPlusKernel, FioKernel, HankelKernel, Radon2DKernel,
                      composed_matvec, dft_apply, fio_entry, hankel1_orders_device, hankel_entry)
from .metrics import OperatorReference, RowSampledReference, estimate_eps_a, estimate_eps_a_info
from .storage import FormatError, load_factors, read_vector, save_factors, write_vector
from .partition import (BlockId, DyadicPartition, QuadtreePartition, block_cols, block_rows, level_geometry,
                        make_partition, make_quadtree_partition)

__all__ = [n for n in dir() if not n.startswith("_")]
__version__ = "0.1.0"
