"""B200-native TT-rounding hot path of arXiv 2011.06532.

Drop-in for the path-relevant public surface of the reference package
``ttpar`` (its __init__.py:10-95): TT construction, add / scale / hadamard,
inner product and norms, left/right orthonormalization, truncated SVD,
TSQR, round_tt with RoundingOptions, the
Kronecker-operator apply and TTPAR1 files -- on device-resident,
mode-sliced TT tensors, computed by hand-written sm_100a CUDA kernels
(paper_2011_06532_b200/csrc, C ABI in include/ttb.h).
"""

from .comm import (Communicator, DistComm, LocalComm, LocalGroup, SerialComm, default_comm, empty_cache,
                   run_local_ranks)
from .errors import (BoundsError, CapabilityError, CapacityError, ContractError, DeadlockError,
                     NumericError, ShapeError, TTError)
from .operator import KroneckerOperator, apply_operator, load_operator, mode2_multiply, save_operator
from .ops import add, add_n, hadamard, inner_product, norm, pivoted_cholesky, round_hadamard, scale
from .parallel import (ROUNDING_VARIANTS, RoundingOptions, TruncatedSVD, TSQRFactor, distribute, gather,
                       orthonormalize, round_tt, round_tt_host, serial_tt, truncated_svd, tsqr_apply_q,
                       tsqr_factor)
from .tensor import DistTTTensor, TTCore, TTTensor, block_bounds, random_tt
from .ttio import load_tt, load_tt_dist, save_tt, save_tt_dist

__version__ = "0.1.0"

__all__ = [
    "BoundsError", "CapabilityError", "CapacityError", "Communicator", "ContractError", "DeadlockError",
    "DistComm", "DistTTTensor", "KroneckerOperator", "LocalComm", "LocalGroup", "NumericError", "ROUNDING_VARIANTS", "RoundingOptions", "SerialComm",
    "ShapeError", "TSQRFactor", "TTCore", "TTError", "TTTensor", "TruncatedSVD", "add", "add_n",
    "apply_operator", "block_bounds", "default_comm", "distribute", "empty_cache", "gather", "hadamard", "inner_product", "load_operator",
    "load_tt", "load_tt_dist", "mode2_multiply", "norm", "pivoted_cholesky",
    "orthonormalize", "random_tt", "round_hadamard", "round_tt", "round_tt_host", "run_local_ranks", "save_operator", "save_tt",
    "save_tt_dist", "scale", "serial_tt", "truncated_svd", "tsqr_apply_q",
    "tsqr_factor", "__version__",
]
