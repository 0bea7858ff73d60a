"""B200-native iterative sketching for overdetermined least squares
(arXiv 2311.04362), a drop-in for the `itsketch` package's north-star path
`iterative_sketching(a, b, cfg, truth)`.

The Python layer mirrors the reference API; all arithmetic runs in the
sm_100a kernels of libitsk_b200.so (see include/itsk_b200.h).
"""

from ._lib import SingularMatrixError
from .embed import SparseSignEmbedding, default_distortion, sparse_sign_new
from .linalg import (
    QrFactors,
    cond_est,
    householder_qr_econ,
    rand_power_norm_est,
    tri_solve_upper,
    tri_solve_upper_transpose,
)
from .lsqr import lsqr, sketch_and_precondition
from .problems import LsProblem, Truth, gen_randsvd, gen_sparse
from .sparse import CsrMatrix
from .solvers import (
    SolveResult,
    SolverConfig,
    SolveTrace,
    damping_params,
    iterative_sketching,
    momentum_params,
    release_workspaces,
    should_stop,
    sketch_and_solve,
)

__all__ = [
    "SingularMatrixError", "SparseSignEmbedding", "default_distortion", "sparse_sign_new",
    "QrFactors", "cond_est", "householder_qr_econ", "rand_power_norm_est", "tri_solve_upper",
    "tri_solve_upper_transpose", "LsProblem", "Truth", "gen_randsvd", "SolveResult", "SolverConfig",
    "SolveTrace", "damping_params", "iterative_sketching", "momentum_params", "release_workspaces",
    "should_stop", "sketch_and_solve", "lsqr", "sketch_and_precondition", "gen_sparse", "CsrMatrix",
]
