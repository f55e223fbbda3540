"""B200-native solve phase for subdomain-deflated Krylov solvers preconditioned
by local smoothed-aggregation AMG (arXiv 1710.03940).

Drop-in for the reference package's solver API (deflamg 0.1.0,
pkg/src/deflamg/__init__.py): ``DeflatedSolver``, ``SolverConfig``,
``SparseMatrix``, the partition helpers and the exception classes.  The solve
runs in hand-written sm_100a kernels behind the C ABI of
``include/dflb200.h`` (``libdflb200.so``, built in-tree).
"""
from .config import SolverConfig
from .errors import (
    BreakdownError,
    CommunicatorError,
    ConfigError,
    DeflamgError,
    DeviceError,
    DimensionError,
    ParseError,
    PartitionError,
    SingularMatrixError,
    StructureError,
)
from .runtime import Partition, partition_contiguous
from .sparse import SparseMatrix

__version__ = "0.1.0"


def __getattr__(name):
    # the solver pulls in the native library; import it lazily so that the
    # pure-host pieces (config, generators) stay importable without it
    if name in ("DeflatedSolver", "solve_deflated"):
        from . import deflation

        return getattr(deflation, name)
    raise AttributeError(name)


__all__ = [
    "DeflatedSolver",
    "solve_deflated",
    "SolverConfig",
    "SparseMatrix",
    "Partition",
    "partition_contiguous",
    "DeflamgError",
    "DimensionError",
    "StructureError",
    "SingularMatrixError",
    "PartitionError",
    "CommunicatorError",
    "BreakdownError",
    "ParseError",
    "ConfigError",
    "DeviceError",
    "__version__",
]
