"""B200-native SKR hot path: greedy similarity sort + GCRO-DR recycling chain.

Drop-in surface of the reference package ``kryrec`` for the hot path
(kryrec/__init__.py): ``greedy_sort``, ``gcrodr_solve``, ``SolverConfig``,
``SolveReport``, ``RecycleSpace``, ``build_preconditioner`` ('none' |
'jacobi' | 'bjacobi' | 'sor' | 'ilu0' | 'icc0'), ``CsrMatrix`` -- plus ``solve_sequence`` (the chained solve of
harness.py:233-260 with the recycle pair resident on the GPU) and
``sharded_greedy_sort`` (multi-GPU). All arithmetic runs in libskr.so
(hand-written sm_100a CUDA); there is no CPU fallback.
"""

from .gcrodr import (
    GcroDrEngine,
    RecycleSpace,
    gcrodr_solve,
    harmonic_ritz_first_cycle,
    harmonic_ritz_subsequent,
)
from .gmres import SolveReport, SolverConfig, gmres_solve
from .precond import (
    BlockJacobiPreconditioner,
    DevicePreconditioner,
    Icc0Preconditioner,
    IdentityPreconditioner,
    Ilu0Preconditioner,
    JacobiPreconditioner,
    Preconditioner,
    SorPreconditioner,
    ZeroPivotError,
    build_device_preconditioner,
    build_preconditioner,
)
from .sequence import (
    ChainState,
    SequenceResult,
    chunk_positions,
    gather_results,
    chain_grid_ctas,
    solve_chains,
    solve_sequence,
    split_chunks,
)
from .dataset import DatasetWriter, export_dataset
from .sorting import (
    ParameterMatrix,
    frobenius_distance,
    greedy_sort,
    greedy_sort_device,
    grouped_sort,
    grouped_sort_device,
    sharded_greedy_sort,
)
from .sparse import CsrMatrix, DeviceCsr, axpy, dot, eye, norm2, spmv

__version__ = "0.1.0"

__all__ = [
    "BlockJacobiPreconditioner", "DevicePreconditioner", "Icc0Preconditioner", "Ilu0Preconditioner",
    "SorPreconditioner", "build_device_preconditioner",
    "ChainState", "CsrMatrix", "DeviceCsr", "GcroDrEngine", "IdentityPreconditioner", "JacobiPreconditioner",
    "ParameterMatrix", "Preconditioner", "RecycleSpace", "SequenceResult", "SolveReport",
    "SolverConfig", "ZeroPivotError", "axpy", "build_preconditioner", "chunk_positions", "dot",
    "eye", "export_dataset", "DatasetWriter", "gather_results", "frobenius_distance", "gcrodr_solve", "gmres_solve", "greedy_sort",
    "greedy_sort_device", "grouped_sort", "grouped_sort_device", "harmonic_ritz_first_cycle", "harmonic_ritz_subsequent", "norm2",
    "sharded_greedy_sort", "chain_grid_ctas", "solve_chains", "solve_sequence", "split_chunks", "spmv",
]
