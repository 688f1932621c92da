"""B200-native solver for entropic unbalanced optimal transport by domain decomposition.

Drop-in for the solve path of the reference ``domdec`` package (arXiv
2410.08859): problem and partition setup, ``domdec_solve``, the returned
basic-cell marginals, dual potentials and primal-dual objective.  All compute
runs in ``libdomdec_b200.so`` (hand-written sm_100a CUDA, C ABI in
``include/domdec_b200.h``); there is no CPU path.
"""

from .grids import (DivergenceSpec, Grid, GridMeasure, GridMismatchError, SparseCellMarginal,
                    TransportProblem, assemble_y_marginal, kl_divergence, truncate_and_rebox)
from .decomposition import (BasicPartition, CompositePartition, Decomposition,
                            build_basic_partition, build_composite_partitions,
                            build_staggered_batches, make_decomposition)

__version__ = "0.1.0"

__all__ = [
    "DivergenceSpec", "Grid", "GridMeasure", "GridMismatchError", "SparseCellMarginal",
    "TransportProblem", "assemble_y_marginal", "kl_divergence", "truncate_and_rebox",
    "BasicPartition", "CompositePartition", "Decomposition", "build_basic_partition",
    "build_composite_partitions", "build_staggered_batches", "make_decomposition",
]
