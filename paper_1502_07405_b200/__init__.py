"""B200-native numeric factorization and solve of the HSS-compressed
multifrontal sparse LU (arXiv 1502.07405), behind the reference's interface.

See DESIGN.md. Numerics run only in the sm_100a kernels of libhssmf_b200.so.
"""
from .api import (  # noqa: F401
    EliminationTree, FrontStat, GridGeometry, GridProblem, HssFactors, HssOptions,
    HssRankExceeded, IoError, KrylovDivergenceError, MfFactors, SingularMatrixError,
    SolveReport, SolverError, SolverOptions, SparseMatrix, front_cluster_tree,
    generate_convdiff3d, generate_grid_problem, gmres, hss_compress, iterative_refinement,
    mf_factor, mf_solve, mf_solve_new, nested_dissection_geometric, ordered_grid,
    ordered_problem, symbolic_factorization, nested_dissection_graph, reorder_tree_separators,
    ordered_graph, read_matrix_market, write_matrix_market, equilibrate_and_permute,
    ScalingState, StructuralSingularError,
)
