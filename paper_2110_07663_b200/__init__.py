"""semlab_b200: B200-native spectral-element pressure-Poisson hot path (arXiv 2110.07663).

The compute path is libsemlab_b200.so (hand-written sm_100a kernels + C++ host behind the
C-ABI of include/semlab_b200.h); this package is the Python mirror of the reference API.
"""
from .semlab import (ASM, ASM_SMOOTHER, COARSE_AMG, COARSE_DIRECT, DIRICHLET, JACOBI_SMOOTHER, NEUMANN, RAS,
                     RAS_SMOOTHER, ChebyParams, ChebyshevSmoother, Context, GmresConfig, GmresStats, HexMesh,
                     LambdaEstimate, LinOp, Pmg, SchwarzSmoother, SemSpace, default_context, estimate_lambda_max,
                     generate_kershaw, gmres_solve, pcg_solve)

__all__ = [
    "ASM", "ASM_SMOOTHER", "COARSE_AMG", "COARSE_DIRECT", "DIRICHLET", "JACOBI_SMOOTHER", "NEUMANN", "RAS",
    "RAS_SMOOTHER", "ChebyParams", "ChebyshevSmoother", "Context", "GmresConfig", "GmresStats", "HexMesh",
    "LambdaEstimate", "LinOp", "Pmg", "SchwarzSmoother", "SemSpace", "default_context", "estimate_lambda_max",
    "generate_kershaw", "gmres_solve", "pcg_solve",
]
