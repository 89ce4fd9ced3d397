"""B200-native SCVT energy/gradient + Lloyd-preconditioned LBFGS (arXiv 1709.06924 hot path).

Drop-in for the reference package `scvtmesh` 0.1.0 on its hot path: the same public names
(`scvtmesh/__init__.py:9-29`) with the per-evaluation work — spherical Delaunay, Voronoi
fans, subdivided quadrature of the density, gradient, Lloyd preconditioner and the LBFGS
vector algebra — executed by hand-written sm_100a CUDA kernels in `libscvtb200.so`
(C ABI: include/scvt_b200.h).  There is no CPU fallback.
"""

from .density import DensityField, density_preset, sample_by_density
from .errors import *  # noqa: F401,F403
from .geometry import (QUADRATURE_RULES, QuadratureRule, composite_nodes, icosahedron_vertices,
                       normalize, random_sphere_points)
from .optimizer import IterationRecord, MinimizeResult, Minimizer, StoppingCriteria, minimize
from .parallel import ShardedMeshEvaluator
from .pipeline import (EvalResult, LevelResult, MeshEvaluator, RunPlan, RunResult,
                       SphericalTriangulation, bisect, bisection_ladder, parallel_iteration, run)

__version__ = "0.1.0"

__all__ = [
    "DensityField",
    "density_preset",
    "sample_by_density",
    "QuadratureRule",
    "QUADRATURE_RULES",
    "composite_nodes",
    "random_sphere_points",
    "icosahedron_vertices",
    "normalize",
    "StoppingCriteria",
    "IterationRecord",
    "MinimizeResult",
    "minimize",
    "Minimizer",
    "MeshEvaluator",
    "ShardedMeshEvaluator",
    "EvalResult",
    "SphericalTriangulation",
    "parallel_iteration",
    "bisect",
    "bisection_ladder",
    "RunPlan",
    "RunResult",
    "LevelResult",
    "run",
    "__version__",
]
