"""paper_1903_07884_b200 -- B200-native hot path of the circulant-preconditioned
voxel VIE (arXiv 1903.07884), drop-in for the reference package ``voxvie``'s
operator / preconditioner / GMRES API.

Hot path (CUDA, sm_100a, via the C-ABI in include/voxvie_b200.h):
  operator.plan_operator / apply_n / apply_system        (reference operator.py)
  circulant.build_one_level / build_reduced_one_level /
            reduce_one_level / build_two_level / build_blocked / *.apply
                                                          (reference circulant.py)
  solver.gmres                                            (reference solver.py)
Host-side setup inputs (grid, kernel assembly, workloads) are plain numpy.
"""

from .grid import MATERIALS, PermittivityMap, Physics, VoxelGrid, homogenize, medium_coefficient
from .kernel import ToeplitzKernel, assemble_kernel
from .operator import apply_n, apply_system, plan_operator

__version__ = "0.1.0"

__all__ = [
    "MATERIALS", "PermittivityMap", "Physics", "ToeplitzKernel", "VoxelGrid",
    "apply_n", "apply_system", "assemble_kernel", "homogenize", "medium_coefficient",
    "plan_operator", "__version__",
]
from .circulant import (  # noqa: E402
    BlockedPrec, Box, OneLevelPrec, Partition, ReducedOneLevelPrec, TwoLevelPrec, build_blocked,
    build_one_level, build_reduced_one_level, build_two_level, partition_boxes, reduce_one_level,
)
from .solver import SolveReport, gmres  # noqa: E402

__all__ += [
    "BlockedPrec", "Box", "OneLevelPrec", "Partition", "ReducedOneLevelPrec", "SolveReport",
    "TwoLevelPrec", "build_blocked", "build_one_level", "build_reduced_one_level", "build_two_level",
    "gmres", "partition_boxes", "reduce_one_level",
]
