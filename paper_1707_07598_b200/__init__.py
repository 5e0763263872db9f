"""B200-native adaptive MSFV forward + gradient (drop-in for msinv's adaptive path).

Public names mirror the reference package's (msinv/__init__.py:3-20) for the
hot path; compute runs in libmsfv.so (sm_100a) through the C-ABI in
include/msfv.h.  Importing this package does not touch the GPU.
"""

from .mesh import TensorMesh, CoarsePartition, create_mesh, create_partition, block_node_sets
from .operators import (
    sigma_map, sigma_deriv, nodal_gradient, edge_cell_map,
    assemble_operator, DiffusionOperator, grad_A_u, grad_A_u_full,
)
from .basis import (
    BasisSpec, MultiscaleBasis, BasisBuilder, generate_bc_lagrange, assemble_basis,
    coarse_hat_values,
)
from .forward import Survey, ReducedState, forward_reduced, AdaptiveSensitivity, sensitivity_adaptive
from .inversion import misfit_ssd, misfit_ssd_dev, AdaptiveReducedProblem
from .models import build_survey
from .enriched import source_family, skeleton_family, local_pca_family, reference_fields
from .fine import (
    forward_full, FullState, FullSensitivity, sensitivity_full, FullProblem, block_cg, IterativeResult,
)
from .gn import gauss_newton_dev, GNSettings, DeviceObjective, DeviceTrace
from .table3 import apply_Yk, apply_Xk, apply_Yk_dev, apply_Xk_dev
from .planar import (
    Mesh2D, Partition2D, create_mesh_2d, create_partition_2d, AdaptiveReducedProblem2D,
    ReducedState2D, Sensitivity2D, cell_survey_2d, config_problem_2d,
)
from .errors import (
    InvalidModelError, FactorizationError, SolverBreakdown,
    StaleBasisError, ReducedSingularError,
)

__version__ = "0.1.0"
