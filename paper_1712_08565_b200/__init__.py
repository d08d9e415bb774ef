"""B200-native MF-WQ hot path: drop-in for the reference igamf operator API.

Names mirror ``igamf/__init__.py:9-31`` for the path this package builds:
setup (spaces, WQ rules, geometry maps), the matrix-free stiffness operator,
the fast-diagonalisation preconditioner, PCG / BiCGStab, and the tensor-Gauss
load vector and L2 / H1 error norms.  Compute runs in
hand-written sm_100a kernels (libmfwq.so, C-ABI in include/mfwq.h).
"""

from .errors import (DegenerateGeometryError, EigenSolveError,
                     IndefiniteOperatorError, WQConstructionError)
from .geometry import GeometryMap, affine_map, identity_map, quarter_ring_map
from .kron import CostMeter, kron_apply, tensor_grid
from .problems import (ManufacturedCase, assemble_rhs, cube_sine_case, h1_relative_error, l2_relative_error,
                       oscillating_case)
from .operators import (COEFF_EVAL_FLOPS, MassOperator, StiffnessOperator, SystemOperator, apply_system,
                        setup_mass, setup_stiffness)
from .solvers import (FDPreconditioner, KrylovReport, bicgstab, cg, stopping_tolerance,
                      univariate_parametric_matrices)
from .splines import (KnotVector, TensorSpace, make_uniform_knots,
                      multi_to_scalar, scalar_to_multi, tensor_space)
from .wq import (EXACTNESS_TOL, TensorRule, WQRule1D, build_tensor_rule,
                 build_wq_rule)

__all__ = [n for n in dir() if not n.startswith("_")]
__version__ = "0.1.0"
