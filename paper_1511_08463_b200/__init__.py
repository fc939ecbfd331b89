"""B200-native (sm_100a, fp64) quasi-static phase-field fracture load step.

Drop-in for the hot path of the reference package ``phasefrac`` (arXiv:1511.08463):
the same solver API (``Material``, ``Discretization``, ``State``, ``SolverConfig``,
``am_solve``, ``oram_n_solve``, ``solve_load_step``, ``run_quasistatic``, ...) with
every numeric step executed by the hand-written CUDA library ``libphasefrac_b200.so``
through its C ABI (include/phasefrac_b200.h).  There is no CPU fallback: without the
library (or a CUDA device) the numeric entry points raise.
"""

__version__ = "0.1.0"

from .linalg import (BreakdownError, InnerSolverError, LinearSolveReport,  # noqa: F401
                     LinearSolverError, SingularOperatorError)
from .model import (C_W, DamageModel, Material, critical_shock, critical_traction,  # noqa: F401
                    internal_length)
from .mesh import (BOUNDARY_TAGS, StructuredMesh, StructuredMesh3D, banded_rect_mesh,  # noqa: F401
                   boundary_dofs, rect_mesh)
from .vi import ActiveSetReport, VIConfig, fb_phi  # noqa: F401
from .fem import (DeviceOperator, DirichletBC, Discretization, EnergyBreakdown,  # noqa: F401
                  State, assemble_energy, assemble_Kaa, assemble_Kua, assemble_Kuu,
                  assemble_load_u, assemble_residual_alpha, assemble_residual_u, combine_bcs)
from .solver import (NonlinearReport, SolverConfig, am_solve, coupled_newton_solve,  # noqa: F401
                     damage_step, elastic_step, first_order_residual, oram_n_solve,
                     residual_norm, solve_load_step)
from .cases import (ProblemSetup, StepFailureError, StepRecord, UnstructuredSetup,  # noqa: F401
                    run_quasistatic, run_quasistatic_unstructured, setup_sent, setup_surfing,
                    setup_thermal_shock, setup_thermal_slab, setup_traction, setup_traction3d,
                    surfing_displacement, thermal_strain)
from .umesh import (UnstructuredMesh, UnstructuredOperators, jittered_box_mesh,  # noqa: F401
                    jittered_rect_mesh)

__all__ = [n for n in dir() if not n.startswith("_")]
