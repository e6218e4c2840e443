"""B200-native (sm_100a, fp64) time-stepping path of the modal DG spherical
shallow-water solver of arXiv 2303.11767, behind the reference's solver API
(/root/reference/pkg/src/dgswe).

    from paper_2303_11767_b200 import (build_latlon_mesh, SpatialOperator,
        swe_sphere_model, tableau, TimeControls, integrate, rk_step,
        default_config, build_case, mass_integral, l2_error)

Device work goes through the C ABI in include/dgswe_b200.h
(libdgswe_b200.so, built in-tree); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .geometry import (BOTTOM, EARTH, LEFT, RIGHT, TOP, Mesh, MassMatrix, NeighborRef,  # noqa: F401
                       PhysicalConstants, Quadrature, Vander, build_latlon_mesh, build_planar_mesh,
                       build_vander, mass_matrix_planar,
                       eval_modal_at_nodes, gauss_legendre, legendre_deriv, legendre_eval,
                       mass_matrix_sphere, min_effective_diameter, project_initial,
                       sphere_row_mass_matrices)
from .physics import (PlanarSWEModel, PositivityError, SphereSWEModel, X_DIR, Y_DIR,  # noqa: F401
                      swe_planar_model, swe_sphere_model)  # noqa: F401
from .monitors import (convergence_rate, l2_error, l2_error_host, mass_integral,  # noqa: F401
                       mass_integral_host)
from .stepping import (ButcherTableau, DivergenceError, StepLog, TimeControls,  # noqa: F401
                       integrate, rk_step, tableau)
from .williamson import (CASE_IDS, CaseConfig, RunSetup, build_case, default_config,  # noqa: F401
                         ic_advection_sine, ic_geostrophic_adjustment, ic_williamson_tc2, ic_williamson_tc5, ic_williamson_tc6,
                         tc5_bottom, tc6_fields)
from .operator import RusanovParams, SpatialOperator, State  # noqa: F401
from .advection import AdvectionModel, AdvectionOperator, AdvState, advection_model  # noqa: F401
from .tracing import LaunchRegion, set_op_recorder  # noqa: F401
