"""B200-native MGRIT semi-Lagrangian hot path (arXiv 2203.13382).

Drop-in mirror of the reference package's operator/driver API
(mgrit_advect/__init__.py:5-20, hot-path subset) backed by hand-written
sm_100a kernels in libmgrit_b200.so (C ABI: include/mgrit_b200.h).
"""

from .core import (Grid1D, Grid2D, TimeGrid, WaveSpeed, get_wave_speed,  # noqa: F401
                   initial_condition, random_state, space_time_norm)
from .mgrit import (ConvergenceReport, GmresConfig, Level, SolverConfig,  # noqa: F401
                    build_hierarchy, c_relax, departures_from_coords, f_relax, set_launch_policy,
                    residual, sequential_reference, solve, solve_sequential,
                    v_cycle)
from .operators import (CorrectionField, DepartureSet1D, DepartureSet2D, ErkScheme,  # noqa: F401
                        ImSD, apply_ImSD, apply_IpSD, corrected_coarse_step, decompose,
                        derivative_stencil, erk_scheme, forward_euler_coarse_step, gmres_solve,
                        interp_weights, sl_step, stencil_extents)

__version__ = "0.2.0"
