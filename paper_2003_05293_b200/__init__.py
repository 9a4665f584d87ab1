"""B200-native CS-WGS multi-spot hologram solver (arXiv 2003.05293).

Drop-in for the hot path of the reference package ``holospots``
(holospots/__init__.py:10-29): the RS / WGS / CS-WGS solvers, the
superpose / forward-projection kernels and the e / u quality report, with
the same names, signatures and exceptions.  Compute runs in hand-written
sm_100a CUDA kernels behind a C ABI (include/holospots_b200.h); there is no
CPU fallback.
"""

from .errors import (DegenerateFieldError, DeviceError, GeometryMismatchError, HoloError,
                     InvalidParameterError, OutOfFieldError, UndefinedUniformityError,
                     ZeroIlluminationError)
from .kernels import (DEFAULT_CHUNK, SpotCoefficients, SpotTables, forward_project,
                      reduce_complex, spot_tables, superpose, warm_up)
from .metrics import (QualityReport, efficiency, quality_report, spot_intensities,
                      target_relative, uniformity)
from .optics import (CompressionPlan, Hologram, Pupil, SpotSet, build_panel, build_pupil, phase_of,
                     spot_phase, wrap_phase)
from .solvers import (PlannedRun, SolverConfig, SolverTrace, StepRecord, WgsState,
                      budget_controller, cswgs, predict_ops, rebalance_weights, rs, solve,
                      solve_batch, wgs, wgs_step)
from .scenarios import (SCENARIO_NAMES, Scenario, cubes_scenario, grid_scenario,
                        load_scenario_file, named_scenario, rotate_points, rotation_sweep)
from .sequences import rotation_sequence, sequence_quality, solve_sequence
from .simulate import FieldImage, probe_intensities, render_plane
from .sweeps import (BenchRecord, BudgetComparison, CellStats, calibrate_ops_per_ms,
                     compare_at_budget, frame_budget_ops, summarize, sweep)
from .slm import PhaseLut, slm_raster, solve_rasters
from ._lib import get_device, get_precision, set_device, set_precision
from .precision import precision
from .workloads import grid_spots, named_spots, random_foci

__version__ = "0.1.0"
