"""B200-native solver for the receding-horizon eco-driving DP of arXiv 2104.01284.

Drop-in for the reference package's DP path (``ecodrive.dp`` / ``ecodrive.mpc``):
same types and entry points, executed by hand-written sm_100a CUDA kernels
behind the C ABI in ``include/eco_b200.h``.  ``plugin.install()`` registers the
``"b200"`` / ``"b200-fp64"`` backend names inside an importable reference
package.  Beyond the reference's single-solve / closed-loop API:
``BatchSolver`` (many scenarios on one road, C4) and ``SlabSolver`` (one grid
split into speed-plane slabs across GPUs, C5).
"""

from .dp import (BACKENDS, CostToGoTable, GridSpec, PenaltyConfig, PolicyTable, SolveContext, SolveResult,
                 StepPlan, ToyInstance, backward_step, build_context, dump_tables, load_tables,
                 make_toy_pack, solve_digests, solve_horizon, solve_toy, table_digest)
from .errors import (InfeasiblePowerError, NativeLibraryError, RouteFormatError, StartStateInfeasibleError,
                     UnknownSignalError, VehicleFormatError, ZeroMeanVelocityError)
from .fixtures import bench_schedule, load_fixture_route, make_vehicle
from .mpc import (ClosedLoopTrajectory, ControlDecision, EcoDrivingMPC, TerminalCostField, TrajectoryStep,
                  build_terminal_cost, field_value, mpc_step, simulate_closed_loop)
from .plant import ActionVector, StateVector, Vehicle
from .route import Route, SignalTiming, SpatSchedule, load_route, next_green_start, phase_at
from .batch import BatchResult, BatchSolver, solve_batch
from .slab import SlabResult, SlabSolver, gather_policies, make_partition
from .harness import BenchReport, DiffReport, compare_solves, diff_backends_run, run_bench
from .io import read_trajectory_csv, summarize, write_summary_json, write_timing_csv, write_trajectory_csv

__version__ = "0.1.0"
