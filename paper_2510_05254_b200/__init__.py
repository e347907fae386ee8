"""paper_2510_05254_b200 -- B200-native NDG right-hand side + Runge-Kutta hot path.

The compute path is libndgx.so (hand-written sm_100a CUDA behind the C ABI in
include/ndgx.h); ``ndgx`` mirrors the reference solver's API on top of it.
"""
from . import report  # noqa: F401
from .ndgx import (ADVECTION, ARITH_EXACT, ARITH_FAST, EULER_ISOTHERMAL, IC_EULER_SUBSONIC, IC_MULTISINE, RK3, RK4, RK6,  # noqa: F401
                   AdvanceResult, Block, BlockDecomposition, ConfigError, CudaError,
                   DecompositionError, EquationModel, InstabilityError, Mesh, NdgError,
                   PhysicsError, RunError, Solver, SolverConfig, StepPlan, StepStats,
                   TransportError, advance, decompose, differentiation_matrix, gauss_lobatto,
                   init_block, init_euler_subsonic, init_multisine, lib, multisine_amplitudes,
                   nccl_unique_id, plan_rank, dump_field, load_field, RankPlan, rk_from_name, serial_rhs, validate, version,
                   l2_error, conserved_totals, run_partitioned, PartitionedResult, WorkerTiming)
