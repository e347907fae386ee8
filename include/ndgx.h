/*
 * ndgx.h -- C ABI of the B200-native NDG right-hand side + Runge-Kutta hot path.
 *
 * Drop-in boundary for the reference solver's stepping loop
 * (/root/reference/proj; paths below are relative to it):
 *
 *   ndgx_create/ndgx_destroy  <- DGOperator ctor (src/solver.cpp:189-210) +
 *                                RKIntegrator ctor (include/ndg/solver.hpp:41-44) +
 *                                HaloSet::allocate (src/solver.cpp:159-164)
 *   ndgx_upload/ndgx_download <- StateField hand-over (include/ndg/grid.hpp:50-56,
 *                                AoS [cell_x][cell_y][cell_z][i][j][k][var])
 *   ndgx_rhs                  <- serial_rhs (src/solver.cpp:442-456) /
 *                                DGOperator::apply (src/solver.cpp:212-308)
 *   ndgx_advance              <- advance (src/solver.cpp:372-440) with StepPlan
 *                                (include/ndg/solver.hpp:168-171), StepStats (:153-158)
 *   ndgx_decompose            <- decompose (src/partition.cpp:44-106)
 *   ndgx_create_partitioned   <- run_partitioned (src/partition.cpp:186-333) as one
 *                                handle over P blocks on 1..8 devices
 *   ndgx_create_rank          <- one worker of run_partitioned per process (NCCL)
 *   ndgx_gauss_lobatto / ndgx_differentiation_matrix
 *                             <- gauss_lobatto / differentiation_matrix
 *                                (src/basis.cpp:32-76, 96-118), host setup inputs
 *   ndgx_init_*               <- init_multisine / init_euler_subsonic
 *                                (src/grid.cpp:135-188), host setup inputs
 *
 * Conventions (mirroring the reference): the caller owns every host buffer;
 * a handle is used by one host thread at a time (like serial advance); all
 * device memory belongs to the handle.  Every entry point returns an
 * ndgx_status; a non-zero status fills the optional ndgx_error, whose code
 * maps 1:1 onto include/ndg/errors.hpp:13-56.
 *
 * There is no CPU fallback: ndgx_create fails with NDGX_ERR_CUDA when no
 * sm_100 device is present.
 */
#ifndef NDGX_H
#define NDGX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NDGX_OK = 0,
  NDGX_ERR_CONFIG = 1,        /* ndg::ConfigError        errors.hpp:13-16 */
  NDGX_ERR_PHYSICS = 2,       /* ndg::PhysicsError       errors.hpp:19-22 */
  NDGX_ERR_INSTABILITY = 3,   /* ndg::InstabilityError   errors.hpp:25-33 (step) */
  NDGX_ERR_DECOMPOSITION = 4, /* ndg::DecompositionError errors.hpp:36-39 */
  NDGX_ERR_TRANSPORT = 5,     /* ndg::TransportError     errors.hpp:42-45 (NCCL/P2P) */
  NDGX_ERR_RUN = 6,           /* ndg::RunError           errors.hpp:48-56 (worker) */
  NDGX_ERR_CUDA = 7           /* device / driver failure (no reference analogue) */
} ndgx_status;

typedef enum { NDGX_ADVECTION = 0, NDGX_EULER_ISOTHERMAL = 1 } ndgx_equation; /* models.hpp:26 */
typedef enum { NDGX_RK3 = 0, NDGX_RK4 = 1, NDGX_RK6 = 2 } ndgx_rk;           /* solver.hpp:20 */

/* Arithmetic mode.  EXACT reproduces the reference's IEEE-754 operation
 * order with no contraction (bit-identical states); FAST lets the kernels
 * contract into FMA (<= 1e-12 relative L2 vs the reference). */
typedef enum { NDGX_ARITH_EXACT = 0, NDGX_ARITH_FAST = 1 } ndgx_arith;

/* Mesh (grid.hpp:18-37) + EquationModel (models.hpp:43-73) +
 * SolverConfig (solver.hpp:142-148).  Axes >= dim are ignored. */
typedef struct {
  int dim;              /* 1..3 */
  int cells[3];         /* cells per axis (global) */
  double length[3];     /* box edge lengths */
  int order;            /* Gauss-Lobatto nodes per axis, 2..8 on the GPU path */
  int equation;         /* ndgx_equation */
  double velocity[3];   /* advection velocity */
  double sound_speed;   /* isothermal Euler a > 0 */
  int rk;               /* ndgx_rk */
  double cfl;           /* (0, 1] */
  double t_end;         /* > 0 */
  /* optional basis, e.g. the caller's own gauss_lobatto/differentiation_matrix
   * (NULL -> computed by ndgx_gauss_lobatto / ndgx_differentiation_matrix) */
  const double* nodes;   /* [order] */
  const double* weights; /* [order] */
  const double* diff;    /* [order*order], diff[l*order+k] = h_k'(xi_l) (basis.hpp:22) */
  int device;            /* CUDA device ordinal */
  int arith;             /* ndgx_arith */
} ndgx_problem;

typedef struct { /* StepStats (solver.hpp:153-158); wall_seconds from CUDA events */
  long steps;
  double dt_min, dt_max, wall_seconds;
} ndgx_stats;

typedef struct {
  int code;        /* ndgx_status */
  long step;       /* InstabilityError::step() */
  int stage;       /* RK stage of a PhysicsError in the operator, else -1 */
  int worker;      /* RunError::worker(), else -1 */
  int cell[3];     /* offending cell (global) for operator PhysicsErrors, else -1 */
  char message[256];
} ndgx_error;

typedef struct ndgx_solver ndgx_solver;

/* Lifecycle. */
int ndgx_create(const ndgx_problem* problem, ndgx_solver** out, ndgx_error* err);
void ndgx_destroy(ndgx_solver* s);

/* State hand-over in the reference AoS layout (FieldShape::index order).
 * host pointers may be pageable or pinned; the permutation to the device
 * layout runs on the GPU. */
int ndgx_upload(ndgx_solver* s, const double* u_aos, ndgx_error* err);
int ndgx_download(ndgx_solver* s, double* u_aos, ndgx_error* err);

/* serial_rhs of the current state into dudt_aos (host, AoS). */
int ndgx_rhs(ndgx_solver* s, double* dudt_aos, ndgx_error* err);

/* advance(config, state, StepPlan{fixed_steps, warmup}): fixed_steps < 0
 * integrates to problem.t_end with the last step shortened.  The state stays
 * on the device (download it afterwards). */
int ndgx_advance(ndgx_solver* s, long fixed_steps, int warmup, ndgx_stats* stats,
                 ndgx_error* err);

/* Sizes. */
int64_t ndgx_dof(const ndgx_solver* s);      /* cells * order^dim * n_var (grid.cpp:72-74) */
size_t ndgx_state_size(const ndgx_solver* s); /* doubles in one state (== dof) */
int ndgx_stages(const ndgx_solver* s);

/* Device-resident stepping for benchmarks: launch `steps` fixed CFL steps
 * on the handle's stream without host synchronisation or error polling
 * (call ndgx_sync to collect errors).  ndgx_stream returns the cudaStream_t. */
int ndgx_launch_steps(ndgx_solver* s, long steps, ndgx_error* err);
int ndgx_sync(ndgx_solver* s, ndgx_stats* stats, ndgx_error* err);
void* ndgx_stream(ndgx_solver* s);
/* Per-stage timing of one step captured in a CUDA graph with event records
 * between the stages (replayed 5 times, mean): ms[i] for stage i (a split
 * stage's interior + boundary shell end to end), ms[stages] the step control. */
int ndgx_profile_step(ndgx_solver* s, float* ms, int n, ndgx_error* err);

/* Host setup inputs (same arithmetic as the reference). */
int ndgx_gauss_lobatto(int order, double* nodes, double* weights);
int ndgx_differentiation_matrix(int order, const double* nodes, double* diff);
int ndgx_init_multisine(const ndgx_problem* p, const double* amplitudes, int n_modes,
                        double* u_aos);
void ndgx_multisine_amplitudes(int n_modes, uint64_t seed, double* out);
int ndgx_init_euler_subsonic(const ndgx_problem* p, double* u_aos);

/* Host diagnostics, summed in the reference's order (bit-identical):
 *   ndgx_l2_error         <- l2_error (src/grid.cpp:190-203), var in [0, nvar)
 *   ndgx_conserved_totals <- conserved_totals (src/grid.cpp:205-213), out[nvar] */
int ndgx_l2_error(const ndgx_problem* p, const double* a_aos, const double* b_aos, int var,
                  double* out);
int ndgx_conserved_totals(const ndgx_problem* p, const double* u_aos, double* out);

/* Block decomposition (partition.cpp:44-106): grid[3]; lo/hi [workers][3];
 * nbr [workers][3][2] (low, high). */
int ndgx_decompose(int dim, const int cells[3], int workers, int grid[3], int* lo, int* hi,
                   int* nbr, ndgx_error* err);

/* ---------------------------------------------------------------- blocks
 * Multi-GPU: one process per GPU, each owning one block of decompose()'s
 * tiling of the global mesh (run_partitioned, src/partition.cpp:186-333,
 * with its in-process Transport (include/ndg/transport.hpp:29-39) replaced by
 * NCCL over NVLink).  Per RK stage each rank packs the stage-input face
 * planes of its split axes, exchanges them with ncclSend/ncclRecv, and the
 * stage kernel reads the received planes for its out-of-block faces; per
 * step one ncclAllReduce(max) of the wavespeed bound (exchange_halos and the
 * alpha barrier, src/partition.cpp:108-131, 236-261).  All of it is captured
 * in the step CUDA graphs.  Results are identical to the single-block run. */
typedef struct {
  int rank, nranks;
  int grid[3];           /* blocks per axis (decompose) */
  int lo[3], hi[3];      /* this rank's global cell range [lo, hi) */
  int split[3];          /* 1: faces along the axis come from the neighbour ranks */
  int nbr[3][2];         /* neighbour rank [axis][low, high] */
  long long plane[3];    /* doubles per face plane along the axis: cross-section cells * face nodes * vars */
} ndgx_rank_plan;

/* Block plan of `rank` (host only, no GPU).  force_exchange != 0 routes every
 * axis through the transport, even a self-periodic one (test hook). */
int ndgx_plan_rank(const ndgx_problem* global, int nranks, int rank, int force_exchange, ndgx_rank_plan* plan,
                   ndgx_error* err);
/* NCCL bootstrap: rank 0 creates the id, the caller broadcasts it (e.g. over
 * torch.distributed), every rank passes it to ndgx_create_rank. */
int ndgx_nccl_unique_id(unsigned char id[128], ndgx_error* err);
/* A solver for this rank's block.  `global` describes the whole mesh; states
 * exchanged with ndgx_upload/ndgx_download are the block's own AoS field. */
int ndgx_create_rank(const ndgx_problem* global, int nranks, int rank, const unsigned char nccl_id[128],
                     int force_exchange, ndgx_solver** out, ndgx_error* err);
int ndgx_get_plan(const ndgx_solver* s, ndgx_rank_plan* plan);
/* Initial conditions of the block [lo, hi) of the global mesh (block AoS). */
int ndgx_init_multisine_block(const ndgx_problem* global, const double* amplitudes, int n_modes, const int lo[3],
                              const int hi[3], double* u_aos);
int ndgx_init_euler_subsonic_block(const ndgx_problem* global, const int lo[3], const int hi[3], double* u_aos);

/* ------------------------------------------------------- partitioned
 * run_partitioned (src/partition.cpp:186-333, include/ndg/partition.hpp:
 * 66-67) in ONE handle: `workers` blocks of decompose()'s tiling, block w on
 * device_ids[w % n_devices] (n_devices 0 / device_ids NULL -> global->device),
 * i.e. SURVEY §8b's (n_devices, device_ids).  Per RK stage each block's pack
 * kernel stores its boundary stage-input planes straight into the neighbour
 * blocks' halo buffers (peer memory over NVLink across GPUs), the interior
 * runs while they land, the boundary shell after; one shared device-side step
 * control gives every block the global wavespeed (the alpha barrier).
 * ndgx_upload/ndgx_download/ndgx_rhs/ndgx_advance on the handle take the
 * GLOBAL AoS field, and every failure is NDGX_ERR_RUN with the reference's
 * message "worker <w>: <what>" and error.worker = w.  force_exchange != 0
 * routes every axis through the halo planes, even with one block (test hook).
 * Results are bit-identical to ndgx_create's single block. */
int ndgx_create_partitioned(const ndgx_problem* global, int workers, int n_devices, const int* device_ids,
                            int force_exchange, ndgx_solver** out, ndgx_error* err);
int ndgx_workers(const ndgx_solver* s);                                   /* blocks in the handle */
int ndgx_get_block(const ndgx_solver* s, int worker, ndgx_rank_plan* plan); /* Block of `worker` */

/* Checkpoint / restart in the reference's field-dump format ("ndgfield 1":
 * text header, then the raw little-endian doubles in FieldShape::index
 * order; dump_field / load_field, src/field_io.cpp:18-72).  dump writes the
 * solver's current state (its block, for a rank solver); load checks the
 * header against the solver's mesh and uploads the payload. */
int ndgx_dump_field(ndgx_solver* s, const char* path, ndgx_error* err);
int ndgx_load_field(ndgx_solver* s, const char* path, ndgx_error* err);

/* Initial conditions and diagnostics on the device,
 * over the handle's current state in HBM (every block of the handle; a rank
 * solver's own block):
 *   ndgx_init_device              <- init_multisine (src/grid.cpp:135-156, ic
 *                                    NDGX_IC_MULTISINE with the amplitudes of
 *                                    multisine_amplitudes, :127-133) /
 *                                    init_euler_subsonic (:162-188) + upload,
 *                                    without a host field or an H2D copy
 *   ndgx_conserved_totals_device  <- conserved_totals (src/grid.cpp:205-213), out[nvar]
 *   ndgx_l2_error_ic_device       <- l2_error(state, init_*(...), var) (src/grid.cpp:190-203),
 *                                    the IC evaluated on the fly (experiments.cpp:112, 508)
 *   ndgx_l1_norm_device           <- l1_norm (src/grid.cpp:215-223)
 * Same ConfigError messages as the reference.  Values follow the reference's
 * expressions (explicit roundings); device sin and the tree-ordered sums make
 * them equal to the host functions to ~1e-16 / ~1e-15 relative. */
typedef enum { NDGX_IC_MULTISINE = 0, NDGX_IC_EULER_SUBSONIC = 1 } ndgx_ic;
int ndgx_init_device(ndgx_solver* s, int ic, const double* amplitudes, int n_modes, ndgx_error* err);
int ndgx_conserved_totals_device(ndgx_solver* s, double* out, ndgx_error* err);
int ndgx_l2_error_ic_device(ndgx_solver* s, int ic, const double* amplitudes, int n_modes, int var, double* out,
                            ndgx_error* err);
int ndgx_l1_norm_device(ndgx_solver* s, int var, double* out, ndgx_error* err);

/* Library identification: "ndgx <version> sm_100a". */
const char* ndgx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NDGX_H */
