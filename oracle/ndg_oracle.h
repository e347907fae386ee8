/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the NDG RHS + RK hot path.
 *
 * A plain-C restatement of the reference solver (/root/reference/proj, the
 * "ndgbench" C++20 code) used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the CHECKER.  The product path
 * (paper_2510_05254_b200/) never links, loads or calls anything in oracle/.
 *
 * Parity pin: every function reproduces the reference's IEEE-754 double
 * arithmetic in source order (the reference build has no -march, hence no
 * FMA; this file is compiled with -ffp-contract=off).  It is checked
 * bit-for-bit against the reference itself compiled from its own sources
 * (oracle/Makefile -> oracle/_ref/libndg_ref.so) and against the FNV-1a
 * digests of SURVEY.md's appendix (tests/golden/).
 */
#ifndef NDG_ORACLE_H
#define NDG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors Mesh (grid.hpp:18-37) + EquationModel (models.hpp:43-73)
 * + SolverConfig (solver.hpp:142-148). */
typedef struct {
  int dim;
  int cells[3];
  double length[3];
  int order;          /* nodes per cell per axis (N) */
  int kind;           /* 0 advection, 1 isothermal Euler */
  double velocity[3]; /* advection */
  double sound_speed; /* Euler */
  int rk;             /* 0 rk3, 1 rk4, 2 rk6 */
  double cfl;
  double t_end;
} ndgo_config;

typedef struct {
  long steps;
  double dt_min, dt_max, wall_seconds;
} ndgo_stats;

/* codes: 0 ok, 1 ConfigError, 2 PhysicsError, 3 InstabilityError,
 *        4 DecompositionError, 6 RunError */
typedef struct {
  int code;
  long step;
  int worker;
  char message[256];
} ndgo_error;

int ndgo_n_var(const ndgo_config* c);
int64_t ndgo_dof(const ndgo_config* c);
size_t ndgo_size(const ndgo_config* c);
size_t ndgo_index(const ndgo_config* c, const int cell[3], const int node[3], int var);
int ndgo_wrap_cell(const ndgo_config* c, int axis, int cell, int offset);

int ndgo_gauss_lobatto(int order, double* nodes, double* weights);
int ndgo_differentiation_matrix(int order, const double* nodes, double* diff);
void ndgo_legendre(int n, double x, double* p, double* dp);

void ndgo_multisine_amplitudes(int n_modes, uint64_t seed, double* out);
uint64_t ndgo_splitmix64_next(uint64_t* state);
int ndgo_init_multisine(const ndgo_config* c, const double* amps, int n_amps, double* out);
int ndgo_init_euler_subsonic(const ndgo_config* c, double* out);

double ndgo_l2_error(const ndgo_config* c, const double* a, const double* b, int var);
void ndgo_conserved_totals(const ndgo_config* c, const double* f, double* totals);
double ndgo_l1_norm(const ndgo_config* c, const double* f, int var);

void ndgo_tableau(int rk, int* stages, double a[7][7], double b[7]);
double ndgo_max_wavespeed_bound(const ndgo_config* c, const double* u, size_t n,
                                ndgo_error* err);
double ndgo_dt_from_alpha(const ndgo_config* c, double alpha);
size_t ndgo_face_trace_size(const ndgo_config* c, const int cells[3], int axis);
void ndgo_pack_face_trace(const ndgo_config* c, const int cells[3], const double* u,
                          int axis, int cell_d, int node_d, double* out);

/* serial_rhs (solver.cpp:442-456): dudt of a periodic field. */
int ndgo_serial_rhs(const ndgo_config* c, const double* u, double* dudt, ndgo_error* err);
/* advance (solver.cpp:372-440): u is overwritten with the final state. */
int ndgo_advance(const ndgo_config* c, double* u, long fixed_steps, int warmup,
                 ndgo_stats* stats, ndgo_error* err);

/* decompose (partition.cpp:44-106). lo/hi: [workers][3]; nbr: [workers][3][2]. */
int ndgo_decompose(const ndgo_config* c, int workers, int grid[3], int* lo, int* hi,
                   int* nbr, ndgo_error* err);

/* FNV-1a 64 over raw bytes (report.cpp:284-293 applied to the state bytes). */
uint64_t ndgo_fnv1a64(const void* data, size_t nbytes);

#ifdef __cplusplus
}
#endif
#endif
