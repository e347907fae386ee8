/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle (checker) for the NDG RHS + RK path.
 * See ndg_oracle.h.  Every function cites the reference lines it restates;
 * paths are relative to /root/reference/proj.  Compile with
 * -ffp-contract=off (no FMA), like the reference build (CMakeLists.txt:1-37).
 */
#include "ndg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static const double kTwoPi = 6.283185307179586476925286766559; /* grid.cpp:12 */

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

static void set_err(ndgo_error* e, int code, long step, const char* msg) {
  if (!e) return;
  e->code = code;
  e->step = step;
  e->worker = -1;
  snprintf(e->message, sizeof(e->message), "%s", msg);
}

/* EquationModel::n_var (models.hpp:40) */
int ndgo_n_var(const ndgo_config* c) { return c->kind == 0 ? 1 : c->dim + 1; }

static int cells_of(const ndgo_config* c, int a) { return a < c->dim ? c->cells[a] : 1; }
static double cell_size(const ndgo_config* c, int a) {
  return (a < c->dim ? c->length[a] : 1.0) / (double)cells_of(c, a); /* grid.hpp:25 */
}

/* Mesh::dof (grid.cpp:72-74) */
int64_t ndgo_dof(const ndgo_config* c) {
  int64_t cells = (int64_t)cells_of(c, 0) * cells_of(c, 1) * cells_of(c, 2);
  int64_t npc = 1;
  for (int a = 0; a < c->dim; ++a) npc *= c->order;
  return cells * npc * ndgo_n_var(c);
}

/* FieldShape::size (grid.cpp:83-87) */
size_t ndgo_size(const ndgo_config* c) {
  size_t s = (size_t)ndgo_n_var(c);
  for (int a = 0; a < c->dim; ++a) s *= (size_t)c->cells[a] * c->order;
  return s;
}

/* FieldShape::index (grid.hpp:50-56) */
size_t ndgo_index(const ndgo_config* c, const int cell[3], const int node[3], int var) {
  size_t idx = 0;
  for (int a = 0; a < c->dim; ++a) idx = idx * c->cells[a] + cell[a];
  for (int a = 0; a < c->dim; ++a) idx = idx * c->order + node[a];
  return idx * ndgo_n_var(c) + var;
}

/* Mesh::wrap_cell (grid.cpp:76-81) */
int ndgo_wrap_cell(const ndgo_config* c, int axis, int cell, int offset) {
  const int n = cells_of(c, axis);
  int w = (cell + offset) % n;
  if (w < 0) w += n;
  return w;
}

/* ---------------------------------------------------------------- basis */

/* legendre (basis.cpp:15-30) */
void ndgo_legendre(int n, double x, double* p_out, double* dp_out) {
  if (n == 0) {
    *p_out = 1.0;
    *dp_out = 0.0;
    return;
  }
  double pm1 = 1.0, p = x, dpm1 = 0.0, dp = 1.0;
  for (int m = 1; m < n; ++m) {
    const double pp1 = ((2 * m + 1) * x * p - m * pm1) / (m + 1);
    const double dpp1 = dpm1 + (2 * m + 1) * p;
    pm1 = p;
    p = pp1;
    dpm1 = dp;
    dp = dpp1;
  }
  *p_out = p;
  *dp_out = dp;
}

/* gauss_lobatto (basis.cpp:32-76) */
int ndgo_gauss_lobatto(int order, double* nodes, double* weights) {
  if (order < 2 || order > 16) return 1;
  const int n = order, deg = order - 1;
  for (int k = 0; k < n; ++k) nodes[k] = 0.0;
  nodes[0] = -1.0;
  nodes[n - 1] = 1.0;
  const double pi = acos(-1.0);
  for (int k = 1; k < n - 1; ++k) {
    double x = -cos(pi * k / deg);
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      ndgo_legendre(deg, x, &p, &dp);
      const double delta = (1.0 - x * x) * dp / (deg * (deg + 1) * p);
      x += delta;
      if (fabs(delta) <= 1e-15) break;
    }
    nodes[k] = x;
  }
  for (int k = 0; k < n / 2; ++k) {
    const double s = 0.5 * (nodes[k] - nodes[n - 1 - k]);
    nodes[k] = s;
    nodes[n - 1 - k] = -s;
  }
  if (n % 2 == 1) nodes[n / 2] = 0.0;
  for (int k = 0; k < n; ++k) {
    double p, dp;
    ndgo_legendre(deg, nodes[k], &p, &dp);
    weights[k] = 2.0 / (n * deg * p * p);
  }
  return 0;
}

/* differentiation_matrix (basis.cpp:96-118): diff[l*n+k] = h_k'(xi_l) */
int ndgo_differentiation_matrix(int order, const double* nodes, double* diff) {
  const int n = order, deg = n - 1;
  double p[16], dp;
  for (int k = 0; k < n; ++k) ndgo_legendre(deg, nodes[k], &p[k], &dp);
  for (int l = 0; l < n; ++l) {
    double rowsum = 0.0;
    for (int k = 0; k < n; ++k) {
      if (k == l) continue;
      const double v = p[l] / (p[k] * (nodes[l] - nodes[k]));
      diff[l * n + k] = v;
      rowsum += v;
    }
    diff[l * n + l] = -rowsum;
  }
  return 0;
}

/* ------------------------------------------------------- ICs/diagnostics */

/* SplitMix64 (rng.hpp:15-33) */
uint64_t ndgo_splitmix64_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* multisine_amplitudes (grid.cpp:127-133) */
void ndgo_multisine_amplitudes(int n_modes, uint64_t seed, double* out) {
  uint64_t s = seed;
  for (int k = 0; k < n_modes; ++k)
    out[k] = (double)(ndgo_splitmix64_next(&s) >> 11) * 0x1.0p-53;
}

/* node_coordinates (grid.cpp:109-125) */
static void node_coords(const ndgo_config* c, const double* gl, const int cell[3],
                        const int node[3], double x[3]) {
  x[0] = x[1] = x[2] = 0.0;
  for (int a = 0; a < c->dim; ++a) {
    const double dx = cell_size(c, a);
    x[a] = cell[a] * dx + 0.5 * dx * (gl[node[a]] + 1.0);
  }
}

/* for_each_node visitor order (grid.cpp:28-48) */
typedef void (*node_fn)(const ndgo_config*, const int cell[3], const int node[3], double w,
                        void* ctx);
static void for_each_node(const ndgo_config* c, const double* weights, node_fn fn,
                          void* ctx) {
  int nc[3] = {1, 1, 1};
  for (int a = 0; a < c->dim; ++a) nc[a] = c->order;
  double jac = 1.0;
  for (int a = 0; a < c->dim; ++a) jac *= 0.5 * cell_size(c, a);
  int cell[3], node[3];
  for (cell[0] = 0; cell[0] < cells_of(c, 0); ++cell[0])
    for (cell[1] = 0; cell[1] < cells_of(c, 1); ++cell[1])
      for (cell[2] = 0; cell[2] < cells_of(c, 2); ++cell[2])
        for (node[0] = 0; node[0] < nc[0]; ++node[0])
          for (node[1] = 0; node[1] < nc[1]; ++node[1])
            for (node[2] = 0; node[2] < nc[2]; ++node[2]) {
              double w = jac;
              for (int a = 0; a < c->dim; ++a) w *= weights[node[a]];
              fn(c, cell, node, w, ctx);
            }
}

typedef struct {
  const double* gl;
  const double* amps;
  int n_amps;
  double* out;
} ms_ctx;

static void ms_visit(const ndgo_config* c, const int cell[3], const int node[3], double w,
                     void* vctx) {
  (void)w;
  ms_ctx* m = (ms_ctx*)vctx;
  double x[3];
  node_coords(c, m->gl, cell, node, x);
  double u = 0.0;
  for (int k = 0; k < m->n_amps; ++k) u += m->amps[k] * sin(kTwoPi * (double)(k + 1) * x[0]);
  m->out[ndgo_index(c, cell, node, 0)] = u;
}

/* init_multisine (grid.cpp:135-156) */
int ndgo_init_multisine(const ndgo_config* c, const double* amps, int n_amps, double* out) {
  if (c->kind != 0 || n_amps < 1) return 1;
  double gl[16], w[16];
  ndgo_gauss_lobatto(c->order, gl, w);
  memset(out, 0, ndgo_size(c) * sizeof(double));
  ms_ctx m = {gl, amps, n_amps, out};
  for_each_node(c, w, ms_visit, &m);
  return 0;
}

static void eu_visit(const ndgo_config* c, const int cell[3], const int node[3], double w,
                     void* vctx) {
  (void)w;
  ms_ctx* m = (ms_ctx*)vctx;
  const double a = c->sound_speed;
  double x[3];
  node_coords(c, m->gl, cell, node, x);
  const double sx = sin(kTwoPi * x[0]);
  const double sy = sin(kTwoPi * x[1]);
  double rho = 1.0 + 0.2 * sx * sy;
  if (c->dim == 3) rho = 1.0 + 0.2 * sx * sy * sin(kTwoPi * x[2]);
  const double ux = 0.5 * a * sy;
  const double uy = 0.5 * a * sx;
  m->out[ndgo_index(c, cell, node, 0)] = rho;
  m->out[ndgo_index(c, cell, node, 1)] = rho * ux;
  m->out[ndgo_index(c, cell, node, 2)] = rho * uy;
  if (c->dim == 3) m->out[ndgo_index(c, cell, node, 3)] = 0.0;
}

/* init_euler_subsonic (grid.cpp:162-188) */
int ndgo_init_euler_subsonic(const ndgo_config* c, double* out) {
  if (c->kind != 1 || c->dim < 2) return 1;
  double gl[16], w[16];
  ndgo_gauss_lobatto(c->order, gl, w);
  memset(out, 0, ndgo_size(c) * sizeof(double));
  ms_ctx m = {gl, NULL, 0, out};
  for_each_node(c, w, eu_visit, &m);
  return 0;
}

typedef struct {
  const double* a;
  const double* b;
  int var;
  double sum;
  double* totals;
  int mode; /* 0 l2, 1 totals, 2 l1 */
} diag_ctx;

static void diag_visit(const ndgo_config* c, const int cell[3], const int node[3], double w,
                       void* vctx) {
  diag_ctx* d = (diag_ctx*)vctx;
  if (d->mode == 0) {
    const size_t i = ndgo_index(c, cell, node, d->var);
    const double df = d->a[i] - d->b[i];
    d->sum += w * df * df;
  } else if (d->mode == 1) {
    for (int v = 0; v < ndgo_n_var(c); ++v)
      d->totals[v] += w * d->a[ndgo_index(c, cell, node, v)];
  } else {
    d->sum += w * fabs(d->a[ndgo_index(c, cell, node, d->var)]);
  }
}

/* l2_error (grid.cpp:190-203) */
double ndgo_l2_error(const ndgo_config* c, const double* a, const double* b, int var) {
  double gl[16], w[16];
  ndgo_gauss_lobatto(c->order, gl, w);
  diag_ctx d = {a, b, var, 0.0, NULL, 0};
  for_each_node(c, w, diag_visit, &d);
  return sqrt(d.sum);
}

/* conserved_totals (grid.cpp:205-213) */
void ndgo_conserved_totals(const ndgo_config* c, const double* f, double* totals) {
  double gl[16], w[16];
  ndgo_gauss_lobatto(c->order, gl, w);
  for (int v = 0; v < ndgo_n_var(c); ++v) totals[v] = 0.0;
  diag_ctx d = {f, NULL, 0, 0.0, totals, 1};
  for_each_node(c, w, diag_visit, &d);
}

/* l1_norm (grid.cpp:215-223) */
double ndgo_l1_norm(const ndgo_config* c, const double* f, int var) {
  double gl[16], w[16];
  ndgo_gauss_lobatto(c->order, gl, w);
  diag_ctx d = {f, NULL, var, 0.0, NULL, 2};
  for_each_node(c, w, diag_visit, &d);
  return d.sum;
}

/* ---------------------------------------------------------------- models */

/* physical_flux (models.cpp:42-57); returns 0 or -1 on nonpositive density */
static int physical_flux(const ndgo_config* c, const double* u, int axis, double* flux) {
  if (c->kind == 0) {
    flux[0] = c->velocity[axis] * u[0];
    return 0;
  }
  const double rho = u[0];
  if (!(rho > 0.0)) return -1;
  const double ua = u[1 + axis] / rho;
  const int nv = ndgo_n_var(c);
  flux[0] = u[1 + axis];
  for (int i = 1; i < nv; ++i) flux[i] = ua * u[i];
  flux[1 + axis] += rho * c->sound_speed * c->sound_speed;
  return 0;
}

/* wavespeed_bound (models.cpp:59-70) */
static int wavespeed_bound(const ndgo_config* c, const double* u, int axis, double* out) {
  if (c->kind == 0) {
    *out = fabs(c->velocity[axis]);
    return 0;
  }
  const double rho = u[0];
  if (!(rho > 0.0)) return -1;
  *out = fabs(u[1 + axis] / rho) + c->sound_speed;
  return 0;
}

/* lax_friedrichs (models.cpp:77-88) with max_wavespeed (:72-75) */
static int lax_friedrichs(const ndgo_config* c, const double* um, const double* up, int axis,
                          double* flux, double* bad_rho) {
  double fm[4], fp[4], am, ap;
  if (physical_flux(c, um, axis, fm)) { *bad_rho = um[0]; return -1; }
  if (physical_flux(c, up, axis, fp)) { *bad_rho = up[0]; return -1; }
  if (wavespeed_bound(c, um, axis, &am)) { *bad_rho = um[0]; return -1; }
  if (wavespeed_bound(c, up, axis, &ap)) { *bad_rho = up[0]; return -1; }
  const double alpha = dmax(am, ap);
  const int nv = ndgo_n_var(c);
  for (int i = 0; i < nv; ++i) flux[i] = 0.5 * (fm[i] + fp[i] - alpha * (up[i] - um[i]));
  return 0;
}

/* --------------------------------------------------------------- solver */

/* make_rk3/4/6 (solver.cpp:17-68) */
void ndgo_tableau(int rk, int* stages, double a[7][7], double b[7]) {
  memset(a, 0, sizeof(double) * 49);
  memset(b, 0, sizeof(double) * 7);
  if (rk == 0) {
    *stages = 3;
    a[1][0] = 1.0 / 3.0;
    a[2][1] = 2.0 / 3.0;
    b[0] = 0.25; b[1] = 0.0; b[2] = 0.75;
  } else if (rk == 1) {
    *stages = 4;
    a[1][0] = 0.5;
    a[2][1] = 0.5;
    a[3][2] = 1.0;
    b[0] = 1.0 / 6.0; b[1] = 1.0 / 3.0; b[2] = 1.0 / 3.0; b[3] = 1.0 / 6.0;
  } else {
    const double q = sqrt(21.0);
    *stages = 7;
    a[1][0] = 1.0;
    a[2][0] = 3.0 / 8.0;
    a[2][1] = 1.0 / 8.0;
    a[3][0] = 8.0 / 27.0;
    a[3][1] = 2.0 / 27.0;
    a[3][2] = 8.0 / 27.0;
    a[4][0] = 3.0 * (3.0 * q - 7.0) / 392.0;
    a[4][1] = -8.0 * (7.0 - q) / 392.0;
    a[4][2] = 48.0 * (7.0 - q) / 392.0;
    a[4][3] = -3.0 * (21.0 - q) / 392.0;
    a[5][0] = -5.0 * (231.0 + 51.0 * q) / 1960.0;
    a[5][1] = -40.0 * (7.0 + q) / 1960.0;
    a[5][2] = -320.0 * q / 1960.0;
    a[5][3] = 3.0 * (21.0 + 121.0 * q) / 1960.0;
    a[5][4] = 392.0 * (6.0 + q) / 1960.0;
    a[6][0] = 15.0 * (22.0 + 7.0 * q) / 180.0;
    a[6][1] = 120.0 / 180.0;
    a[6][2] = 40.0 * (7.0 * q - 5.0) / 180.0;
    a[6][3] = -63.0 * (3.0 * q - 2.0) / 180.0;
    a[6][4] = -14.0 * (49.0 + 9.0 * q) / 180.0;
    a[6][5] = 70.0 * (7.0 - q) / 180.0;
    b[0] = 9.0 / 180.0; b[1] = 0.0; b[2] = 64.0 / 180.0; b[3] = 0.0;
    b[4] = 49.0 / 180.0; b[5] = 49.0 / 180.0; b[6] = 9.0 / 180.0;
  }
}

typedef struct {
  int axes[2];
  int count;
  int cells0, cells1, nodes0, nodes1;
} transverse_t;

/* transverse_of (solver.cpp:78-92), on a (possibly block-local) shape */
static transverse_t transverse_of(int dim, const int cells[3], int order, int axis) {
  transverse_t t = {{-1, -1}, 0, 1, 1, 1, 1};
  for (int a = 0; a < dim; ++a)
    if (a != axis) t.axes[t.count++] = a;
  if (t.count > 0) { t.cells0 = cells[t.axes[0]]; t.nodes0 = order; }
  if (t.count > 1) { t.cells1 = cells[t.axes[1]]; t.nodes1 = order; }
  return t;
}

typedef struct {
  size_t cell[3];
  size_t node[3];
} strides_t;

/* strides_of (solver.cpp:99-111) */
static strides_t strides_of(int dim, const int cells[3], int order, int nv) {
  strides_t st;
  memset(&st, 0, sizeof(st));
  size_t acc = (size_t)nv;
  for (int a = dim - 1; a >= 0; --a) { st.node[a] = acc; acc *= (size_t)order; }
  for (int a = dim - 1; a >= 0; --a) { st.cell[a] = acc; acc *= (size_t)cells[a]; }
  return st;
}

/* face_trace_size (solver.cpp:153-157) */
size_t ndgo_face_trace_size(const ndgo_config* c, const int cells[3], int axis) {
  transverse_t t = transverse_of(c->dim, cells, c->order, axis);
  return (size_t)t.cells0 * t.cells1 * t.nodes0 * t.nodes1 * ndgo_n_var(c);
}

/* pack_face_trace (solver.cpp:166-187) */
void ndgo_pack_face_trace(const ndgo_config* c, const int cells[3], const double* u,
                          int axis, int cell_d, int node_d, double* out) {
  const transverse_t t = transverse_of(c->dim, cells, c->order, axis);
  const strides_t st = strides_of(c->dim, cells, c->order, ndgo_n_var(c));
  const int nv = ndgo_n_var(c);
  size_t pos = 0;
  const size_t fixed = cell_d * st.cell[axis] + node_d * st.node[axis];
  for (int c0 = 0; c0 < t.cells0; ++c0)
    for (int c1 = 0; c1 < t.cells1; ++c1) {
      size_t cell_base = fixed;
      if (t.count > 0) cell_base += c0 * st.cell[t.axes[0]];
      if (t.count > 1) cell_base += c1 * st.cell[t.axes[1]];
      for (int a0 = 0; a0 < t.nodes0; ++a0)
        for (int a1 = 0; a1 < t.nodes1; ++a1) {
          size_t base = cell_base;
          if (t.count > 0) base += a0 * st.node[t.axes[0]];
          if (t.count > 1) base += a1 * st.node[t.axes[1]];
          for (int v = 0; v < nv; ++v) out[pos++] = u[base + v];
        }
    }
}

/* DGOperator (solver.cpp:189-210) baked per-axis matrices */
typedef struct {
  int n;
  double kernel[3][256];
  double lift[3];
} dgop_t;

static void dgop_build(const ndgo_config* c, dgop_t* op) {
  double gl[16], w[16], D[256];
  const int n = c->order;
  ndgo_gauss_lobatto(n, gl, w);
  ndgo_differentiation_matrix(n, gl, D);
  op->n = n;
  for (int d = 0; d < c->dim; ++d) {
    const double dx = cell_size(c, d);
    for (int k = 0; k < n; ++k)
      for (int l = 0; l < n; ++l) op->kernel[d][k * n + l] = 2.0 * D[l * n + k] * w[l] / (dx * w[k]);
    op->lift[d] = 2.0 / (dx * w[0]);
  }
}

/* DGOperator::apply (solver.cpp:212-308). shape cells = cells[] (block-local);
 * halo_low/high[d] are face planes in pack_face_trace order. */
static int dgop_apply(const ndgo_config* c, const dgop_t* op, const int cells[3],
                      const double* u, double* const halo_low[3], double* const halo_high[3],
                      double* dudt, size_t n_total, ndgo_error* err) {
  memset(dudt, 0, n_total * sizeof(double));
  const int N = c->order, nv = ndgo_n_var(c);
  const strides_t st = strides_of(c->dim, cells, N, nv);
  double fline[16 * 4], fhat[4], bad = 0.0;
  char msg[200];
  for (int d = 0; d < c->dim; ++d) {
    const double* K = op->kernel[d];
    const double lift = op->lift[d];
    const size_t sd = st.node[d];
    const transverse_t t = transverse_of(c->dim, cells, N, d);
    const int md = cells[d];
    for (int cd = 0; cd < md; ++cd)
      for (int c0 = 0; c0 < t.cells0; ++c0)
        for (int c1 = 0; c1 < t.cells1; ++c1) {
          size_t cell_base = cd * st.cell[d];
          if (t.count > 0) cell_base += c0 * st.cell[t.axes[0]];
          if (t.count > 1) cell_base += c1 * st.cell[t.axes[1]];
          for (int a0 = 0; a0 < t.nodes0; ++a0)
            for (int a1 = 0; a1 < t.nodes1; ++a1) {
              size_t base = cell_base;
              if (t.count > 0) base += a0 * st.node[t.axes[0]];
              if (t.count > 1) base += a1 * st.node[t.axes[1]];
              for (int l = 0; l < N; ++l) {
                if (physical_flux(c, &u[base + l * sd], d, &fline[l * nv])) {
                  int cell[3] = {0, 0, 0};
                  cell[d] = cd;
                  if (t.count > 0) cell[t.axes[0]] = c0;
                  if (t.count > 1) cell[t.axes[1]] = c1;
                  snprintf(msg, sizeof(msg),
                           "nonpositive density %f in flux evaluation at cell (%d,%d,%d)",
                           u[base + l * sd], cell[0], cell[1], cell[2]);
                  set_err(err, 2, 0, msg);
                  return 2;
                }
              }
              for (int k = 0; k < N; ++k) {
                double* out = &dudt[base + k * sd];
                const double* krow = &K[k * N];
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                for (int l = 0; l < N; ++l) {
                  const double kl = krow[l];
                  const double* f = &fline[l * nv];
                  for (int v = 0; v < nv; ++v) acc[v] += kl * f[v];
                }
                for (int v = 0; v < nv; ++v) out[v] += acc[v];
              }
            }
        }
    for (int f = 0; f <= md; ++f) {
      const int has_left = f > 0, has_right = f < md;
      size_t pos = 0;
      for (int c0 = 0; c0 < t.cells0; ++c0)
        for (int c1 = 0; c1 < t.cells1; ++c1) {
          size_t tcell = 0;
          if (t.count > 0) tcell += c0 * st.cell[t.axes[0]];
          if (t.count > 1) tcell += c1 * st.cell[t.axes[1]];
          const size_t left_base = has_left ? tcell + (f - 1) * st.cell[d] + (N - 1) * sd : 0;
          const size_t right_base = has_right ? tcell + f * st.cell[d] : 0;
          for (int a0 = 0; a0 < t.nodes0; ++a0)
            for (int a1 = 0; a1 < t.nodes1; ++a1) {
              size_t noff = 0;
              if (t.count > 0) noff += a0 * st.node[t.axes[0]];
              if (t.count > 1) noff += a1 * st.node[t.axes[1]];
              const double* um = has_left ? &u[left_base + noff] : &halo_low[d][pos];
              const double* up = has_right ? &u[right_base + noff] : &halo_high[d][pos];
              if (lax_friedrichs(c, um, up, d, fhat, &bad)) {
                snprintf(msg, sizeof(msg),
                         "nonpositive density %f in flux evaluation at face %d axis %d", bad, f,
                         d);
                set_err(err, 2, 0, msg);
                return 2;
              }
              if (has_left) {
                double* out = &dudt[left_base + noff];
                for (int v = 0; v < nv; ++v) out[v] -= lift * fhat[v];
              }
              if (has_right) {
                double* out = &dudt[right_base + noff];
                for (int v = 0; v < nv; ++v) out[v] += lift * fhat[v];
              }
              pos += nv;
            }
        }
    }
  }
  return 0;
}

/* max_wavespeed_bound (solver.cpp:310-334) */
double ndgo_max_wavespeed_bound(const ndgo_config* c, const double* u, size_t n,
                                ndgo_error* err) {
  if (c->kind == 0) {
    double alpha = 0.0;
    for (int d = 0; d < c->dim; ++d) alpha = dmax(alpha, fabs(c->velocity[d]));
    return alpha;
  }
  const int nv = ndgo_n_var(c);
  const double a = c->sound_speed;
  double alpha = 0.0;
  for (size_t i = 0; i < n; i += nv) {
    const double rho = u[i];
    if (!(rho > 0.0)) {
      char msg[160];
      snprintf(msg, sizeof(msg), "nonpositive density %f in time-step estimate", rho);
      set_err(err, 2, 0, msg);
      return -1.0;
    }
    double m = 0.0;
    for (int d = 0; d < c->dim; ++d) m = dmax(m, fabs(u[i + 1 + d]));
    alpha = dmax(alpha, m / rho + a);
  }
  return alpha;
}

/* dt_from_alpha (solver.cpp:336-341) */
double ndgo_dt_from_alpha(const ndgo_config* c, double alpha) {
  if (alpha <= 0.0) return INFINITY;
  double h = cell_size(c, 0);
  for (int d = 1; d < c->dim; ++d) h = dmin(h, cell_size(c, d));
  return c->cfl * h / (alpha * (2 * c->order - 1));
}

typedef struct {
  const ndgo_config* c;
  const dgop_t* op;
  int cells[3];
  double* halo_low[3];
  double* halo_high[3];
  size_t n;
} serial_rhs_t;

/* the serial rhs lambda of advance (solver.cpp:386-393) */
static int serial_rhs_apply(serial_rhs_t* s, const double* state, double* dudt,
                            ndgo_error* err) {
  const ndgo_config* c = s->c;
  for (int d = 0; d < c->dim; ++d) {
    ndgo_pack_face_trace(c, s->cells, state, d, s->cells[d] - 1, c->order - 1, s->halo_low[d]);
    ndgo_pack_face_trace(c, s->cells, state, d, 0, 0, s->halo_high[d]);
  }
  return dgop_apply(c, s->op, s->cells, state, s->halo_low, s->halo_high, dudt, s->n, err);
}

static int serial_setup(const ndgo_config* c, dgop_t* op, serial_rhs_t* s) {
  dgop_build(c, op);
  s->c = c;
  s->op = op;
  for (int a = 0; a < 3; ++a) s->cells[a] = cells_of(c, a);
  s->n = ndgo_size(c);
  for (int d = 0; d < 3; ++d) {
    s->halo_low[d] = s->halo_high[d] = NULL;
    if (d < c->dim) {
      const size_t fs = ndgo_face_trace_size(c, s->cells, d);
      s->halo_low[d] = (double*)calloc(fs, sizeof(double));
      s->halo_high[d] = (double*)calloc(fs, sizeof(double));
    }
  }
  return 0;
}

static void serial_teardown(serial_rhs_t* s) {
  for (int d = 0; d < 3; ++d) {
    free(s->halo_low[d]);
    free(s->halo_high[d]);
  }
}

/* serial_rhs (solver.cpp:442-456) */
int ndgo_serial_rhs(const ndgo_config* c, const double* u, double* dudt, ndgo_error* err) {
  dgop_t* op = (dgop_t*)malloc(sizeof(dgop_t));
  serial_rhs_t s;
  serial_setup(c, op, &s);
  const int rc = serial_rhs_apply(&s, u, dudt, err);
  serial_teardown(&s);
  free(op);
  return rc;
}

/* RKIntegrator::step (solver.hpp:49-76) */
typedef struct {
  int stages;
  double a[7][7], b[7];
  double* k[7];
  double* stage;
  size_t n;
} rk_t;

static int rk_step(rk_t* r, double* u, double dt, serial_rhs_t* s, ndgo_error* err) {
  const size_t n = r->n;
  for (int i = 0; i < r->stages; ++i) {
    const double* arg = u;
    if (i > 0) {
      memcpy(r->stage, u, n * sizeof(double));
      for (int j = 0; j < i; ++j) {
        const double aij = r->a[i][j];
        if (aij == 0.0) continue;
        const double* kj = r->k[j];
        double* st = r->stage;
        for (size_t m = 0; m < n; ++m) st[m] += aij * kj[m];
      }
      arg = r->stage;
    }
    const int rc = serial_rhs_apply(s, arg, r->k[i], err);
    if (rc) return rc;
    double* ki = r->k[i];
    for (size_t m = 0; m < n; ++m) ki[m] *= dt;
  }
  for (int i = 0; i < r->stages; ++i) {
    const double bi = r->b[i];
    if (bi == 0.0) continue;
    const double* ki = r->k[i];
    for (size_t m = 0; m < n; ++m) u[m] += bi * ki[m];
  }
  return 0;
}

static int check_finite(const double* u, size_t n, long step, ndgo_error* err) {
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(u[i])) {
      char msg[96];
      snprintf(msg, sizeof(msg), "non-finite state after step %ld", step);
      set_err(err, 3, step, msg);
      return 3;
    }
  }
  return 0;
}

/* validate (solver.cpp:349-357) */
static int validate(const ndgo_config* c, ndgo_error* err) {
  if (!(c->cfl > 0.0) || c->cfl > 1.0) { set_err(err, 1, 0, "cfl must lie in (0, 1]"); return 1; }
  if (!(c->t_end > 0.0)) { set_err(err, 1, 0, "t_end must be positive"); return 1; }
  return 0;
}

/* advance (solver.cpp:372-440) */
int ndgo_advance(const ndgo_config* c, double* u, long fixed_steps, int warmup,
                 ndgo_stats* stats, ndgo_error* err) {
  if (validate(c, err)) return 1;
  dgop_t* op = (dgop_t*)malloc(sizeof(dgop_t));
  serial_rhs_t s;
  serial_setup(c, op, &s);
  const size_t n = s.n;
  rk_t r;
  ndgo_tableau(c->rk, &r.stages, r.a, r.b);
  r.n = n;
  r.stage = (double*)calloc(n, sizeof(double));
  for (int i = 0; i < 7; ++i) r.k[i] = i < r.stages ? (double*)calloc(n, sizeof(double)) : NULL;
  int rc = 0;
  stats->steps = 0;
  stats->dt_min = INFINITY;
  stats->dt_max = 0.0;
  stats->wall_seconds = 0.0;
  if (warmup) {
    double* scratch = (double*)malloc(n * sizeof(double));
    memcpy(scratch, u, n * sizeof(double));
    const double alpha = ndgo_max_wavespeed_bound(c, scratch, n, err);
    if (alpha < 0.0) rc = 2;
    if (!rc) {
      double dt = ndgo_dt_from_alpha(c, alpha);
      if (!isfinite(dt)) dt = c->t_end;
      rc = rk_step(&r, scratch, dt, &s, err);
    }
    free(scratch);
  }
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  if (!rc && fixed_steps >= 0) {
    for (long st = 0; st < fixed_steps && !rc; ++st) {
      const double alpha = ndgo_max_wavespeed_bound(c, u, n, err);
      if (alpha < 0.0) { rc = 2; break; }
      const double dt = ndgo_dt_from_alpha(c, alpha);
      if (!isfinite(dt)) {
        set_err(err, 1, 0, "fixed-step run requires a positive wavespeed");
        rc = 1;
        break;
      }
      rc = rk_step(&r, u, dt, &s, err);
      if (rc) break;
      rc = check_finite(u, n, st + 1, err);
      if (rc) break;
      ++stats->steps;
      stats->dt_min = dmin(stats->dt_min, dt);
      stats->dt_max = dmax(stats->dt_max, dt);
    }
  } else if (!rc) {
    double t = 0.0;
    while (t < c->t_end) {
      const double alpha = ndgo_max_wavespeed_bound(c, u, n, err);
      if (alpha < 0.0) { rc = 2; break; }
      const double stable = ndgo_dt_from_alpha(c, alpha);
      const double remaining = c->t_end - t;
      const int last = remaining <= stable;
      const double dt = last ? remaining : stable;
      rc = rk_step(&r, u, dt, &s, err);
      if (rc) break;
      rc = check_finite(u, n, stats->steps + 1, err);
      if (rc) break;
      ++stats->steps;
      stats->dt_min = dmin(stats->dt_min, dt);
      stats->dt_max = dmax(stats->dt_max, dt);
      if (last) break;
      t += dt;
    }
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  stats->wall_seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  free(r.stage);
  for (int i = 0; i < 7; ++i) free(r.k[i]);
  serial_teardown(&s);
  free(op);
  return rc;
}

/* ----------------------------------------------------------- partition */

static int64_t interface_cost(const ndgo_config* c, const int grid[3]) {
  int64_t cost = 0; /* partition.cpp:22-34 */
  for (int d = 0; d < c->dim; ++d) {
    int64_t cross = 1;
    for (int e = 0; e < c->dim; ++e)
      if (e != d) cross *= c->cells[e];
    cost += (int64_t)grid[d] * cross;
  }
  return cost;
}

static int range_start(int cells, int parts, int index) { /* partition.cpp:36-40 */
  const int base = cells / parts, rem = cells % parts;
  return index * base + (index < rem ? index : rem);
}

static int grid_less(const int a[3], const int b[3]) {
  for (int i = 0; i < 3; ++i) {
    if (a[i] < b[i]) return 1;
    if (a[i] > b[i]) return 0;
  }
  return 0;
}

/* decompose (partition.cpp:44-106) */
int ndgo_decompose(const ndgo_config* c, int workers, int grid[3], int* lo, int* hi, int* nbr,
                   ndgo_error* err) {
  if (workers < 1) { set_err(err, 4, 0, "worker count must be >= 1"); return 4; }
  int found = 0, best[3] = {1, 1, 1};
  int64_t best_cost = 0;
  int cells[3];
  for (int a = 0; a < 3; ++a) cells[a] = cells_of(c, a);
  for (int px = 1; px <= workers; ++px) {
    if (workers % px) continue;
    const int rest = workers / px;
    for (int py = 1; py <= rest; ++py) {
      if (rest % py) continue;
      const int g[3] = {px, py, rest / py};
      int ok = 1;
      for (int d = 0; d < 3; ++d) {
        if (d >= c->dim && g[d] != 1) ok = 0;
        if (g[d] > cells[d]) ok = 0;
      }
      if (!ok) continue;
      const int64_t cost = interface_cost(c, g);
      if (!found || cost < best_cost || (cost == best_cost && grid_less(g, best))) {
        found = 1;
        memcpy(best, g, sizeof(best));
        best_cost = cost;
      }
    }
  }
  if (!found) {
    set_err(err, 4, 0, "no factorization of workers fits the cell grid");
    return 4;
  }
  memcpy(grid, best, sizeof(best));
  for (int gx = 0; gx < best[0]; ++gx)
    for (int gy = 0; gy < best[1]; ++gy)
      for (int gz = 0; gz < best[2]; ++gz) {
        const int w = (gx * best[1] + gy) * best[2] + gz;
        const int coord[3] = {gx, gy, gz};
        for (int d = 0; d < 3; ++d) {
          lo[w * 3 + d] = range_start(cells[d], best[d], coord[d]);
          hi[w * 3 + d] = range_start(cells[d], best[d], coord[d] + 1);
        }
        for (int d = 0; d < 3; ++d) {
          int cc[3] = {gx, gy, gz};
          cc[d] = (coord[d] + best[d] - 1) % best[d];
          nbr[(w * 3 + d) * 2 + 0] = (cc[0] * best[1] + cc[1]) * best[2] + cc[2];
          cc[d] = (coord[d] + 1) % best[d];
          nbr[(w * 3 + d) * 2 + 1] = (cc[0] * best[1] + cc[1]) * best[2] + cc[2];
        }
      }
  return 0;
}

uint64_t ndgo_fnv1a64(const void* data, size_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xCBF29CE484222325ULL;
  for (size_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ULL;
  }
  return h;
}
