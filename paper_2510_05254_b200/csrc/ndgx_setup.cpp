// ndgx_setup.cpp -- host setup inputs of the GPU path: Gauss-Lobatto basis,
// operator coefficients, RK tableaus, initial conditions, decomposition.
//
// These run once per problem on the host and must produce exactly the
// reference's doubles (the operator matrices K_d feed every stage), so they
// follow the reference's expression order and are compiled with
// -ffp-contract=off.  Paths relative to /root/reference/proj.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "ndgx.h"
#include "ndgx_setup.h"

namespace ndgx {

// legendre (src/basis.cpp:15-30)
void legendre(int n, double x, double* p_out, double* dp_out) {
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

// Butcher tableaus (src/solver.cpp:17-68)
void rk_tableau(int rk, int* stages, double a[7][7], double b[7]) {
  std::memset(a, 0, sizeof(double) * 49);
  std::memset(b, 0, sizeof(double) * 7);
  if (rk == NDGX_RK3) {
    *stages = 3;
    a[1][0] = 1.0 / 3.0;
    a[2][1] = 2.0 / 3.0;
    b[0] = 0.25;
    b[2] = 0.75;
  } else if (rk == NDGX_RK4) {
    *stages = 4;
    a[1][0] = 0.5;
    a[2][1] = 0.5;
    a[3][2] = 1.0;
    b[0] = 1.0 / 6.0;
    b[1] = 1.0 / 3.0;
    b[2] = 1.0 / 3.0;
    b[3] = 1.0 / 6.0;
  } else {
    const double q = std::sqrt(21.0);
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
    b[0] = 9.0 / 180.0;
    b[2] = 64.0 / 180.0;
    b[4] = 49.0 / 180.0;
    b[5] = 49.0 / 180.0;
    b[6] = 9.0 / 180.0;
  }
}

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;  // src/grid.cpp:12

int cells_of(const ndgx_problem* p, int a) { return a < p->dim ? p->cells[a] : 1; }
double cell_size(const ndgx_problem* p, int a) {
  return (a < p->dim ? p->length[a] : 1.0) / static_cast<double>(cells_of(p, a));
}

size_t aos_index(const ndgx_problem* p, int nv, const int cell[3], const int node[3], int var) {
  size_t idx = 0;  // FieldShape::index (include/ndg/grid.hpp:50-56)
  for (int a = 0; a < p->dim; ++a) idx = idx * p->cells[a] + cell[a];
  for (int a = 0; a < p->dim; ++a) idx = idx * p->order + node[a];
  return idx * nv + var;
}

// Parallel over the outermost cell axis; every node is independent, so the
// result is identical to the reference's sequential for_each_node
// (src/grid.cpp:28-48).
template <typename Fn>
void for_each_node_parallel(const ndgx_problem* p, Fn&& fn) {
  const int n = p->order;
  int nc[3] = {1, 1, 1};
  for (int a = 0; a < p->dim; ++a) nc[a] = n;
  const int c0 = cells_of(p, 0);
  const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  const int workers = static_cast<int>(std::min<unsigned>(hw, static_cast<unsigned>(c0)));
  auto run = [&](int lo, int hi) {
    int cell[3], node[3];
    for (cell[0] = lo; cell[0] < hi; ++cell[0])
      for (cell[1] = 0; cell[1] < cells_of(p, 1); ++cell[1])
        for (cell[2] = 0; cell[2] < cells_of(p, 2); ++cell[2])
          for (node[0] = 0; node[0] < nc[0]; ++node[0])
            for (node[1] = 0; node[1] < nc[1]; ++node[1])
              for (node[2] = 0; node[2] < nc[2]; ++node[2]) fn(cell, node);
  };
  if (workers <= 1 || static_cast<int64_t>(c0) * cells_of(p, 1) * cells_of(p, 2) < 4096) {
    run(0, c0);
    return;
  }
  std::vector<std::thread> th;
  for (int w = 0; w < workers; ++w) {
    const int lo = static_cast<int>(static_cast<int64_t>(c0) * w / workers);
    const int hi = static_cast<int>(static_cast<int64_t>(c0) * (w + 1) / workers);
    th.emplace_back(run, lo, hi);
  }
  for (auto& t : th) t.join();
}

// for_each_node (src/grid.cpp:28-48), sequential, with its quadrature weight
// jac * prod_a w[node_a] formed in the same order (for order-dependent sums).
template <typename Fn>
void for_each_node_weighted(const ndgx_problem* p, const double* w, Fn&& fn) {
  int nc[3] = {1, 1, 1};
  for (int a = 0; a < p->dim; ++a) nc[a] = p->order;
  double jac = 1.0;
  for (int a = 0; a < p->dim; ++a) jac *= 0.5 * cell_size(p, a);
  int cell[3], node[3];
  for (cell[0] = 0; cell[0] < cells_of(p, 0); ++cell[0])
    for (cell[1] = 0; cell[1] < cells_of(p, 1); ++cell[1])
      for (cell[2] = 0; cell[2] < cells_of(p, 2); ++cell[2])
        for (node[0] = 0; node[0] < nc[0]; ++node[0])
          for (node[1] = 0; node[1] < nc[1]; ++node[1])
            for (node[2] = 0; node[2] < nc[2]; ++node[2]) {
              double wt = jac;
              for (int a = 0; a < p->dim; ++a) wt *= w[node[a]];
              fn(cell, node, wt);
            }
}

void node_coords(const ndgx_problem* p, const double* gl,const int cell[3], const int node[3],
                 double x[3]) {
  x[0] = x[1] = x[2] = 0.0;  // node_coordinates (src/grid.cpp:109-125)
  for (int a = 0; a < p->dim; ++a) {
    const double dx = cell_size(p, a);
    x[a] = cell[a] * dx + 0.5 * dx * (gl[node[a]] + 1.0);
  }
}

int64_t interface_cost(int dim, const int cells[3], const int grid[3]) {
  int64_t cost = 0;  // src/partition.cpp:22-34
  for (int d = 0; d < dim; ++d) {
    int64_t cross = 1;
    for (int e = 0; e < dim; ++e)
      if (e != d) cross *= cells[e];
    cost += static_cast<int64_t>(grid[d]) * cross;
  }
  return cost;
}

int range_start(int cells, int parts, int index) {  // src/partition.cpp:36-40
  const int base = cells / parts, rem = cells % parts;
  return index * base + std::min(index, rem);
}

}  // namespace

void build_operator(const ndgx_problem* p, const double* nodes, const double* weights,
                    const double* diff, double K[3][64], double lift[3]) {
  const int n = p->order;  // DGOperator ctor (src/solver.cpp:189-210)
  for (int d = 0; d < 3; ++d) {
    for (int q = 0; q < 64; ++q) K[d][q] = 0.0;
    lift[d] = 0.0;
  }
  for (int d = 0; d < p->dim; ++d) {
    const double dx = cell_size(p, d);
    for (int k = 0; k < n; ++k)
      for (int l = 0; l < n; ++l) K[d][k * n + l] = 2.0 * diff[l * n + k] * weights[l] / (dx * weights[k]);
    lift[d] = 2.0 / (dx * weights[0]);
  }
}

double dt_numerator(const ndgx_problem* p) {
  double h = cell_size(p, 0);  // dt_from_alpha (src/solver.cpp:336-341)
  for (int d = 1; d < p->dim; ++d) h = std::min(h, cell_size(p, d));
  return p->cfl * h;
}

}  // namespace ndgx

using namespace ndgx;

namespace ndgx {
namespace {
template <typename Fn>
void for_each_block_node(const ndgx_problem* p, const int lo[3], const int hi[3], Fn&& fn) {
  ndgx_problem local = *p;
  for (int a = 0; a < 3; ++a) local.cells[a] = a < p->dim ? hi[a] - lo[a] : 1;
  for_each_node_parallel(&local, [&](const int cell[3], const int node[3]) {
    const int g[3] = {cell[0] + (p->dim > 0 ? lo[0] : 0), cell[1] + (p->dim > 1 ? lo[1] : 0),
                      cell[2] + (p->dim > 2 ? lo[2] : 0)};
    fn(&local, cell, g, node);
  });
}
bool block_ok(const ndgx_problem* p, const int lo[3], const int hi[3]) {
  for (int a = 0; a < p->dim; ++a)
    if (lo[a] < 0 || hi[a] > p->cells[a] || lo[a] >= hi[a]) return false;
  return true;
}
}  // namespace
}  // namespace ndgx

extern "C" {

// gauss_lobatto (src/basis.cpp:32-76)
int ndgx_gauss_lobatto(int order, double* nodes, double* weights) {
  if (order < 2 || order > 16) return NDGX_ERR_CONFIG;
  const int n = order, deg = order - 1;
  for (int k = 0; k < n; ++k) nodes[k] = 0.0;
  nodes[0] = -1.0;
  nodes[n - 1] = 1.0;
  const double pi = std::acos(-1.0);
  for (int k = 1; k < n - 1; ++k) {
    double x = -std::cos(pi * k / deg);
    for (int it = 0; it < 100; ++it) {
      double pv, dp;
      legendre(deg, x, &pv, &dp);
      const double delta = (1.0 - x * x) * dp / (deg * (deg + 1) * pv);
      x += delta;
      if (std::abs(delta) <= 1e-15) break;
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
    double pv, dp;
    legendre(deg, nodes[k], &pv, &dp);
    weights[k] = 2.0 / (n * deg * pv * pv);
  }
  return NDGX_OK;
}

// differentiation_matrix (src/basis.cpp:96-118)
int ndgx_differentiation_matrix(int order, const double* nodes, double* diff) {
  if (order < 2 || order > 16) return NDGX_ERR_CONFIG;
  const int n = order, deg = n - 1;
  double pk[16], dp;
  for (int k = 0; k < n; ++k) legendre(deg, nodes[k], &pk[k], &dp);
  for (int l = 0; l < n; ++l) {
    double rowsum = 0.0;
    for (int k = 0; k < n; ++k) {
      if (k == l) continue;
      const double v = pk[l] / (pk[k] * (nodes[l] - nodes[k]));
      diff[l * n + k] = v;
      rowsum += v;
    }
    diff[l * n + l] = -rowsum;
  }
  return NDGX_OK;
}

// multisine_amplitudes (src/grid.cpp:127-133) with SplitMix64 (include/ndg/rng.hpp:15-33)
void ndgx_multisine_amplitudes(int n_modes, uint64_t seed, double* out) {
  uint64_t state = seed;
  for (int k = 0; k < n_modes; ++k) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    out[k] = static_cast<double>(z >> 11) * 0x1.0p-53;
  }
}

// init_multisine (src/grid.cpp:135-156)
int ndgx_init_multisine(const ndgx_problem* p, const double* amps, int n_modes, double* u) {
  if (p->equation != NDGX_ADVECTION || n_modes < 1) return NDGX_ERR_CONFIG;
  double gl[16], w[16];
  if (ndgx_gauss_lobatto(p->order, gl, w)) return NDGX_ERR_CONFIG;
  for_each_node_parallel(p, [&](const int cell[3], const int node[3]) {
    double x[3];
    node_coords(p, gl, cell, node, x);
    double v = 0.0;
    for (int k = 0; k < n_modes; ++k) v += amps[k] * std::sin(kTwoPi * static_cast<double>(k + 1) * x[0]);
    u[aos_index(p, 1, cell, node, 0)] = v;
  });
  return NDGX_OK;
}

// The same initial conditions restricted to the block [lo, hi) of the global
// mesh `p`, written in the block's own AoS layout: every node value is the
// global one (node coordinates come from the global cell index), so a
// decomposed run starts from exactly the slices of the global field.

int ndgx_init_multisine_block(const ndgx_problem* p, const double* amps, int n_modes, const int lo[3],
                              const int hi[3], double* u) {
  if (p->equation != NDGX_ADVECTION || n_modes < 1 || !block_ok(p, lo, hi)) return NDGX_ERR_CONFIG;
  double gl[16], w[16];
  if (ndgx_gauss_lobatto(p->order, gl, w)) return NDGX_ERR_CONFIG;
  for_each_block_node(p, lo, hi, [&](const ndgx_problem* lp, const int cell[3], const int g[3], const int node[3]) {
    double x[3];
    node_coords(p, gl, g, node, x);
    double v = 0.0;
    for (int k = 0; k < n_modes; ++k) v += amps[k] * std::sin(kTwoPi * static_cast<double>(k + 1) * x[0]);
    u[aos_index(lp, 1, cell, node, 0)] = v;
  });
  return NDGX_OK;
}

int ndgx_init_euler_subsonic_block(const ndgx_problem* p, const int lo[3], const int hi[3], double* u) {
  if (p->equation != NDGX_EULER_ISOTHERMAL || p->dim < 2 || !block_ok(p, lo, hi)) return NDGX_ERR_CONFIG;
  double gl[16], w[16];
  if (ndgx_gauss_lobatto(p->order, gl, w)) return NDGX_ERR_CONFIG;
  const int nv = p->dim + 1;
  const double a = p->sound_speed;
  for_each_block_node(p, lo, hi, [&](const ndgx_problem* lp, const int cell[3], const int g[3], const int node[3]) {
    double x[3];
    node_coords(p, gl, g, node, x);
    const double sx = std::sin(kTwoPi * x[0]);
    const double sy = std::sin(kTwoPi * x[1]);
    double rho = 1.0 + 0.2 * sx * sy;
    if (p->dim == 3) rho = 1.0 + 0.2 * sx * sy * std::sin(kTwoPi * x[2]);
    const double ux = 0.5 * a * sy;
    const double uy = 0.5 * a * sx;
    u[aos_index(lp, nv, cell, node, 0)] = rho;
    u[aos_index(lp, nv, cell, node, 1)] = rho * ux;
    u[aos_index(lp, nv, cell, node, 2)] = rho * uy;
    if (p->dim == 3) u[aos_index(lp, nv, cell, node, 3)] = 0.0;
  });
  return NDGX_OK;
}

// init_euler_subsonic (src/grid.cpp:162-188)
int ndgx_init_euler_subsonic(const ndgx_problem* p, double* u) {
  if (p->equation != NDGX_EULER_ISOTHERMAL || p->dim < 2) return NDGX_ERR_CONFIG;
  double gl[16], w[16];
  if (ndgx_gauss_lobatto(p->order, gl, w)) return NDGX_ERR_CONFIG;
  const int nv = p->dim + 1;
  const double a = p->sound_speed;
  for_each_node_parallel(p, [&](const int cell[3], const int node[3]) {
    double x[3];
    node_coords(p, gl, cell, node, x);
    const double sx = std::sin(kTwoPi * x[0]);
    const double sy = std::sin(kTwoPi * x[1]);
    double rho = 1.0 + 0.2 * sx * sy;
    if (p->dim == 3) rho = 1.0 + 0.2 * sx * sy * std::sin(kTwoPi * x[2]);
    const double ux = 0.5 * a * sy;
    const double uy = 0.5 * a * sx;
    u[aos_index(p, nv, cell, node, 0)] = rho;
    u[aos_index(p, nv, cell, node, 1)] = rho * ux;
    u[aos_index(p, nv, cell, node, 2)] = rho * uy;
    if (p->dim == 3) u[aos_index(p, nv, cell, node, 3)] = 0.0;
  });
  return NDGX_OK;
}

// l2_error (src/grid.cpp:190-203): sequential in for_each_node order
// (src/grid.cpp:28-48) with the same weight products, so the sum is the
// reference's bit for bit.  Host diagnostics for the convergence experiments.
int ndgx_l2_error(const ndgx_problem* p, const double* a, const double* b, int var, double* out) {
  double gl[16], w[16];
  if (!p || !a || !b || !out || ndgx_gauss_lobatto(p->order, gl, w)) return NDGX_ERR_CONFIG;
  const int nv = p->equation == NDGX_ADVECTION ? 1 : p->dim + 1;
  if (var < 0 || var >= nv) return NDGX_ERR_CONFIG;
  double sum = 0.0;
  for_each_node_weighted(p, w, [&](const int cell[3], const int node[3], double wt) {
    const size_t i = aos_index(p, nv, cell, node, var);
    const double d = a[i] - b[i];
    sum += wt * d * d;
  });
  *out = std::sqrt(sum);
  return NDGX_OK;
}

// conserved_totals (src/grid.cpp:205-213): out[nvar]
int ndgx_conserved_totals(const ndgx_problem* p, const double* u, double* out) {
  double gl[16], w[16];
  if (!p || !u || !out || ndgx_gauss_lobatto(p->order, gl, w)) return NDGX_ERR_CONFIG;
  const int nv = p->equation == NDGX_ADVECTION ? 1 : p->dim + 1;
  for (int v = 0; v < nv; ++v) out[v] = 0.0;
  for_each_node_weighted(p, w, [&](const int cell[3], const int node[3], double wt) {
    for (int v = 0; v < nv; ++v) out[v] += wt * u[aos_index(p, nv, cell, node, v)];
  });
  return NDGX_OK;
}

// decompose (src/partition.cpp:44-106)
int ndgx_decompose(int dim, const int cells_in[3], int workers, int grid[3], int* lo, int* hi,
                   int* nbr, ndgx_error* err) {
  auto fail = [&](const char* msg) {
    if (err) {
      std::memset(err, 0, sizeof(*err));
      err->code = NDGX_ERR_DECOMPOSITION;
      err->stage = -1;
      err->worker = -1;
      std::snprintf(err->message, sizeof(err->message), "%s", msg);
    }
    return static_cast<int>(NDGX_ERR_DECOMPOSITION);
  };
  if (workers < 1) {
    char m[96];
    std::snprintf(m, sizeof(m), "worker count must be >= 1, got %d", workers);
    return fail(m);
  }
  int cells[3];
  for (int a = 0; a < 3; ++a) cells[a] = a < dim ? cells_in[a] : 1;
  bool found = false;
  int best[3] = {1, 1, 1};
  int64_t best_cost = 0;
  for (int px = 1; px <= workers; ++px) {
    if (workers % px) continue;
    const int rest = workers / px;
    for (int py = 1; py <= rest; ++py) {
      if (rest % py) continue;
      const int g[3] = {px, py, rest / py};
      bool ok = true;
      for (int d = 0; d < 3; ++d) {
        if (d >= dim && g[d] != 1) ok = false;
        if (g[d] > cells[d]) ok = false;
      }
      if (!ok) continue;
      const int64_t cost = interface_cost(dim, cells, g);
      const bool less = std::lexicographical_compare(g, g + 3, best, best + 3);
      if (!found || cost < best_cost || (cost == best_cost && less)) {
        found = true;
        std::copy(g, g + 3, best);
        best_cost = cost;
      }
    }
  }
  if (!found) {
    char m[200];
    std::snprintf(m, sizeof(m),
                  "no factorization of %d workers fits a %dx%dx%d cell grid with at least one "
                  "cell per block per axis",
                  workers, cells[0], cells[1], cells[2]);
    return fail(m);
  }
  std::copy(best, best + 3, grid);
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
          int c[3] = {gx, gy, gz};
          c[d] = (coord[d] + best[d] - 1) % best[d];
          nbr[(w * 3 + d) * 2 + 0] = (c[0] * best[1] + c[1]) * best[2] + c[2];
          c[d] = (coord[d] + 1) % best[d];
          nbr[(w * 3 + d) * 2 + 1] = (c[0] * best[1] + c[1]) * best[2] + c[2];
        }
      }
  if (err) err->code = NDGX_OK;
  return NDGX_OK;
}

}  // extern "C"
