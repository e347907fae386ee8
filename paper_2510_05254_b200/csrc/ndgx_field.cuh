// ndgx_field.cuh -- initial conditions and diagnostics on the device.
//
// Reference (paths relative to /root/reference/proj):
//   node_coordinates     src/grid.cpp:109-125   x_a = cell_a dx_a + 0.5 dx_a (xi_node + 1)
//   init_multisine       src/grid.cpp:135-156   u = sum_k A_k sin(2 pi (k + 1) x)
//   init_euler_subsonic  src/grid.cpp:162-188   rho = 1 + 0.2 sx sy (sz), m = rho (0.5 a sy, 0.5 a sx, 0)
//   for_each_node        src/grid.cpp:28-48     w = jac * prod_a weight(node_a), jac = prod_a 0.5 dx_a
//   l2_error             src/grid.cpp:190-203   sqrt(sum w (a - b)^2)
//   conserved_totals     src/grid.cpp:205-213   sum w u_v
//   l1_norm              src/grid.cpp:215-223   sum w |u|
//
// The kernels write / read the solver's own device layout
// (a[(e * NV + v) * NPE + n], block-local e, n = i + N (j + N k)), so a C5
// field (6.4 GB) is generated in HBM without a host array or an H2D copy.
// Every expression keeps the reference's operation order with explicit _rn
// roundings; only sin differs (CUDA's libdevice sin vs glibc, <= 2 ulp), so
// device ICs match the host ones to ~1e-16 relative.  The reductions sum in a
// fixed tree order (per-thread grid-stride partials, a CTA tree, the CTA
// partials in index order on the host): deterministic, and equal to the
// reference's sequential sums to rounding (~1e-15 relative).
#pragma once

#include <cuda_runtime.h>

namespace ndgx {

constexpr double kTwoPiDev = 6.283185307179586476925286766559;  // src/grid.cpp:12
constexpr int kMaxModes = 256;

struct FieldArgs {
  double* u;               // device-layout state of one block
  int dim, N, nv, npe;
  int cells[3], goff[3];   // the block and its offset in the global mesh
  double dx[3];            // global cell sizes length / gcells (grid.hpp:27)
  double nodes[8], weights[8];
  double jac;              // prod_a 0.5 dx_a (src/grid.cpp:33-34)
  double sound_speed;
  int ic;                  // 0 multisine, 1 euler subsonic, -1 none
  int n_modes;
  const double* amps;      // device copy of the multisine amplitudes
  int var;                 // diagnostics: the variable of l2 / l1
  int what;                // 0 totals, 1 l2 vs the IC, 2 l1
};

// (e, n) -> global cell and node index
__device__ __forceinline__ void field_cell(const FieldArgs& a, long long e, int n, int cell[3], int node[3]) {
  const int c0 = a.cells[0], c1 = a.cells[1];
  cell[0] = (int)(e % c0) + a.goff[0];
  cell[1] = (int)((e / c0) % c1) + a.goff[1];
  cell[2] = (int)(e / ((long long)c0 * c1)) + a.goff[2];
  node[0] = n % a.N;
  node[1] = a.dim > 1 ? (n / a.N) % a.N : 0;
  node[2] = a.dim > 2 ? n / (a.N * a.N) : 0;
}

// the initial condition at one node, every variable (out[nv])
__device__ __forceinline__ void ic_values(const FieldArgs& a, const int cell[3], const int node[3], double* out) {
  double x[3] = {0.0, 0.0, 0.0};
  for (int d = 0; d < a.dim; ++d)
    x[d] = __dadd_rn(__dmul_rn((double)cell[d], a.dx[d]),
                     __dmul_rn(__dmul_rn(0.5, a.dx[d]), __dadd_rn(a.nodes[node[d]], 1.0)));
  if (a.ic == 0) {
    double v = 0.0;
    for (int k = 0; k < a.n_modes; ++k)
      v = __dadd_rn(v, __dmul_rn(a.amps[k], sin(__dmul_rn(__dmul_rn(kTwoPiDev, (double)(k + 1)), x[0]))));
    out[0] = v;
  } else {
    const double sx = sin(__dmul_rn(kTwoPiDev, x[0]));
    const double sy = sin(__dmul_rn(kTwoPiDev, x[1]));
    double rho = __dadd_rn(1.0, __dmul_rn(__dmul_rn(0.2, sx), sy));
    if (a.dim == 3) rho = __dadd_rn(1.0, __dmul_rn(__dmul_rn(__dmul_rn(0.2, sx), sy), sin(__dmul_rn(kTwoPiDev, x[2]))));
    const double ux = __dmul_rn(__dmul_rn(0.5, a.sound_speed), sy);
    const double uy = __dmul_rn(__dmul_rn(0.5, a.sound_speed), sx);
    out[0] = rho;
    out[1] = __dmul_rn(rho, ux);
    out[2] = __dmul_rn(rho, uy);
    if (a.dim == 3) out[3] = 0.0;
  }
}

// one thread per node of the block: every variable of the IC
__global__ void __launch_bounds__(256) init_field_kernel(const FieldArgs a) {
  const long long nodes = (long long)a.cells[0] * a.cells[1] * a.cells[2] * a.npe;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nodes;
       q += (long long)gridDim.x * blockDim.x) {
    const long long e = q / a.npe;
    const int n = (int)(q - e * a.npe);
    int cell[3], node[3];
    field_cell(a, e, n, cell, node);
    double v[4];
    ic_values(a, cell, node, v);
    for (int w = 0; w < a.nv; ++w) a.u[(e * a.nv + w) * a.npe + n] = v[w];
  }
}

// Weighted sums over the block: what 0 -> sum w u_v (v < nv), 1 -> sum w
// (u_var - IC_var)^2, 2 -> sum w |u_var|; one partial per CTA per output
// (partial[blockIdx.x * nout + k]).
__global__ void __launch_bounds__(256) diag_kernel(const FieldArgs a, double* partial) {
  __shared__ double red[4][8];
  const int nout = a.what == 0 ? a.nv : 1;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const long long nodes = (long long)a.cells[0] * a.cells[1] * a.cells[2] * a.npe;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nodes;
       q += (long long)gridDim.x * blockDim.x) {
    const long long e = q / a.npe;
    const int n = (int)(q - e * a.npe);
    int cell[3], node[3];
    field_cell(a, e, n, cell, node);
    double w = a.jac;
    for (int d = 0; d < a.dim; ++d) w = __dmul_rn(w, a.weights[node[d]]);
    const double* u = a.u + e * a.nv * a.npe + n;
    if (a.what == 0) {
      for (int v = 0; v < a.nv; ++v) acc[v] = __dadd_rn(acc[v], __dmul_rn(w, u[(size_t)v * a.npe]));
    } else if (a.what == 1) {
      double ic[4];
      ic_values(a, cell, node, ic);
      const double d = __dsub_rn(u[(size_t)a.var * a.npe], ic[a.var]);
      acc[0] = __dadd_rn(acc[0], __dmul_rn(__dmul_rn(w, d), d));
    } else {
      acc[0] = __dadd_rn(acc[0], __dmul_rn(w, fabs(u[(size_t)a.var * a.npe])));
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = 0; k < nout; ++k) {
    double v = acc[k];
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) red[k][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < nout; ++k) {
      double s = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s = __dadd_rn(s, red[k][q]);
      partial[blockIdx.x * nout + k] = s;
    }
}

}  // namespace ndgx
