// ndgx_device.cuh -- sm_100a kernels of the fused NDG RHS + RK stage update.
//
// Reference semantics (paths relative to /root/reference/proj):
//   volume term      src/solver.cpp:229-262   (per axis, K-row dot, out += acc)
//   face term        src/solver.cpp:264-306   (LF flux, -/+ lift)
//   physical flux    src/models.cpp:42-57, wavespeed :59-75, LF :77-88
//   RK stage update  include/ndg/solver.hpp:49-76
//   CFL alpha scan   src/solver.cpp:310-334, dt_from_alpha :336-341
//   finite check     src/solver.cpp:361-368
//
// Device layout (SoA, node-fastest, element-blocked):
//   a[((e * NV + v) * NPE) + n],  e = cx + C0*(cy + C1*cz),  n = i + N*(j + N*k)
// so one element's variable is NPE contiguous doubles (512 B at 2D N=8 and
// at 3D N=4) and each x-line is N contiguous doubles.
//
// The fused stage kernel (ndgx_stage.cuh) runs one element per warp over a
// persistent grid (see there).  This file holds the shared arithmetic
// (reference operation order), the step-control kernels, the wavespeed scan,
// the face-plane packing of multi-block runs and the layout permutation.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace ndgx {

constexpr int kMaxOrder = 8;
constexpr int kMaxTerms = 6;
constexpr int kMaxRanges = 6;  // boundary shell of a 3D block: two slabs per axis
constexpr unsigned long long kNoError = ~0ull;

// Error-key phases, ordered like the reference's execution within a step.
enum : int {
  kPhaseScan = 0,        // max_wavespeed_bound PhysicsError (solver.cpp:325-328)
  kPhaseZeroSpeed = 1,   // fixed-step ConfigError (solver.cpp:411-413)
  kPhaseStage0 = 2,      // 2 + stage: operator PhysicsError (solver.cpp:258-261)
  kPhaseInstability = 9  // check_finite InstabilityError (solver.cpp:361-368)
};

__host__ __device__ inline unsigned long long error_key(long long step, int phase,
                                                        long long cell, int node) {
  return ((unsigned long long)(step & 0xFFFFF) << 44) | ((unsigned long long)(phase & 0xF) << 40) |
         ((unsigned long long)(cell & 0xFFFFFFF) << 12) | (unsigned long long)(node & 0xFFF);
}

// Device-resident step control (advance, solver.cpp:405-436).
struct Control {
  unsigned long long alpha_bits;  // running max wavespeed of the current state (>= 0)
  unsigned long long any_err;     // 1 once any error was recorded; max-reduced with alpha_bits
                                  // across ranks so every rank stops at the same step
  unsigned long long err_key;     // first error in reference execution order
  double dt;
  double t;
  double dt_min;
  double dt_max;
  long long steps;                // steps begun
  int skip;                       // current step inactive (done / error)
  int done;                       // t_end reached
  int aborted;                    // multi-rank: some rank failed, this one stopped with it
};

struct StepParams {
  Control* ctl;
  long long fixed_steps;  // < 0: t_end mode
  double t_end;
  double cflh;            // cfl * min_d dx_d  (dt_from_alpha numerator)
  double two_n_minus_1;   // (2N - 1)
  double const_alpha;     // advection: max_d |a_d|; < 0 for Euler (scanned)
  int warmup;             // warm-up step: non-finite dt -> t_end, no stats
  int ranked;             // multi-rank solver: any_err (all-reduced) stops every rank
};

// Stage signatures of the supported tableaus (make_rk3/4/6, solver.cpp:17-68):
// (number of K_j read, bit t set when ku[t] enters U_s (a != 0), bit t set
// when ku[t] enters the last stage's S (b != 0)).  Kernels are instantiated
// per signature so the term loops are fully resolved at compile time.
struct StageSig {
  int nu, am, bm;
};
constexpr StageSig kSigs[] = {{0, 0, 0},  {1, 1, 0},  {2, 2, 1},  {3, 4, 7},  {2, 3, 0},
                              {3, 7, 0},  {4, 15, 0}, {5, 31, 0}, {6, 63, 53}};
constexpr int kNumSigs = 9;

struct StageArgs {
  const double* u;                 // u^n
  // ku[0..nu): the K_j this stage reads (ascending j).  Stage input U_s =
  // u + sum over t with bit t of amask of ca[t] * ku[t] (a_sj != 0,
  // solver.hpp:55-62); at the last stage S = u + sum over bit t of bmask of
  // cb[t] * ku[t] (b_j != 0, solver.hpp:69-75); both in ascending j order.
  const double* ku[kMaxTerms];
  int nu, amask, bmask;
  double ca[kMaxTerms], cb[kMaxTerms];
  double* out;                     // K_s, or u_new at the last stage
  Control* ctl;
  double b_last;
  int is_last;
  int rhs_only;                    // serial_rhs: dt := 1, no step control
  int phase;                       // kPhaseStage0 + stage
  int scan_alpha;                  // last stage of an Euler run: reduce next alpha
  int cells[3];                    // local block
  int gcells[3];                   // global mesh (error cell naming)
  int goff[3];                     // block offset in the global mesh
  double sound_speed;
  double vel[3];
  double lift[3];
  double K[3][kMaxOrder * kMaxOrder];  // K_d[k*N + l] (solver.cpp:203-207)
  int depth;                       // per-warp ring depth (elements in flight + 1); 0: direct loads
  int sig;                         // index into kSigs (host bookkeeping)
  // multi-block: stage-input face planes received from the neighbour across
  // [axis][side] (side 0 low, 1 high), layout [cross-section cell][var][face node];
  // null -> periodic wrap inside this block
  const double* ext[3][2];
  // element ranges of this launch, one per blockIdx.y: e = rng[q][0],
  // rng[q][0] + rng[q][2], ... < rng[q][1] (the whole block; or the interior
  // / the boundary shell when a stage is split around its halo exchange:
  // contiguous runs, whole x-columns at stride C0), and the region filter:
  // 0 every element of the ranges, 1 only those inside the box
  // [inner[0], inner[1]), 2 only those outside it, 3 like 1 where the
  // range's rows all lie inside the box in y and z (only x is tested)
  int rng[kMaxRanges][3];
  int region;
  int inner[2][3];
  int block_id;                    // worker / rank: names the block in InstabilityError keys
};

// ------------------------------------------------------------- arithmetic
template <bool EXACT>
struct Ar;

template <>
struct Ar<true> {  // reference IEEE order, no contraction
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double mac(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));
  }
};

template <>
struct Ar<false> {  // contracted
  static __device__ __forceinline__ double add(double a, double b) { return a + b; }
  static __device__ __forceinline__ double sub(double a, double b) { return a - b; }
  static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
  static __device__ __forceinline__ double div(double a, double b) { return a / b; }
  static __device__ __forceinline__ double mac(double acc, double a, double b) {
    return fma(a, b, acc);
  }
};

__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }

// F_axis(u) and the one-sided wavespeed bound (models.cpp:42-70).
// With rinv >= 0 (contracted mode only) u_a / rho is formed as u_a * (1 / rho),
// sharing one reciprocal between the axes of a node.
template <int DIM, int KIND, bool EXACT>
__device__ __forceinline__ void flux(const StageArgs& p, const double* u, int axis, double* f,
                                     double& speed, double rinv = -1.0) {
  using A = Ar<EXACT>;
  if (KIND == 0) {
    f[0] = A::mul(p.vel[axis], u[0]);
    speed = fabs(p.vel[axis]);
  } else {
    constexpr int NV = DIM + 1;
    const double rho = u[0];
    // m_axis by selects: `axis` may be a run-time value, and a dynamic index
    // into u[] / f[] would put both arrays in local memory
    double ma = u[1];
    if (axis == 1) ma = u[2];
    if (DIM > 2 && axis == 2) ma = u[DIM > 2 ? 3 : 1];
    const double ua = (!EXACT && rinv >= 0.0) ? ma * rinv : A::div(ma, rho);
    const double pr = A::mul(A::mul(rho, p.sound_speed), p.sound_speed);
    f[0] = ma;
#pragma unroll
    for (int i = 1; i < NV; ++i) {
      f[i] = A::mul(ua, u[i]);
      if (i == 1 + axis) f[i] = A::add(f[i], pr);
    }
    speed = A::add(fabs(ua), p.sound_speed);
  }
}

// Lax-Friedrichs flux from both one-sided fluxes and speeds (models.cpp:77-88).
template <int NV, bool EXACT>
__device__ __forceinline__ void lax_friedrichs(const double* um, const double* up,
                                               const double* fm, const double* fp, double sm,
                                               double sp, double* fhat) {
  using A = Ar<EXACT>;
  const double alpha = dmax(sm, sp);
#pragma unroll
  for (int v = 0; v < NV; ++v)
    fhat[v] = A::mul(0.5, A::sub(A::add(fm[v], fp[v]), A::mul(alpha, A::sub(up[v], um[v]))));
}

__device__ __forceinline__ void record_error(Control* ctl, unsigned long long key) {
  if (key < *(volatile unsigned long long*)&ctl->err_key) atomicMin(&ctl->err_key, key);
  if (*(volatile unsigned long long*)&ctl->any_err == 0ull) atomicMax(&ctl->any_err, 1ull);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// 0 + x as the reference's dudt.assign(0) followed by out += acc: x, except
// -0 becomes +0.  Done on the integer pipe instead of a DADD.
__device__ __forceinline__ double zero_plus(double x) {
  const long long b = __double_as_longlong(x);
  return (b << 1) == 0 ? 0.0 : x;
}

}  // namespace ndgx

#include "ndgx_stage.cuh"

namespace ndgx {

// ============================================================ alpha scan
// max_wavespeed_bound over a device-layout state (solver.cpp:310-334).
// Error keys name the cell globally (block offset goff, global extents g1, g2),
// like the stage kernels' keys.
template <int DIM>
__global__ void alpha_scan_kernel(const double* __restrict__ u, int c0, int c1, int c2, int order,
                                  double a, Control* ctl, long long step_for_error, int3 goff, int g1, int g2) {
  constexpr int NV = DIM + 1;
  const int npe = DIM == 2 ? order * order : order * order * order;
  const long long n_elem = (long long)c0 * c1 * c2;
  const long long total = n_elem * npe;
  double alpha = 0.0;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long e = q / npe;
    const int n = (int)(q - e * npe);
    const double* base = u + e * NV * npe + n;
    const double rho = base[0];
    if (!(rho > 0.0)) {
      const int cx = (int)(e % c0), cy = (int)((e / c0) % c1), cz = (int)(e / ((long long)c0 * c1));
      const int i = n % order, j = (n / order) % order, k = n / (order * order);
      const int an = DIM == 2 ? i * order + j : (i * order + j) * order + k;
      record_error(ctl, error_key(step_for_error, kPhaseScan,
                                  ((long long)(cx + goff.x) * g1 + cy + goff.y) * g2 + cz + goff.z, an));
      continue;
    }
    double m = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) m = dmax(m, fabs(base[(size_t)(1 + d) * npe]));
    alpha = dmax(alpha, __dadd_rn(__ddiv_rn(m, rho), a));
  }
  alpha = warp_max(alpha);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = alpha;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) m = dmax(m, red[w]);
    atomicMax(&ctl->alpha_bits, (unsigned long long)__double_as_longlong(m));
  }
}

// ============================================================ step control
// One thread: dt_from_alpha (solver.cpp:336-341) + the fixed-step / t_end
// loop bookkeeping of advance (solver.cpp:407-436), without host round trips.
static __global__ void step_begin_kernel(StepParams sp) {
  Control* c = sp.ctl;
  if (c->done) {
    c->skip = 1;
    return;
  }
  // completion first: an error recorded by the final step's trailing scan
  // (the next step's wavespeed) must not abort a run that is already over
  const bool fixed = sp.fixed_steps >= 0;
  if ((fixed && c->steps >= sp.fixed_steps) || (!fixed && !(c->t < sp.t_end))) {
    c->done = 1;
    c->skip = 1;
    return;
  }
  if (sp.ranked ? c->any_err != 0ull : c->err_key != kNoError) {
    // a rank solver stops on the all-reduced flag, so every rank -- the
    // failing one included -- stops at this same step (run_partitioned:
    // "stopped by failure elsewhere", src/partition.cpp:239-241)
    if (sp.ranked) c->aborted = 1;
    c->skip = 1;
    return;
  }
  const double alpha = sp.const_alpha >= 0.0 ? sp.const_alpha : __longlong_as_double((long long)c->alpha_bits);
  const double stable = (alpha <= 0.0) ? __longlong_as_double(0x7ff0000000000000LL)
                                       : __ddiv_rn(sp.cflh, __dmul_rn(alpha, sp.two_n_minus_1));
  double dt;
  if (sp.warmup) {
    dt = isfinite(stable) ? stable : sp.t_end;
    c->steps = 1;
    c->done = 1;  // a warm-up is exactly one step
  } else {
    const long long step = ++c->steps;
    if (fixed) {
      if (!isfinite(stable)) {
        atomicMin(&c->err_key, error_key(step, kPhaseZeroSpeed, 0, 0));
        c->skip = 1;
        return;
      }
      dt = stable;
    } else {
      const double remaining = __dsub_rn(sp.t_end, c->t);
      const bool last = remaining <= stable;
      dt = last ? remaining : stable;
      if (last) c->done = 1;
      else c->t = __dadd_rn(c->t, dt);
    }
    c->dt_min = (dt < c->dt_min) ? dt : c->dt_min;
    c->dt_max = (c->dt_max < dt) ? dt : c->dt_max;
  }
  c->dt = dt;
  c->skip = 0;
  c->alpha_bits = 0ull;  // this step's last-stage epilogue accumulates the next alpha
}

// ====================================================== in-graph timing
// The global nanosecond timer into the next slot of out: launched between the
// stages of captured steps, consecutive stamps bracket each stage as it runs
// in the timed graph (events recorded inside a graph cannot be timed).
static __global__ void stamp_kernel(unsigned long long* out, unsigned int* count) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  out[atomicAdd(count, 1u)] = t;
}

// ===================================================== layout permutation
// AoS (FieldShape::index, grid.hpp:50-56) <-> device SoA element-blocked.
template <bool TO_DEVICE>
__global__ void permute_kernel(const double* __restrict__ src, double* __restrict__ dst,
                               int dim, int c0, int c1, int c2, int order, int nv,
                               long long total) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    // q enumerates the device layout: ((e*nv + v)*npe + n)
    int npe = order;
    if (dim > 1) npe *= order;
    if (dim > 2) npe *= order;
    const long long n = q % npe;
    const long long ev = q / npe;
    const int v = (int)(ev % nv);
    const long long e = ev / nv;
    const int cx = (int)(e % c0);
    const long long r = e / c0;
    const int cy = (int)(r % c1);
    const int cz = (int)(r / c1);
    const int i = (int)(n % order);
    const int j = dim > 1 ? (int)((n / order) % order) : 0;
    const int k = dim > 2 ? (int)(n / ((long long)order * order)) : 0;
    long long idx = cx;
    if (dim > 1) idx = idx * c1 + cy;
    if (dim > 2) idx = idx * c2 + cz;
    idx = idx * order + i;
    if (dim > 1) idx = idx * order + j;
    if (dim > 2) idx = idx * order + k;
    idx = idx * nv + v;
    if (TO_DEVICE) dst[q] = src[idx];
    else dst[idx] = src[q];
  }
}

// ===================================================== face-plane packing
// The stage-input traces of a block's boundary faces along its split axes,
// for the neighbour ranks (pack_face_trace + exchange_halos, src/solver.cpp:
// 166-187, src/partition.cpp:108-131): plane [d][side] holds U_s = u + sum
// a K_j (the stage kernel's combination, same arithmetic) at the face nodes
// of the cells with c_d = 0 (side 0) or C_d - 1 (side 1), laid out
// [cross-section cell][var][face node] -- the layout StageArgs::ext reads.
struct PackArgs {
  const double* u;
  const double* ku[kMaxTerms];
  double ca[kMaxTerms];
  int nu, amask;
  int dim, order, nv, npe;
  int cells[3];
  int split[3];
  long long plane[3];    // doubles per plane
  double* snd[3][2];
  Control* ctl;
  int rhs_only;
};

template <bool EXACT>
__global__ void pack_kernel(const __grid_constant__ PackArgs p) {
  using A = Ar<EXACT>;
  if (!p.rhs_only && (*(volatile int*)&p.ctl->skip || *(volatile unsigned long long*)&p.ctl->err_key != kNoError))
    return;
  const int N = p.order;
  const int L = p.dim == 1 ? 1 : (p.dim == 2 ? N : N * N);
  long long total = 0;
  for (int d = 0; d < 3; ++d) total += p.split[d] ? 2 * p.plane[d] : 0;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    long long r = q;
    int d = 0;
    for (; d < 3; ++d) {
      const long long sz = p.split[d] ? 2 * p.plane[d] : 0;
      if (r < sz) break;
      r -= sz;
    }
    const int side = (int)(r / p.plane[d]);
    r -= side * p.plane[d];
    const int t = (int)(r % L);
    const long long xv = r / L;
    const int v = (int)(xv % p.nv);
    const long long xs = xv / p.nv;
    // cross-section cell -> block cell
    int c[3];
    const int a1 = d == 0 ? 1 : 0, a2 = d == 2 ? 1 : 2;
    c[a1] = (int)(xs % p.cells[a1]);
    c[a2] = (int)(xs / p.cells[a1]);
    c[d] = side ? p.cells[d] - 1 : 0;
    const int k = side ? N - 1 : 0;
    int n;  // node(d, t, k)
    if (d == 0) n = k + N * t;
    else if (d == 1) n = (t % N) + N * (k + N * (t / N));
    else n = t + N * N * k;
    const size_t e = (size_t)c[0] + (size_t)p.cells[0] * ((size_t)c[1] + (size_t)p.cells[1] * c[2]);
    const size_t g = (e * p.nv + v) * p.npe + n;
    double U = p.u[g];
    for (int j = 0; j < p.nu; ++j)
      if (p.amask >> j & 1) U = A::mac(U, p.ca[j], p.ku[j][g]);
    p.snd[d][side][r] = U;
  }
}

}  // namespace ndgx
