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
// One CTA owns a tile of TE consecutive x-cells.  Phase X: one thread per
// x-line loads the stage input U_s = u + sum_j a_sj K_j (on the fly, in the
// reference's term order), evaluates every axis' flux at its nodes, applies
// the x volume term from registers and the x faces (in-tile neighbours via
// shared memory, others from global/L2).  Phase Y (and Z) re-partition the
// tile into y-lines (z-lines) through shared memory and add their volume and
// face terms in the reference's per-node order vol_x, face_x, vol_y, face_y,
// vol_z, face_z.  The owner of the last phase runs the RK epilogue:
// K_s = dt * dudt (stored), or at the last stage u_new = S + b_s K_s with
// S = u + sum_{j<s} b_j K_j formed in phase X -- plus the finite check and
// the next step's wavespeed max-reduction (warp shuffle -> block -> atomicMax).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ndgx {

constexpr int kMaxOrder = 8;
constexpr int kMaxTerms = 6;
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
  unsigned long long err_key;     // first error in reference execution order
  double dt;
  double t;
  double dt_min;
  double dt_max;
  long long steps;                // steps begun
  int skip;                       // current step inactive (done / error)
  int done;                       // t_end reached
};

struct StepParams {
  Control* ctl;
  long long fixed_steps;  // < 0: t_end mode
  double t_end;
  double cflh;            // cfl * min_d dx_d  (dt_from_alpha numerator)
  double two_n_minus_1;   // (2N - 1)
  double const_alpha;     // advection: max_d |a_d|; < 0 for Euler (scanned)
  int warmup;             // warm-up step: non-finite dt -> t_end, no stats
};

struct StageArgs {
  const double* u;                 // u^n
  // union of the K_j read by this stage (ascending j): the stage input uses
  // those with bit t of amask (coefficient ca[t] = a_sj != 0), the last
  // stage's S = u + sum b_j K_j those with bit t of bmask (cb[t] = b_j != 0)
  const double* ku[kMaxTerms];
  double ca[kMaxTerms];
  double cb[kMaxTerms];
  int nu, amask, bmask;
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

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

template <int DIM, int N, int KIND>
struct Geo {
  static constexpr int NV = (KIND == 0) ? 1 : DIM + 1;
  static constexpr int L = (DIM == 1) ? 1 : (DIM == 2 ? N : N * N);  // lines per element per axis
  static constexpr int NPE = L * N;                                   // nodes per element
  static constexpr int LP = L * (N + 1);  // padded shared-memory stride of one element variable
  // element tile TX x TY x TZ (powers of two), ~128 line-owner threads
  static constexpr int TE = 1 << ilog2((128 / L) < 1 ? 1 : (128 / L));
  static constexpr int LG = ilog2(TE);
  static constexpr int LX = DIM == 1 ? LG : (DIM == 2 ? (LG + 1) / 2 : (LG + 2) / 3);
  static constexpr int LY = DIM == 1 ? 0 : (DIM == 2 ? LG - LX : (LG - LX + 1) / 2);
  static constexpr int LZ = LG - LX - LY;
  static constexpr int TX = 1 << LX, TY = 1 << LY, TZ = 1 << LZ;
  static constexpr int THREADS = TE * L;
  static constexpr int PAIR = (N % 2 == 0) ? 2 : 1;  // doubles per prepass load
  // halo faces per tile side along axis d = TE / T_d
  static constexpr int HF0 = TE / TX, HF1 = TE / TY, HF2 = TE / TZ;
  static constexpr int HOFF1 = 2 * HF0 * NV * L;
  static constexpr int HOFF2 = HOFF1 + (DIM > 1 ? 2 * HF1 * NV * L : 0);
  static constexpr int HSIZE = HOFF2 + (DIM > 2 ? 2 * HF2 * NV * L : 0);
  // shared memory carve-up (doubles)
  static constexpr int ARR = TE * NV * LP;
  static constexpr int OFF_U = 0;                           // U_s, later the partial dudt P
  static constexpr int OFF_F = OFF_U + ARR;                 // F_axis for axes 1..DIM-1
  static constexpr int OFF_T = OFF_F + (DIM - 1) * ARR;     // own U traces, axes 1..DIM-1
  static constexpr int OFF_H = OFF_T + (DIM - 1) * TE * 2 * (NV + 1) * L;  // halo U_s
  static constexpr int OFF_R = OFF_H + HSIZE;               // reduction scratch
  static constexpr int SMEM_BASE = (OFF_R + 32) * 8;
  static constexpr int SMEM_LAST = SMEM_BASE;
  // CTAs per SM allowed by shared memory (228 KB/SM, 1 KB reserved per CTA);
  // registers are capped so they never become the tighter limit
  static constexpr int CTAS_SMEM = 232448 / (SMEM_BASE + 1024);
  static constexpr int MINB = CTAS_SMEM < 1 ? 1 : (CTAS_SMEM > 8 ? 8 : CTAS_SMEM);

  // node index of position k along `axis` for transverse line index tr
  static __device__ __forceinline__ int node(int axis, int tr, int k) {
    if (axis == 0) return k + N * tr;
    if (axis == 1) return (tr % N) + N * (k + N * (tr / N));
    return tr + N * N * k;
  }
  // padded shared-memory slot of node n: x-lines padded to N+1 doubles, so
  // x-line owners (lane stride N+1) and y/z-line owners (unit stride) are
  // both bank-conflict free
  static __device__ __forceinline__ int sn(int n) { return n + n / N; }
  // AoS node order inside a cell (grid.hpp:50-56): i slowest
  static __device__ __forceinline__ int aos_node(int n) {
    const int i = n % N;
    if (DIM == 1) return i;
    const int j = (n / N) % N;
    if (DIM == 2) return i * N + j;
    return (i * N + j) * N + n / (N * N);
  }
  static __device__ __forceinline__ int halo_off(int axis) {
    return axis == 0 ? 0 : (axis == 1 ? HOFF1 : HOFF2);
  }
  static __device__ __forceinline__ int halo_faces(int axis) {
    return axis == 0 ? HF0 : (axis == 1 ? HF1 : HF2);
  }
};

// F_axis(u) and the one-sided wavespeed bound (models.cpp:42-70).
template <int DIM, int KIND, bool EXACT>
__device__ __forceinline__ void flux(const StageArgs& p, const double* u, int axis, double* f,
                                     double& speed) {
  using A = Ar<EXACT>;
  if (KIND == 0) {
    f[0] = A::mul(p.vel[axis], u[0]);
    speed = fabs(p.vel[axis]);
  } else {
    constexpr int NV = DIM + 1;
    const double rho = u[0];
    const double ua = A::div(u[1 + axis], rho);
    f[0] = u[1 + axis];
#pragma unroll
    for (int i = 1; i < NV; ++i) f[i] = A::mul(ua, u[i]);
    f[1 + axis] = A::add(f[1 + axis], A::mul(A::mul(rho, p.sound_speed), p.sound_speed));
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

template <int PAIR>
struct Vec;
template <>
struct Vec<1> {
  double x;
  // coherent loads: at the last stage one term may alias the output slot
  static __device__ __forceinline__ Vec ld(const double* p) { return Vec{*p}; }
};
template <>
struct Vec<2> {
  double x, y;
  static __device__ __forceinline__ Vec ld(const double* p) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    return Vec{v.x, v.y};
  }
};

// Tile geometry shared by the prepass and the line phases.
struct TileCtx {
  int x0, y0, z0;     // tile origin (cells)
  int vx, vy, vz;     // valid extent of the tile along each axis
};

// TMA bulk prefetch of [p, p+bytes) into L2 (sm_90+), 16-byte granular.
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  const size_t a0 = reinterpret_cast<size_t>(p) & ~size_t(15);
  const size_t a1 = (reinterpret_cast<size_t>(p) + bytes + 15) & ~size_t(15);
  size_t a = a0;
  while (a < a1) {
    const unsigned n = (unsigned)((a1 - a) > (size_t)(1u << 20) ? (1u << 20) : (a1 - a));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
    a += n;
  }
}

// Prefetch the input rows (u and the union terms) of tile `tile` into L2.
template <int DIM, int N, int KIND>
__device__ __forceinline__ void prefetch_tile(const StageArgs& p, int tile) {
  using G = Geo<DIM, N, KIND>;
  constexpr int NV = G::NV, NPE = G::NPE;
  const int C0 = p.cells[0], C1 = p.cells[1], C2 = p.cells[2];
  const int ntx = (C0 + G::TX - 1) / G::TX, nty = (C1 + G::TY - 1) / G::TY;
  const int x0 = (tile % ntx) * G::TX, y0 = ((tile / ntx) % nty) * G::TY, z0 = (tile / (ntx * nty)) * G::TZ;
  const int vx = min(G::TX, C0 - x0), vy = min(G::TY, C1 - y0), vz = min(G::TZ, C2 - z0);
  const size_t row_bytes = (size_t)vx * NV * NPE * sizeof(double);
  for (int r = 0; r < vy * vz; ++r) {
    const int y = y0 + r % vy, z = z0 + r / vy;
    const size_t off = ((size_t)x0 + (size_t)C0 * ((size_t)y + (size_t)C1 * z)) * NV * NPE;
    prefetch_l2(p.u + off, row_bytes);
    for (int t = 0; t < p.nu; ++t) prefetch_l2(p.ku[t] + off, row_bytes);
  }
}

// ------------------------------------------------------------ prepass
// Node-parallel, coalesced, all terms in flight: U_s = u + sum a_sj K_j for
// every node of the tile into padded shared memory, and at the last stage
// S = u + sum b_j K_j straight into the output array (read back by the
// epilogue from L2; the slot is never read by other CTAs in that stage).
// Then the out-of-tile neighbours' face planes into the halo.
// Full warps only (THREADS need not be a multiple of 32); each warp takes
// elements el = warp + NW*m (an element's NV*NPE doubles are contiguous in
// HBM), lanes take PAIR-sized chunks, and (element, chunk) work is flattened
// and batched so that ~8 double2 loads are in flight per lane.
template <int DIM, int N, int KIND, bool EXACT, int NU>
__device__ __forceinline__ void prepass(const StageArgs& p, const TileCtx& tc, double* smem) {
  using G = Geo<DIM, N, KIND>;
  using A = Ar<EXACT>;
  constexpr int NV = G::NV, NPE = G::NPE, LP = G::LP, TE = G::TE, PAIR = G::PAIR, L = G::L;
  constexpr int NW = G::THREADS / 32;      // full warps (>= 2 for every instantiation)
  constexpr int CH = NV * NPE / PAIR;      // chunks per element
  constexpr int CNT = (CH + 31) / 32;      // chunks per lane per element
  constexpr int EPW = (TE + NW - 1) / NW;  // elements per warp
  constexpr int J = EPW * CNT;             // work items per lane
  // the prepass runs before the register-heavy line phases: spend the
  // kernel's register allowance on loads in flight (4 registers per double2)
  constexpr int REGCAP = 65536 / (G::THREADS * G::MINB) > 255 ? 255 : 65536 / (G::THREADS * G::MINB);
  constexpr int BUDGET = (REGCAP - 48) / 4 < 2 ? 2 : (REGCAP - 48) / 4;
  constexpr int CB0 = BUDGET / (1 + NU) < 1 ? 1 : BUDGET / (1 + NU);
  constexpr int CB = CB0 < J ? CB0 : J;    // items per load batch
  static_assert(NW >= 1, "stage kernel needs at least one full warp");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= NW) return;  // the partial warp (if any) only joins the barriers
  const int C0 = p.cells[0], C1 = p.cells[1];
  double* sU = smem + G::OFF_U;
  const bool last = p.is_last;

#pragma unroll
  for (int j0 = 0; j0 < J; j0 += CB) {
    Vec<PAIR> uu[CB], kk[CB][NU > 0 ? NU : 1];
    size_t ga[CB];
    bool ok[CB];
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int j = j0 + b;
      const int el = warp + NW * (j / CNT), c = j % CNT;
      const int ex = el % G::TX, ey = (el / G::TX) % G::TY, ez = el / (G::TX * G::TY);
      ok[b] = j < J && el < TE && ex < tc.vx && ey < tc.vy && ez < tc.vz &&
              (CH % 32 == 0 || lane + 32 * c < CH);
      const size_t e = (size_t)(tc.x0 + ex) + (size_t)C0 * ((size_t)(tc.y0 + ey) + (size_t)C1 * (tc.z0 + ez));
      ga[b] = e * NV * NPE + (size_t)(lane + 32 * c) * PAIR;
      if (ok[b]) {
        uu[b] = Vec<PAIR>::ld(p.u + ga[b]);
#pragma unroll
        for (int t = 0; t < NU; ++t) kk[b][t] = Vec<PAIR>::ld(p.ku[t] + ga[b]);
      }
    }
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      if (!ok[b]) continue;
      const int j = j0 + b;
      const int el = warp + NW * (j / CNT), c = j % CNT;
      const int r = (lane + 32 * c) * PAIR;
      const int v = r / NPE, n = r - v * NPE;
      const int sa = (el * NV + v) * LP + G::sn(n);
      double U0 = uu[b].x, S0 = uu[b].x;
#pragma unroll
      for (int t = 0; t < NU; ++t) {
        if (p.amask >> t & 1) U0 = A::mac(U0, p.ca[t], kk[b][t].x);
        if (last && (p.bmask >> t & 1)) S0 = A::mac(S0, p.cb[t], kk[b][t].x);
      }
      sU[sa] = U0;
      if constexpr (PAIR == 2) {
        double U1 = uu[b].y, S1 = uu[b].y;
#pragma unroll
        for (int t = 0; t < NU; ++t) {
          if (p.amask >> t & 1) U1 = A::mac(U1, p.ca[t], kk[b][t].y);
          if (last && (p.bmask >> t & 1)) S1 = A::mac(S1, p.cb[t], kk[b][t].y);
        }
        sU[sa + 1] = U1;  // n and n+1 share an x-line (N even)
        if (last) *reinterpret_cast<double2*>(p.out + ga[b]) = make_double2(S0, S1);
      } else {
        if (last) p.out[ga[b]] = S0;
      }
    }
  }

  // halo: the face plane of each out-of-tile neighbour (always loaded, also
  // when the periodic wrap lands inside the tile -- the values are identical)
  constexpr int HV = NV * L;              // values per face plane
  constexpr int HC = (HV + 31) / 32;      // chunks per lane per face
  constexpr int NF0 = 2 * G::HF0, NF1 = DIM > 1 ? 2 * G::HF1 : 0, NF2 = DIM > 2 ? 2 * G::HF2 : 0;
  constexpr int NF = NF0 + NF1 + NF2;
  constexpr int FPW = (NF + NW - 1) / NW;
  constexpr int HJ = FPW * HC;
  constexpr int HB = CB0 < HJ ? CB0 : HJ;
  double* sH = smem + G::OFF_H;
#pragma unroll
  for (int j0 = 0; j0 < HJ; j0 += HB) {
    double hu[HB], hk[HB][NU > 0 ? NU : 1];
    int hd[HB];
    bool ok[HB];
#pragma unroll
    for (int b = 0; b < HB; ++b) {
      const int j = j0 + b;
      const int fq = warp + NW * (j / HC), cc = j % HC;
      const int q = lane + 32 * cc;  // q = v * L + t
      int axis, f2;
      if (fq < NF0) { axis = 0; f2 = fq; }
      else if (fq < NF0 + NF1) { axis = 1; f2 = fq - NF0; }
      else { axis = 2; f2 = fq - NF0 - NF1; }
      const int nf = axis == 0 ? G::HF0 : (axis == 1 ? G::HF1 : G::HF2);
      const int side = f2 / nf, f = f2 - side * nf;
      int ex, ey, ez;
      if (axis == 0) { ey = f % G::TY; ez = f / G::TY; ex = side ? tc.vx - 1 : 0; }
      else if (axis == 1) { ex = f % G::TX; ez = f / G::TX; ey = side ? tc.vy - 1 : 0; }
      else { ex = f % G::TX; ey = f / G::TX; ez = side ? tc.vz - 1 : 0; }
      ok[b] = j < HJ && fq < NF && ex < tc.vx && ey < tc.vy && ez < tc.vz && (HV % 32 == 0 || q < HV);
      int cc3[3] = {tc.x0 + ex, tc.y0 + ey, tc.z0 + ez};
      const int cn = p.cells[axis];
      cc3[axis] = side ? (cc3[axis] + 1 == cn ? 0 : cc3[axis] + 1) : (cc3[axis] == 0 ? cn - 1 : cc3[axis] - 1);
      const size_t gb = ((size_t)cc3[0] + (size_t)C0 * ((size_t)cc3[1] + (size_t)C1 * cc3[2])) * NV * NPE;
      const int v = q / L, t = q - v * L;
      const size_t g = gb + (size_t)v * NPE + G::node(axis, t, side ? 0 : N - 1);
      hd[b] = G::halo_off(axis) + (side * nf + f) * HV + q;
      if (ok[b]) {
        hu[b] = __ldg(p.u + g);
#pragma unroll
        for (int tt = 0; tt < NU; ++tt) hk[b][tt] = __ldg(p.ku[tt] + g);
      }
    }
#pragma unroll
    for (int b = 0; b < HB; ++b) {
      if (!ok[b]) continue;
      double U0 = hu[b];
#pragma unroll
      for (int tt = 0; tt < NU; ++tt)
        if (p.amask >> tt & 1) U0 = A::mac(U0, p.ca[tt], hk[b][tt]);
      sH[hd[b]] = U0;
    }
  }
}

// ============================================================ stage kernel
template <int DIM, int N, int KIND, bool EXACT>
__global__ void __launch_bounds__(Geo<DIM, N, KIND>::THREADS, Geo<DIM, N, KIND>::MINB)
stage_kernel(const __grid_constant__ StageArgs p) {
  using G = Geo<DIM, N, KIND>;
  using A = Ar<EXACT>;
  constexpr int NV = G::NV, L = G::L, NPE = G::NPE, LP = G::LP, TE = G::TE;
  constexpr int NT = NV + 1;  // trace slots per face node: U (NV) + one-sided wavespeed
  extern __shared__ double smem[];

  Control* ctl = p.ctl;
  // inactive step, or an earlier stage already failed: keep the inputs of the
  // failing stage intact for the host's error report
  if (!p.rhs_only && (*(volatile int*)&ctl->skip ||
                      *(volatile unsigned long long*)&ctl->err_key != kNoError))
    return;

  const int C0 = p.cells[0], C1 = p.cells[1], C2 = p.cells[2];
  const int ntx = (C0 + G::TX - 1) / G::TX, nty = (C1 + G::TY - 1) / G::TY;
  const int ntiles = ntx * nty * ((C2 + G::TZ - 1) / G::TZ);
  const double dt = p.rhs_only ? 1.0 : ctl->dt;
  const long long step = p.rhs_only ? 0 : ctl->steps;
  double alpha = 0.0;  // running max wavespeed of this CTA (last stage)
  if (threadIdx.x == 0 && blockIdx.x < ntiles) prefetch_tile<DIM, N, KIND>(p, blockIdx.x);

  // persistent CTAs: tiles bid, bid + grid, ...; the next tile's inputs are
  // prefetched into L2 by TMA while this one computes
  for (int bid = blockIdx.x; bid < ntiles; bid += gridDim.x) {
  if (threadIdx.x == 0 && bid + (int)gridDim.x < ntiles) prefetch_tile<DIM, N, KIND>(p, bid + gridDim.x);
  TileCtx tc;
  tc.x0 = (bid % ntx) * G::TX;
  tc.y0 = ((bid / ntx) % nty) * G::TY;
  tc.z0 = (bid / (ntx * nty)) * G::TZ;
  tc.vx = min(G::TX, C0 - tc.x0);
  tc.vy = min(G::TY, C1 - tc.y0);
  tc.vz = min(G::TZ, C2 - tc.z0);

  const int tid = threadIdx.x;
  const int el = tid / L;
  const int tr = tid - el * L;  // transverse line index (same count for every axis)
  const int ex = el % G::TX, ey = (el / G::TX) % G::TY, ez = el / (G::TX * G::TY);
  const bool valid = ex < tc.vx && ey < tc.vy && ez < tc.vz;
  const int cx = tc.x0 + ex, cy = tc.y0 + ey, cz = tc.z0 + ez;
  const size_t e = (size_t)cx + (size_t)C0 * ((size_t)cy + (size_t)C1 * cz);
  const size_t ebase = e * NV * NPE;
  const int tj = DIM > 1 ? tr % N : 0, tk = DIM > 2 ? tr / N : 0;  // x-line's (j, k)

  double* sU = smem + G::OFF_U;  // [TE][NV][LP]  U_s, then P
  double* sF = smem + G::OFF_F;  // [DIM-1][TE][NV][LP]
  double* sT = smem + G::OFF_T;  // [DIM-1][TE][2][NT][L]
  double* sH = smem + G::OFF_H;  // halo

  // padded shared slot of the node at position k along `axis` of line tr:
  // sbase(axis) + k * sstride(axis)
  auto sbase = [&](int axis) -> int {
    if (axis == 0) return tr * (N + 1);
    if (axis == 1) return tj /*= i0*/ + (N + 1) * N * tk;
    return tj + (N + 1) * tk;  // axis 2: tr = i0 + N*i1
  };
  auto sstride = [](int axis) -> int { return axis == 0 ? 1 : (axis == 1 ? N + 1 : (N + 1) * N); };
  auto gbase = [&](int axis) -> int {  // node index of k = 0
    if (axis == 0) return tr * N;
    if (axis == 1) return tj + N * N * tk;
    return tr;
  };
  auto gstride = [](int axis) -> int { return axis == 0 ? 1 : (axis == 1 ? N : N * N); };
  auto trc = [&](int axis, int elx, int side, int v, int t) -> double& {  // axis >= 1
    return sT[((((axis - 1) * TE + elx) * 2 + side) * NT + v) * L + t];
  };
  auto halo = [&](int axis, int side, int f, int v, int t) -> double {
    return sH[G::halo_off(axis) + ((side * G::halo_faces(axis) + f) * NV + v) * L + t];
  };
  auto aos_cell = [&](int x, int y, int z) -> long long {  // global AoS cell index
    const long long gx = x + p.goff[0], gy = y + p.goff[1], gz = z + p.goff[2];
    return (gx * p.gcells[1] + gy) * (long long)p.gcells[2] + gz;
  };

  // ---------------------------------------------------------------- prepass
  switch (p.nu) {
    case 0: prepass<DIM, N, KIND, EXACT, 0>(p, tc, smem); break;
    case 1: prepass<DIM, N, KIND, EXACT, 1>(p, tc, smem); break;
    case 2: prepass<DIM, N, KIND, EXACT, 2>(p, tc, smem); break;
    case 3: prepass<DIM, N, KIND, EXACT, 3>(p, tc, smem); break;
    case 4: prepass<DIM, N, KIND, EXACT, 4>(p, tc, smem); break;
    case 5: prepass<DIM, N, KIND, EXACT, 5>(p, tc, smem); break;
    default: prepass<DIM, N, KIND, EXACT, 6>(p, tc, smem); break;
  }
  __syncthreads();

  // ---------------------------------------------------------------- phase X
  double D[NV][N];
  const int xl = el * NV * LP + sbase(0);  // this x-line in sU / sF / sS
  if (valid) {
    double U[NV][N];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int i = 0; i < N; ++i) U[v][i] = sU[xl + v * LP + i];
    // fluxes at every node of the line, every axis
    double FX[NV][N];
    double s_lo = 0.0, s_hi = 0.0;
    const bool yb = DIM > 1 && (tj == 0 || tj == N - 1);
    const bool zb = DIM > 2 && (tk == 0 || tk == N - 1);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double un[NV], f[NV], sp;
      if (KIND == 1 && !(U[0][i] > 0.0)) {
        // first bad node of the reference's x-volume traversal: (cell, (j,k), i)
        const int nkey = (DIM == 1) ? i : (DIM == 2 ? tj * N + i : (tj * N + tk) * N + i);
        record_error(ctl, error_key(step, p.phase, aos_cell(cx, cy, cz), nkey));
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) un[v] = U[v][i];
      flux<DIM, KIND, EXACT>(p, un, 0, f, sp);
#pragma unroll
      for (int v = 0; v < NV; ++v) FX[v][i] = f[v];
      if (i == 0) s_lo = sp;
      if (i == N - 1) s_hi = sp;
#pragma unroll
      for (int d = 1; d < DIM; ++d) {
        flux<DIM, KIND, EXACT>(p, un, d, f, sp);
#pragma unroll
        for (int v = 0; v < NV; ++v) sF[(d - 1) * G::ARR + xl + v * LP + i] = f[v];
        // own face traces (state + one-sided speed) for the y/z phases
        if (d == 1 && yb) {
#pragma unroll
          for (int v = 0; v < NV; ++v) trc(1, el, tj == 0 ? 0 : 1, v, i + N * tk) = un[v];
          trc(1, el, tj == 0 ? 0 : 1, NV, i + N * tk) = sp;
        }
        if (d == 2 && zb) {
#pragma unroll
          for (int v = 0; v < NV; ++v) trc(2, el, tk == 0 ? 0 : 1, v, i + N * tj) = un[v];
          trc(2, el, tk == 0 ? 0 : 1, NV, i + N * tj) = sp;
        }
      }
    }
    // x faces (solver.cpp:268-306): face at i=0 (we are its + side) and at
    // i=N-1 (we are its - side); the minus state is always the lower cell.
    // The fluxes are formed first so U can retire before the volume term.
    double fh_lo[NV], fh_hi[NV];
    {
      double nb_lo[NV], nb_hi[NV];
      const int fx = ey + G::TY * ez;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        nb_lo[v] = ex > 0 ? sU[xl - NV * LP + v * LP + (N - 1)] : halo(0, 0, fx, v, tr);
        nb_hi[v] = ex < tc.vx - 1 ? sU[xl + NV * LP + v * LP] : halo(0, 1, fx, v, tr);
      }
      double fo[NV], fn[NV], sn, uo[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) { fo[v] = FX[v][0]; uo[v] = U[v][0]; }
      flux<DIM, KIND, EXACT>(p, nb_lo, 0, fn, sn);
      lax_friedrichs<NV, EXACT>(nb_lo, uo, fn, fo, sn, s_lo, fh_lo);
#pragma unroll
      for (int v = 0; v < NV; ++v) { fo[v] = FX[v][N - 1]; uo[v] = U[v][N - 1]; }
      flux<DIM, KIND, EXACT>(p, nb_hi, 0, fn, sn);
      lax_friedrichs<NV, EXACT>(uo, nb_hi, fo, fn, s_hi, sn, fh_hi);
    }
    // volume x: out(=0) += sum_l K[k][l] F_l (solver.cpp:246-256), then the
    // lifted face fluxes: out += lift F^ at i=0, out -= lift F^ at i=N-1
    const double lift = p.lift[0];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) acc = A::mac(acc, p.K[0][k * N + l], FX[v][l]);
        D[v][k] = zero_plus(acc);
      }
      D[v][0] = A::add(D[v][0], A::mul(lift, fh_lo[v]));
      D[v][N - 1] = A::sub(D[v][N - 1], A::mul(lift, fh_hi[v]));
    }
  }
  if (DIM > 1) {
    __syncthreads();  // every x-face read of sU is done: sU becomes P
    if (valid) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int i = 0; i < N; ++i) sU[xl + v * LP + i] = D[v][i];
    }
  }

  // -------------------------------------------------------- phases Y and Z
#pragma unroll
  for (int axis = 1; axis < DIM; ++axis) {
    __syncthreads();
    if (valid) {
      const int ab = el * NV * LP + sbase(axis);
      const int as = sstride(axis);
      const double* Fa = sF + (axis - 1) * G::ARR + ab;
      // faces along this axis first (own traces; neighbours from the tile or
      // the halo), so that only one variable's flux line is live at a time
      const int ea = axis == 1 ? ey : ez;
      const int va = axis == 1 ? tc.vy : tc.vz;
      const int step_el = axis == 1 ? G::TX : G::TX * G::TY;
      const int fidx = axis == 1 ? ex + G::TX * ez : ex + G::TX * ey;
      double fh_lo[NV], fh_hi[NV];
      {
        double a_lo[NV], a_hi[NV], nb_lo[NV], nb_hi[NV], fo[NV], fn[NV], sn;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          a_lo[v] = trc(axis, el, 0, v, tr);
          a_hi[v] = trc(axis, el, 1, v, tr);
          nb_lo[v] = ea > 0 ? trc(axis, el - step_el, 1, v, tr) : halo(axis, 0, fidx, v, tr);
          nb_hi[v] = ea < va - 1 ? trc(axis, el + step_el, 0, v, tr) : halo(axis, 1, fidx, v, tr);
        }
        const double so_lo = trc(axis, el, 0, NV, tr), so_hi = trc(axis, el, 1, NV, tr);
        flux<DIM, KIND, EXACT>(p, nb_lo, axis, fn, sn);
#pragma unroll
        for (int v = 0; v < NV; ++v) fo[v] = Fa[v * LP];
        lax_friedrichs<NV, EXACT>(nb_lo, a_lo, fn, fo, sn, so_lo, fh_lo);
        flux<DIM, KIND, EXACT>(p, nb_hi, axis, fn, sn);
#pragma unroll
        for (int v = 0; v < NV; ++v) fo[v] = Fa[v * LP + (N - 1) * as];
        lax_friedrichs<NV, EXACT>(a_hi, nb_hi, fo, fn, so_hi, sn, fh_hi);
      }
      // volume: partial + sum_l K[k][l] F_l, then the lifted face fluxes
      const double lift = p.lift[axis];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double F[N];
#pragma unroll
        for (int k = 0; k < N; ++k) F[k] = Fa[v * LP + k * as];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = A::mac(acc, p.K[axis][k * N + l], F[l]);
          D[v][k] = A::add(sU[ab + v * LP + k * as], acc);
        }
        D[v][0] = A::add(D[v][0], A::mul(lift, fh_lo[v]));
        D[v][N - 1] = A::sub(D[v][N - 1], A::mul(lift, fh_hi[v]));
      }
      if (axis < DIM - 1) {
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int k = 0; k < N; ++k) sU[ab + v * LP + k * as] = D[v][k];
      }
    }
  }

  // ------------------------------------------------------------ epilogue
  constexpr int FA = DIM - 1;  // axis of the final owner
  if (valid) {
    double* gout = p.out + ebase + gbase(FA);
    const int gs = gstride(FA);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double kv[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) kv[v] = A::mul(D[v][k], dt);  // k_i *= dt (solver.hpp:66-67)
      if (!p.is_last) {
#pragma unroll
        for (int v = 0; v < NV; ++v) gout[v * NPE + k * gs] = kv[v];
      } else {
        double un[NV];
        bool finite = true;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          // S was stored into this slot by the prepass of this CTA (a plain load, not __ldg)
          un[v] = A::mac(gout[v * NPE + k * gs], p.b_last, kv[v]);  // u += b_i k_i (solver.hpp:69-75)
          gout[v * NPE + k * gs] = un[v];
          finite = finite && isfinite(un[v]);
        }
        if (!finite) record_error(ctl, error_key(step, kPhaseInstability, 0, 0));
        if (KIND == 1 && p.scan_alpha) {
          // the next step's max_wavespeed_bound (solver.cpp:323-332), fused
          if (!(un[0] > 0.0)) {
            record_error(ctl, error_key(step + 1, kPhaseScan, aos_cell(cx, cy, cz),
                                        G::aos_node(gbase(FA) + k * gs)));
          } else {
            double m = 0.0;
#pragma unroll
            for (int d = 0; d < DIM; ++d) m = dmax(m, fabs(un[1 + d]));
            alpha = dmax(alpha, A::add(A::div(m, un[0]), p.sound_speed));
          }
        }
      }
    }
  }
  __syncthreads();  // shared memory is reused by the next tile
  }  // tile loop

  if (KIND == 1 && p.is_last && p.scan_alpha) {
    double* sR = smem + G::OFF_R;
    // block max of the non-negative wavespeeds on their IEEE bit patterns
    // (valid for partial warps), then one global atomic per CTA
    unsigned long long* red = reinterpret_cast<unsigned long long*>(sR);
    __syncthreads();
    if (threadIdx.x == 0) red[0] = 0ull;
    __syncthreads();
    atomicMax(red, (unsigned long long)__double_as_longlong(alpha));
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&ctl->alpha_bits, red[0]);
  }
}

// ============================================================ alpha scan
// max_wavespeed_bound over a device-layout state (solver.cpp:310-334).
template <int DIM>
__global__ void alpha_scan_kernel(const double* __restrict__ u, int c0, int c1, int c2, int order,
                                  double a, Control* ctl, long long step_for_error) {
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
                                  ((long long)cx * c1 + cy) * c2 + cz, an));
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
  if (c->err_key != kNoError || c->done) {
    c->skip = 1;
    return;
  }
  const bool fixed = sp.fixed_steps >= 0;
  if ((fixed && c->steps >= sp.fixed_steps) || (!fixed && !(c->t < sp.t_end))) {
    c->done = 1;
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

}  // namespace ndgx
