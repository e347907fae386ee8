// ndgx_stage.cuh -- the fused NDG right-hand side + RK stage kernel (sm_100a).
//
// Reference semantics (paths relative to /root/reference/proj):
//   stage input      include/ndg/solver.hpp:52-63   U_s = u + sum_j a_sj K_j (j order, a_sj != 0)
//   volume term      src/solver.cpp:229-262         out += sum_l K_d[k][l] F_d(U_l), per axis
//   face term        src/solver.cpp:264-306         out -/+= lift_d * LF(U-, U+)
//   flux / speed     src/models.cpp:42-88
//   RK epilogue      include/ndg/solver.hpp:64-75   K_s = dt*dudt; u += b_j K_j (j order)
//   CFL alpha        src/solver.cpp:310-334         fused into the last stage's epilogue
//   finite check     src/solver.cpp:361-368
//
// Execution model: a persistent grid of warps, no CTA barriers during the
// element work (__syncwarp only).  By default one element per warp; elements
// are walked x fastest so neighbouring warps work on neighbouring elements
// and face-neighbour reads hit L2.  Per element, warp-locally:
//   1  node phase: each lane forms the stage input U_s = u + sum a K at its
//      nodes straight from HBM (all of a lane's loads in flight together);
//   2  face phase: the Lax-Friedrichs flux at every face node, the
//      neighbour's stage input from HBM (or the received multi-block plane);
//   3  output phase: the volume quadrature, the lifted face fluxes and the
//      RK epilogue (K_s = dt*dudt, or u_new = S + b_s K_s, finite check,
//      next-step wavespeed), stored straight to HBM.
// HBM traffic is the compulsory one array pass per input and output.
//
// Bodies:
//   2D N=8, FAST (the flagship, element_2d8_fast): FP64 tensor cores,
//             mma.sync.m8n8k4.f64 -- lane = 4r + c evaluates fluxes at nodes
//             (i = 2c + h, j = r), exactly its B fragments of D_x = K_x F_x; one
//             warp-local transpose gives the A fragments of D_y = F_y K_y^T.
//             Runs of 2 x-adjacent elements per warp (u-only and last stages)
//             take the x-lo neighbour from the previous element's slab.
//             2D Euler N = 5..7 and advection N = 7 run it zero-padded to the
//             8 x 8 grid (NDGX_MMA2_ORDERS[_ADV]).
//   3D N=4, FAST (element_3d4_lines): lanes own whole x / y / z lines of a
//             swizzled U slab (conflict-free along every axis); z-runs per
//             warp carry the z-hi face flux to the next element.
//   generic (every other shape, and EXACT everywhere): the reference's loop
//             structure; EXACT in its operation order with _rn intrinsics
//             (bit-identical), FAST with contracted FMAs.  Small elements run
//             G::EPW to a warp (G::GL lanes each); 2D orders 6-8 (and 3D 6-8)
//             sum the volume by whole-line tasks, the 2D order-8 exact body
//             by half-line tasks.
#pragma once

namespace ndgx {

// Stage signatures (kSigs index) that take the 3D order-4 tensor-core body:
// all of them since the per-signature register caps (stage_minb) let the
// many-term RK6 stages keep their face loads in flight (C4, 128^3: the 2..5
// term stages 6.75 / 7.55 / 8.24 / 9.31 ms vs 8.51 / 9.14 / 9.87 / 11.53 ms in
// the generic body).
#ifndef NDGX_LINEG
#define NDGX_LINEG 1  // generic 2D bodies: volume sums by whole-line tasks
#endif
#ifndef NDGX_LINE8
#define NDGX_LINE8 1  // 2D order-8 exact body: volume sums by line tasks
#endif
#ifndef NDGX_GPF
#define NDGX_GPF 1  // generic body: all of a lane's node loads issued before any combination
#endif
#ifndef NDGX_DT2
#define NDGX_DT2 1  // flagship Euler, stages without b-terms: transposed volume product (outputs at own node pair)
#endif
#ifndef NDGX_DT2_LAST
#define NDGX_DT2_LAST 0  // (tuning) the transposed product in the last stages too
#endif
#ifndef NDGX_YTR2
#define NDGX_YTR2 1  // flagship: y-face traces as one 16-byte store per variable
#endif
#ifndef NDGX_GEN_UTRACE
#define NDGX_GEN_UTRACE 1  // generic body: face traces hold U only (flux and speed recomputed at the face)
#endif
#ifndef NDGX_LINES3
#define NDGX_LINES3 1  // 3D order-4 contracted stages: line-task body (1) or the tensor-core body (0)
#endif
#ifndef NDGX_MMA3_SIGS
#define NDGX_MMA3_SIGS 0x1FF
#endif
// bit N: the contracted 2D order-N (N < 8) stages run the flagship body
// zero-padded to 8 x 8 nodes.  Measured at 1e8 DOF against the generic body
// (profiles/r02/padded_mma_orders.jsonl): Euler o5 / o6 / o7 7.6 / 8.5 /
// 7.1e10 -> 8.1e10 / 1.19e11 / 1.40e11; advection o7 6.0e10 -> 1.30e11,
// o5 even, o6 1.02e11 -> 8.1e10 (its 4-lane groups win there)
#ifndef NDGX_MMA2_ORDERS
#define NDGX_MMA2_ORDERS 0x0E0  // Euler
#endif
#ifndef NDGX_MMA2_ORDERS_ADV
#define NDGX_MMA2_ORDERS_ADV 0x080  // advection
#endif

template <int DIM, int N, int KIND>
struct Geo {
  static constexpr int NV = (KIND == 0) ? 1 : DIM + 1;
  static constexpr int L = (DIM == 1) ? 1 : (DIM == 2 ? N : N * N);  // lines per element per axis
  static constexpr int NPE = L * N;                                   // nodes per element
  static constexpr int NM = (NPE + 31) / 32;                          // nodes per lane
  static constexpr int FACES = 2 * DIM;
  static constexpr int FN = FACES * L;                                // face nodes per element
  static constexpr int FM = (FN + 31) / 32;                           // face nodes per lane
  static constexpr int HW = 2 * NV + 1;                               // trace: U[NV], F[NV], speed
  static constexpr int TW = NDGX_GEN_UTRACE ? NV : HW;                // generic trace record width (U only)
  // shared memory: [mbarriers WARPS*MAXD][scratch RED] then per warp a slab
  // (doubles): fluxes [DIM][NV][NPE] | traces [face][HW][L] | face fluxes
  // [face][NV][L], followed by the warp's ring of D element slots, each
  // holding u and the NU K_j of one element ([array][var][node], TMA-filled)
  static constexpr int OFF_T = DIM * NV * NPE;
  static constexpr int OFF_H = OFF_T + FACES * TW * L;
  static constexpr int WSLAB = ((OFF_H + FACES * NV * L) + 1) & ~1;
  // warps per CTA: 4, fewer where four generic slabs exceed ~190 KB (3D
  // order 7: 3 warps, order 8: 2 -- one element is 63 / 89 KB of slab)
  static constexpr int WARPS = WSLAB * 4 <= 24000 ? 4 : (24000 / WSLAB < 1 ? 1 : 24000 / WSLAB);
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int MAXD = 4;                                      // max ring depth per warp
  static constexpr int RED = 2 * WARPS;                      // block reduction scratch (doubles)
  // the generic body's operator rows K_d[k][.] in shared memory, rows padded
  // to N + 1 doubles: lanes reading different rows k hit different banks (a
  // per-lane index into the kernel parameters serialises in the constant cache)
  static constexpr int KROW = N + 1;
  static constexpr int KSM = ((DIM * N * KROW) + 1) & ~1;
  static constexpr int HEAD = WARPS * MAXD + RED + KSM;      // 8-byte words before the slabs
  static constexpr int CHUNK = NV * NPE;                     // one array of one element (doubles)
  // generic body: lanes per element (GL) and elements per warp (EPW).  Small
  // elements share a warp so the node and face passes keep the lanes busy:
  // 2D o4 / o5 / o6 8 lanes (2 / 4 / 5 node passes, 2 / 3 / 3 face passes),
  // 2D o6 advection and o2 / o3 4 lanes, 1D 4-8 lanes, 3D o2 8 lanes.
  // Measured at 1e8 DOF (profiles/r02/order_sweep_*.jsonl): 2D Euler o4 16
  // lanes 9.4e10, 8 lanes 1.03e11; 2D advection o6 8 lanes 6.5e10, 4 lanes 9.2e10.
  static constexpr int group_lanes() {
    return DIM == 1 ? (N <= 4 ? 4 : 8)
                    : (DIM == 2 ? (N <= 3 || (N == 6 && KIND == 0) ? 4 : (N <= 6 ? 8 : 32)) : (N == 2 ? 8 : 32));
  }
#ifdef NDGX_GL
  static constexpr int GL = NDGX_GL;  // tuning builds of one instance
#else
  static constexpr int GL = group_lanes();
#endif
  static constexpr int EPW = 32 / GL;
  // per-group slab stride: WSLAB padded so that the EPW groups' slabs start
  // 16/EPW doubles apart modulo the 32 banks (with equal alignment every
  // group hit the same banks: 2D o4 had 40 of 78 shared wavefronts excessive)
#ifndef NDGX_GPAD
#define NDGX_GPAD 1
#endif
  static constexpr int GSTRIDE =
      (EPW == 1 || NDGX_GPAD == 0) ? WSLAB : WSLAB + ((16 / EPW) - (WSLAB % 16) + 16) % 16;
  // (measured, profiles/r02/loworder_pad_ab.jsonl: 2D Euler o2 9.4e10 -> 1.03e11, o4 1.05e11 -> 1.19e11,
  //  o5 +3%; with U-only trace records 3D o2 Euler needs it too: its slab became a multiple of 16)
  static constexpr int NMG = (NPE + GL - 1) / GL;            // node passes of a lane
  static constexpr int FMG = (FN + GL - 1) / GL;             // face passes of a lane
  static constexpr bool TMA_OK = (CHUNK % 2) == 0 && GL == 32;  // 16-byte element chunks, one element per warp
#ifdef NDGX_NO_MMA  // A/B builds: the contracted generic (scalar DFMA) body instead of the tensor-core bodies
  static constexpr bool MMA = false, MMA3 = false;
#else
  // FAST-mode tensor-core volume (2D): order 8, and the orders in
  // NDGX_MMA2_ORDERS zero-padded to the 8 x 8 node grid of the same body
  static constexpr bool MMA =
      (DIM == 2 && (N == 8 || (N >= 5 && (((KIND == 1 ? NDGX_MMA2_ORDERS : NDGX_MMA2_ORDERS_ADV) >> N) & 1) != 0)));
  static constexpr bool MMA3 = (DIM == 3 && N == 4);         // FAST-mode tensor-core volume (3D)
#endif
  // one face node per lane: the ring slot also carries the element's face
  // neighbour values ([array][var][lane], cp.async), so no load is on demand
  static constexpr bool FACE_PF = (FM == 1);
  static constexpr int SLOT1 = CHUNK + (FACE_PF ? 32 * NV : 0);  // ring doubles per input array
  // tensor-core bodies: 2D stages only F_y (F_x stays in registers as MMA
  // fragments); 3D stages F_x, F_y, F_z (F_x becomes the accumulator) and
  // keeps face traces of U and speed only.  Both add S at the last stage.
  static constexpr __host__ __device__ int wslab(bool mma, bool last) {
    return mma ? (MMA3 ? (NDGX_LINES3 ? (4 + (last ? 1 : 0)) * NV * NPE  // line body: U | three dudt parts | S
                                      : (((3 + (last ? 1 : 0)) * NV * NPE + FACES * (NV + 1) * L + FACES * NV * L + 1) & ~1))
                       : (((1 + (last ? 1 : 0)) * NV * 64 + FACES * HW * 8 + FACES * NV * 8 + 1) & ~1))
               : EPW * GSTRIDE;
  }
  // which body a (arith, signature) kernel runs: the 2D N=8 / 3D N=4
  // tensor-core bodies (contracted mode; 3D for the NDGX_MMA3_SIGS stages)
  static constexpr __host__ __device__ bool mma_body(bool exact, int sig) {
    return !exact && (MMA || (MMA3 && ((NDGX_MMA3_SIGS >> sig) & 1) != 0));
  }
  static constexpr int smem_bytes(int nu, int depth, bool mma, bool last) {
    return (HEAD + WARPS * (wslab(mma, last) + depth * (1 + nu) * SLOT1)) * 8;
  }

  // node index of position k along `axis` on transverse line t
  static __device__ __forceinline__ int node(int axis, int t, int k) {
    if (axis == 0) return k + N * t;
    if (axis == 1) return (t % N) + N * (k + N * (t / N));
    return t + N * N * k;
  }
  // position along `axis` and transverse line index of node n
  static __device__ __forceinline__ int pos_of(int axis, int n) {
    if (axis == 0) return n % N;
    if (axis == 1) return (n / N) % N;
    return n / (N * N);
  }
  static __device__ __forceinline__ int line_of(int axis, int n) {
    if (axis == 0) return n / N;
    if (axis == 1) return (n % N) + N * (n / (N * N));
    return n % (N * N);
  }
  // AoS node order inside a cell (grid.hpp:50-56): i slowest
  static __device__ __forceinline__ int aos_node(int n) {
    const int i = n % N;
    if (DIM == 1) return i;
    const int j = (n / N) % N;
    if (DIM == 2) return i * N + j;
    return (i * N + j) * N + n / (N * N);
  }
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* q) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(q));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
// the one arrival of a TMA-filled barrier, registering the bytes the copies complete
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(b)),
               "r"(bytes)
               : "memory");
}
// Wait for the phase of parity `parity`.  A watchdog turns a lost completion
// into a trapped kernel (a CUDA error) instead of a hung device.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  uint32_t polls = 0;
  long long t0 = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (!done && (++polls & 4095u) == 0) {
      if (t0 == 0) {
        t0 = clock64();
      } else if (clock64() - t0 > (1ll << 31)) {
        printf("ndgx watchdog: block %d thread %d stuck on mbarrier %u (parity %u)\n", (int)blockIdx.x,
               (int)threadIdx.x, smem_u32(b), parity);
        __trap();
      }
    }
  } while (!done);
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 1/x to ~1 ulp for the contracted mode: the MUFU 64-bit reciprocal seed plus
// two Newton steps (an IEEE division costs several times more).  Non-positive
// x only occurs in a failing run (PhysicsError), where any value will do.
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(PENDING) : "memory");
}

// D(8x8) += A(8x4, row) * B(4x8, col) in FP64 on the tensor cores
__device__ __forceinline__ void dmma_8x8x4(double a, double b, double& c0, double& c1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// U_s = u + sum_{t in amask} ca[t] ku[t] and (when `with_s`) S = u +
// sum_{t in bmask} cb[t] ku[t], each in the reference's term order.
template <bool EXACT, int NU, int AM, int BM>
__device__ __forceinline__ void combine_g(const StageArgs& p, size_t g, bool with_s, double& U, double& S) {
  using A = Ar<EXACT>;
  // issue every load first so they are all in flight together
  double k[NU > 0 ? NU : 1];
#pragma unroll
  for (int t = 0; t < NU; ++t) k[t] = __ldg(p.ku[t] + g);
  const double u = __ldg(p.u + g);
  U = u;
#pragma unroll
  for (int t = 0; t < NU; ++t)
    if ((AM >> t & 1) != 0) U = A::mac(U, p.ca[t], k[t]);
  S = u;
  if (with_s) {
#pragma unroll
    for (int t = 0; t < NU; ++t)
      if ((BM >> t & 1) != 0) S = A::mac(S, p.cb[t], k[t]);
  }
}

// The same combination from an element slot in shared memory: array a at
// src[a * stride] (0 = u, 1 + t = ku[t]).
template <bool EXACT, int NU, int AM, int BM>
__device__ __forceinline__ void combine_s(const StageArgs& p, const double* src, int stride, bool with_s, double& U,
                                          double& S) {
  using A = Ar<EXACT>;
  const double u = src[0];
  U = u;
#pragma unroll
  for (int t = 0; t < NU; ++t)
    if ((AM >> t & 1) != 0) U = A::mac(U, p.ca[t], src[(1 + t) * stride]);
  S = u;
  if (with_s) {
#pragma unroll
    for (int t = 0; t < NU; ++t)
      if ((BM >> t & 1) != 0) S = A::mac(S, p.cb[t], src[(1 + t) * stride]);
  }
}

// U_s at two adjacent nodes (16-byte aligned) of one variable, from the ring
// slot (`ring`) or HBM: one 16-byte load per input array.
template <int NU, int AM, int BM = 0>
__device__ __forceinline__ void combine_pair(const StageArgs& p, bool ring, const double* s, size_t g, int stride,
                                             double& U0, double& U1, double* S0 = nullptr, double* S1 = nullptr) {
  double2 k[NU > 0 ? NU : 1];
  double2 u;
  if (ring) {
    u = *reinterpret_cast<const double2*>(s);
#pragma unroll
    for (int t = 0; t < NU; ++t) k[t] = *reinterpret_cast<const double2*>(s + (1 + t) * stride);
  } else {
    u = __ldg(reinterpret_cast<const double2*>(p.u + g));
#pragma unroll
    for (int t = 0; t < NU; ++t) k[t] = __ldg(reinterpret_cast<const double2*>(p.ku[t] + g));
  }
  U0 = u.x;
  U1 = u.y;
#pragma unroll
  for (int t = 0; t < NU; ++t)
    if ((AM >> t & 1) != 0) {
      U0 = fma(p.ca[t], k[t].x, U0);
      U1 = fma(p.ca[t], k[t].y, U1);
    }
  if (S0 != nullptr) {  // last stage: S = u + sum b_j K_j from the same loads
    double a = u.x, b = u.y;
#pragma unroll
    for (int t = 0; t < NU; ++t)
      if ((BM >> t & 1) != 0) {
        a = fma(p.cb[t], k[t].x, a);
        b = fma(p.cb[t], k[t].y, b);
      }
    *S0 = a;
    *S1 = b;
  }
}

// ------------------------------------------------------------ 3D order-4 body
// One element of the 3D, N = 4, contracted-arithmetic stage (the C4 shape).
// Per axis d the volume term is D_d[k][line] = sum_l K_d[k][l] F_d[l][line]
// over the 16 lines of the axis, two m8n8k4 MMAs (lines 0-7, 8-15; rows
// 4-7 of A are zero), with the running sum over axes carried through the
// MMA accumulator input from shared memory (F_x's slots hold it).
struct Lane4 {
  double k[3];  // K_d[r][c] (0 for r >= 4)
};

// Runs (RA = 0: x, 2: z; -1: none): a warp visiting consecutive elements
// along axis RA reuses the previous element's hi-face flux as this
// element's lo-face flux (`prev`): the two face-flux slots of that axis
// alternate with `par`, so the hi slot of one element is the lo slot of the
// next.  Bitwise the same value: LF(U-, U+) of the same two stage inputs.
template <int KIND, int NU, int AM, int BM, int RA = -1>
__device__ __forceinline__ void element_3d4_fast(const StageArgs& p, const Lane4& ln, int lane, int e, int cx,
                                                 int cy, int cz, double* sF, double* sT, double* sH, double dt,
                                                 long long step, double& alpha, bool prev = false, int par = 0) {
  constexpr int N = 4, NPE = 64, L = 16, DIM = 3;
  constexpr int NV = KIND == 0 ? 1 : 4;
  constexpr int TW = NV + 1;  // trace record: U (+1 spare slot); flux and speed are recomputed at the face
  constexpr int CHUNK = NV * NPE;
  constexpr bool LAST = BM != 0;
  using G = Geo<3, 4, KIND>;
  const int C0 = p.cells[0], C1 = p.cells[1], C2 = p.cells[2];
  const size_t ebase = (size_t)e * CHUNK;
  const double a2 = KIND == 1 ? p.sound_speed : 0.0;
  const int r = lane >> 2, c = lane & 3;
  double* sS = sF + 3 * NV * NPE;  // last stage: S at the nodes
  // XOR-swizzled slab slots (pairs n, n + 1 stay adjacent): F_x / running
  // dudt / S with bits 3, 4 folded into bits 2, 3 (the accumulator patterns of
  // axes 0 and 2 lose their 2- and 4-way conflicts), F_z with the z plane
  // folded into bits 2, 3 (the B-operand reads of axis 2: 4-way -> none)
  auto sw = [](int d, int n) { return d == 0 ? n ^ ((n >> 1) & 12) : (d == 2 ? n ^ (((n >> 4) & 3) << 2) : n); };

  // flux of U along axis d and the one-sided speed (models.cpp:42-70), contracted
  auto fluxd = [&](const double* U, int d, double* F, double& sp) {
    if (KIND == 0) {
      F[0] = p.vel[d] * U[0];
      sp = fabs(p.vel[d]);
    } else {
      const double rinv = fast_rcp(U[0]);
      const double md = d == 0 ? U[1] : (d == 1 ? U[2] : U[NV - 1]);  // selects, not a dynamic index
      const double ua = md * rinv;
      const double pr = U[0] * a2 * a2;
      F[0] = md;
#pragma unroll
      for (int q = 1; q < NV; ++q) F[q] = q == 1 + d ? fma(ua, U[q], pr) : ua * U[q];
      sp = fabs(ua) + a2;
    }
  };

  // ---------------------------------------------------------- nodes (pair 2 lane, 2 lane + 1)
  {
    const int n0 = 2 * lane;
    double Up[2][NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const size_t g = ebase + v * NPE + n0;
      double2 k[1 + NU];
      k[0] = __ldg(reinterpret_cast<const double2*>(p.u + g));
#pragma unroll
      for (int t = 0; t < NU; ++t) k[1 + t] = __ldg(reinterpret_cast<const double2*>(p.ku[t] + g));
      double u0 = k[0].x, u1 = k[0].y;
#pragma unroll
      for (int t = 0; t < NU; ++t)
        if ((AM >> t & 1) != 0) {
          u0 = fma(p.ca[t], k[1 + t].x, u0);
          u1 = fma(p.ca[t], k[1 + t].y, u1);
        }
      Up[0][v] = u0;
      Up[1][v] = u1;
      if (LAST) {
        double s0 = k[0].x, s1 = k[0].y;
#pragma unroll
        for (int t = 0; t < NU; ++t)
          if ((BM >> t & 1) != 0) {
            s0 = fma(p.cb[t], k[1 + t].x, s0);
            s1 = fma(p.cb[t], k[1 + t].y, s1);
          }
        *reinterpret_cast<double2*>(sS + v * NPE + sw(0, n0)) = make_double2(s0, s1);
      }
    }
    double Fp[DIM][2][NV];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = n0 + h;
      if (KIND == 1 && !(Up[h][0] > 0.0)) {
        const int i = n & 3, j = (n >> 2) & 3, kk = n >> 4;
        const long long gx = cx + p.goff[0], gy = cy + p.goff[1], gz = cz + p.goff[2];
        record_error(p.ctl, error_key(step, p.phase, (gx * p.gcells[1] + gy) * (long long)p.gcells[2] + gz,
                                      (j * N + kk) * N + i));
      }
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double sp;
        fluxd(Up[h], d, Fp[d][h], sp);
        const int pos = G::pos_of(d, n);
        if (pos == 0 || pos == N - 1) {
          double* t = sT + ((2 * d + (pos == 0 ? 0 : 1)) * TW) * L + G::line_of(d, n);
#pragma unroll
          for (int v = 0; v < NV; ++v) t[v * L] = Up[h][v];
        }
      }
    }
#pragma unroll
    for (int d = 0; d < DIM; ++d)
#pragma unroll
      for (int v = 0; v < NV; ++v)
        *reinterpret_cast<double2*>(sF + (d * NV + v) * NPE + sw(d, n0)) = make_double2(Fp[d][0][v], Fp[d][1][v]);
  }
  __syncwarp();

  // ---------------------------------------------------------- faces (96 nodes, 3 per lane)
  // iteration m: axis d = m, lanes 0-15 the lo face, 16-31 the hi face
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    const int d = m, side = lane >> 4, t = lane & 15;
    const int f = 2 * d + side;                              // trace slot
    const int fh = 2 * d + (d == RA ? (side ^ par) : side);  // face-flux slot
    if (d == RA && prev && side == 0) continue;              // the previous element's hi-face flux
    const int ca = d == 0 ? cx : (d == 1 ? cy : cz);
    const int cn = d == 0 ? C0 : (d == 1 ? C1 : C2);
    const bool bnd = side ? (ca == cn - 1) : (ca == 0);
    const double* ext = p.ext[d][side];
    double Un[NV];
    if (bnd && ext != nullptr) {
      const size_t xs = d == 0 ? (size_t)cy + (size_t)C1 * cz
                               : (d == 1 ? (size_t)cx + (size_t)C0 * cz : (size_t)cx + (size_t)C0 * cy);
#pragma unroll
      for (int v = 0; v < NV; ++v) Un[v] = __ldg(ext + (xs * NV + v) * L + t);
    } else {
      const int stride = d == 0 ? 1 : (d == 1 ? C0 : C0 * C1);
      const int en = side ? (bnd ? e - (cn - 1) * stride : e + stride) : (bnd ? e + (cn - 1) * stride : e - stride);
      const size_t g = (size_t)en * CHUNK + G::node(d, t, side ? 0 : N - 1);
      // all of this node's loads in flight first, then the combination
      double raw[1 + NU][NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        raw[0][v] = __ldg(p.u + g + v * NPE);
#pragma unroll
        for (int a = 0; a < NU; ++a)
          if ((AM >> a & 1) != 0) raw[1 + a][v] = __ldg(p.ku[a] + g + v * NPE);
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        Un[v] = raw[0][v];
#pragma unroll
        for (int a = 0; a < NU; ++a)
          if ((AM >> a & 1) != 0) Un[v] = fma(p.ca[a], raw[1 + a][v], Un[v]);
      }
    }
    double Uo[NV];
    const double* tr = sT + (f * TW) * L + t;
#pragma unroll
    for (int v = 0; v < NV; ++v) Uo[v] = tr[v * L];
    double Fo[NV], Fn[NV], so, sn;  // own side recomputed from its U trace
    fluxd(Uo, d, Fo, so);
    fluxd(Un, d, Fn, sn);
    const double al = dmax(so, sn);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      // minus state = lower cell along d (solver.cpp:268-306; models.cpp:77-88)
      const double um = side ? Uo[v] : Un[v], up = side ? Un[v] : Uo[v];
      const double fm = side ? Fo[v] : Fn[v], fp = side ? Fn[v] : Fo[v];
      // explicit roundings: every code path (either side, run or not) gives
      // the same bits, so a reused hi-face flux equals a recomputed lo one
      sH[(fh * NV + v) * L + t] = __dmul_rn(0.5, fma(-al, __dsub_rn(up, um), __dadd_rn(fm, fp)));
    }
  }
  __syncwarp();

  // ---------------------------------------------------------- volume on the tensor cores
  double* acc = sF;  // F_x's slots become the running dudt
  const bool krow = r < N;
  const int rr = r & 3;  // rows 4-7 of the MMA are zero rows: their lanes mirror rows 0-3 (results unused)
#pragma unroll
  for (int d = 0; d < DIM - 1; ++d) {
    if (d > 0) __syncwarp();  // the previous axis' partial sums are stored
#pragma unroll
    for (int v = 0; v < NV; ++v) {
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int q0 = sw(0, G::node(d, 8 * g + 2 * c, rr)), q1 = sw(0, G::node(d, 8 * g + 2 * c + 1, rr));
        double c0 = 0.0, c1 = 0.0;
        if (d > 0) {
          c0 = acc[v * NPE + q0];
          c1 = acc[v * NPE + q1];
        }
        const double b = sF[(d * NV + v) * NPE + sw(d, G::node(d, 8 * g + r, c))];
        dmma_8x8x4(ln.k[d], b, c0, c1);
        __syncwarp();  // B/C reads of this group precede the in-place stores
        if (krow) {
          acc[v * NPE + q0] = c0;
          acc[v * NPE + q1] = c1;
        }
      }
    }
  }
  __syncwarp();
  // final axis (z): outputs of line group g at nodes o0 = 8g + 2c + 16 rr and
  // o0 + 1; the g = 1 results move to lanes 16-31, so every lane finishes one
  // output pair per variable (lifted faces and the RK epilogue, branch-free)
  const int gl = lane >> 4;                       // this lane's line group
  const int o0 = 8 * gl + 2 * c + 16 * rr;
  const int qa = sw(0, o0), qb = sw(0, o0 + 1);
  const int jj = 2 * gl + (c >> 1), i0 = (2 * c) & 3;
  constexpr int X0 = 0, Y0 = 2, Z0 = 4;
  const int xl = X0 + (RA == 0 ? par : 0), zl = Z0 + (RA == 2 ? par : 0);  // run-axis slots alternate
  // face-lift coefficients of the two outputs (0 off the face)
  const double xc0 = (c & 1) == 0 ? p.lift[0] : 0.0, xc1 = (c & 1) != 0 ? -p.lift[0] : 0.0;
  const double yc = gl == 0 ? (c < 2 ? p.lift[1] : 0.0) : (c >= 2 ? -p.lift[1] : 0.0);
  const double zc = rr == 0 ? p.lift[2] : (rr == N - 1 ? -p.lift[2] : 0.0);
  const double* hx0 = sH + xl * NV * L + jj + 4 * rr;
  const double* hx1 = sH + (2 * X0 + 1 - xl) * NV * L + jj + 4 * rr;
  const double* hy = sH + (Y0 + gl) * NV * L + i0 + 4 * rr;
  const double* hz = sH + (rr == 0 ? zl : 2 * Z0 + 1 - zl) * NV * L + i0 + 4 * jj;
  double* gout = p.out + ebase + o0;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double c0[2], c1[2];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      c0[g] = acc[v * NPE + sw(0, G::node(2, 8 * g + 2 * c, rr))];
      c1[g] = acc[v * NPE + sw(0, G::node(2, 8 * g + 2 * c + 1, rr))];
      const double b = sF[(2 * NV + v) * NPE + sw(2, G::node(2, 8 * g + r, c))];
      dmma_8x8x4(ln.k[2], b, c0[g], c1[g]);
    }
    const double y0 = __shfl_sync(0xffffffffu, c0[1], lane & 15), y1 = __shfl_sync(0xffffffffu, c1[1], lane & 15);
    double d0 = gl ? y0 : c0[0], d1 = gl ? y1 : c1[0];
    d0 = fma(xc0, hx0[v * L], d0);
    d1 = fma(xc1, hx1[v * L], d1);
    d0 = fma(yc, hy[v * L], d0);
    d1 = fma(yc, hy[v * L + 1], d1);
    d0 = fma(zc, hz[v * L], d0);
    d1 = fma(zc, hz[v * L + 1], d1);
    const double k0 = d0 * dt, k1 = d1 * dt;
    if (!LAST) {
      *reinterpret_cast<double2*>(gout + v * NPE) = make_double2(k0, k1);
    } else {
      __syncwarp();  // every lane's accumulator reads of v precede the u_new stores
      const double u0 = fma(p.b_last, k0, sS[v * NPE + qa]);
      const double u1 = fma(p.b_last, k1, sS[v * NPE + qb]);
      *reinterpret_cast<double2*>(gout + v * NPE) = make_double2(u0, u1);
      acc[v * NPE + qa] = u0;  // u_new for the finite check / next alpha
      acc[v * NPE + qb] = u1;
    }
  }
  if (LAST) {
    __syncwarp();
    // node-parallel over the lane's own pair: finite check and next alpha
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = 2 * lane + h;
      double un[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) un[v] = acc[v * NPE + sw(0, n)];
      double sum = un[0];
#pragma unroll
      for (int v = 1; v < NV; ++v) sum += un[v];
      if (!isfinite(sum)) record_error(p.ctl, error_key(step, kPhaseInstability, p.block_id, 0));
      if (KIND == 1 && p.scan_alpha) {
        if (!(un[0] > 0.0)) {
          const long long gx = cx + p.goff[0], gy = cy + p.goff[1], gz = cz + p.goff[2];
          record_error(p.ctl, error_key(step + 1, kPhaseScan, (gx * p.gcells[1] + gy) * (long long)p.gcells[2] + gz,
                                        G::aos_node(n)));
        } else {
          double mm = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) mm = dmax(mm, fabs(un[1 + d]));
          alpha = dmax(alpha, __dadd_rn(__ddiv_rn(mm, un[0]), p.sound_speed));  // == alpha_scan_kernel
        }
      }
    }
  }
  __syncwarp();  // this element's slab reads precede the next element's writes
}

// ------------------------------------------------------------ 3D order-4 line body
// The C4 shape (3D, N = 4, contracted) by LINE TASKS instead of tensor-core
// tiles.  The tensor-core body moves every flux through shared memory in the
// MMA operand layouts and carries the running dudt across the three axes
// through shared memory: ~420 shared wavefronts per element, and the L1 pipe
// at 95% bounds it.  Here a lane owns whole lines:
//   1  nodes: each lane forms U_s at its node pair (16-byte loads) and stores
//      it once into a swizzled U slab;
//   2  lines: 48 tasks (16 lines per axis), lanes 0-15 the x lines and 16-31
//      the y lines, then lanes 0-15 the z lines.  A task reads its line's 4
//      nodes, computes the Lax-Friedrichs flux at the line's two ends (its
//      face nodes: own flux = the end node's flux, neighbour from HBM / the
//      received plane), the 4 node fluxes, D = K F (16 FMA per variable) and
//      the lifted end fluxes, and stores the axis's dudt part;
//   3  epilogue: each lane sums the three axis parts at its node pair.
// About 160 shared wavefronts per element.  K_d = (dx_0 / dx_d) K_0 (exactly
// K_0 on the equal-spacing meshes): every lane uses K_0 as constant-bank
// operands and scales by r_d = lift_d / lift_0.  In a z-run the z lines stay
// on lanes 0-15, so the z-lo face flux is the previous element's z-hi flux
// carried in registers (`hc`), bitwise the value a recomputation gives.
//
// Slab swizzle: node n = i + 4 j + 16 k sits at n ^ (k | k << 2) (i ^= k,
// j ^= k): every plane of fixed i, j or k maps onto 16 distinct double
// banks, so line reads and writes along any axis are conflict-free.
__device__ __forceinline__ int sw3(int n) {
  const int k = n >> 4;
  return n ^ (k | (k << 2));
}

template <int KIND, int NU, int AM, int BM>
__device__ __forceinline__ void element_3d4_lines(const StageArgs& p, int lane, int e, int cx, int cy, int cz,
                                                  double* sU, double* sD, double dt, long long step, double& alpha,
                                                  bool prev, double (&hc)[KIND == 0 ? 1 : 4], double rdy, double rdz,
                                                  bool scaled) {
  constexpr int N = 4, NPE = 64, L = 16, DIM = 3;
  constexpr int NV = KIND == 0 ? 1 : 4;
  constexpr int CHUNK = NV * NPE;
  constexpr bool LAST = BM != 0;
  using G = Geo<3, 4, KIND>;
  const int C0 = p.cells[0], C1 = p.cells[1], C2 = p.cells[2];
  const size_t ebase = (size_t)e * CHUNK;
  const double a2 = KIND == 1 ? p.sound_speed : 0.0;

  // flux of U along axis d and the one-sided speed (models.cpp:42-70), contracted
  auto fluxd = [&](const double* U, int d, double* F, double& sp) {
    if (KIND == 0) {
      const double vd = d == 0 ? p.vel[0] : (d == 1 ? p.vel[1] : p.vel[2]);
      F[0] = vd * U[0];
      sp = fabs(vd);
    } else {
      const double rinv = fast_rcp(U[0]);
      // m_d by value selects (d is a run-time value in the x/y round: an
      // address select would put the line arrays in local memory)
      double md = U[1];
      if (d == 1) md = U[2];
      if (d == 2) md = U[NV - 1];
      const double ua = md * rinv;
      const double pr = U[0] * a2 * a2;
      F[0] = md;
#pragma unroll
      for (int q = 1; q < NV; ++q) F[q] = fma(ua, U[q], q == 1 + d ? pr : 0.0);  // (no U[1 + d] index)
      sp = fabs(ua) + a2;
    }
  };

  // ---------------------------------------------------------- 1: nodes (pair 2 lane, 2 lane + 1)
  const int n0 = 2 * lane;
  const int s0 = sw3(n0), s1 = sw3(n0 + 1);  // the pair's slab slots (one 16-byte unit, halves swapped for odd k)
  double* sS = sD + 3 * NV * NPE;  // last stage: S at the node pairs (slab, not registers)
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const size_t g = ebase + v * NPE + n0;
    double2 k[1 + NU];
    k[0] = __ldg(reinterpret_cast<const double2*>(p.u + g));
#pragma unroll
    for (int t = 0; t < NU; ++t) k[1 + t] = __ldg(reinterpret_cast<const double2*>(p.ku[t] + g));
    double ua = k[0].x, ub = k[0].y;
#pragma unroll
    for (int t = 0; t < NU; ++t)
      if ((AM >> t & 1) != 0) {
        ua = fma(p.ca[t], k[1 + t].x, ua);
        ub = fma(p.ca[t], k[1 + t].y, ub);
      }
    if (LAST) {
      double s0 = k[0].x, s1 = k[0].y;
#pragma unroll
      for (int t = 0; t < NU; ++t)
        if ((BM >> t & 1) != 0) {
          s0 = fma(p.cb[t], k[1 + t].x, s0);
          s1 = fma(p.cb[t], k[1 + t].y, s1);
        }
      *reinterpret_cast<double2*>(sS + v * NPE + n0) = make_double2(s0, s1);
    }
    if (KIND == 1 && v == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!((h ? ub : ua) > 0.0)) {
          const int n = n0 + h, i = n & 3, j = (n >> 2) & 3, kk = n >> 4;
          const long long gx = cx + p.goff[0], gy = cy + p.goff[1], gz = cz + p.goff[2];
          record_error(p.ctl, error_key(step, p.phase, (gx * p.gcells[1] + gy) * (long long)p.gcells[2] + gz,
                                        (j * N + kk) * N + i));
        }
      }
    }
    sU[v * NPE + s0] = ua;  // two 8-byte stores: cheaper than selecting the halves
    sU[v * NPE + s1] = ub;
  }
  __syncwarp();

  // ---------------------------------------------------------- 2: line tasks
  // task (d, t): line t of axis d; lanes 0-15 x, 16-31 y, then lanes 0-15 z
  // off[q]: slab slot of the line's node at position q; rd = lift_d / lift_0
  auto line_task = [&](const int d, const int t, const int (&off)[4], const double rd, const bool reuse_lo) {
    // the line's end nodes first (their fluxes serve the faces), the inner two after
    double Ul[4][NV], F[4][NV], sp[4];
#pragma unroll
    for (int q = 0; q < 4; q += 3) {
#pragma unroll
      for (int v = 0; v < NV; ++v) Ul[q][v] = sU[v * NPE + off[q]];
      fluxd(Ul[q], d, F[q], sp[q]);
    }
    // the line's end faces: lo (side 0) at q = 0, hi (side 1) at q = 3
    double H[2][NV];
    const int ca = d == 0 ? cx : (d == 1 ? cy : cz);
    const int cn = d == 0 ? C0 : (d == 1 ? C1 : C2);
    const int stride = d == 0 ? 1 : (d == 1 ? C0 : C0 * C1);
    // LF flux at the end face `side` (0: lo, own node q = 0; 1: hi, q = 3)
    auto end_face = [&](const int side, const double* Uo, const double* Fo, const double so, double* Hs) {
      const bool bnd = side ? (ca == cn - 1) : (ca == 0);
      const double* ext = d == 0 ? p.ext[0][side] : (d == 1 ? p.ext[1][side] : p.ext[2][side]);
      double Un[NV];
      if (bnd && ext != nullptr) {
        const size_t xs = d == 0 ? (size_t)cy + (size_t)C1 * cz
                                 : (d == 1 ? (size_t)cx + (size_t)C0 * cz : (size_t)cx + (size_t)C0 * cy);
#pragma unroll
        for (int v = 0; v < NV; ++v) Un[v] = __ldg(ext + (xs * NV + v) * L + t);
      } else {
        const int en = side ? (bnd ? e - (cn - 1) * stride : e + stride) : (bnd ? e + (cn - 1) * stride : e - stride);
        const size_t g = (size_t)en * CHUNK + G::node(d, t, side ? 0 : N - 1);
        // combined as the loads arrive (the scheduler keeps as many in
        // flight as the register cap allows)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          Un[v] = __ldg(p.u + g + v * NPE);
#pragma unroll
          for (int a = 0; a < NU; ++a)
            if ((AM >> a & 1) != 0) Un[v] = fma(p.ca[a], __ldg(p.ku[a] + g + v * NPE), Un[v]);
        }
      }
      double Fn[NV], sn;
      fluxd(Un, d, Fn, sn);
      const double al = dmax(so, sn);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        // minus state = lower cell along d (solver.cpp:268-306; models.cpp:77-88)
        const double um = side ? Uo[v] : Un[v], up = side ? Un[v] : Uo[v];
        const double fm = side ? Fo[v] : Fn[v], fp = side ? Fn[v] : Fo[v];
        // explicit roundings: the same bits from either side of the face
        Hs[v] = __dmul_rn(0.5, fma(-al, __dsub_rn(up, um), __dadd_rn(fm, fp)));
      }
    };
    if (reuse_lo) {
#pragma unroll
      for (int v = 0; v < NV; ++v) H[0][v] = hc[v];
    } else {
      end_face(0, Ul[0], F[0], sp[0], H[0]);
    }
    end_face(1, Ul[3], F[3], sp[3], H[1]);
#pragma unroll
    for (int q = 1; q < 3; ++q) {
#pragma unroll
      for (int v = 0; v < NV; ++v) Ul[q][v] = sU[v * NPE + off[q]];
      fluxd(Ul[q], d, F[q], sp[q]);
    }
    // D_d = r_d (K_0 F + lifted end fluxes), K_d = r_d K_0 with r_d = lift_d / lift_0
    double* out = sD + d * NV * NPE;
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double acc = p.K[0][k * 4] * F[0][v];
#pragma unroll
        for (int l = 1; l < 4; ++l) acc = fma(p.K[0][k * 4 + l], F[l][v], acc);
        if (k == 0) acc = fma(p.lift[0], H[0][v], acc);
        if (k == 3) acc = fma(-p.lift[0], H[1][v], acc);
        out[v * NPE + off[k]] = scaled ? acc * rd : acc;  // (warp-uniform: rd == 1 on equal spacing)
      }
    if (d == 2) {
#pragma unroll
      for (int v = 0; v < NV; ++v) hc[v] = H[1][v];  // the next z element's lo-face flux
    }
  };
  {
    // round 1: x line t = j + 4k at slots 16k + 4(j^k) + (q^k); y line t = i + 4k at 16k + 4(q^k) + (i^k)
    const int d = lane >> 4, t = lane & 15, c = t >> 2, w = t & 3;
    const int base = 16 * c + (d == 0 ? 4 * (w ^ c) : (w ^ c)), m = d == 0 ? 1 : 4;
    const int off[4] = {base + m * c, base + m * (1 ^ c), base + m * (2 ^ c), base + m * (3 ^ c)};
    line_task(d, t, off, d == 0 ? 1.0 : rdy, false);
  }
  __syncwarp();  // keeps the two rounds apart in the schedule (their live sets do not add up)
  {
    // round 2: the z lines, each split over two lanes: lane t (half 0) the
    // lo face and outputs q = 0, 1, lane t + 16 (half 1) the hi face and
    // q = 2, 3; both read the line and form its 4 fluxes.  Line t = i + 4j
    // sits at slots 16q + 4(j^q) + (i^q).  The z-hi flux carried along the
    // run lives on the half-1 lane; the half-0 lane takes it by a shuffle.
    constexpr int d = 2;
    const int t = lane & 15, half = lane >> 4, i = t & 3, j = t >> 2;
    double hprev[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) hprev[v] = __shfl_xor_sync(0xffffffffu, hc[v], 16);
    double Ul[4][NV], F[4][NV], sp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int v = 0; v < NV; ++v) Ul[q][v] = sU[v * NPE + 16 * q + 4 * (j ^ q) + (i ^ q)];
      fluxd(Ul[q], d, F[q], sp[q]);
    }
    double Uo[NV], Fo[NV];  // this half's end node (value selects: no dynamic index)
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      Uo[v] = half ? Ul[3][v] : Ul[0][v];
      Fo[v] = half ? F[3][v] : F[0][v];
    }
    const double so = half ? sp[3] : sp[0];
    double H[NV];
    // the lo face of a run's inner element: the carried flux; else computed
    const bool take = half == 0 && prev;
    const bool bnd = half ? (cz == C2 - 1) : (cz == 0);
    const double* ext = half ? p.ext[2][1] : p.ext[2][0];
    double Un[NV];
    if (!take) {
      if (bnd && ext != nullptr) {
        const size_t xs = (size_t)cx + (size_t)C0 * cy;
#pragma unroll
        for (int v = 0; v < NV; ++v) Un[v] = __ldg(ext + (xs * NV + v) * L + t);
      } else {
        const int stride = C0 * C1;
        const int en = half ? (bnd ? e - (C2 - 1) * stride : e + stride) : (bnd ? e + (C2 - 1) * stride : e - stride);
        const size_t g = (size_t)en * CHUNK + t + (half ? 0 : 48);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          Un[v] = __ldg(p.u + g + v * NPE);
#pragma unroll
          for (int a = 0; a < NU; ++a)
            if ((AM >> a & 1) != 0) Un[v] = fma(p.ca[a], __ldg(p.ku[a] + g + v * NPE), Un[v]);
        }
      }
      double Fn[NV], sn;
      fluxd(Un, d, Fn, sn);
      const double al = dmax(so, sn);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        // minus state = lower cell along z (solver.cpp:268-306; models.cpp:77-88)
        const double um = half ? Uo[v] : Un[v], up = half ? Un[v] : Uo[v];
        const double fm = half ? Fo[v] : Fn[v], fp = half ? Fn[v] : Fo[v];
        H[v] = __dmul_rn(0.5, fma(-al, __dsub_rn(up, um), __dadd_rn(fm, fp)));
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (take) H[v] = hprev[v];
      if (half) hc[v] = H[v];  // the next z element's lo-face flux (taken by lane t)
    }
    // outputs q = 2 half + s: K_2 rows by value selects, the own face lifted
    // onto q = 0 (half 0) or q = 3 (half 1)
    const double ca0 = half ? 0.0 : p.lift[0], cb1 = half ? -p.lift[0] : 0.0;
    double* out = sD + d * NV * NPE;
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      double kr[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) kr[l] = half ? p.K[0][(2 + s2) * 4 + l] : p.K[0][s2 * 4 + l];
      const int q = 2 * half + s2;
      const int slot = 16 * q + 4 * (j ^ q) + (i ^ q);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double acc = kr[0] * F[0][v];
#pragma unroll
        for (int l = 1; l < 4; ++l) acc = fma(kr[l], F[l][v], acc);
        acc = fma(s2 == 0 ? ca0 : cb1, H[v], acc);
        out[v * NPE + slot] = scaled ? acc * rdz : acc;
      }
    }
  }
  __syncwarp();

  // ---------------------------------------------------------- 3: epilogue at the node pair
  double un[2][NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double dv[2];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double w0 = sD[(d * NV + v) * NPE + s0], w1 = sD[(d * NV + v) * NPE + s1];
      dv[0] = d == 0 ? w0 : dv[0] + w0;
      dv[1] = d == 0 ? w1 : dv[1] + w1;
    }
    const double k0 = dv[0] * dt, k1 = dv[1] * dt;
    double* gout = p.out + ebase + v * NPE + n0;
    if (!LAST) {
      *reinterpret_cast<double2*>(gout) = make_double2(k0, k1);
    } else {
      const double2 S = *reinterpret_cast<const double2*>(sS + v * NPE + n0);
      un[0][v] = fma(p.b_last, k0, S.x);
      un[1][v] = fma(p.b_last, k1, S.y);
      *reinterpret_cast<double2*>(gout) = make_double2(un[0][v], un[1][v]);
    }
  }
  if (LAST) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double sum = un[h][0];
#pragma unroll
      for (int v = 1; v < NV; ++v) sum += un[h][v];
      if (!isfinite(sum)) record_error(p.ctl, error_key(step, kPhaseInstability, p.block_id, 0));
      if (KIND == 1 && p.scan_alpha) {
        if (!(un[h][0] > 0.0)) {
          const long long gx = cx + p.goff[0], gy = cy + p.goff[1], gz = cz + p.goff[2];
          record_error(p.ctl, error_key(step + 1, kPhaseScan, (gx * p.gcells[1] + gy) * (long long)p.gcells[2] + gz,
                                        G::aos_node(n0 + h)));
        } else {
          double mm = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) mm = dmax(mm, fabs(un[h][1 + d]));
          alpha = dmax(alpha, __dadd_rn(__ddiv_rn(mm, un[h][0]), p.sound_speed));  // == alpha_scan_kernel
        }
      }
    }
  }
  __syncwarp();  // this element's slab reads precede the next element's writes
}

// ------------------------------------------------------------ flagship body
// One element of the 2D, N = 8, contracted-arithmetic stage (the benchmark
// shape), written for issue efficiency: lane constants are hoisted by the
// caller (Lane8), global accesses use per-element base pointers with
// immediate offsets, and the only branches are warp-uniform.
struct Lane8 {
  int r, c;              // lane = 4r + c
  int n0;                // flux nodes (i = 2c + h, j = r): n0 and n0 + 1 (adjacent)
  int f, t;              // face lane: face f (x-lo, x-hi, y-lo, y-hi), face node t
  int nb_node;           // the neighbour element's node facing this face lane
  int o0;                // output node s = 0: (i = r, j = 2c); s = 1 is o0 + 8
  double xco, yco0, yco1;  // face-lift coefficients of the output nodes
  int xf;                // x face (0 / 1) feeding the output row r
  double kx[2], ky[2];   // K_x[r][2c+h], K_y[r][2c+h] (k-step h pairs l = 2c + h)
  int n0s, a0s, a1s;     // swizzled slab slots of n0 and of the A / output nodes o0, o0 + 8
  // order N < 8 on the padded 8 x 8 grid (slab slots keep the padded index
  // i + 8 j; padded nodes carry zero fluxes, padded K rows / columns are 0)
  int g0;                // global node of the flux node (2c, r): i + N j
  int og0, og1;          // global nodes of the output nodes (r, 2c), (r, 2c + 1)
  int vm;                // valid bits: 1, 2 flux nodes h = 0, 1; 4, 8 output nodes s = 0, 1; 16 face node t
  int yf0, yf1;          // y face (2 lo / 3 hi) lifted into output s = 0 / 1
  double yco1p;          // its coefficient for s = 1 (yco0 for s = 0)
  // transposed output (NDGX_DT2): the lane's outputs are its own flux nodes
  // (i = 2c + s, j = r); the y face of row r is shared, the x face is per s
  double gco;            // y-face lift coefficient of row r (0 inside)
  int gf;                // its face (2 lo / 3 hi)
  double fco0, fco1;     // x-face lift coefficients of outputs s = 0 / 1
  int ff0, ff1;          // their faces (0 lo / 1 hi)
};

// Slab slot of node n = i + 8 j for the flagship's F_y and S arrays: the
// 16-byte unit n / 2 is XORed with 2 ((j / 2) mod 4).  The node-phase stores
// (double2 at i = 2c, j = r) stay conflict-free and the transposed reads
// (i = r, j = 2c or 2c + 1, by lanes 4r + c) hit eight distinct bank quads
// per half-warp instead of two (a 4-way conflict unswizzled).
__host__ __device__ constexpr int swz8(int n) { return n ^ (((n >> 4) & 3) << 2); }

// One element's raw inputs for the flagship body, loaded one element ahead
// (NDGX_PF2: the advection stages, whose warps otherwise wait one full
// memory latency per element): the lane's node pair of every input array
// and its face node's neighbour values.
template <int NV, int NU>
struct Pre8 {
  double2 node[NV][1 + NU];
  double face[1 + NU][NV];
};

// The loads of element_2d8_fast (order 8, no ring, no slab reuse), issued
// into `q` without waiting for them.
template <int KIND, int NU>
__device__ __forceinline__ void preload_2d8(const StageArgs& p, const Lane8& ln, int e, int cx, int cy,
                                            Pre8<KIND == 0 ? 1 : 3, NU>& q) {
  constexpr int NV = KIND == 0 ? 1 : 3, NPE = 64, N = 8, CHUNK = NV * NPE;
  const int C0 = p.cells[0], C1 = p.cells[1];
  const int f = ln.f, d = f >> 1, side = f & 1;
  const bool bnd = d == 0 ? (side ? cx == C0 - 1 : cx == 0) : (side ? cy == C1 - 1 : cy == 0);
  const double* ext = p.ext[d][side];
  if (bnd && ext != nullptr) {
    const size_t xs = d == 0 ? (size_t)cy : (size_t)cx;
#pragma unroll
    for (int v = 0; v < NV; ++v) q.face[0][v] = __ldg(ext + (xs * NV + v) * N + ln.t);
  } else {
    const int step_d = d == 0 ? 1 : C0;
    const int span = d == 0 ? C0 : C1;
    const int en = side ? (bnd ? e - (span - 1) * step_d : e + step_d) : (bnd ? e + (span - 1) * step_d : e - step_d);
    const size_t g = (size_t)en * CHUNK + ln.nb_node;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      q.face[0][v] = __ldg(p.u + g + v * NPE);
#pragma unroll
      for (int a = 0; a < NU; ++a) q.face[1 + a][v] = __ldg(p.ku[a] + g + v * NPE);
    }
  }
  const size_t ebase = (size_t)e * CHUNK;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const size_t g = ebase + v * NPE + ln.n0;
    q.node[v][0] = __ldg(reinterpret_cast<const double2*>(p.u + g));
#pragma unroll
    for (int t = 0; t < NU; ++t) q.node[v][1 + t] = __ldg(reinterpret_cast<const double2*>(p.ku[t] + g));
  }
}

template <int N, int KIND, int NU, int AM, int BM, int SIG, bool PRE = false>
__device__ __forceinline__ void element_2d8_fast(const StageArgs& p, const Lane8& ln, int lane, int e, int cx,
                                                 int cy, const double* src, const double* fsrc, bool ring_,
                                                 double* sF, double* sT, double* sH, double dt, bool last,
                                                 long long step, double& alpha, bool reuse_lo = false,
                                                 const Pre8<KIND == 0 ? 1 : 3, NU>* pre = nullptr) {
  // N < 8: the same body on the zero-padded 8 x 8 grid (slab index i + 8 j)
  constexpr bool PAD = N < 8;
  constexpr int NPE = N * N, L = 8;
  const bool ring = !PAD && ring_;  // (no TMA ring: odd or unaligned element chunks)
  constexpr int NV = KIND == 0 ? 1 : 3;
  constexpr int HW = 2 * NV + 1;
  constexpr int CHUNK = NV * NPE;
  using A = Ar<false>;
  const int C0 = p.cells[0], C1 = p.cells[1];
  const size_t ebase = (size_t)e * CHUNK;
  const double a2 = KIND == 1 ? p.sound_speed : 0.0;

  // face neighbour loads first, so they are in flight together with the
  // node loads (one memory latency per element instead of two)
  const int f = ln.f, d = f >> 1, side = f & 1;
  const bool bnd = d == 0 ? (side ? cx == C0 - 1 : cx == 0) : (side ? cy == C1 - 1 : cy == 0);
  const double* ext = p.ext[d][side];
  const bool from_ext = bnd && ext != nullptr;
  // x-lo face of an element that follows its x-lo neighbour in the warp's
  // run: the neighbour's stage input at (7, t) is its own x-hi trace, still
  // in the slab (read before this element's node phase overwrites it)
  const bool from_prev = reuse_lo && f == 0;
  double Uprev[NV];
  if (from_prev) {
#pragma unroll
    for (int v = 0; v < NV; ++v) Uprev[v] = sT[(HW + v) * L + ln.t];
  }
  if (reuse_lo) __syncwarp();  // read before the node phase's trace stores
  double Nraw[1 + NU][NV];
  if constexpr (PRE) {
#pragma unroll
    for (int a = 0; a < 1 + NU; ++a)
#pragma unroll
      for (int v = 0; v < NV; ++v) Nraw[a][v] = pre->face[a][v];
  } else if (!ring && !from_prev) {
    if (from_ext) {
      const size_t xs = d == 0 ? (size_t)cy : (size_t)cx;
#pragma unroll
      for (int v = 0; v < NV; ++v) Nraw[0][v] = __ldg(ext + (xs * NV + v) * N + (PAD ? (ln.vm & 16 ? ln.t : 0) : ln.t));
    } else {
      const int step_d = d == 0 ? 1 : C0;
      const int span = d == 0 ? C0 : C1;
      const int en = side ? (bnd ? e - (span - 1) * step_d : e + step_d) : (bnd ? e + (span - 1) * step_d : e - step_d);
      const size_t g = (size_t)en * CHUNK + ln.nb_node;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        Nraw[0][v] = __ldg(p.u + g + v * NPE);
#pragma unroll
        for (int a = 0; a < NU; ++a) Nraw[1 + a][v] = __ldg(p.ku[a] + g + v * NPE);
      }
    }
  }

  // ---------------------------------------------------------- nodes
  double Bx[2][NV], Fyp[2][NV];
  // both nodes of the lane at once: one 16-byte load per (array, var)
  double Up[2][NV];
  double* sS = sF + NV * 64;  // last stage: S at the flux nodes, read back at the output nodes
  if constexpr (PAD) {
    // scalar loads (the node pairs of odd N are not 16-byte aligned); a
    // padded node gets rho = 1, momentum 0 (finite fluxes, zeroed below)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool ok = (ln.vm >> h & 1) != 0;
      double Sh[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double Uv = (KIND == 1 && v == 0) ? 1.0 : 0.0, Sv = 0.0;
        if (ok) combine_g<false, NU, AM, BM>(p, ebase + v * NPE + ln.g0 + h, last, Uv, Sv);
        Up[h][v] = Uv;
        Sh[v] = Sv;
      }
      if (last) {
#pragma unroll
        for (int v = 0; v < NV; ++v) sS[v * 64 + ln.n0s + h] = Sh[v];
      }
    }
  } else if constexpr (PRE) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double2* k = pre->node[v];
      double u0 = k[0].x, u1 = k[0].y;
#pragma unroll
      for (int t = 0; t < NU; ++t)
        if ((AM >> t & 1) != 0) {
          u0 = fma(p.ca[t], k[1 + t].x, u0);
          u1 = fma(p.ca[t], k[1 + t].y, u1);
        }
      Up[0][v] = u0;
      Up[1][v] = u1;
      if (last) {  // S = u + sum b_j K_j (combine_pair's expressions)
        double a = k[0].x, b = k[0].y;
#pragma unroll
        for (int t = 0; t < NU; ++t)
          if ((BM >> t & 1) != 0) {
            a = fma(p.cb[t], k[1 + t].x, a);
            b = fma(p.cb[t], k[1 + t].y, b);
          }
        *reinterpret_cast<double2*>(sS + v * NPE + ln.n0s) = make_double2(a, b);
      }
    }
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (last) {
        double S0, S1;
        combine_pair<NU, AM, BM>(p, ring, src + v * NPE + ln.n0, ebase + v * NPE + ln.n0, CHUNK, Up[0][v],
                                 Up[1][v], &S0, &S1);
        *reinterpret_cast<double2*>(sS + v * NPE + ln.n0s) = make_double2(S0, S1);
      } else {
        combine_pair<NU, AM>(p, ring, src + v * NPE + ln.n0, ebase + v * NPE + ln.n0, CHUNK, Up[0][v], Up[1][v]);
      }
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int n = ln.n0 + h;
    const bool ok = !PAD || (ln.vm >> h & 1) != 0;
    double U[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) U[v] = Up[h][v];
    double Fx[NV], Fy[NV], sx, sy;
    if (KIND == 0) {
      Fx[0] = p.vel[0] * U[0];
      Fy[0] = p.vel[1] * U[0];
      sx = fabs(p.vel[0]);
      sy = fabs(p.vel[1]);
    } else {
      if (!(U[0] > 0.0)) {  // (padded nodes hold rho = 1)
        const int i = n & 7, j = n >> 3;
        const long long gx = cx + p.goff[0], gy = cy + p.goff[1];
        record_error(p.ctl, error_key(step, p.phase, (gx * p.gcells[1] + gy) * (long long)p.gcells[2], j * N + i));
      }
      const double rinv = fast_rcp(U[0]);
      const double ux = U[1] * rinv, uy = U[2] * rinv;
      const double pr = U[0] * a2 * a2;  // (rho a) a
      Fx[0] = U[1];
      Fx[1] = fma(ux, U[1], pr);
      Fx[2] = ux * U[2];
      Fy[0] = U[2];
      Fy[1] = uy * U[1];
      Fy[2] = fma(uy, U[2], pr);
      sx = fabs(ux) + a2;
      sy = fabs(uy) + a2;
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      Bx[h][v] = ok ? Fx[v] : 0.0;
      Fyp[h][v] = ok ? Fy[v] : 0.0;
    }
    // face traces, U only (the face lane recomputes flux and speed, cheaper
    // than the partial-warp shared stores of keeping them): x faces at
    // i = 2c + h = 0 / 7, y faces at j = r = 0 / 7
    const int i = 2 * ln.c + h;
    if ((i == 0 || i == N - 1) && (!PAD || ln.r < N)) {
      double* t = sT + (i == 0 ? 0 : HW) * L + ln.r;
#pragma unroll
      for (int v = 0; v < NV; ++v) t[v * L] = U[v];
    }
#if !NDGX_YTR2
    if (ln.r == 0 || ln.r == N - 1) {
      double* t = sT + ((ln.r == 0 ? 2 : 3) * HW) * L + i;
#pragma unroll
      for (int v = 0; v < NV; ++v) t[v * L] = U[v];
    }
#endif
  }
#if NDGX_YTR2
  // y-face traces of both nodes at once (i = 2c, 2c + 1 are adjacent slots):
  // one 16-byte store per variable by the r = 0 / 7 lanes
  if (ln.r == 0 || ln.r == N - 1) {
    double* t = sT + ((ln.r == 0 ? 2 : 3) * HW) * L + 2 * ln.c;
#pragma unroll
    for (int v = 0; v < NV; ++v) *reinterpret_cast<double2*>(t + v * L) = make_double2(Up[0][v], Up[1][v]);
  }
#endif
#pragma unroll
  for (int v = 0; v < NV; ++v)
    *reinterpret_cast<double2*>(sF + v * 64 + ln.n0s) = make_double2(Fyp[0][v], Fyp[1][v]);
  __syncwarp();

  // ---------------------------------------------------------- faces
  {
    double Un[NV];
    if (from_prev) {
#pragma unroll
      for (int v = 0; v < NV; ++v) Un[v] = Uprev[v];
    } else if (from_ext) {
#pragma unroll
      for (int v = 0; v < NV; ++v) Un[v] = ring ? fsrc[v * 32 + lane] : Nraw[0][v];
    } else if (ring) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double S;
        combine_s<false, NU, AM, BM>(p, fsrc + v * 32 + lane, NV * 32, false, Un[v], S);
      }
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        Un[v] = Nraw[0][v];
#pragma unroll
        for (int a = 0; a < NU; ++a)
          if ((AM >> a & 1) != 0) Un[v] = fma(p.ca[a], Nraw[1 + a][v], Un[v]);
      }
    }
    // flux along d and one-sided speed (models.cpp:42-70), the node phase's expressions
    auto fluxd = [&](const double* W, double* F, double& sp) {
      if (KIND == 0) {
        F[0] = p.vel[d] * W[0];
        sp = fabs(p.vel[d]);
      } else {
        const double rinv = fast_rcp(W[0]);
        const double md = d == 0 ? W[1] : W[2];  // a select, not a (local-memory) dynamic index
        const double ua = md * rinv;
        const double pr = W[0] * a2 * a2;
        F[0] = md;
        F[1] = d == 0 ? fma(ua, W[1], pr) : ua * W[1];
        F[2] = d == 0 ? ua * W[2] : fma(ua, W[2], pr);
        sp = fabs(ua) + a2;
      }
    };
    const double* own = sT + (f * HW) * L + ln.t;
    double Fn[NV], sn;
    fluxd(Un, Fn, sn);
    {
      double Uo[NV], Fo[NV], so;  // this element's side, from its U trace
#pragma unroll
      for (int v = 0; v < NV; ++v) Uo[v] = own[v * L];
      fluxd(Uo, Fo, so);
      const double al = dmax(so, sn);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        // minus state = lower cell along d (solver.cpp:268-306; models.cpp:77-88)
        const double um = side ? Uo[v] : Un[v], up = side ? Un[v] : Uo[v];
        const double fm = side ? Fo[v] : Fn[v], fp = side ? Fn[v] : Fo[v];
        sH[(f * NV + v) * L + ln.t] = 0.5 * ((fm + fp) - al * (up - um));
      }
    }
  }
  __syncwarp();

  // ---------------------------------------------------------- volume + epilogue
  double* gout = p.out + ebase;
  double un[2][NV];
  // Euler stages without b-terms: D^T = F_x^T K_x^T + K_y F_y^T, the same
  // fragments with the operands swapped, so the accumulator holds D at the
  // lane's own flux nodes (i = 2c + s, j = r), n0 and n0 + 1: one 16-byte
  // store per variable instead of two 8-byte ones.  Measured (profiles/r02/
  // dt2_ab.jsonl): C3 2.237 -> 2.184 ms/step, C5 18.45 -> 17.90; the last
  // stages (more spills: C5 6.35 -> 6.89 ms) and advection (C2 1-term stages
  // 0.069 -> 0.079 ms) lose, so they keep D.
  constexpr bool DT = NDGX_DT2 != 0 && KIND == 1 && (BM == 0 || NDGX_DT2_LAST != 0);
  const int on0 = DT ? ln.n0 : ln.o0;  // output node s: on0 + s * ostep (slab index i + 8 j)
  constexpr int ostep = DT ? 1 : 8;
  if constexpr (DT) {
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double d0 = 0.0, d1 = 0.0;
    dmma_8x8x4(Bx[0][v], ln.kx[0], d0, d1);  // A = F_x^T (own fluxes), B = K_x^T
    dmma_8x8x4(Bx[1][v], ln.kx[1], d0, d1);
    const double* Fy = sF + v * 64;
    dmma_8x8x4(ln.ky[0], Fy[ln.a0s], d0, d1);  // A = K_y, B = F_y^T (F_y[i=r][j=2c+h])
    dmma_8x8x4(ln.ky[1], Fy[ln.a1s], d0, d1);
    // lifted face fluxes: y faces on rows r = 0 / N-1 (line i), x faces on
    // columns i = 0 / N-1 (line j = r)
    const double* hy = sH + (ln.gf * NV + v) * L + 2 * ln.c;
    d0 = fma(ln.gco, hy[0], d0);
    d1 = fma(ln.gco, hy[1], d1);
    d0 = fma(ln.fco0, sH[((PAD ? ln.ff0 : 0) * NV + v) * L + ln.r], d0);
    d1 = fma(ln.fco1, sH[((PAD ? ln.ff1 : 1) * NV + v) * L + ln.r], d1);
    double o0 = d0 * dt, o1 = d1 * dt;
    if (last) {
      const double2 S = *reinterpret_cast<const double2*>(sS + v * 64 + ln.n0s);
      o0 = fma(p.b_last, o0, S.x);
      o1 = fma(p.b_last, o1, S.y);
    }
    if constexpr (PAD) {
      if (ln.vm & 1) gout[v * NPE + ln.g0] = o0;
      if (ln.vm & 2) gout[v * NPE + ln.g0 + 1] = o1;
      // a padded output node: rho = 1, momentum 0 (finite; its wavespeed a
      // is below every real node's, so the alpha max is unchanged)
      un[0][v] = (ln.vm & 1) ? o0 : (v == 0 ? 1.0 : 0.0);
      un[1][v] = (ln.vm & 2) ? o1 : (v == 0 ? 1.0 : 0.0);
    } else {
      *reinterpret_cast<double2*>(gout + v * NPE + ln.n0) = make_double2(o0, o1);
      un[0][v] = o0;
      un[1][v] = o1;
    }
  }
  } else {
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double d0 = 0.0, d1 = 0.0;
    dmma_8x8x4(ln.kx[0], Bx[0][v], d0, d1);  // D_x = K_x F_x
    dmma_8x8x4(ln.kx[1], Bx[1][v], d0, d1);
    const double* Fy = sF + v * 64;
    dmma_8x8x4(Fy[ln.a0s], ln.ky[0], d0, d1);  // += F_y K_y^T, A = F_y[i=r][j=2c+h]
    dmma_8x8x4(Fy[ln.a1s], ln.ky[1], d0, d1);
    // lifted face fluxes: x faces on rows r = 0 / N-1 (line j), y faces on
    // columns j = 0 (s = 0 of c = 0) / N-1 (N = 8: s = 1 of c = 3) (line i = r)
    const double* hx = sH + (ln.xf * NV + v) * L + 2 * ln.c;
    d0 = fma(ln.xco, hx[0], d0);
    d1 = fma(ln.xco, hx[1], d1);
    if constexpr (PAD) {
      d0 = fma(ln.yco0, sH[(ln.yf0 * NV + v) * L + ln.r], d0);
      d1 = fma(ln.yco1p, sH[(ln.yf1 * NV + v) * L + ln.r], d1);
    } else {
      d0 = fma(ln.yco0, sH[(2 * NV + v) * L + ln.r], d0);
      d1 = fma(ln.yco1, sH[(3 * NV + v) * L + ln.r], d1);
    }
    const double k0 = d0 * dt, k1 = d1 * dt;
    const int o0 = PAD ? ln.og0 : ln.o0, o1 = PAD ? ln.og1 : ln.o0 + 8;
    const bool w0 = !PAD || (ln.vm & 4) != 0, w1 = !PAD || (ln.vm & 8) != 0;
    if (!last) {
      if (w0) gout[v * NPE + o0] = k0;
      if (w1) gout[v * NPE + o1] = k1;
    } else {
      const double S0 = sS[v * 64 + ln.a0s], S1 = sS[v * 64 + ln.a1s];
      un[0][v] = fma(p.b_last, k0, S0);
      un[1][v] = fma(p.b_last, k1, S1);
      if (w0) gout[v * NPE + o0] = un[0][v];
      if (w1) gout[v * NPE + o1] = un[1][v];
      // a padded output node: rho = 1, momentum 0 (finite; its wavespeed a
      // is below every real node's, so the alpha max is unchanged)
      if (!w0) un[0][v] = v == 0 ? 1.0 : 0.0;
      if (!w1) un[1][v] = v == 0 ? 1.0 : 0.0;
    }
  }
  }
  if (last) {
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      double sum = un[s2][0];  // non-finite iff some component is
#pragma unroll
      for (int v = 1; v < NV; ++v) sum += un[s2][v];
      if (!isfinite(sum)) record_error(p.ctl, error_key(step, kPhaseInstability, p.block_id, 0));
      if (KIND == 1 && p.scan_alpha) {
        if (!(un[s2][0] > 0.0)) {
          const int n = on0 + ostep * s2;
          const long long gx = cx + p.goff[0], gy = cy + p.goff[1];
          record_error(p.ctl, error_key(step + 1, kPhaseScan, (gx * p.gcells[1] + gy) * (long long)p.gcells[2],
                                        (n & 7) * N + (n >> 3)));
        } else {
          // the same IEEE expression as alpha_scan_kernel, so a restarted run
          // (whose first alpha comes from the scan) reproduces dt bit for bit
          const double mm = dmax(fabs(un[s2][1]), fabs(un[s2][2]));
          alpha = dmax(alpha, __dadd_rn(__ddiv_rn(mm, un[s2][0]), p.sound_speed));
        }
      }
    }
  }
  __syncwarp();  // this element's slab reads precede the next element's writes
}

// ============================================================ stage kernel
// Resident CTAs per SM the register allocation is capped for (4 warps each):
// 4 (<= 128 registers, 16 warps) by default -- capping at 80 for 24 warps
// measured 25% slower on the flagship (less load-level parallelism per warp).
// The 3D order-4 Euler line body (C4) is measured per signature, per-stage
// minima of repeated runs at caps 2..5 (profiles/r02/c4_zsplit_regcap.jsonl):
// 4 (<= 128 registers, 16 warps) for the u-only and 1..5-term RK6 stages
// (3.73 / 4.62 / 5.42 / 6.22 / 7.36 / 8.87 ms), 2 (<= 255 registers: every
// K_j load of a face node in flight) for the 7-array last stage (10.35 ms vs
// 12.22 at 3 and 13.93 at 4).
__host__ __device__ constexpr int stage_minb(int dim, int n, int kind, bool exact, int sig) {
#ifdef NDGX_MINB
  return NDGX_MINB + 0 * (dim + n + kind + (exact ? 1 : 0) + sig);
#else
#ifndef NDGX_MINB3
#define NDGX_MINB3 0x244443344ull  // per signature, one hex digit each (sig 8 ... sig 0)
#endif
#ifndef NDGX_MINB2
#define NDGX_MINB2 0x444  // the 2D order-8 Euler flagship, same classes: last (bm != 0) | others | u-only
#endif
#ifndef NDGX_MINBP
#define NDGX_MINBP 0x555  // the padded flagship body (2D Euler o5-o7), the same classes
#endif
#ifndef NDGX_MINBA
#define NDGX_MINBA 0x445  // the 2D order-8 advection flagship (C2), the same classes
#endif
  // (generic bodies: 2D o4 5 CTAs, 1.03e11 -> 1.05e11 Euler; 2D o6 Euler 3 CTAs, 7.2e10 -> 7.9e10;
  //  2D o5 advection 5 CTAs, 7.6e10 -> 8.1e10.  The advection flagship's u-only
  //  stage at 5 CTAs: C2 stage 0 0.0505 -> 0.0463 ms (profiles/r02/c2_caps_after_prefetch.jsonl).  The padded flagship body at 5 CTAs:
  //  Euler o5 / o6 / o7 8.1 / 11.9 / 13.9e10 -> 9.0 / 12.2 / 15.5e10, profiles/r02/padded_mma_tune.jsonl)
  return (dim == 3 && n == 4 && kind == 1 && !exact)
             ? (int)((NDGX_MINB3 >> (4 * sig)) & 15)
         : (dim == 2 && n == 8 && kind == 1 && !exact)
             ? (sig == 0 ? (NDGX_MINB2 & 15)
                         : ((kSigs[sig].bm != 0) ? (NDGX_MINB2 >> 8 & 15) : (NDGX_MINB2 >> 4 & 15)))
         : (dim == 2 && n == 8 && kind == 0 && !exact)
             ? (sig == 0 ? (NDGX_MINBA & 15)
                         : ((kSigs[sig].bm != 0) ? (NDGX_MINBA >> 8 & 15) : (NDGX_MINBA >> 4 & 15)))
         : (dim == 2 && n >= 5 && n < 8 && ((NDGX_MMA2_ORDERS >> n) & 1) != 0 && kind == 1 && !exact)
             ? (sig == 0 ? (NDGX_MINBP & 15)
                         : ((kSigs[sig].bm != 0) ? (NDGX_MINBP >> 8 & 15) : (NDGX_MINBP >> 4 & 15)))
         : (dim == 2 && n == 5 && kind == 0 && !exact) ? 5
         : (dim == 2 && n == 4 && !exact) ? 5
         : (dim == 2 && n == 6 && kind == 1 && !exact) ? 3
                                                        : 4;
#endif
}

// SIG indexes kSigs: the stage's term structure (p.nu, p.amask, p.bmask) at
// compile time, so the term loops resolve without predicates
template <int DIM, int N, int KIND, bool EXACT, int SIG, bool XF = false>
__global__ void __launch_bounds__(Geo<DIM, N, KIND>::THREADS, stage_minb(DIM, N, KIND, EXACT, SIG))
stage_kernel(const __grid_constant__ StageArgs p) {
  using G = Geo<DIM, N, KIND>;
  using A = Ar<EXACT>;
  constexpr int NV = G::NV, L = G::L, NPE = G::NPE, HW = G::HW;
  constexpr bool USE_MMA = G::MMA && !EXACT;
  constexpr bool USE_MMA3 = G::MMA3 && G::mma_body(EXACT, SIG);
  constexpr int NU = kSigs[SIG].nu, AM = kSigs[SIG].am, BM = kSigs[SIG].bm;
  // generic body: face traces hold U only; the face lane recomputes its own
  // side's flux and speed (fewer partial-warp shared stores)
  constexpr bool GEN_UTRACE = NDGX_GEN_UTRACE != 0;
  extern __shared__ __align__(16) double smem[];

  Control* ctl = p.ctl;
  // inactive step, or an earlier stage already failed: keep the inputs of the
  // failing stage intact for the host's error report
  if (!p.rhs_only && (*(volatile int*)&ctl->skip || *(volatile unsigned long long*)&ctl->err_key != kNoError))
    return;

  const int C0 = p.cells[0], C1 = p.cells[1], C2 = p.cells[2];
  // this CTA's element range (blockIdx.y): e = begin, begin + stride, ... < end
  const int e_lo = p.rng[blockIdx.y][0], nelem = p.rng[blockIdx.y][1];  // element counts are < 2^31
  const int e_stride = p.rng[blockIdx.y][2];
  // the last stage is exactly the signature with b-terms (kSigs), so the
  // epilogue variant is resolved at compile time
  constexpr bool last = kSigs[SIG].bm != 0;
  const double dt = p.rhs_only ? 1.0 : ctl->dt;
  const long long step = p.rhs_only ? 0 : ctl->steps;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  constexpr int SLOT = (1 + NU) * G::SLOT1;  // one ring slot (doubles): arrays | face neighbour values
  const int depth = G::TMA_OK ? p.depth : 0;  // 0: the node phase reads HBM directly
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + wib * G::MAXD;
  constexpr bool LASTC = kSigs[SIG].bm != 0;
  constexpr int WSL = G::wslab(USE_MMA || USE_MMA3, LASTC);
  // slab: fluxes (2D MMA: F_y; 3D MMA: F_x|F_y|F_z) | S (last stage) | traces | face fluxes
  constexpr int OFFT = USE_MMA ? (1 + (LASTC ? 1 : 0)) * NV * 64  // (2D: the padded 8 x 8 grid)
                               : (USE_MMA3 ? (3 + (LASTC ? 1 : 0)) * NV * NPE : G::OFF_T);
  constexpr int TRW = USE_MMA3 ? NV + 1 : (USE_MMA ? HW : G::TW);  // trace record width
  constexpr int LS = USE_MMA ? 8 : L;                              // trace slots per face
  double* sF = smem + G::HEAD + wib * (WSL + depth * SLOT);
  double* sT = sF + OFFT;                                    // [face][TRW][LS]
  double* sH = sT + G::FACES * TRW * LS;                     // [face][NV][LS]
  double* ring = sF + WSL;                                   // [depth][1+NU][NV][NPE] | faces
  const long long nwarps = (long long)gridDim.x * G::WARPS;
  double alpha = 0.0;
  if (lane == 0)
    for (int q = 0; q < depth; ++q) mbar_init(&bar[q], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // K rows for the generic body (one CTA barrier per launch, before any element)
  double* const sK = smem + G::WARPS * G::MAXD + G::RED;
  if constexpr (!USE_MMA && !USE_MMA3) {
    for (int q = threadIdx.x; q < DIM * N * N; q += G::THREADS) {
      const int d = q / (N * N), r = q - d * N * N;
      sK[(d * N + r / N) * G::KROW + r % N] = p.K[d][r];
    }
    __syncthreads();
  }
  __syncwarp();
  // lane 0 streams element ee's u and K_j into ring slot q with one bulk copy each
  // element ee = (ex, ey, ez): lane 0 streams its u and K_j into ring slot q
  // with one bulk copy each; with FACE_PF every face lane also copies its
  // neighbour face node (or the received plane) with cp.async (one group)
  auto issue = [&](int ee, int ex, int ey, int ez, int q) {
    double* dst = ring + q * SLOT;
    const size_t off = (size_t)ee * G::CHUNK;
    if (lane == 0) {
      mbar_arrive_expect_tx(&bar[q], (uint32_t)((1 + NU) * G::CHUNK * 8));
      bulk_g2s(dst, p.u + off, G::CHUNK * 8, &bar[q]);
#pragma unroll
      for (int t = 0; t < NU; ++t) bulk_g2s(dst + (1 + t) * G::CHUNK, p.ku[t] + off, G::CHUNK * 8, &bar[q]);
    }
    if constexpr (G::FACE_PF) {
      double* fr = dst + (1 + NU) * G::CHUNK;  // [array][var][lane]
      if (lane < G::FN) {
        const int f = lane / L, t = lane - f * L;
        const int d = f >> 1, side = f & 1;
        const int ca = d == 0 ? ex : (d == 1 ? ey : ez);
        const int cn = d == 0 ? C0 : (d == 1 ? C1 : C2);
        const bool boundary = side ? (ca == cn - 1) : (ca == 0);
        if (boundary && p.ext[d][side] != nullptr) {
          const size_t xs = d == 0 ? (size_t)ey + (size_t)C1 * ez
                                   : (d == 1 ? (size_t)ex + (size_t)C0 * ez : (size_t)ex + (size_t)C0 * ey);
#pragma unroll
          for (int v = 0; v < NV; ++v) cp_async8(fr + v * 32 + lane, p.ext[d][side] + (xs * NV + v) * L + t);
        } else {
          const int stride = d == 0 ? 1 : (d == 1 ? C0 : C0 * C1);
          const int en = side ? (ca + 1 == cn ? ee - (cn - 1) * stride : ee + stride)
                              : (ca == 0 ? ee + (cn - 1) * stride : ee - stride);
          const size_t g = (size_t)en * (NV * NPE) + G::node(d, t, side ? 0 : N - 1);
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            cp_async8(fr + v * 32 + lane, p.u + g + (size_t)v * NPE);
#pragma unroll
            for (int a = 0; a < NU; ++a) cp_async8(fr + ((1 + a) * NV + v) * 32 + lane, p.ku[a] + g + (size_t)v * NPE);
          }
        }
      }
      cp_async_commit();
    }
  };

  // MMA lane roles (2D, the 8 x 8 grid): lane = 4r + c
  const int r = lane >> 2, c = lane & 3;
  double hc3[KIND == 0 ? 1 : 4] = {};  // line body: the z-hi face flux carried along a z-run
  const double rdy3 = DIM == 3 ? p.lift[1] / p.lift[0] : 1.0, rdz3 = DIM == 3 ? p.lift[2] / p.lift[0] : 1.0;
  const bool scaled3 = DIM == 3 && !(rdy3 == 1.0 && rdz3 == 1.0);  // unequal spacing: K_d = r_d K_0
  Lane4 ln4{};
  if constexpr (USE_MMA3) {
    for (int d = 0; d < 3; ++d) ln4.k[d] = r < 4 ? p.K[d][r * 4 + c] : 0.0;
  }
  Lane8 ln8{};
  if constexpr (USE_MMA) {
    ln8.r = r;
    ln8.c = c;
    ln8.n0 = 2 * c + 8 * r;
    ln8.f = lane >> 3;
    ln8.t = lane & 7;
    const int tn = ln8.t < N ? ln8.t : 0;  // (a padded face lane reads node 0's address)
    // the neighbour's facing node: x-lo (N-1, t), x-hi (0, t), y-lo (t, N-1), y-hi (t, 0)
    ln8.nb_node = ln8.f == 0 ? N - 1 + N * tn : (ln8.f == 1 ? N * tn : (ln8.f == 2 ? tn + N * (N - 1) : tn));
    ln8.o0 = r + 16 * c;
    ln8.n0s = swz8(ln8.n0);
    ln8.a0s = swz8(ln8.o0);
    ln8.a1s = swz8(ln8.o0 + 8);
    ln8.xco = r == 0 ? p.lift[0] : (r == N - 1 ? -p.lift[0] : 0.0);
    ln8.xf = r == N - 1 ? 1 : 0;
    ln8.yco0 = c == 0 ? p.lift[1] : 0.0;
    ln8.yco1 = c == 3 ? -p.lift[1] : 0.0;
    for (int h = 0; h < 2; ++h) {
      const bool in = r < N && 2 * c + h < N;
      ln8.kx[h] = in ? p.K[0][r * N + 2 * c + h] : 0.0;
      ln8.ky[h] = in ? p.K[1][r * N + 2 * c + h] : 0.0;
    }
    if constexpr (N < 8) {
      ln8.g0 = 2 * c + N * r;
      ln8.og0 = r + N * 2 * c;
      ln8.og1 = ln8.og0 + N;
      ln8.vm = (r < N && 2 * c < N ? 5 : 0) | (r < N && 2 * c + 1 < N ? 10 : 0) | (ln8.t < N ? 16 : 0);
      // y faces: output (r, j = 2c + s) takes the lo face at j = 0, the hi face at j = N - 1
      ln8.yf0 = 2 * c == N - 1 ? 3 : 2;
      ln8.yf1 = 2 * c + 1 == N - 1 ? 3 : 2;
      ln8.yco0 = 2 * c == 0 ? p.lift[1] : (2 * c == N - 1 ? -p.lift[1] : 0.0);
      ln8.yco1p = 2 * c + 1 == N - 1 ? -p.lift[1] : 0.0;
    }
    ln8.gco = r == 0 ? p.lift[1] : (r == N - 1 ? -p.lift[1] : 0.0);
    ln8.gf = r == N - 1 ? 3 : 2;
    ln8.fco0 = 2 * c == 0 ? p.lift[0] : (2 * c == N - 1 ? -p.lift[0] : 0.0);
    ln8.fco1 = 2 * c + 1 == N - 1 ? -p.lift[0] : 0.0;
    ln8.ff0 = 2 * c == N - 1 ? 1 : 0;
    ln8.ff1 = 1;
  }

  // element e = cx + C0 (cy + C1 cz), advanced by the total warp count times
  // the range stride with an incremental (x, y, z) counter
  const int nw = (int)nwarps;
  const int es = nw * e_stride;  // element step (< 2^31: ranges stay inside the block)
  const int sx = es % C0, sy = (es / C0) % C1, sz = es / (C0 * C1);
  int e = e_lo + ((int)blockIdx.x * G::WARPS + wib) * e_stride;
  int cx = e % C0, cy = (e / C0) % C1, cz = e / (C0 * C1);
  auto step_coords = [&](int& x, int& y, int& z) {
    x += sx;
    int carry = x >= C0;
    x -= carry ? C0 : 0;
    y += sy + carry;
    carry = y >= C1;
    y -= carry ? C1 : 0;
    z += sz + carry;
  };
  // region filter of a split stage (StageArgs::region): the interior launch
  // takes only the elements inside p.inner (no face on a split axis), the
  // boundary launch only those outside it
  auto skipped = [&](int x, int y, int z) -> bool {
    if (p.region == 0) return false;
    const bool in = x >= p.inner[0][0] && x < p.inner[1][0] && y >= p.inner[0][1] && y < p.inner[1][1] &&
                    z >= p.inner[0][2] && z < p.inner[1][2];
    return in == (p.region == 2);  // regions 1 and 3 take the inside
  };
  // the element `depth - 1` iterations ahead (the next one to issue)
  int ae = e, ax = cx, ay = cy, az = cz;
  for (int q = 0; q + 1 < depth; ++q) {
    if (ae < nelem) issue(ae, ax, ay, az, q);
    else if (G::FACE_PF) cp_async_commit();  // keep one group per slot
    ae += es;
    step_coords(ax, ay, az);
  }
  int slot = 0;
  uint32_t parity = 0;
#ifndef NDGX_XRUN
#define NDGX_XRUN 2  // run length (C3 2.228 vs 2.246 ms/step at 4, 2.284 at 8; C5 18.32 vs 18.46 at 4)
#endif
  // (measured per stage: a win for the Euler last stage, 0.96 -> 0.83 ms on
  // C3, whose x-lo reuse saves two arrays' face loads; a loss elsewhere)
#ifndef NDGX_XRUN_SIGS
#define NDGX_XRUN_SIGS 0x108  // the last stages (bm != 0); the u-only stage had them (0.50 -> 0.48 ms)
#endif                        // until one-ahead loads beat them (NDGX_PF2_SIGS below)
  if constexpr (USE_MMA && NDGX_XRUN > 1 && KIND == 1 && ((NDGX_XRUN_SIGS >> SIG) & 1) != 0) {
    // (unfiltered contiguous launches, or x-filtered ones in the XF
    // instantiation: a region test inside the runs perturbs this
    // register-capped body, so the unfiltered kernel carries none)
    if (depth == 0 && e_stride == 1 && p.region == (XF ? 3 : 0)) {
      // runs of XR consecutive x elements per warp (run ρ -> warp ρ mod nw)
      const int X0 = XF ? p.inner[0][0] : 0, X1 = XF ? p.inner[1][0] : C0;
      constexpr int XR = NDGX_XRUN;
      const long long S = (long long)nw * XR;  // run stride
      const int tx = (int)(S % C0), ty = (int)((S / C0) % C1), tz = (int)(S / ((long long)C0 * C1));
      int rb = e_lo + ((int)blockIdx.x * G::WARPS + wib) * XR;
      int rx = rb % C0, ry = (rb / C0) % C1, rz = rb / (C0 * C1);
      for (; rb < nelem; rb += (int)S) {
        int x = rx, y = ry, z = rz;
        for (int k = 0; k < XR && rb + k < nelem; ++k) {
          // region 3: the rows of the range are interior, only x in [X0, X1) is
          // taken, and the x-lo neighbour is in the slab for x > X0
          if (!XF || (x >= X0 && x < X1))
            element_2d8_fast<N, KIND, NU, AM, BM, SIG>(p, ln8, lane, rb + k, x, y, ring, nullptr, false, sF, sT, sH,
                                                    dt, last, step, alpha, k > 0 && x > X0);
          if (++x == C0) {
            x = 0;
            if (++y == C1) {
              y = 0;
              ++z;
            }
          }
        }
        rx += tx;
        int carry = rx >= C0;
        rx -= carry ? C0 : 0;
        ry += ty + carry;
        carry = ry >= C1;
        ry -= carry ? C1 : 0;
        rz += tz + carry;
      }
      e = nelem;  // done: skip the element loop below
    }
  }
  // The generic body (exact mode, and the contracted shapes without a
  // tensor-core body).  Small elements are processed G::GL lanes per element,
  // G::EPW elements per warp (lane group `grp`, lane `sub` in the group):
  // every lane of a group runs the one-element code with `sub` for `lane`
  // and GL for 32, on its own slab.  `act` false: the lane only keeps the
  // warp's barriers (no element, or one the launch's region skips).
  auto generic_element = [&](const int e, const int cx, const int cy, const int cz, const double* src,
                             const double* fsrc, const bool act) {
    constexpr int GL = G::GL;
    // the 2D order-8 exact body sums its volume terms by line tasks (phase 3)
    constexpr bool LINE8 = NDGX_LINE8 != 0 && EXACT && DIM == 2 && N == 8 && GL == 32;
    // 2D orders 6-7 (and odd-order advection) sum by whole-line tasks
    // (NDGX_LINEG; profiles/r02/lineg_ab.jsonl: 2D Euler o6 8.1e10 -> 8.6e10,
    // advection o6 9.1e10 -> 1.0e11, o7 5.3e10 -> 6.2e10; a loss for o2/o4 and
    // for Euler o3/o5, which keep the per-node sums)
#ifndef NDGX_LINEG3
#define NDGX_LINEG3 0x1C0  // 3D orders (bit N) taking the whole-line volume: 6-8 (o6 1.7e10 -> 2.0e10; o3 and exact o4 lose 15-19%)
#endif
    constexpr bool LINEG = NDGX_LINEG != 0 && !LINE8 &&
                           ((DIM == 2 && (N >= 6 || (KIND == 0 && (N & 1) != 0))) ||
                            (DIM == 3 && ((NDGX_LINEG3 >> N) & 1) != 0));
    // F_x / x-part slot of node (i, j): 8 j + (i ^ j) -- an x line read at a
    // fixed position by 8 lanes (8 lines) covers 8 distinct banks
    auto sx8 = [](int n) { return (n & ~7) | ((n ^ (n >> 3)) & 7); };
    const int sub = GL == 32 ? lane : (lane & (GL - 1)), grp = GL == 32 ? 0 : lane / GL;
    double* const gF = sF + grp * G::GSTRIDE;
    double* const gT = gF + G::OFF_T;
    double* const gH = gF + G::OFF_H;
    const size_t ebase = (size_t)e * NV * NPE;
    auto aos_cell = [&]() -> long long {  // global AoS cell index of this element
      const long long gx = cx + p.goff[0], gy = cy + p.goff[1], gz = cz + p.goff[2];
      return (gx * p.gcells[1] + gy) * (long long)p.gcells[2] + gz;
    };

    // ------------------------------------------------ 1: nodes
    // lane's nodes: n = sub + GL m
    double Sn[G::NMG][NV];  // last stage: S at the lane's nodes
#if NDGX_GPF
    // direct loads: every node's raw values first (one memory latency for
    // all of the lane's nodes instead of one per node).  Measured
    // (profiles/r02/generic_prefetch_ab.jsonl): the 2D order-8 exact body (the
    // drop-in's default mode on C3) 8.95e10 -> 9.6e10; a loss for the other
    // shapes (2D o4/o6 fast -5..-8%, 3D o4 exact -6%), which keep the plain loads
    constexpr bool GPF = DIM == 2 && N == 8;
    double rawn[G::NMG][NV][1 + NU];
    if (GPF && depth == 0) {
#pragma unroll
      for (int m = 0; m < G::NMG; ++m) {
        const int n = sub + GL * m;
        if (!act || n >= NPE) continue;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const size_t g = ebase + (size_t)v * NPE + n;
          rawn[m][v][0] = __ldg(p.u + g);
#pragma unroll
          for (int t = 0; t < NU; ++t) rawn[m][v][1 + t] = __ldg(p.ku[t] + g);
        }
      }
    }
#endif
#pragma unroll
    for (int m = 0; m < G::NMG; ++m) {
      const int n = sub + GL * m;
      if (!act || n >= NPE) continue;
      double U[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double S;
        if (depth > 0)
          combine_s<EXACT, NU, AM, BM>(p, src + v * NPE + n, G::CHUNK, last, U[v], S);
        else
#if NDGX_GPF
        if (GPF)
          combine_s<EXACT, NU, AM, BM>(p, rawn[m][v], 1, last, U[v], S);
        else
#endif
          combine_g<EXACT, NU, AM, BM>(p, ebase + (size_t)v * NPE + n, last, U[v], S);
        Sn[m][v] = S;
      }
      if (KIND == 1 && !(U[0] > 0.0)) {
        // first bad node of the reference's x-volume traversal: (cell, (j,k), i)
        const int i = n % N, j = (n / N) % N, k = n / (N * N);
        const int nkey = (DIM == 2) ? j * N + i : (j * N + k) * N + i;
        record_error(ctl, error_key(step, p.phase, aos_cell(), nkey));
      }
      const double rinv = (!EXACT && KIND == 1) ? fast_rcp(U[0]) : -1.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double F[NV], sp;
        flux<DIM, KIND, EXACT>(p, U, d, F, sp, rinv);
#pragma unroll
        for (int v = 0; v < NV; ++v) gF[(d * NV + v) * NPE + (LINE8 && d == 0 ? sx8(n) : n)] = F[v];
        const int k = G::pos_of(d, n);
        if (k == 0 || k == N - 1) {
          double* t = gT + ((2 * d + (k == 0 ? 0 : 1)) * G::TW) * L + G::line_of(d, n);
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            t[v * L] = U[v];
            if (!GEN_UTRACE) t[(NV + v) * L] = F[v];
          }
          if (!GEN_UTRACE) t[2 * NV * L] = sp;
        }
      }
    }
    __syncwarp();

    // ------------------------------------------------ 2: face fluxes
#pragma unroll
    for (int m = 0; m < G::FMG; ++m) {
      const int q = sub + GL * m;
      if (!act || q >= G::FN) continue;
      const int f = q / L, t = q - f * L;
      const int d = f >> 1, side = f & 1;
      const double* own = gT + (f * G::TW) * L + t;
      // neighbour across (d, side): periodic wrap in this block, or the received plane
      const int ca = d == 0 ? cx : (d == 1 ? cy : cz);
      const int cn = d == 0 ? C0 : (d == 1 ? C1 : C2);
      const bool boundary = side ? (ca == cn - 1) : (ca == 0);
      double Un[NV];
      if (G::FACE_PF && depth > 0) {
        const bool ext = boundary && p.ext[d][side] != nullptr;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double S;
          if (ext) Un[v] = fsrc[v * 32 + lane];
          else combine_s<EXACT, NU, AM, BM>(p, fsrc + v * 32 + lane, NV * 32, false, Un[v], S);
        }
      } else if (boundary && p.ext[d][side] != nullptr) {
        const size_t xs = d == 0 ? (size_t)cy + (size_t)C1 * cz
                                 : (d == 1 ? (size_t)cx + (size_t)C0 * cz : (size_t)cx + (size_t)C0 * cy);
#pragma unroll
        for (int v = 0; v < NV; ++v) Un[v] = __ldg(p.ext[d][side] + (xs * NV + v) * L + t);
      } else {
        // neighbour element index: e -/+ stride_d, wrapped periodically
        const int stride = d == 0 ? 1 : (d == 1 ? C0 : C0 * C1);
        const int en = side ? (ca + 1 == cn ? e - (cn - 1) * stride : e + stride)
                            : (ca == 0 ? e + (cn - 1) * stride : e - stride);
        const size_t g = (size_t)en * (NV * NPE) + G::node(d, t, side ? 0 : N - 1);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double S;
          combine_g<EXACT, NU, AM, BM>(p, g + (size_t)v * NPE, false, Un[v], S);
        }
      }
      double Fn[NV], sn;
      flux<DIM, KIND, EXACT>(p, Un, d, Fn, sn, (!EXACT && KIND == 1) ? fast_rcp(Un[0]) : -1.0);
      // this element's side: U from the trace, flux and speed recomputed
      // (the same function of the same U as in the node phase)
      double Uo[NV], Fo[NV], so;
#pragma unroll
      for (int v = 0; v < NV; ++v) Uo[v] = own[v * L];
      if (GEN_UTRACE) {
        flux<DIM, KIND, EXACT>(p, Uo, d, Fo, so, (!EXACT && KIND == 1) ? fast_rcp(Uo[0]) : -1.0);
      } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) Fo[v] = own[(NV + v) * L];
        so = own[2 * NV * L];
      }
      const double a = dmax(side ? so : sn, side ? sn : so);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        // minus state = lower cell along d (solver.cpp:268-306; models.cpp:77-88)
        const double um = side ? Uo[v] : Un[v], up = side ? Un[v] : Uo[v];
        const double fm = side ? Fo[v] : Fn[v], fp = side ? Fn[v] : Fo[v];
        gH[(f * NV + v) * L + t] = A::mul(0.5, A::sub(A::add(fm, fp), A::mul(a, A::sub(up, um))));
      }
    }
    __syncwarp();

    // ------------------------------------------------ 3: volume, faces, epilogue
    // 2D order 8, exact: the volume sums by line tasks.  Lane = (axis d =
    // lane / 16, line t, half): outputs k = 4 half .. 4 half + 3 of line t,
    // every variable, each sum in the reference's order (one pass over the
    // line's 8 fluxes instead of 8 slab reads per output and axis).  The x
    // part (with its lifted faces) and the bare y sum go back into the flux
    // slab; each node owner then finishes D = Dx + Sy + y lifts exactly as
    // the per-node loop below does, so the states stay bit-identical.
    if constexpr (LINEG) {
      // general 2D shapes: whole lines, task q = sub + GL r (x lines t = q,
      // y lines t = q - N); each F slot is read only by its own line's task,
      // so the parts go back in place as they are formed
#pragma unroll
      for (int q0 = 0; q0 < DIM * L; q0 += GL) {
        const int q = q0 + sub;
        if (act && q < DIM * L) {
          const int d = q / L, t = q - d * L;
          double* Fd = gF + d * NV * NPE;
          double fl[NV][N];
#pragma unroll
          for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int l = 0; l < N; ++l) fl[v][l] = Fd[v * NPE + G::node(d, t, l)];
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const double* Kr = sK + (d * N + k) * G::KROW;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              double acc = A::mul(Kr[0], fl[v][0]);
#pragma unroll
              for (int l = 1; l < N; ++l) acc = A::mac(acc, Kr[l], fl[v][l]);
              if (d == 0) {
                acc = zero_plus(acc);
                if (k == 0) acc = A::add(acc, A::mul(p.lift[0], gH[(0 * NV + v) * L + t]));
                if (k == N - 1) acc = A::sub(acc, A::mul(p.lift[0], gH[(1 * NV + v) * L + t]));
              }
              Fd[v * NPE + G::node(d, t, k)] = acc;
            }
          }
        }
      }
      __syncwarp();
    }
    if constexpr (LINE8) {
      const int d = lane >> 4, t = (lane >> 1) & 7, half = lane & 1;
      double fl[NV][N];
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int l = 0; l < N; ++l) fl[v][l] = gF[(d * NV + v) * NPE + (d == 0 ? sx8(l + 8 * t) : t + 8 * l)];
      double res[4][NV];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        // the halves interleave (k = 2 kk + half): the in-place stores below
        // then hit 16 distinct bank pairs per half-warp (k = 4 half + kk put
        // both halves on the same pairs: 4 wavefronts per store, 2 excessive)
        const int k = 2 * kk + half;
        const double* Kr = sK + (d * N + k) * G::KROW;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double acc = A::mul(Kr[0], fl[v][0]);
#pragma unroll
          for (int l = 1; l < N; ++l) acc = A::mac(acc, Kr[l], fl[v][l]);
          if (d == 0) {
            acc = zero_plus(acc);
            if (k == 0) acc = A::add(acc, A::mul(p.lift[0], gH[(0 * NV + v) * L + t]));
            if (k == N - 1) acc = A::sub(acc, A::mul(p.lift[0], gH[(1 * NV + v) * L + t]));
          }
          res[kk][v] = acc;
        }
      }
      __syncwarp();  // every line's flux reads precede the in-place stores
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int k = 2 * kk + half;
#pragma unroll
        for (int v = 0; v < NV; ++v) gF[(d * NV + v) * NPE + (d == 0 ? sx8(k + 8 * t) : t + 8 * k)] = res[kk][v];
      }
      __syncwarp();
    }
#pragma unroll
    for (int m = 0; m < G::NMG; ++m) {
      const int n = sub + GL * m;
      if (!act || n >= NPE) continue;
      double un[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double D = 0.0;
        if constexpr (LINE8 || LINEG) {
          // D = x part (with x lifts), then per further axis: + its sum, its lifts
          D = gF[v * NPE + (LINE8 ? sx8(n) : n)];
#pragma unroll
          for (int d = 1; d < DIM; ++d) {
            const int k = G::pos_of(d, n), t = G::line_of(d, n);
            D = A::add(D, gF[(d * NV + v) * NPE + n]);
            if (k == 0) D = A::add(D, A::mul(p.lift[d], gH[((2 * d) * NV + v) * L + t]));
            if (k == N - 1) D = A::sub(D, A::mul(p.lift[d], gH[((2 * d + 1) * NV + v) * L + t]));
          }
        }
#pragma unroll
        for (int d = 0; d < (LINE8 || LINEG ? 0 : DIM); ++d) {
          const int k = G::pos_of(d, n), t = G::line_of(d, n);
          const double* Fl = gF + (d * NV + v) * NPE;
          const double* Kr = sK + (d * N + k) * G::KROW;
          // 0 + K0 F0 + K1 F1 + ...: the leading 0 + only normalises a -0,
          // which zero_plus (axis 0) or the add onto dudt (axes > 0) reproduces
          double acc = A::mul(Kr[0], Fl[G::node(d, t, 0)]);
#pragma unroll
          for (int l = 1; l < N; ++l) acc = A::mac(acc, Kr[l], Fl[G::node(d, t, l)]);
          D = d == 0 ? zero_plus(acc) : A::add(D, acc);
          if (k == 0) D = A::add(D, A::mul(p.lift[d], gH[((2 * d) * NV + v) * L + t]));
          if (k == N - 1) D = A::sub(D, A::mul(p.lift[d], gH[((2 * d + 1) * NV + v) * L + t]));
        }
        const size_t gi = ebase + (size_t)v * NPE + n;
        const double kv = A::mul(D, dt);  // k_i *= dt (solver.hpp:66-67)
        if (!last) {
          p.out[gi] = kv;
        } else {
          un[v] = p.b_last != 0.0 ? A::mac(Sn[m][v], p.b_last, kv) : Sn[m][v];
          p.out[gi] = un[v];
        }
      }
      if (last) {
        bool fin = true;
#pragma unroll
        for (int v = 0; v < NV; ++v) fin = fin && isfinite(un[v]);
        if (!fin) record_error(ctl, error_key(step, kPhaseInstability, p.block_id, 0));
        if (KIND == 1 && p.scan_alpha) {
          if (!(un[0] > 0.0)) {
            record_error(ctl, error_key(step + 1, kPhaseScan, aos_cell(), G::aos_node(n)));
          } else {
            double mm = 0.0;
#pragma unroll
            for (int d = 0; d < DIM; ++d) mm = dmax(mm, fabs(un[1 + d]));
            alpha = dmax(alpha, __dadd_rn(__ddiv_rn(mm, un[0]), p.sound_speed));
          }
        }
      }
    }
    __syncwarp();  // this element's slab reads precede the next element's writes
  };


#ifndef NDGX_RUN3
#define NDGX_RUN3 2  // 3D traversal of whole-plane launches: 0 element order, 1 x-runs, 2 z-runs
#endif
#ifndef NDGX_RUNLEN3
#define NDGX_RUNLEN3 8  // z-run length: DRAM bytes per C4 step 1.13x the algorithmic (1.17x at 16, 1.12x at 4), same time
#endif
#ifndef NDGX_YB3
#define NDGX_YB3 8
#endif
#ifndef NDGX_REUSE3
#define NDGX_REUSE3 1
#endif
  // 3D: runs of consecutive elements along z (x-runs: along x, in y-blocks of
  // NDGX_YB3 rows) per warp.  In element order (x fastest) the z neighbour
  // is C0*C1 elements away and, at the many-term RK6 stages, falls out of L2
  // before it is read again (C4 stage 5: 1.5x the compulsory DRAM bytes).
  // In a z-run the z neighbours are this warp's previous and next elements,
  // and the tensor-core body takes the lo-face flux from the previous one.
  if constexpr (DIM == 3 && NDGX_RUN3 != 0 && G::GL == 32) {
    const int plane = C0 * C1;
    if (depth == 0 && e_stride == 1 && p.region == 0 && e_lo % plane == 0 && nelem % plane == 0 && nelem > e_lo) {
      const int z0 = e_lo / plane, nz = nelem / plane - z0;
      const int w0 = (int)blockIdx.x * G::WARPS + wib;
      auto visit = [&](int x, int y, int z, bool prev, int par) {
        const int ee = x + C0 * (y + C1 * z);
        if constexpr (USE_MMA3 && NDGX_LINES3 != 0)
          element_3d4_lines<KIND, NU, AM, BM>(p, lane, ee, x, y, z, sF, sF + NV * NPE, dt, step, alpha,
                                              NDGX_RUN3 == 2 && NDGX_REUSE3 != 0 && prev, hc3, rdy3, rdz3,
                                              scaled3);
        else if constexpr (USE_MMA3)
          element_3d4_fast<KIND, NU, AM, BM, NDGX_RUN3 == 2 ? 2 : 0>(p, ln4, lane, ee, x, y, z, sF, sT, sH, dt, step,
                                                                    alpha, NDGX_REUSE3 != 0 && prev, par);
        else
          generic_element(ee, x, y, z, nullptr, nullptr, true);
      };
      if (NDGX_RUN3 == 2) {
        const int ZR = nz < NDGX_RUNLEN3 ? nz : NDGX_RUNLEN3;
        const int nzc = (nz + ZR - 1) / ZR;
        for (int rho = w0; rho < plane * nzc; rho += nw) {
          const int zc = rho / plane, xy = rho - zc * plane;
          const int y = xy / C0, x = xy - y * C0;
          const int zb = z0 + zc * ZR, ze = min(zb + ZR, z0 + nz);
          for (int z = zb; z < ze; ++z) visit(x, y, z, z > zb, (z - zb) & 1);
        }
      } else {
        const int XR = C0 < NDGX_RUNLEN3 ? C0 : NDGX_RUNLEN3;
        const int nxc = (C0 + XR - 1) / XR;
        const int YB = (C1 % NDGX_YB3 == 0) ? NDGX_YB3 : C1;
        const int nruns = nxc * C1 * nz;
        for (int rho = w0; rho < nruns; rho += nw) {
          int q = rho / nxc;
          const int xc = rho - q * nxc;
          const int yy = q % YB;
          q /= YB;
          const int z = z0 + q % nz, yb = q / nz;
          const int y = yb * YB + yy, xb = xc * XR, xe = min(xb + XR, C0);
          for (int x = xb; x < xe; ++x) visit(x, y, z, x > xb, (x - xb) & 1);
        }
      }
      e = nelem;  // done: skip the element loop below
    }
  }

  // generic body with several elements per warp: chunks of EPW consecutive
  // range elements, chunk c -> warp c mod nw
  if constexpr (G::GL < 32 && !USE_MMA) {
    const int grp = lane / G::GL;
    const long long cnt = ((long long)nelem - e_lo + e_stride - 1) / e_stride;  // elements of this range
    for (long long c = (long long)blockIdx.x * G::WARPS + wib; c * G::EPW < cnt; c += nw) {
      const long long k = c * G::EPW + grp;
      const bool have = k < cnt;
      const int ee = (int)(e_lo + (have ? k : 0) * e_stride);
      const int x = ee % C0, y = (ee / C0) % C1, z = ee / (C0 * C1);
      generic_element(ee, x, y, z, nullptr, nullptr, have && !skipped(x, y, z));
    }
    e = nelem;  // done: skip the element loop below
  }
#ifndef NDGX_PF2
#define NDGX_PF2 1
#endif
  // advection flagship: each element's loads issued one element ahead (two
  // register buffers, alternating), so a warp's memory latency overlaps the
  // previous element's work.  Measured (profiles/r02/c2_prefetch_ab.jsonl):
  // C2 0.277 -> 0.241 ms/step, advection o8 at 1e8 DOF 1.54e11 -> 1.80e11.
  // The Euler u-only stage waits on its node loads (35% of its samples at
  // the first use of U) and takes it too, in place of its x-runs: C3 2.173 ->
  // 2.145, C5 17.74 -> 17.58 ms/step (medians of 5, c3_stage0_prefetch_ab.jsonl).
  // The other Euler stages are L1/LSU-bound and lose (C3 2.168 -> 2.193 ms
  // at 3 CTAs/SM, spills at 4: negative/c3_c5_euler_prefetch.jsonl).
#ifndef NDGX_PF2_EULER
#define NDGX_PF2_EULER 1
#endif
#ifndef NDGX_PF2_SIGS
#define NDGX_PF2_SIGS 0x1  // the Euler signatures it applies to: the u-only stage
#endif
  if constexpr (USE_MMA && N == 8 && NDGX_PF2 != 0 && NU <= 3 &&  // (5+ arrays spill)
                (KIND == 0 || (NDGX_PF2_EULER != 0 && ((NDGX_PF2_SIGS >> SIG) & 1) != 0 &&
                               ((NDGX_XRUN_SIGS >> SIG) & 1) == 0))) {
    if (depth == 0 && p.region == 0) {
      Pre8<NV, NU> qa, qb;
      if (e < nelem) preload_2d8<KIND, NU>(p, ln8, e, cx, cy, qa);
      while (e < nelem) {
        int x2 = cx, y2 = cy, z2 = cz;
        step_coords(x2, y2, z2);
        const int e2 = e + es;
        if (e2 < nelem) preload_2d8<KIND, NU>(p, ln8, e2, x2, y2, qb);
        element_2d8_fast<N, KIND, NU, AM, BM, SIG, true>(p, ln8, lane, e, cx, cy, nullptr, nullptr, false, sF, sT, sH,
                                                         dt, last, step, alpha, false, &qa);
        e = e2;
        cx = x2;
        cy = y2;
        cz = z2;
        if (e >= nelem) break;
        step_coords(x2, y2, z2);
        const int e3 = e + es;
        if (e3 < nelem) preload_2d8<KIND, NU>(p, ln8, e3, x2, y2, qa);
        element_2d8_fast<N, KIND, NU, AM, BM, SIG, true>(p, ln8, lane, e, cx, cy, nullptr, nullptr, false, sF, sT, sH,
                                                         dt, last, step, alpha, false, &qb);
        e = e3;
        cx = x2;
        cy = y2;
        cz = z2;
      }
    }
  }
  for (; e < nelem; e += es) {
    const double* src = ring + slot * SLOT;  // this element's u and K_j (when depth > 0)
    const double* fsrc = src + (1 + NU) * G::CHUNK;  // its face neighbour values (FACE_PF)
    if (depth > 0) {
      // keep depth-1 elements in flight: refill the slot the previous element used
      if (ae < nelem) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads first
        issue(ae, ax, ay, az, (slot + depth - 1) % depth);
      } else if (G::FACE_PF) {
        cp_async_commit();
      }
      ae += es;
      step_coords(ax, ay, az);
      mbar_wait(&bar[slot], parity);
      if constexpr (G::FACE_PF) {
        // this element's group is the oldest of the depth in flight
        if (depth == 2) cp_async_wait<1>();
        else if (depth == 3) cp_async_wait<2>();
        else cp_async_wait<3>();
      }
    }
    if (skipped(cx, cy, cz)) {  // not in this launch's region (its ring slot is consumed unread)
      if (depth > 0 && ++slot == depth) {
        slot = 0;
        parity ^= 1;
      }
      step_coords(cx, cy, cz);
      continue;
    }
    if constexpr (USE_MMA3 && NDGX_LINES3 != 0) {
      element_3d4_lines<KIND, NU, AM, BM>(p, lane, e, cx, cy, cz, sF, sF + NV * NPE, dt, step, alpha, false, hc3, rdy3,
                                          rdz3, scaled3);
      step_coords(cx, cy, cz);
      continue;
    } else if constexpr (USE_MMA3) {
      element_3d4_fast<KIND, NU, AM, BM>(p, ln4, lane, e, cx, cy, cz, sF, sT, sH, dt, step, alpha);
      step_coords(cx, cy, cz);
      continue;
    }
    if constexpr (USE_MMA) {
      element_2d8_fast<N, KIND, NU, AM, BM, SIG>(p, ln8, lane, e, cx, cy, src, fsrc, depth > 0, sF, sT, sH, dt, last, step,
                                         alpha);
      if (depth > 0 && ++slot == depth) {
        slot = 0;
        parity ^= 1;
      }
      step_coords(cx, cy, cz);
      continue;
    }
    generic_element(e, cx, cy, cz, src, fsrc, true);
    if (depth > 0 && ++slot == depth) {
      slot = 0;
      parity ^= 1;
    }
    step_coords(cx, cy, cz);
  }
  if constexpr (G::FACE_PF) cp_async_wait<0>();  // no copy outlives the kernel

  if (KIND == 1 && last && p.scan_alpha) {
    // block max of the non-negative wavespeeds on their IEEE bit patterns
    alpha = warp_max(alpha);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(smem) + G::WARPS * G::MAXD;
    if (lane == 0) red[wib] = (unsigned long long)__double_as_longlong(alpha);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long mx = 0ull;
      for (int q = 0; q < G::WARPS; ++q) mx = red[q] > mx ? red[q] : mx;
      atomicMax(&ctl->alpha_bits, mx);
    }
  }
}

}  // namespace ndgx
