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
// Execution model: ONE ELEMENT PER WARP.  Every warp of a persistent grid
// walks elements e = warp_id, warp_id + total_warps, ... (x fastest, so
// neighbouring warps work on neighbouring elements and face-neighbour reads
// hit L2) and runs, warp-locally with only __syncwarp between the steps:
//   1  node phase: each lane forms the stage input U_s = u + sum a K at its
//      nodes straight from HBM (all of a lane's loads in flight together),
//      the flux along every axis and the one-sided speeds; fluxes go to a
//      warp-private shared-memory slab, face nodes also to a trace slab
//   2  face phase: one lane per face node loads the neighbour element's face
//      node (or the received multi-block plane), forms its stage input, flux
//      and speed, and the Lax-Friedrichs flux of every variable
//   3  output phase: the volume quadrature of every axis, the lifted face
//      fluxes and the RK epilogue (K_s = dt*dudt, or u_new = S + b_s K_s,
//      finite check, next-step wavespeed), stored straight to HBM.
// No block barriers, no producer warps: latency is hidden by the many
// independent warps per SM, and HBM traffic is the compulsory one array pass
// per input and output (neighbour face nodes are L2 hits).
//
// Two volume back-ends:
//   EXACT     the reference's operation order with _rn intrinsics (bit-
//             identical states): per output node and axis, 0 + K0 F0 + ...,
//             added once, faces after each axis.
//   FAST, 2D N=8 (the flagship)  FP64 tensor cores, mma.sync.m8n8k4.f64: with
//             lane = 4r + c the lane evaluates fluxes at nodes (i=c+4h, j=r),
//             which are exactly its B fragments of D_x = K_x F_x; one
//             warp-local transpose gives the A fragments of D_y = F_y K_y^T,
//             accumulated onto D_x, and both land on nodes (i=r, j=2c+s).
//   FAST, other shapes: the exact loop structure with contracted FMAs.
#pragma once

namespace ndgx {

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
  static constexpr int WARPS = 4;                                     // warps per CTA
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int MAXD = 4;                                      // max ring depth per warp
  // shared memory: [mbarriers WARPS*MAXD][scratch RED] then per warp a slab
  // (doubles): fluxes [DIM][NV][NPE] | traces [face][HW][L] | face fluxes
  // [face][NV][L], followed by the warp's ring of D element slots, each
  // holding u and the NU K_j of one element ([array][var][node], TMA-filled)
  static constexpr int OFF_T = DIM * NV * NPE;
  static constexpr int OFF_H = OFF_T + FACES * HW * L;
  static constexpr int WSLAB = ((OFF_H + FACES * NV * L) + 1) & ~1;
  static constexpr int RED = 2 * WARPS;                      // block reduction scratch (doubles)
  static constexpr int HEAD = WARPS * MAXD + RED;            // 8-byte words before the slabs
  static constexpr int CHUNK = NV * NPE;                     // one array of one element (doubles)
  static constexpr bool TMA_OK = (CHUNK % 2) == 0;           // 16-byte element chunks
  static constexpr bool MMA = (DIM == 2 && N == 8);          // FAST-mode tensor-core volume
  static constexpr int smem_bytes(int nu, int depth) { return (HEAD + WARPS * (WSLAB + depth * (1 + nu) * CHUNK)) * 8; }

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

// ============================================================ stage kernel
// SIG indexes kSigs: the stage's term structure (p.nu, p.amask, p.bmask) at
// compile time, so the term loops resolve without predicates
template <int DIM, int N, int KIND, bool EXACT, int SIG>
__global__ void __launch_bounds__(Geo<DIM, N, KIND>::THREADS, 4)
stage_kernel(const __grid_constant__ StageArgs p) {
  using G = Geo<DIM, N, KIND>;
  using A = Ar<EXACT>;
  constexpr int NV = G::NV, L = G::L, NPE = G::NPE, HW = G::HW;
  constexpr bool USE_MMA = G::MMA && !EXACT;
  constexpr int NU = kSigs[SIG].nu, AM = kSigs[SIG].am, BM = kSigs[SIG].bm;
  extern __shared__ __align__(16) double smem[];

  Control* ctl = p.ctl;
  // inactive step, or an earlier stage already failed: keep the inputs of the
  // failing stage intact for the host's error report
  if (!p.rhs_only && (*(volatile int*)&ctl->skip || *(volatile unsigned long long*)&ctl->err_key != kNoError))
    return;

  const int C0 = p.cells[0], C1 = p.cells[1], C2 = p.cells[2];
  const long long nelem = (long long)C0 * C1 * C2;
  const bool last = p.is_last != 0;
  const double dt = p.rhs_only ? 1.0 : ctl->dt;
  const long long step = p.rhs_only ? 0 : ctl->steps;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  constexpr int SLOT = (1 + NU) * G::CHUNK;  // one ring slot (doubles)
  const int depth = G::TMA_OK ? p.depth : 0;  // 0: the node phase reads HBM directly
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + wib * G::MAXD;
  double* sF = smem + G::HEAD + wib * (G::WSLAB + depth * SLOT);  // [DIM][NV][NPE]
  double* sT = sF + G::OFF_T;                                     // [face][HW][L]
  double* sH = sF + G::OFF_H;                                     // [face][NV][L]
  double* ring = sF + G::WSLAB;                                   // [depth][1+NU][NV][NPE]
  const long long nwarps = (long long)gridDim.x * G::WARPS;
  double alpha = 0.0;
  if (lane == 0)
    for (int q = 0; q < depth; ++q) mbar_init(&bar[q], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  // lane 0 streams element ee's u and K_j into ring slot q with one bulk copy each
  auto issue = [&](long long ee, int q) {
    double* dst = ring + q * SLOT;
    const size_t off = (size_t)ee * G::CHUNK;
    mbar_arrive_expect_tx(&bar[q], (uint32_t)(SLOT * 8));
    bulk_g2s(dst, p.u + off, G::CHUNK * 8, &bar[q]);
#pragma unroll
    for (int t = 0; t < NU; ++t) bulk_g2s(dst + (1 + t) * G::CHUNK, p.ku[t] + off, G::CHUNK * 8, &bar[q]);
  };

  // MMA lane roles (2D N=8): lane = 4r + c
  const int r = lane >> 2, c = lane & 3;
  double kx[2] = {0.0, 0.0}, ky[2] = {0.0, 0.0};
  if constexpr (USE_MMA) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      kx[h] = p.K[0][r * N + c + 4 * h];  // A of D_x = K_x F_x: K_x[k=r][i=c+4h]
      ky[h] = p.K[1][r * N + c + 4 * h];  // B of D_y = F_y K_y^T: K_y[k=r][j=c+4h]
    }
  }

  // element e = cx + C0 (cy + C1 cz), advanced by the total warp count with
  // an incremental (x, y, z) counter (element counts are < 2^31)
  const int nw = (int)nwarps;
  const int sx = nw % C0, sy = (nw / C0) % C1, sz = nw / (C0 * C1);
  int e = (int)blockIdx.x * G::WARPS + wib;
  int cx = e % C0, cy = (e / C0) % C1, cz = e / (C0 * C1);
  if (lane == 0)
    for (int q = 0; q + 1 < depth; ++q)
      if (e + (long long)q * nw < nelem) issue(e + (long long)q * nw, q);
  int slot = 0;
  uint32_t parity = 0;
  for (; e < nelem; e += nw) {
    const size_t ebase = (size_t)e * NV * NPE;
    const double* src = ring + slot * SLOT;  // this element's u and K_j (when depth > 0)
    if (depth > 0) {
      // keep depth-1 elements in flight: refill the slot the previous element used
      const long long ahead = e + (long long)(depth - 1) * nw;
      if (lane == 0 && ahead < nelem) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads first
        issue(ahead, (slot + depth - 1) % depth);
      }
      mbar_wait(&bar[slot], parity);
    }
    auto aos_cell = [&]() -> long long {  // global AoS cell index of this element
      const long long gx = cx + p.goff[0], gy = cy + p.goff[1], gz = cz + p.goff[2];
      return (gx * p.gcells[1] + gy) * (long long)p.gcells[2] + gz;
    };

    // ------------------------------------------------ 1: nodes
    // lane's nodes: n = lane + 32m (generic) or n = (c + 4h) + 8r (MMA)
    double Bx[G::NM][NV];  // MMA: F_x at the lane's nodes = B fragments of D_x
    double Sn[G::NM][NV];  // last stage: S at the lane's output nodes (generic)
#pragma unroll
    for (int m = 0; m < G::NM; ++m) {
      const int n = USE_MMA ? (c + 4 * m) + N * r : lane + 32 * m;
      if (n >= NPE) continue;
      double U[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double S;
        if (depth > 0)
          combine_s<EXACT, NU, AM, BM>(p, src + v * NPE + n, G::CHUNK, last && !USE_MMA, U[v], S);
        else
          combine_g<EXACT, NU, AM, BM>(p, ebase + (size_t)v * NPE + n, last && !USE_MMA, U[v], S);
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
        if (USE_MMA && d == 0) {
#pragma unroll
          for (int v = 0; v < NV; ++v) Bx[m][v] = F[v];
        } else {
#pragma unroll
          for (int v = 0; v < NV; ++v) sF[(d * NV + v) * NPE + n] = F[v];
        }
        const int k = G::pos_of(d, n);
        if (k == 0 || k == N - 1) {
          double* t = sT + ((2 * d + (k == 0 ? 0 : 1)) * HW) * L + G::line_of(d, n);
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            t[v * L] = U[v];
            t[(NV + v) * L] = F[v];
          }
          t[2 * NV * L] = sp;
        }
      }
    }
    __syncwarp();

    // ------------------------------------------------ 2: face fluxes
#pragma unroll
    for (int m = 0; m < G::FM; ++m) {
      const int q = lane + 32 * m;
      if (q >= G::FN) continue;
      const int f = q / L, t = q - f * L;
      const int d = f >> 1, side = f & 1;
      const double* own = sT + (f * HW) * L + t;
      // neighbour across (d, side): periodic wrap in this block, or the received plane
      const int ca = d == 0 ? cx : (d == 1 ? cy : cz);
      const int cn = d == 0 ? C0 : (d == 1 ? C1 : C2);
      const bool boundary = side ? (ca == cn - 1) : (ca == 0);
      double Un[NV];
      if (boundary && p.ext[d][side] != nullptr) {
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
      const double so = own[2 * NV * L];
      const double a = dmax(side ? so : sn, side ? sn : so);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        // minus state = lower cell along d (solver.cpp:268-306; models.cpp:77-88)
        const double um = side ? own[v * L] : Un[v], up = side ? Un[v] : own[v * L];
        const double fm = side ? own[(NV + v) * L] : Fn[v], fp = side ? Fn[v] : own[(NV + v) * L];
        sH[(f * NV + v) * L + t] = A::mul(0.5, A::sub(A::add(fm, fp), A::mul(a, A::sub(up, um))));
      }
    }
    __syncwarp();

    // ------------------------------------------------ 3: volume, faces, epilogue
    if constexpr (USE_MMA) {
      // outputs at nodes (i = r, j = 2c + s), all variables
      const double xco = r == 0 ? p.lift[0] : (r == N - 1 ? -p.lift[0] : 0.0);
      const int xf = r == N - 1 ? 1 : 0;
      const double yco[2] = {c == 0 ? p.lift[1] : 0.0, c == 3 ? -p.lift[1] : 0.0};
      const int yf[2] = {2, 3};
      double un[2][NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double d0 = 0.0, d1 = 0.0;
        dmma_8x8x4(kx[0], Bx[0][v], d0, d1);  // D_x = K_x F_x
        dmma_8x8x4(kx[1], Bx[1][v], d0, d1);
        const double* Fy = sF + (1 * NV + v) * NPE;
        dmma_8x8x4(Fy[r + N * c], ky[0], d0, d1);        // += F_y K_y^T, A = F_y[i=r][j=c]
        dmma_8x8x4(Fy[r + N * (c + 4)], ky[1], d0, d1);  // A = F_y[i=r][j=c+4]
        double dv[2] = {d0, d1};
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          const int j = 2 * c + s2;
          // lifted face fluxes, branch-free: x faces at i = 0 / N-1 (line j),
          // y faces at j = 0 / N-1 (line i = r); interior nodes add 0 * (a face value)
          dv[s2] = fma(xco, sH[(xf * NV + v) * L + j], dv[s2]);
          dv[s2] = fma(yco[s2], sH[(yf[s2] * NV + v) * L + r], dv[s2]);
          const size_t gi = ebase + (size_t)v * NPE + r + N * j;
          const double kv = dv[s2] * dt;
          if (!last) {
            p.out[gi] = kv;
          } else {
            double S, Uu;
            const int ln = v * NPE + r + N * j;
            if (depth > 0)
              combine_s<EXACT, NU, AM, BM>(p, src + ln, G::CHUNK, true, Uu, S);
            else
              combine_g<EXACT, NU, AM, BM>(p, ebase + ln, true, Uu, S);
            un[s2][v] = fma(p.b_last, kv, S);
            p.out[gi] = un[s2][v];
          }
        }
      }
      if (last) {
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          double sum = un[s2][0];  // non-finite iff some component is
#pragma unroll
          for (int v = 1; v < NV; ++v) sum += un[s2][v];
          if (!isfinite(sum)) record_error(ctl, error_key(step, kPhaseInstability, 0, 0));
          if (KIND == 1 && p.scan_alpha) {
            const int n = r + N * (2 * c + s2);
            if (!(un[s2][0] > 0.0)) {
              record_error(ctl, error_key(step + 1, kPhaseScan, aos_cell(), G::aos_node(n)));
            } else {
              double mm = 0.0;
#pragma unroll
              for (int d = 0; d < DIM; ++d) mm = dmax(mm, fabs(un[s2][1 + d]));
              alpha = dmax(alpha, fma(mm, fast_rcp(un[s2][0]), p.sound_speed));  // contracted mode
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < G::NM; ++m) {
        const int n = lane + 32 * m;
        if (n >= NPE) continue;
        double un[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double D = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            const int k = G::pos_of(d, n), t = G::line_of(d, n);
            const double* Fl = sF + (d * NV + v) * NPE;
            const double* Kr = &p.K[d][k * N];
            // 0 + K0 F0 + K1 F1 + ...: the leading 0 + only normalises a -0,
            // which zero_plus (axis 0) or the add onto dudt (axes > 0) reproduces
            double acc = A::mul(Kr[0], Fl[G::node(d, t, 0)]);
#pragma unroll
            for (int l = 1; l < N; ++l) acc = A::mac(acc, Kr[l], Fl[G::node(d, t, l)]);
            D = d == 0 ? zero_plus(acc) : A::add(D, acc);
            if (k == 0) D = A::add(D, A::mul(p.lift[d], sH[((2 * d) * NV + v) * L + t]));
            if (k == N - 1) D = A::sub(D, A::mul(p.lift[d], sH[((2 * d + 1) * NV + v) * L + t]));
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
          if (!fin) record_error(ctl, error_key(step, kPhaseInstability, 0, 0));
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
    }
    __syncwarp();  // this element's slab reads precede the next element's writes
    if (depth > 0 && ++slot == depth) {
      slot = 0;
      parity ^= 1;
    }
    cx += sx;
    int carry = cx >= C0;
    cx -= carry ? C0 : 0;
    cy += sy + carry;
    carry = cy >= C1;
    cy -= carry ? C1 : 0;
    cz += sz + carry;
  }

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
