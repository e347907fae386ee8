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
// Per node, the reference accumulates dudt in the order vol_x, face_x, vol_y,
// face_y, vol_z, face_z, each volume contribution formed from 0 in l order
// and added once.  EXACT=true reproduces that order with _rn intrinsics (no
// contraction) so states are bit-identical to the reference; EXACT=false
// evaluates the volume quadrature on the FP64 tensor cores
// (mma.sync.m8n8k4.f64: D[k][line] = sum_l K[k][l] F[l][line] + D_prev) and
// contracts the rest into FMAs (<= 1e-12 relative L2).
//
// Execution model (persistent CTAs, tiles round-robin, x fastest):
//   producer warp: per tile, one lane issues TMA bulk copies
//     (cp.async.bulk + mbarrier complete_tx) of the tile's rows of u and of
//     every K_j the stage reads into the MAIN ring; all lanes issue
//     register-free cp.async copies of the neighbour face nodes into the HALO
//     ring, one tile ahead; once a tile's copies land they form its halo
//     records (stage input, flux along the face normal, one-sided speed).
//   4 consumer warps, separated by a named barrier:
//     A  node-parallel: U_s (and S at the last stage) from the main ring,
//        F_d(U_s) for every axis, face traces (U_s, speed) -> shared memory;
//        the main slot is released right after
//     X/Y/Z  per axis: volume quadrature of every (line, var) plus the
//        Lax-Friedrichs flux at the two line ends, lifted into the end nodes;
//        the last axis runs the RK epilogue and stores K_s (or u_new)
//     E  (last stage, Euler) node-parallel next-step wavespeed reduction
// Shared memory is padded (one double per x-line) so x-line owners (lane
// stride N+1) and y/z-line owners (unit lane stride) are bank-conflict free.
#pragma once

namespace ndgx {

constexpr int c_pow2floor(int x) { return x < 2 ? 1 : 2 * c_pow2floor(x / 2); }
constexpr int c_max(int a, int b) { return a > b ? a : b; }
constexpr int c_min(int a, int b) { return a < b ? a : b; }
constexpr int c_round16(int x) { return (x + 15) & ~15; }  // doubles -> 128-byte multiple

template <int DIM, int N, int KIND>
struct Geo {
  static constexpr int NV = (KIND == 0) ? 1 : DIM + 1;
  static constexpr int L = (DIM == 1) ? 1 : (DIM == 2 ? N : N * N);  // lines per element per axis
  static constexpr int NPE = L * N;                                   // nodes per element
  static constexpr int LP = L * (N + 1);  // padded smem doubles of one element variable
  static constexpr int NCONS = 128;       // consumer threads (4 warps)
  static constexpr int NPROD = 64;        // producer threads (2 warps)
  static constexpr int THREADS = NCONS + NPROD;
  // elements per tile: ~128-160 (line, var) work items per axis
  static constexpr int TE_RAW = c_pow2floor(c_max(1, 160 / (L * NV)));
  static constexpr int TE = DIM == 1 ? 128
                            : DIM == 2 ? c_min(16, TE_RAW)
                                       : (NPE * NV > 512 ? 1 : (NPE * NV > 256 ? 2 : c_max(4, c_min(8, TE_RAW))));
  static constexpr int TX = DIM == 3 ? (TE >= 2 ? 2 : 1) : TE;
  static constexpr int TY = DIM == 3 ? (TE >= 4 ? 2 : 1) : 1;
  static constexpr int TZ = TE / (TX * TY);
  static constexpr int NF0 = TE / TX, NF1 = TE / TY, NF2 = TE / TZ;  // face cross-sections per axis
  static constexpr int HW = 2 * NV + 1;  // halo record: U[NV], F[NV], speed
  // halo records (halo ring slot): [axis][side][f][HW][L]
  static constexpr int HOFF1 = 2 * NF0 * HW * L;
  static constexpr int HOFF2 = HOFF1 + (DIM > 1 ? 2 * NF1 * HW * L : 0);
  static constexpr int HALO = c_round16(HOFF2 + (DIM > 2 ? 2 * NF2 * HW * L : 0));
  static constexpr int HITEMS = 2 * L * (NF0 + (DIM > 1 ? NF1 : 0) + (DIM > 2 ? NF2 : 0));  // halo nodes
  static constexpr int RAW1 = c_round16(HITEMS * NV);  // raw halo doubles per input array
  static constexpr int ARR = TE * NV * LP;             // one padded tile array
  static constexpr int TILE_ARR = TE * NV * NPE;       // one dense tile array (main ring)
  static constexpr int LI = TE * NV * L;               // (line, var) items per axis
  // work area (doubles): F_d (F_0 becomes dudt) | face traces | S | scratch
  static constexpr int TR = DIM * TE * 2 * HW * L;  // face traces [axis][el][side][U, F, speed][t]
  // face fluxes [axis][g = 0..T_d][f][v][t] (face g of a line is its element position)
  static constexpr int FOFF1 = (TX + 1) * NF0 * NV * L;
  static constexpr int FOFF2 = FOFF1 + (DIM > 1 ? (TY + 1) * NF1 * NV * L : 0);
  static constexpr int FH = FOFF2 + (DIM > 2 ? (TZ + 1) * NF2 * NV * L : 0);
  static constexpr int FJ0 = (TX + 1) * NF0 * L, FJ1 = DIM > 1 ? (TY + 1) * NF1 * L : 0,
                       FJ2 = DIM > 2 ? (TZ + 1) * NF2 * L : 0;  // face nodes per axis
  static constexpr int OFF_F = 0;
  static constexpr int OFF_T = OFF_F + DIM * ARR;
  static constexpr int OFF_B = OFF_T + TR;
  static constexpr int OFF_FH = OFF_B + ARR;
  static constexpr int OFF_RED = OFF_FH + FH;
  static constexpr int WORK = c_round16(OFF_RED + 32);
  static constexpr int BAR_BYTES = 128;                // 16 mbarrier slots
  static constexpr bool TMA_OK = (NV * NPE) % 2 == 0;  // 16-byte element rows
  static constexpr int KH = (N + 3) / 4;               // k4 MMA steps per line

  static __device__ __forceinline__ int sn(int n) { return n + n / N; }  // padded slot
  // node index of position k along `axis` on transverse line t
  static __device__ __forceinline__ int node(int axis, int t, int k) {
    if (axis == 0) return k + N * t;
    if (axis == 1) return (t % N) + N * (k + N * (t / N));
    return t + N * N * k;
  }
  // padded slot of position k on line t: lbase(axis, t) + k * lstride(axis)
  static __device__ __forceinline__ int lbase(int axis, int t) {
    if (axis == 0) return t * (N + 1);
    if (axis == 1) return (t % N) + (N + 1) * N * (t / N);
    return (t % N) + (N + 1) * (t / N);
  }
  static __device__ __forceinline__ int lstride(int axis) { return axis == 0 ? 1 : (axis == 1 ? N + 1 : (N + 1) * N); }
  static __device__ __forceinline__ int estride(int axis) { return axis == 0 ? 1 : (axis == 1 ? TX : TX * TY); }
  static __device__ __forceinline__ int nf(int axis) { return axis == 0 ? NF0 : (axis == 1 ? NF1 : NF2); }
  static __device__ __forceinline__ int hoff(int axis) { return axis == 0 ? 0 : (axis == 1 ? HOFF1 : HOFF2); }
  static __device__ __forceinline__ int foff(int axis) { return axis == 0 ? 0 : (axis == 1 ? FOFF1 : FOFF2); }
  // tile element from (axis, position along axis, cross-section f)
  static __device__ __forceinline__ int el_of(int axis, int pos, int f) {
    if (axis == 0) return pos + TX * f;                           // f = ey + TY*ez
    if (axis == 1) return (f % TX) + TX * (pos + TY * (f / TX));  // f = ex + TX*ez
    return f + TX * TY * pos;                                     // f = ex + TX*ey
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
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// the one arrival of a TMA-filled barrier, registering the bytes the copies will complete
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b))
               : "memory");
}
// Wait for the phase of parity `parity` to complete.  A watchdog turns a
// pipeline deadlock into a trapped kernel (reported as a CUDA error) instead
// of a hung device: no legitimate wait lasts anywhere near 2^31 cycles.
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
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(PENDING) : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// D(8x8) += A(8x4, row) * B(4x8, col) in FP64 on the tensor cores
__device__ __forceinline__ void dmma_8x8x4(double a, double b, double& c0, double& c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Tile geometry of tile index `tile` (x fastest).
struct TileCtx {
  int x0, y0, z0;  // origin (cells)
  int v0, v1, v2;  // valid extent along each axis
  __device__ __forceinline__ int vd(int axis) const { return axis == 0 ? v0 : (axis == 1 ? v1 : v2); }
};

template <int DIM, int N, int KIND>
__device__ __forceinline__ TileCtx tile_ctx(const StageArgs& p, int tile) {
  using G = Geo<DIM, N, KIND>;
  const int ntx = (p.cells[0] + G::TX - 1) / G::TX, nty = (p.cells[1] + G::TY - 1) / G::TY;
  TileCtx tc;
  tc.x0 = (tile % ntx) * G::TX;
  tc.y0 = ((tile / ntx) % nty) * G::TY;
  tc.z0 = (tile / (ntx * nty)) * G::TZ;
  tc.v0 = min(G::TX, p.cells[0] - tc.x0);
  tc.v1 = min(G::TY, p.cells[1] - tc.y0);
  tc.v2 = min(G::TZ, p.cells[2] - tc.z0);
  return tc;
}

// U_s = u + sum ca[t] arr[ia[t]] and (last stage) S = u + sum cb[t] arr[ib[t]],
// each in the reference's term order; `ld(a)` reads input array a (0 = u).
template <bool EXACT, typename Ld>
__device__ __forceinline__ void combine(const StageArgs& p, bool last, Ld ld, double& U, double& S) {
  using A = Ar<EXACT>;
  const double u = ld(0);
  U = u;
#pragma unroll
  for (int t = 0; t < kMaxTerms; ++t)
    if (t < p.nA) U = A::mac(U, p.ca[t], ld(p.ia[t]));
  S = u;
  if (last) {
#pragma unroll
    for (int t = 0; t < kMaxTerms; ++t)
      if (t < p.nB) S = A::mac(S, p.cb[t], ld(p.ib[t]));
  }
}

// One variable of the Lax-Friedrichs flux (models.cpp:77-88) from both sides'
// state, flux and one-sided speed: 0.5 * ((fm + fp) - max(sm, sp) * (up - um)).
template <bool EXACT>
__device__ __forceinline__ double lf1(double um, double up, double fm, double fp, double sm, double sp) {
  using A = Ar<EXACT>;
  return A::mul(0.5, A::sub(A::add(fm, fp), A::mul(dmax(sm, sp), A::sub(up, um))));
}

// ------------------------------------------------------------ producer
// Halo node q of the tile: (axis, side, cross-section f, face node t).
struct HaloItem {
  int axis, side, f, t;
  bool valid, ext;  // ext: read the received multi-block plane instead of u / K_j
  int c0, c1, c2;   // neighbour cell (after periodic wrap), or this block's boundary cell when ext
};

template <int DIM, int N, int KIND>
__device__ __forceinline__ HaloItem halo_item(const StageArgs& p, const TileCtx& tc, int q) {
  using G = Geo<DIM, N, KIND>;
  constexpr int L = G::L;
  constexpr int I0 = 2 * G::NF0 * L, I1 = DIM > 1 ? 2 * G::NF1 * L : 0;
  HaloItem h;
  int r;
  if (q < I0) { h.axis = 0; r = q; }
  else if (q < I0 + I1) { h.axis = 1; r = q - I0; }
  else { h.axis = 2; r = q - I0 - I1; }
  h.t = r % L;
  const int fs = r / L;
  const int nfa = G::nf(h.axis);
  h.side = fs / nfa;
  h.f = fs - h.side * nfa;
  // the tile element on this face: position 0 (low) or the last valid one (high)
  const int pos = h.side ? tc.vd(h.axis) - 1 : 0;
  const int el = G::el_of(h.axis, pos, h.f);
  const int ex = el % G::TX, ey = (el / G::TX) % G::TY, ez = el / (G::TX * G::TY);
  h.valid = ex < tc.v0 && ey < tc.v1 && ez < tc.v2;
  h.c0 = tc.x0 + ex;
  h.c1 = tc.y0 + ey;
  h.c2 = tc.z0 + ez;
  const int ca = h.axis == 0 ? h.c0 : (h.axis == 1 ? h.c1 : h.c2);
  const int cn = h.axis == 0 ? p.cells[0] : (h.axis == 1 ? p.cells[1] : p.cells[2]);
  const bool boundary = h.side ? (ca == cn - 1) : (ca == 0);
  h.ext = boundary && p.ext[h.axis][h.side] != nullptr;
  if (!h.ext) {
    const int cw = h.side ? (ca + 1 == cn ? 0 : ca + 1) : (ca == 0 ? cn - 1 : ca - 1);
    if (h.axis == 0) h.c0 = cw;
    else if (h.axis == 1) h.c1 = cw;
    else h.c2 = cw;
  }
  return h;
}

// Each producer thread handles halo nodes q = ptid + NPROD*m in both passes,
// so it only ever reads back its own copies (no producer-wide barrier).
// Pass 1: register-free cp.async copies of the halo nodes' u and K_j values
// (or of the received plane) into the slot's raw area [q][array][var].
template <int DIM, int N, int KIND>
__device__ __forceinline__ void halo_issue(const StageArgs& p, const TileCtx& tc, double* raw, int ptid) {
  using G = Geo<DIM, N, KIND>;
  constexpr int NV = G::NV, L = G::L, NPE = G::NPE;
  const int C0 = p.cells[0], C1 = p.cells[1];
  const int na = 1 + p.nu;
#pragma unroll 1
  for (int q = ptid; q < G::HITEMS; q += G::NPROD) {
    const HaloItem h = halo_item<DIM, N, KIND>(p, tc, q);
    if (!h.valid) continue;
    double* r = raw + q * na * NV;
    if (h.ext) {
      const size_t xs = h.axis == 0 ? (size_t)h.c1 + (size_t)C1 * h.c2
                                    : (h.axis == 1 ? (size_t)h.c0 + (size_t)C0 * h.c2
                                                   : (size_t)h.c0 + (size_t)C0 * h.c1);
      const double* e = p.ext[h.axis][h.side];
#pragma unroll
      for (int v = 0; v < NV; ++v) cp_async8(r + v, e + (xs * NV + v) * L + h.t);
    } else {
      const size_t gb = ((size_t)h.c0 + (size_t)C0 * ((size_t)h.c1 + (size_t)C1 * h.c2)) * NV * NPE +
                        G::node(h.axis, h.t, h.side ? 0 : N - 1);
#pragma unroll 1
      for (int a = 0; a < na; ++a) {
        const double* src = (a == 0 ? p.u : p.ku[a - 1]) + gb;
#pragma unroll
        for (int v = 0; v < NV; ++v) cp_async8(r + a * NV + v, src + (size_t)v * NPE);
      }
    }
  }
  cp_async_commit();
}

// Pass 2 (after the copies landed): stage input, flux along the face normal
// and one-sided wavespeed of every halo node -> records [axis][side][f][HW][L].
template <int DIM, int N, int KIND, bool EXACT>
__device__ __forceinline__ void halo_finish(const StageArgs& p, const TileCtx& tc, double* halo, const double* raw,
                                            int ptid) {
  using G = Geo<DIM, N, KIND>;
  constexpr int NV = G::NV, L = G::L;
  const int na = 1 + p.nu;
#pragma unroll 1
  for (int q = ptid; q < G::HITEMS; q += G::NPROD) {
    const HaloItem h = halo_item<DIM, N, KIND>(p, tc, q);
    if (!h.valid) continue;
    const double* r = raw + q * na * NV;
    double U[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (h.ext) {
        U[v] = r[v];
      } else {
        double S;
        combine<EXACT>(p, false, [&](int a) { return r[a * NV + v]; }, U[v], S);
      }
    }
    double F[NV], sp;
    flux<DIM, KIND, EXACT>(p, U, h.axis, F, sp);
    double* o = halo + G::hoff(h.axis) + (h.side * G::nf(h.axis) + h.f) * G::HW * L + h.t;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      o[v * L] = U[v];
      o[(NV + v) * L] = F[v];
    }
    o[2 * NV * L] = sp;
  }
}

// ------------------------------------------------------------ consumers
// Shared-memory views of the consumer work area and the current halo slot.
template <int DIM, int N, int KIND>
struct Work {
  using G = Geo<DIM, N, KIND>;
  double* F;           // [DIM][TE][NV][LP]; F_0 becomes dudt (then u_new for the alpha scan)
  double* T;           // [DIM][TE][2][HW][L] face traces: U_s, F_axis, one-sided speed
  double* B;           // [TE][NV][LP] S at the last stage
  double* FH;          // face fluxes [axis][g][f][v][t]
  const double* halo;  // halo records of the current tile
  __device__ __forceinline__ double& tr(int axis, int el, int side, int r, int t) const {
    return T[(((axis * G::TE + el) * 2 + side) * G::HW + r) * G::L + t];
  }
  __device__ __forceinline__ const double& hr(int axis, int side, int f, int r, int t) const {
    return halo[G::hoff(axis) + ((side * G::nf(axis) + f) * G::HW + r) * G::L + t];
  }
};

// Phase F: the Lax-Friedrichs flux (all variables) of every face node of the
// tile, from the face traces (phase A) or the halo records; face g along
// `axis` separates tile positions g-1 and g (g = 0 / v_axis: the halo).
template <int DIM, int N, int KIND, bool EXACT>
__device__ __forceinline__ void face_phase(const Work<DIM, N, KIND>& w, const TileCtx& tc, int tid) {
  using G = Geo<DIM, N, KIND>;
  constexpr int NV = G::NV, L = G::L;
#pragma unroll 1
  for (int q = tid; q < G::FJ0 + G::FJ1 + G::FJ2; q += G::NCONS) {
    int axis, r;
    if (q < G::FJ0) { axis = 0; r = q; }
    else if (q < G::FJ0 + G::FJ1) { axis = 1; r = q - G::FJ0; }
    else { axis = 2; r = q - G::FJ0 - G::FJ1; }
    const int t = r % L;
    const int nfa = G::nf(axis);
    const int gf = r / L;
    const int g = gf / nfa, f = gf - g * nfa;
    const int va = tc.vd(axis);
    const int el0 = G::el_of(axis, 0, f);
    const int ex = el0 % G::TX, ey = (el0 / G::TX) % G::TY, ez = el0 / (G::TX * G::TY);
    if (g > va || ex >= tc.v0 || ey >= tc.v1 || ez >= tc.v2) continue;
    // minus (lower) side: element g-1's high trace, or the low halo
    const double* m = g == 0 ? &w.hr(axis, 0, f, 0, t) : &w.tr(axis, G::el_of(axis, g - 1, f), 1, 0, t);
    const double* pl = g == va ? &w.hr(axis, 1, f, 0, t) : &w.tr(axis, G::el_of(axis, g, f), 0, 0, t);
    const double alpha = dmax(m[2 * NV * L], pl[2 * NV * L]);
    double* o = w.FH + G::foff(axis) + (g * nfa + f) * NV * L + t;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      using A = Ar<EXACT>;
      // 0.5 * ((fm + fp) - alpha * (up - um))  (models.cpp:77-88)
      o[v * L] = A::mul(0.5, A::sub(A::add(m[(NV + v) * L], pl[(NV + v) * L]), A::mul(alpha, A::sub(pl[v * L], m[v * L]))));
    }
  }
}

struct LineItem {
  int el, t, v, pos, f;
  bool valid;
};

template <int DIM, int N, int KIND>
__device__ __forceinline__ LineItem line_item(const TileCtx& tc, int axis, int q) {
  using G = Geo<DIM, N, KIND>;
  LineItem li;
  li.t = q % G::L;
  li.v = (q / G::L) % G::NV;
  li.el = q / (G::L * G::NV);
  const int ex = li.el % G::TX, ey = (li.el / G::TX) % G::TY, ez = li.el / (G::TX * G::TY);
  li.valid = q < G::LI && ex < tc.v0 && ey < tc.v1 && ez < tc.v2;
  li.pos = axis == 0 ? ex : (axis == 1 ? ey : ez);
  li.f = axis == 0 ? ey + G::TY * ez : (axis == 1 ? ex + G::TX * ez : ex + G::TX * ey);
  return li;
}

template <int DIM, int N, int KIND>
__device__ __forceinline__ size_t elem_index(const StageArgs& p, const TileCtx& tc, int el) {
  using G = Geo<DIM, N, KIND>;
  return (size_t)(tc.x0 + el % G::TX) +
         (size_t)p.cells[0] * ((size_t)(tc.y0 + (el / G::TX) % G::TY) + (size_t)p.cells[1] * (tc.z0 + el / (G::TX * G::TY)));
}

// ============================================================ stage kernel
template <int DIM, int N, int KIND, bool EXACT>
__global__ void __launch_bounds__(Geo<DIM, N, KIND>::THREADS, 2)
stage_kernel(const __grid_constant__ StageArgs p) {
  using G = Geo<DIM, N, KIND>;
  using A = Ar<EXACT>;
  constexpr int NV = G::NV, NPE = G::NPE, LP = G::LP, TE = G::TE, NC = G::NCONS;
  extern __shared__ __align__(128) unsigned char smem_raw[];

  Control* ctl = p.ctl;
  // inactive step, or an earlier stage already failed: keep the inputs of the
  // failing stage intact for the host's error report
  if (!p.rhs_only && (*(volatile int*)&ctl->skip || *(volatile unsigned long long*)&ctl->err_key != kNoError))
    return;

  const int C0 = p.cells[0], C1 = p.cells[1], C2 = p.cells[2];
  const int ntiles = ((C0 + G::TX - 1) / G::TX) * ((C1 + G::TY - 1) / G::TY) * ((C2 + G::TZ - 1) / G::TZ);
  const bool last = p.is_last != 0;
  const int na = 1 + p.nu;
  const int dm = p.dm, dh = p.dh;
  const int main_sz = na * G::TILE_ARR;
  const int hslot_sz = G::HALO + na * G::RAW1;  // halo records | raw halo values

  uint64_t* mfull = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* mempty = mfull + 4;
  uint64_t* hfull = mfull + 8;
  uint64_t* hempty = mfull + 12;
  double* work = reinterpret_cast<double*>(smem_raw + G::BAR_BYTES);
  double* hring = work + G::WORK;
  double* mring = hring + dh * hslot_sz;

  if (threadIdx.x == 0) {
    for (int s = 0; s < dm; ++s) {
      mbar_init(&mfull[s], 1);
      mbar_init(&mempty[s], NC);
    }
    for (int s = 0; s < dh; ++s) {
      mbar_init(&hfull[s], G::NPROD);
      mbar_init(&hempty[s], NC);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int my_tiles = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  // tile j of this CTA is blockIdx.x + j * gridDim.x, walked with an
  // incremental (x, y, z) tile counter instead of per-tile divisions
  const int ntx = (C0 + G::TX - 1) / G::TX, nty = (C1 + G::TY - 1) / G::TY;
  const int gx = (int)gridDim.x % ntx, gy = ((int)gridDim.x / ntx) % nty, gz = (int)gridDim.x / (ntx * nty);
  auto tile_first = [&](int& tx, int& ty, int& tz) {
    tx = (int)blockIdx.x % ntx;
    ty = ((int)blockIdx.x / ntx) % nty;
    tz = (int)blockIdx.x / (ntx * nty);
  };
  auto tile_next = [&](int& tx, int& ty, int& tz) {
    tx += gx;
    int c = tx >= ntx;
    tx -= c ? ntx : 0;
    ty += gy + c;
    c = ty >= nty;
    ty -= c ? nty : 0;
    tz += gz + c;
  };
  auto make_tc = [&](int tx, int ty, int tz) {
    TileCtx tc;
    tc.x0 = tx * G::TX;
    tc.y0 = ty * G::TY;
    tc.z0 = tz * G::TZ;
    tc.v0 = min(G::TX, C0 - tc.x0);
    tc.v1 = min(G::TY, C1 - tc.y0);
    tc.v2 = min(G::TZ, C2 - tc.z0);
    return tc;
  };
  if (warp >= NC / 32) {
    // ------------------------------------------------------------ producer
    const int ptid = threadIdx.x - NC;
    // issue: one tile's main-ring TMA copies and halo cp.async copies
    auto issue = [&](const TileCtx& tc, int hs, uint32_t hpar, int ms, uint32_t mpar) {
      mbar_wait(&hempty[hs], hpar ^ 1);
      if (p.ring_main) {
        mbar_wait(&mempty[ms], mpar ^ 1);
        if (ptid == 0) {
          double* slot = mring + ms * main_sz;
          const uint32_t row = (uint32_t)tc.v0 * NV * NPE * 8u;
          const int rows = tc.v1 * tc.v2;
          mbar_arrive_expect_tx(&mfull[ms], row * (uint32_t)rows * (uint32_t)na);
          for (int a = 0; a < na; ++a) {
            const double* src = a == 0 ? p.u : p.ku[a - 1];
            for (int r = 0; r < rows; ++r) {
              const int ey = r % tc.v1, ez = r / tc.v1;
              const size_t e0 = (size_t)tc.x0 + (size_t)C0 * ((size_t)(tc.y0 + ey) + (size_t)C1 * (tc.z0 + ez));
              bulk_g2s(slot + a * G::TILE_ARR + (size_t)G::TX * (ey + G::TY * ez) * NV * NPE,
                       src + e0 * NV * NPE, row, &mfull[ms]);
            }
          }
        }
      }
      halo_issue<DIM, N, KIND>(p, tc, hring + hs * hslot_sz + G::HALO, ptid);
    };
    int tx, ty, tz;  // tile being finished
    tile_first(tx, ty, tz);
    int nx = tx, ny = ty, nz = tz;  // next tile to issue
    int hs_i = 0, ms_i = 0;         // slots of the next issue
    uint32_t hp_i = 0, mp_i = 0;    // their use parities
    auto advance_issue = [&]() {
      tile_next(nx, ny, nz);
      if (++hs_i == dh) { hs_i = 0; hp_i ^= 1; }
      if (++ms_i == dm) { ms_i = 0; mp_i ^= 1; }
    };
    if (my_tiles > 0) {
      issue(make_tc(nx, ny, nz), hs_i, hp_i, ms_i, mp_i);
      advance_issue();
    }
    int hs = 0;
    for (int j = 0; j < my_tiles; ++j) {
      // one tile ahead: the next tile's copies are in flight while this one finishes
      if (j + 1 < my_tiles) {
        issue(make_tc(nx, ny, nz), hs_i, hp_i, ms_i, mp_i);
        advance_issue();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      const TileCtx tc = make_tc(tx, ty, tz);
      double* hslot = hring + hs * hslot_sz;
      halo_finish<DIM, N, KIND, EXACT>(p, tc, hslot, hslot + G::HALO, ptid);
      mbar_arrive(&hfull[hs]);
      if (++hs == dh) hs = 0;
      tile_next(tx, ty, tz);
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int tid = threadIdx.x;
  const double dt = p.rhs_only ? 1.0 : ctl->dt;
  const long long step = p.rhs_only ? 0 : ctl->steps;
  double alpha = 0.0;
  Work<DIM, N, KIND> w;
  w.F = work + G::OFF_F;
  w.T = work + G::OFF_T;
  w.B = work + G::OFF_B;
  w.FH = work + G::OFF_FH;
  auto aos_cell = [&](int x, int y, int z) -> long long {  // global AoS cell index
    const long long gx = x + p.goff[0], gy = y + p.goff[1], gz = z + p.goff[2];
    return (gx * p.gcells[1] + gy) * (long long)p.gcells[2] + gz;
  };

  int tx, ty, tz;
  tile_first(tx, ty, tz);
  int hs = 0, ms = 0;
  uint32_t hpar = 0, mpar = 0;
  for (int it = 0; it < my_tiles; ++it) {
    if (it > 0) {
      tile_next(tx, ty, tz);
      if (++hs == dh) { hs = 0; hpar ^= 1; }
      if (++ms == dm) { ms = 0; mpar ^= 1; }
    }
    const TileCtx tc = make_tc(tx, ty, tz);
    w.halo = hring + hs * hslot_sz;
    const double* mslot = mring + ms * main_sz;
    if (it > 0) consumer_sync();  // the previous tile's readers of the work area are done
    if (p.ring_main) mbar_wait(&mfull[ms], mpar);

    // ------------------------------------------------ A: stage input + fluxes
#pragma unroll 2
    for (int q = tid; q < TE * NPE; q += NC) {
      const int el = q / NPE, n = q - el * NPE;
      const int ex = el % G::TX, ey = (el / G::TX) % G::TY, ez = el / (G::TX * G::TY);
      if (ex >= tc.v0 || ey >= tc.v1 || ez >= tc.v2) continue;
      const int sl = G::sn(n);
      double U[NV];
      if (p.ring_main) {
        const double* src = mslot + el * NV * NPE + n;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double S;
          combine<EXACT>(p, last, [&](int a) { return src[a * G::TILE_ARR + v * NPE]; }, U[v], S);
          if (last) w.B[(el * NV + v) * LP + sl] = S;
        }
      } else {
        const size_t g = elem_index<DIM, N, KIND>(p, tc, el) * NV * NPE + n;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double S;
          const size_t gv = g + (size_t)v * NPE;
          combine<EXACT>(p, last, [&](int a) { return __ldg((a == 0 ? p.u : p.ku[a - 1]) + gv); }, U[v], S);
          if (last) w.B[(el * NV + v) * LP + sl] = S;
        }
      }
      const int i = n % N, j = (n / N) % N, k = n / (N * N);
      if (KIND == 1 && !(U[0] > 0.0)) {
        // first bad node of the reference's x-volume traversal: (cell, (j,k), i)
        const int nkey = (DIM == 2) ? j * N + i : (j * N + k) * N + i;
        record_error(ctl, error_key(step, p.phase, aos_cell(tc.x0 + ex, tc.y0 + ey, tc.z0 + ez), nkey));
      }
      const double rinv = (!EXACT && KIND == 1) ? 1.0 / U[0] : -1.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double F[NV], sp;
        flux<DIM, KIND, EXACT>(p, U, d, F, sp, rinv);
#pragma unroll
        for (int v = 0; v < NV; ++v) w.F[((d * TE + el) * NV + v) * LP + sl] = F[v];
        const int pd = d == 0 ? i : (d == 1 ? j : k);
        if (pd == 0 || pd == N - 1) {
          const int t = d == 0 ? j + N * k : (d == 1 ? i + N * k : i + N * j);
          const int side = pd == 0 ? 0 : 1;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            w.tr(d, el, side, v, t) = U[v];
            w.tr(d, el, side, NV + v, t) = F[v];
          }
          w.tr(d, el, side, 2 * NV, t) = sp;
        }
      }
    }
    if (p.ring_main) mbar_arrive(&mempty[ms]);  // main slot consumed
    mbar_wait(&hfull[hs], hpar);                // halo records of this tile
    consumer_sync();

    // ------------------------------------------------ F: face fluxes
    face_phase<DIM, N, KIND, EXACT>(w, tc, tid);
    consumer_sync();
    mbar_arrive(&hempty[hs]);  // halo records of this tile no longer read

    // ------------------------------------------------ X/Y/Z: volume + lift
#pragma unroll
    for (int axis = 0; axis < DIM; ++axis) {
      if (axis > 0) consumer_sync();
      const double lift = p.lift[axis];
      const int as = G::lstride(axis);
      const bool final_axis = axis == DIM - 1;
      const double* Fa = w.F + axis * G::ARR;
      const double* fha = w.FH + G::foff(axis);
      const int nfa = G::nf(axis);
      if constexpr (EXACT) {
        // (line, var) per thread, the reference's sequential quadrature order
#pragma unroll 1
        for (int q = tid; q < G::LI; q += NC) {
          const LineItem li = line_item<DIM, N, KIND>(tc, axis, q);
          if (!li.valid) continue;
          const int lb = (li.el * NV + li.v) * LP + G::lbase(axis, li.t);
          double Fl[N];
#pragma unroll
          for (int l = 0; l < N; ++l) Fl[l] = Fa[lb + l * as];
          double D[N];
#pragma unroll
          for (int k = 0; k < N; ++k) {
            // 0 + K0 F0 + K1 F1 + ...: the leading 0 + only normalises a -0,
            // which zero_plus (axis 0) or the add onto dudt (axes > 0) reproduces
            double acc = A::mul(p.K[axis][k * N], Fl[0]);
#pragma unroll
            for (int l = 1; l < N; ++l) acc = A::mac(acc, p.K[axis][k * N + l], Fl[l]);
            D[k] = axis == 0 ? zero_plus(acc) : A::add(w.F[lb + k * as], acc);
          }
          const double* fh = fha + (li.pos * nfa + li.f) * NV * G::L + li.v * G::L + li.t;
          D[0] = A::add(D[0], A::mul(lift, fh[0]));                        // + side of face pos
          D[N - 1] = A::sub(D[N - 1], A::mul(lift, fh[nfa * NV * G::L]));  // - side of face pos+1
          if (!final_axis) {
#pragma unroll
            for (int k = 0; k < N; ++k) w.F[lb + k * as] = D[k];
          } else {
            double* gout = p.out + (elem_index<DIM, N, KIND>(p, tc, li.el) * NV + li.v) * NPE;
#pragma unroll
            for (int k = 0; k < N; ++k) {
              const int n = G::node(axis, li.t, k);
              const double kv = A::mul(D[k], dt);  // k_i *= dt (solver.hpp:66-67)
              if (!last) {
                gout[n] = kv;
              } else {
                const double un = p.b_last != 0.0 ? A::mac(w.B[lb + k * as], p.b_last, kv) : w.B[lb + k * as];
                gout[n] = un;
                if (!isfinite(un)) record_error(ctl, error_key(step, kPhaseInstability, 0, 0));
                if (KIND == 1 && p.scan_alpha) w.F[lb + k * as] = un;
              }
            }
          }
        }
      } else {
        // FP64 tensor cores: groups of 8 (line, var) items, D[k][line] =
        // sum_l K[k][l] F[l][line] (+ dudt so far) with m8n8k4 MMAs
        const int r = lane >> 2, c = lane & 3;
        double afr[G::KH];
#pragma unroll
        for (int h = 0; h < G::KH; ++h) {
          const int l = c + 4 * h;
          afr[h] = (r < N && l < N) ? p.K[axis][r * N + l] : 0.0;
        }
        const bool krow = r < N;
        if constexpr (G::L % 8 == 0) {
          // each group is 8 consecutive lines t0..t0+7 of one (element, var)
          constexpr int GPL = G::L / 8;
#pragma unroll 1
          for (int g = warp; g < G::LI / 8; g += NC / 32) {
            const int ev = g / GPL;  // el * NV + v
            const int t0 = (g - ev * GPL) * 8;
            const int el = ev / NV, v = ev - el * NV;
            const int ex = el % G::TX, ey = (el / G::TX) % G::TY, ez = el / (G::TX * G::TY);
            if (ex >= tc.v0 || ey >= tc.v1 || ez >= tc.v2) continue;  // warp-uniform
            const int base = ev * LP;
            const int lbb = base + G::lbase(axis, t0 + r);
            const int lb0 = base + G::lbase(axis, t0 + 2 * c);
            const int lb1 = base + G::lbase(axis, t0 + 2 * c + 1);
            double c0 = 0.0, c1 = 0.0;
            if (axis > 0 && krow) {
              c0 = w.F[lb0 + r * as];
              c1 = w.F[lb1 + r * as];
            }
#pragma unroll
            for (int h = 0; h < G::KH; ++h) {
              const int l = c + 4 * h;
              const double b = l < N ? Fa[lbb + l * as] : 0.0;
              dmma_8x8x4(afr[h], b, c0, c1);
            }
            __syncwarp();  // every lane's B/C reads of this group precede the in-place stores
            if (krow) {
              const int pos = axis == 0 ? ex : (axis == 1 ? ey : ez);
              const int f = axis == 0 ? ey + G::TY * ez : (axis == 1 ? ex + G::TX * ez : ex + G::TX * ey);
              if (r == 0 || r == N - 1) {
                // node 0 is the + side of face pos, node N-1 the - side of face pos+1
                const double* fh = fha + ((pos + (r == 0 ? 0 : 1)) * nfa + f) * NV * G::L + v * G::L + t0 + 2 * c;
                const double sg = r == 0 ? lift : -lift;
                c0 = fma(sg, fh[0], c0);
                c1 = fma(sg, fh[1], c1);
              }
              if (!final_axis) {
                w.F[lb0 + r * as] = c0;
                w.F[lb1 + r * as] = c1;
              } else {
                double* gout = p.out + (elem_index<DIM, N, KIND>(p, tc, el) * NV + v) * NPE;
                const int n0 = G::node(axis, t0 + 2 * c, r), n1 = G::node(axis, t0 + 2 * c + 1, r);
                const double k0 = c0 * dt, k1 = c1 * dt;
                if (!last) {
                  gout[n0] = k0;
                  gout[n1] = k1;
                } else {
                  const double u0 = fma(p.b_last, k0, w.B[lb0 + r * as]);
                  const double u1 = fma(p.b_last, k1, w.B[lb1 + r * as]);
                  gout[n0] = u0;
                  gout[n1] = u1;
                  if (!isfinite(u0) || !isfinite(u1)) record_error(ctl, error_key(step, kPhaseInstability, 0, 0));
                  if (KIND == 1 && p.scan_alpha) {
                    w.F[lb0 + r * as] = u0;
                    w.F[lb1 + r * as] = u1;
                  }
                }
              }
            }
          }
        } else {
#pragma unroll 1
        for (int g = warp; g * 8 < G::LI; g += NC / 32) {
          // B fragment: F[l = c + 4h][line = r]; C fragment: lines 2c, 2c+1 at node k = r
          const LineItem lbi = line_item<DIM, N, KIND>(tc, axis, g * 8 + r);
          const LineItem l0 = line_item<DIM, N, KIND>(tc, axis, g * 8 + 2 * c);
          const LineItem l1 = line_item<DIM, N, KIND>(tc, axis, g * 8 + 2 * c + 1);
          const int lbb = (lbi.el * NV + lbi.v) * LP + G::lbase(axis, lbi.t);
          const int lb0 = (l0.el * NV + l0.v) * LP + G::lbase(axis, l0.t);
          const int lb1 = (l1.el * NV + l1.v) * LP + G::lbase(axis, l1.t);
          double c0 = 0.0, c1 = 0.0;
          if (axis > 0 && krow) {
            if (l0.valid) c0 = w.F[lb0 + r * as];
            if (l1.valid) c1 = w.F[lb1 + r * as];
          }
#pragma unroll
          for (int h = 0; h < G::KH; ++h) {
            const int l = c + 4 * h;
            const double b = (lbi.valid && l < N) ? Fa[lbb + l * as] : 0.0;
            dmma_8x8x4(afr[h], b, c0, c1);
          }
          __syncwarp();  // every lane's B/C reads of this group precede the in-place stores
          if (krow) {
            // lifted face fluxes at the line ends: node 0 is the + side of face pos,
            // node N-1 the - side of face pos+1
            if (r == 0 || r == N - 1) {
              const double sg = r == 0 ? lift : -lift;
              const int gofs = r == 0 ? 0 : nfa * NV * G::L;
              if (l0.valid) c0 = fma(sg, fha[(l0.pos * nfa + l0.f) * NV * G::L + l0.v * G::L + l0.t + gofs], c0);
              if (l1.valid) c1 = fma(sg, fha[(l1.pos * nfa + l1.f) * NV * G::L + l1.v * G::L + l1.t + gofs], c1);
            }
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              const LineItem& li = s2 ? l1 : l0;
              const int lbs = s2 ? lb1 : lb0;
              const double dv = s2 ? c1 : c0;
              if (!li.valid) continue;
              if (!final_axis) {
                w.F[lbs + r * as] = dv;
              } else {
                const size_t gi = (elem_index<DIM, N, KIND>(p, tc, li.el) * NV + li.v) * NPE + G::node(axis, li.t, r);
                const double kv = dv * dt;
                if (!last) {
                  p.out[gi] = kv;
                } else {
                  const double un = fma(p.b_last, kv, w.B[lbs + r * as]);
                  p.out[gi] = un;
                  if (!isfinite(un)) record_error(ctl, error_key(step, kPhaseInstability, 0, 0));
                  if (KIND == 1 && p.scan_alpha) w.F[lbs + r * as] = un;
                }
              }
            }
          }
        }
        }
      }
    }

    // ------------------------------------------------ E: next step's alpha
    if (KIND == 1 && last && p.scan_alpha) {
      consumer_sync();
#pragma unroll 1
      for (int q = tid; q < TE * NPE; q += NC) {
        const int el = q / NPE, n = q - el * NPE;
        const int ex = el % G::TX, ey = (el / G::TX) % G::TY, ez = el / (G::TX * G::TY);
        if (ex >= tc.v0 || ey >= tc.v1 || ez >= tc.v2) continue;
        const int sl = G::sn(n);
        double un[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) un[v] = w.F[(el * NV + v) * LP + sl];
        if (!(un[0] > 0.0)) {
          record_error(ctl, error_key(step + 1, kPhaseScan, aos_cell(tc.x0 + ex, tc.y0 + ey, tc.z0 + ez),
                                      G::aos_node(n)));
        } else {
          double m = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) m = dmax(m, fabs(un[1 + d]));
          alpha = dmax(alpha, __dadd_rn(__ddiv_rn(m, un[0]), p.sound_speed));  // == alpha_scan_kernel
        }
      }
    }
  }  // tile loop

  if (KIND == 1 && last && p.scan_alpha) {
    // block max of the non-negative wavespeeds on their IEEE bit patterns
    alpha = warp_max(alpha);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(work + G::OFF_RED);
    consumer_sync();
    if (lane == 0) red[warp] = (unsigned long long)__double_as_longlong(alpha);
    consumer_sync();
    if (tid == 0) {
      unsigned long long m = 0ull;
      for (int q = 0; q < NC / 32; ++q) m = red[q] > m ? red[q] : m;
      atomicMax(&ctl->alpha_bits, m);
    }
  }
}

}  // namespace ndgx
