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
// and added once; EXACT=true reproduces that order with _rn intrinsics (no
// contraction), so states are bit-identical to the reference.
//
// Execution model (one persistent CTA per SM slot, tiles round-robin):
//   warp NCONS/32 (producer): per tile, one elected lane issues TMA bulk
//     copies (cp.async.bulk.shared::cluster.global + mbarrier complete_tx) of
//     the tile's rows of u and every K_j the stage reads into a ring slot; the
//     32 lanes then build the tile's face halo (neighbour face nodes: stage
//     input, flux along the face normal, one-sided wavespeed) from global/L2
//     or from a received multi-block plane, and arrive on the slot's mbarrier.
//   warps 0..3 (consumers), separated by a named barrier:
//     A  node-parallel: U_s (and S = u + sum b_j K_j at the last stage) from
//        the ring, F_d(U_s) and the one-sided speed for every axis -> smem
//     F  face-node-parallel: Lax-Friedrichs flux of every face of the tile
//     X/Y/Z  (line, var)-parallel: the axis' volume quadrature from the flux
//        line in registers, plus the lifted face fluxes at the line ends;
//        the last axis runs the RK epilogue and stores K_s (or u_new)
//     E  (last stage, Euler) node-parallel finite/alpha reduction
// Shared memory is padded so that x-line owners (lane stride N+1) and y/z-line
// owners (unit lane stride) are bank-conflict free.
#pragma once

namespace ndgx {

constexpr int c_pow2floor(int x) { return x < 2 ? 1 : 2 * c_pow2floor(x / 2); }
constexpr int c_max(int a, int b) { return a > b ? a : b; }
constexpr int c_min(int a, int b) { return a < b ? a : b; }

template <int DIM, int N, int KIND>
struct Geo {
  static constexpr int NV = (KIND == 0) ? 1 : DIM + 1;
  static constexpr int L = (DIM == 1) ? 1 : (DIM == 2 ? N : N * N);  // lines per element per axis
  static constexpr int NPE = L * N;                                   // nodes per element
  static constexpr int LP = L * (N + 1);  // padded smem doubles of one element variable
  static constexpr int NCONS = 128;       // consumer threads (4 warps)
  static constexpr int THREADS = NCONS + 32;
  // elements per tile: ~128-160 (line, var) work items per tile
  static constexpr int TE_RAW = c_pow2floor(c_max(1, 160 / (L * NV)));
  static constexpr int TE = DIM == 1 ? 128
                            : DIM == 2 ? c_min(16, TE_RAW)
                                       : (NPE * NV > 512 ? 1 : (NPE * NV > 256 ? 2 : c_max(4, c_min(8, TE_RAW))));
  static constexpr int TX = DIM == 3 ? (TE >= 2 ? 2 : 1) : TE;
  static constexpr int TY = DIM == 3 ? (TE >= 4 ? 2 : 1) : 1;
  static constexpr int TZ = TE / (TX * TY);
  static constexpr int NF0 = TE / TX, NF1 = TE / TY, NF2 = TE / TZ;  // face cross-sections per axis
  static constexpr int HW = 2 * NV + 1;  // halo record: U[NV], F[NV], speed
  // halo (in the ring slot): [axis][side][f][HW][L]
  static constexpr int HOFF1 = 2 * NF0 * HW * L;
  static constexpr int HOFF2 = HOFF1 + (DIM > 1 ? 2 * NF1 * HW * L : 0);
  static constexpr int HALO = ((HOFF2 + (DIM > 2 ? 2 * NF2 * HW * L : 0)) + 15) & ~15;  // 128-byte multiple
  static constexpr int HITEMS = 2 * L * (NF0 + (DIM > 1 ? NF1 : 0) + (DIM > 2 ? NF2 : 0));  // halo nodes
  static constexpr int RAW1 = ((HITEMS * NV) + 15) & ~15;  // raw halo doubles per input array
  // face fluxes: [axis][g = 0..T_d][f][v][L]
  static constexpr int FOFF1 = (TX + 1) * NF0 * NV * L;
  static constexpr int FOFF2 = FOFF1 + (DIM > 1 ? (TY + 1) * NF1 * NV * L : 0);
  static constexpr int FH = FOFF2 + (DIM > 2 ? (TZ + 1) * NF2 * NV * L : 0);
  static constexpr int ARR = TE * NV * LP;  // one padded tile array
  static constexpr int TILE_ARR = TE * NV * NPE;  // one dense tile array (ring)
  // work area (doubles): U_s | F_d (d < DIM; F_0 becomes dudt) | speed_d | S | face fluxes | scratch
  static constexpr int OFF_U = 0;
  static constexpr int OFF_F = OFF_U + ARR;
  static constexpr int OFF_S = OFF_F + DIM * ARR;
  static constexpr int OFF_B = OFF_S + DIM * TE * LP;
  static constexpr int OFF_FH = OFF_B + ARR;
  static constexpr int OFF_RED = OFF_FH + FH;
  static constexpr int WORK = ((OFF_RED + 32) + 15) & ~15;  // 128-byte multiple
  static constexpr int BAR_BYTES = 128;                      // 4 mbarriers, padded
  static constexpr bool TMA_OK = (NV * NPE) % 2 == 0;        // 16-byte element rows

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
  static __device__ __forceinline__ int lstride(int axis) {
    return axis == 0 ? 1 : (axis == 1 ? N + 1 : (N + 1) * N);
  }
  static __device__ __forceinline__ int tdim(int axis) { return axis == 0 ? TX : (axis == 1 ? TY : TZ); }
  static __device__ __forceinline__ int nf(int axis) { return axis == 0 ? NF0 : (axis == 1 ? NF1 : NF2); }
  static __device__ __forceinline__ int hoff(int axis) { return axis == 0 ? 0 : (axis == 1 ? HOFF1 : HOFF2); }
  static __device__ __forceinline__ int foff(int axis) { return axis == 0 ? 0 : (axis == 1 ? FOFF1 : FOFF2); }
  // tile element from (axis, position along axis, cross-section f)
  static __device__ __forceinline__ int el_of(int axis, int pos, int f) {
    if (axis == 0) return pos + TX * f;                       // f = ey + TY*ez
    if (axis == 1) return (f % TX) + TX * (pos + TY * (f / TX));  // f = ex + TX*ez
    return f + TX * TY * pos;                                 // f = ex + TX*ey
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
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
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
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

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

// stage input (and, at the last stage, S) of one variable from u and the K_j
// in the reference's term order; `ld(a)` returns array a (0 = u, 1 + t = ku[t])
template <bool EXACT, typename Ld>
__device__ __forceinline__ void combine(const StageArgs& p, bool last, Ld ld, double& U, double& S) {
  using A = Ar<EXACT>;
  U = ld(0);
  S = U;
#pragma unroll
  for (int t = 0; t < kMaxTerms; ++t) {
    if (t < p.nu) {
      const double k = ld(1 + t);
      if (p.amask >> t & 1) U = A::mac(U, p.ca[t], k);
      if (last && (p.bmask >> t & 1)) S = A::mac(S, p.cb[t], k);
    }
  }
}

// ------------------------------------------------------------ producer
// Halo node q of the tile: (axis, side, cross-section f, face node t).
template <int DIM, int N, int KIND>
struct HaloItem {
  int axis, side, f, t;
  bool valid;
  int c[3];  // neighbour cell (after periodic wrap) -- or this block's boundary cell when ext
  bool ext;  // read the received multi-block plane instead of u / K_j
};

template <int DIM, int N, int KIND>
__device__ __forceinline__ HaloItem<DIM, N, KIND> halo_item(const StageArgs& p, const TileCtx& tc, int q) {
  using G = Geo<DIM, N, KIND>;
  constexpr int L = G::L;
  constexpr int I0 = 2 * G::NF0 * L, I1 = DIM > 1 ? 2 * G::NF1 * L : 0;
  HaloItem<DIM, N, KIND> h;
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
  int c0 = tc.x0 + ex, c1 = tc.y0 + ey, c2 = tc.z0 + ez;
  const int ca = h.axis == 0 ? c0 : (h.axis == 1 ? c1 : c2);
  const int cn = h.axis == 0 ? p.cells[0] : (h.axis == 1 ? p.cells[1] : p.cells[2]);
  const bool boundary = h.side ? (ca == cn - 1) : (ca == 0);
  h.ext = boundary && p.ext[h.axis][h.side] != nullptr;
  if (!h.ext) {
    const int cw = h.side ? (ca + 1 == cn ? 0 : ca + 1) : (ca == 0 ? cn - 1 : ca - 1);
    if (h.axis == 0) c0 = cw;
    else if (h.axis == 1) c1 = cw;
    else c2 = cw;
  }
  h.c[0] = c0;
  h.c[1] = c1;
  h.c[2] = c2;
  return h;
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// The tile's face halo, built by the producer warp in two passes so that the
// whole tile costs one memory latency: (1) every lane issues register-free
// cp.async copies of its halo nodes' u and K_j values (or of the received
// plane) into the slot's raw area [q][a][v]; (2) after the copies land, each
// lane forms the stage input, the flux along the face normal and the
// one-sided wavespeed into the halo records [axis][side][f][HW][L].
template <int DIM, int N, int KIND, bool EXACT>
__device__ __forceinline__ void produce_halo(const StageArgs& p, const TileCtx& tc, double* halo, double* raw,
                                             int lane) {
  using G = Geo<DIM, N, KIND>;
  constexpr int NV = G::NV, L = G::L, NPE = G::NPE;
  const int C0 = p.cells[0], C1 = p.cells[1];
  const int na = 1 + p.nu;
#pragma unroll 1
  for (int q = lane; q < G::HITEMS; q += 32) {
    const HaloItem<DIM, N, KIND> h = halo_item<DIM, N, KIND>(p, tc, q);
    if (!h.valid) continue;
    double* r = raw + q * na * NV;
    if (h.ext) {
      // received plane: [cross-section cell][var][face node]
      const size_t xs = h.axis == 0 ? (size_t)h.c[1] + (size_t)C1 * h.c[2]
                                    : (h.axis == 1 ? (size_t)h.c[0] + (size_t)C0 * h.c[2]
                                                   : (size_t)h.c[0] + (size_t)C0 * h.c[1]);
      const double* e = p.ext[h.axis][h.side];
#pragma unroll
      for (int v = 0; v < NV; ++v) cp_async8(r + v, e + (xs * NV + v) * L + h.t);
    } else {
      const size_t gb = ((size_t)h.c[0] + (size_t)C0 * ((size_t)h.c[1] + (size_t)C1 * h.c[2])) * NV * NPE +
                        G::node(h.axis, h.t, h.side ? 0 : N - 1);
      for (int a = 0; a < na; ++a) {
        const double* src = (a == 0 ? p.u : p.ku[a - 1]) + gb;
#pragma unroll
        for (int v = 0; v < NV; ++v) cp_async8(r + a * NV + v, src + (size_t)v * NPE);
      }
    }
  }
  cp_async_wait_all();
  __syncwarp();
#pragma unroll 1
  for (int q = lane; q < G::HITEMS; q += 32) {
    const HaloItem<DIM, N, KIND> h = halo_item<DIM, N, KIND>(p, tc, q);
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

// ============================================================ stage kernel
template <int DIM, int N, int KIND, bool EXACT>
__global__ void __launch_bounds__(Geo<DIM, N, KIND>::THREADS, 3)
stage_kernel(const __grid_constant__ StageArgs p) {
  using G = Geo<DIM, N, KIND>;
  using A = Ar<EXACT>;
  constexpr int NV = G::NV, L = G::L, NPE = G::NPE, LP = G::LP, TE = G::TE, NC = G::NCONS;
  extern __shared__ __align__(128) unsigned char smem_raw[];

  Control* ctl = p.ctl;
  // inactive step, or an earlier stage already failed: keep the inputs of the
  // failing stage intact for the host's error report
  if (!p.rhs_only && (*(volatile int*)&ctl->skip || *(volatile unsigned long long*)&ctl->err_key != kNoError))
    return;

  const int C0 = p.cells[0], C1 = p.cells[1], C2 = p.cells[2];
  const int ntiles = ((C0 + G::TX - 1) / G::TX) * ((C1 + G::TY - 1) / G::TY) * ((C2 + G::TZ - 1) / G::TZ);
  const bool last = p.is_last != 0;
  const int depth = p.depth;
  const int main_sz = p.ring_main ? (1 + p.nu) * G::TILE_ARR : 0;
  const int slot_sz = main_sz + G::HALO + (1 + p.nu) * G::RAW1;  // main | halo records | raw halo

  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + 2;
  double* work = reinterpret_cast<double*>(smem_raw + G::BAR_BYTES);
  double* ring = work + G::WORK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < depth; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], NC);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == NC / 32) {
    // ------------------------------------------------------------ producer
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int s = it % depth;
      const uint32_t use = it / depth;
      mbar_wait(&empty[s], (use & 1) ^ 1);  // slot released by the consumers
      const TileCtx tc = tile_ctx<DIM, N, KIND>(p, tile);
      double* slot = ring + s * slot_sz;
      if (p.ring_main && lane == 0) {
        const uint32_t row = (uint32_t)tc.v0 * NV * NPE * 8u;
        const int rows = tc.v1 * tc.v2;
        mbar_expect_tx(&full[s], row * (uint32_t)rows * (uint32_t)(1 + p.nu));
        for (int a = 0; a <= p.nu; ++a) {
          const double* src = a == 0 ? p.u : p.ku[a - 1];
          for (int r = 0; r < rows; ++r) {
            const int ey = r % tc.v1, ez = r / tc.v1;
            const size_t e0 = (size_t)tc.x0 + (size_t)C0 * ((size_t)(tc.y0 + ey) + (size_t)C1 * (tc.z0 + ez));
            bulk_g2s(slot + a * G::TILE_ARR + (size_t)G::TX * (ey + G::TY * ez) * NV * NPE, src + e0 * NV * NPE,
                     row, &full[s]);
          }
        }
      }
      produce_halo<DIM, N, KIND, EXACT>(p, tc, slot + main_sz, slot + main_sz + G::HALO, lane);
      __syncwarp();
      mbar_arrive(&full[s]);
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int tid = threadIdx.x;
  const double dt = p.rhs_only ? 1.0 : ctl->dt;
  const long long step = p.rhs_only ? 0 : ctl->steps;
  double alpha = 0.0;
  double* sU = work + G::OFF_U;    // [TE][NV][LP]
  double* sF = work + G::OFF_F;    // [DIM][TE][NV][LP]; F_0 becomes dudt
  double* sS = work + G::OFF_S;    // [DIM][TE][LP] one-sided speeds
  double* sB = work + G::OFF_B;    // [TE][NV][LP] S at the last stage, then u_new
  double* sFh = work + G::OFF_FH;  // face fluxes
  auto aos_cell = [&](int x, int y, int z) -> long long {  // global AoS cell index
    const long long gx = x + p.goff[0], gy = y + p.goff[1], gz = z + p.goff[2];
    return (gx * p.gcells[1] + gy) * (long long)p.gcells[2] + gz;
  };

  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % depth;
    const uint32_t use = it / depth;
    const TileCtx tc = tile_ctx<DIM, N, KIND>(p, tile);
    const double* slot = ring + s * slot_sz;
    const double* halo = slot + main_sz;
    if (it > 0) consumer_sync();  // previous tile's readers of the work area are done
    mbar_wait(&full[s], use & 1);

    // ------------------------------------------------ A: stage input + fluxes
#pragma unroll 2
    for (int q = tid; q < TE * NPE; q += NC) {
      const int el = q / NPE, n = q - el * NPE;
      const int ex = el % G::TX, ey = (el / G::TX) % G::TY, ez = el / (G::TX * G::TY);
      if (ex >= tc.v0 || ey >= tc.v1 || ez >= tc.v2) continue;
      const int sl = G::sn(n);
      double U[NV];
      if (p.ring_main) {
        const double* src = slot + el * NV * NPE + n;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double S;
          combine<EXACT>(p, last, [&](int a) { return src[a * G::TILE_ARR + v * NPE]; }, U[v], S);
          sU[(el * NV + v) * LP + sl] = U[v];
          if (last) sB[(el * NV + v) * LP + sl] = S;
        }
      } else {
        const size_t e = (size_t)(tc.x0 + ex) + (size_t)C0 * ((size_t)(tc.y0 + ey) + (size_t)C1 * (tc.z0 + ez));
        const size_t g = e * NV * NPE + n;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double S;
          const size_t gv = g + (size_t)v * NPE;
          combine<EXACT>(p, last, [&](int a) { return __ldg((a == 0 ? p.u : p.ku[a - 1]) + gv); }, U[v], S);
          sU[(el * NV + v) * LP + sl] = U[v];
          if (last) sB[(el * NV + v) * LP + sl] = S;
        }
      }
      if (KIND == 1 && !(U[0] > 0.0)) {
        // first bad node of the reference's x-volume traversal: (cell, (j,k), i)
        const int i = n % N, j = (n / N) % N, k = n / (N * N);
        const int nkey = (DIM == 2) ? j * N + i : (j * N + k) * N + i;
        record_error(ctl, error_key(step, p.phase, aos_cell(tc.x0 + ex, tc.y0 + ey, tc.z0 + ez), nkey));
      }
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double F[NV], sp;
        flux<DIM, KIND, EXACT>(p, U, d, F, sp);
#pragma unroll
        for (int v = 0; v < NV; ++v) sF[((d * TE + el) * NV + v) * LP + sl] = F[v];
        sS[(d * TE + el) * LP + sl] = sp;
      }
    }
    consumer_sync();

    // ------------------------------------------------ F: face fluxes
    {
      constexpr int J0 = (G::TX + 1) * G::NF0 * L;
      constexpr int J1 = DIM > 1 ? (G::TY + 1) * G::NF1 * L : 0;
      constexpr int J2 = DIM > 2 ? (G::TZ + 1) * G::NF2 * L : 0;
#pragma unroll 1
      for (int q = tid; q < J0 + J1 + J2; q += NC) {
        int axis, r;
        if (q < J0) { axis = 0; r = q; }
        else if (q < J0 + J1) { axis = 1; r = q - J0; }
        else { axis = 2; r = q - J0 - J1; }
        const int t = r % L;
        const int nfa = G::nf(axis);
        const int gf = r / L;
        const int g = gf / nfa, f = gf - g * nfa;
        const int va = tc.vd(axis);
        if (g > va) continue;
        {  // cross-section validity
          const int el0 = G::el_of(axis, 0, f);
          const int ex = el0 % G::TX, ey = (el0 / G::TX) % G::TY, ez = el0 / (G::TX * G::TY);
          if (ex >= tc.v0 || ey >= tc.v1 || ez >= tc.v2) continue;
        }
        double um[NV], up[NV], fm[NV], fp[NV], sm, spp;
        if (g == 0) {
          const double* h = halo + G::hoff(axis) + f * G::HW * L + t;
#pragma unroll
          for (int v = 0; v < NV; ++v) { um[v] = h[v * L]; fm[v] = h[(NV + v) * L]; }
          sm = h[2 * NV * L];
        } else {
          const int el = G::el_of(axis, g - 1, f);
          const int sl = G::sn(G::node(axis, t, N - 1));
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            um[v] = sU[(el * NV + v) * LP + sl];
            fm[v] = sF[((axis * TE + el) * NV + v) * LP + sl];
          }
          sm = sS[(axis * TE + el) * LP + sl];
        }
        if (g == va) {
          const double* h = halo + G::hoff(axis) + (nfa + f) * G::HW * L + t;
#pragma unroll
          for (int v = 0; v < NV; ++v) { up[v] = h[v * L]; fp[v] = h[(NV + v) * L]; }
          spp = h[2 * NV * L];
        } else {
          const int el = G::el_of(axis, g, f);
          const int sl = G::sn(G::node(axis, t, 0));
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            up[v] = sU[(el * NV + v) * LP + sl];
            fp[v] = sF[((axis * TE + el) * NV + v) * LP + sl];
          }
          spp = sS[(axis * TE + el) * LP + sl];
        }
        double fh[NV];
        lax_friedrichs<NV, EXACT>(um, up, fm, fp, sm, spp, fh);
        double* o = sFh + G::foff(axis) + (g * nfa + f) * NV * L + t;
#pragma unroll
        for (int v = 0; v < NV; ++v) o[v * L] = fh[v];
      }
    }
    consumer_sync();
    mbar_arrive(&empty[s]);  // ring slot (tile arrays + halo) no longer read

    // ------------------------------------------------ X/Y/Z: volume + lift
#pragma unroll
    for (int axis = 0; axis < DIM; ++axis) {
      if (axis > 0) consumer_sync();
      const double lift = p.lift[axis];
      const int as = G::lstride(axis);
      const bool final_axis = axis == DIM - 1;
#pragma unroll 1
      for (int q = tid; q < TE * NV * L; q += NC) {
        const int t = q % L;
        const int v = (q / L) % NV;
        const int el = q / (L * NV);
        const int ex = el % G::TX, ey = (el / G::TX) % G::TY, ez = el / (G::TX * G::TY);
        if (ex >= tc.v0 || ey >= tc.v1 || ez >= tc.v2) continue;
        const int lb = (el * NV + v) * LP + G::lbase(axis, t);
        const double* Fa = sF + axis * G::ARR + lb;
        double* Dp = sF + lb;  // dudt lives in F_0's slots
        double Fl[N];
#pragma unroll
        for (int l = 0; l < N; ++l) Fl[l] = Fa[l * as];
        double D[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = A::mac(acc, p.K[axis][k * N + l], Fl[l]);
          D[k] = axis == 0 ? zero_plus(acc) : A::add(Dp[k * as], acc);
        }
        const int pos = axis == 0 ? ex : (axis == 1 ? ey : ez);
        const int f = axis == 0 ? ey + G::TY * ez : (axis == 1 ? ex + G::TX * ez : ex + G::TX * ey);
        const int nfa = G::nf(axis);
        const double* fh = sFh + G::foff(axis) + v * L + t;
        D[0] = A::add(D[0], A::mul(lift, fh[(pos * nfa + f) * NV * L]));
        D[N - 1] = A::sub(D[N - 1], A::mul(lift, fh[((pos + 1) * nfa + f) * NV * L]));
        if (!final_axis) {
#pragma unroll
          for (int k = 0; k < N; ++k) Dp[k * as] = D[k];
        } else {
          // RK epilogue (solver.hpp:64-75)
          const size_t e = (size_t)(tc.x0 + ex) + (size_t)C0 * ((size_t)(tc.y0 + ey) + (size_t)C1 * (tc.z0 + ez));
          double* gout = p.out + (e * NV + v) * NPE;
          const double* Sb = sB + lb;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const int n = G::node(axis, t, k);
            const double kv = A::mul(D[k], dt);  // k_i *= dt
            if (!last) {
              gout[n] = kv;
            } else {
              const double un = p.b_last != 0.0 ? A::mac(Sb[k * as], p.b_last, kv) : Sb[k * as];
              gout[n] = un;
              if (!isfinite(un)) record_error(ctl, error_key(step, kPhaseInstability, 0, 0));
              if (KIND == 1 && p.scan_alpha) Dp[k * as] = un;
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
        for (int v = 0; v < NV; ++v) un[v] = sF[(el * NV + v) * LP + sl];
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
      for (int w = 0; w < NC / 32; ++w) m = red[w] > m ? red[w] : m;
      atomicMax(&ctl->alpha_bits, m);
    }
  }
}

}  // namespace ndgx
