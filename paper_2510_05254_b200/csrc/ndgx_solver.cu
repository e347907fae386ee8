// ndgx_solver.cu -- the C ABI (include/ndgx.h): device state, step loop,
// CUDA-graph capture, halo exchange, error mapping onto the reference's
// exception taxonomy.
//
// Reference (paths relative to /root/reference/proj):
//   advance            src/solver.cpp:372-440     -> ndgx_advance
//   serial_rhs         src/solver.cpp:442-456     -> ndgx_rhs
//   RKIntegrator       include/ndg/solver.hpp:39-82 (buffers :41-44)
//   run_partitioned    src/partition.cpp:186-333  -> ndgx_create_partitioned + ndgx_advance
//   exchange_halos     src/partition.cpp:108-129  -> pack_kernel + peer stores / NCCL
//   errors             include/ndg/errors.hpp:13-56
//
// A handle owns one or more BLOCKS of decompose()'s tiling of the mesh:
//   * ndgx_create            one block = the whole mesh, periodic wrap inside it
//   * ndgx_create_rank       one block of a multi-process run; halos over NCCL
//   * ndgx_create_partitioned  P blocks in this process (run_partitioned's
//                            workers) on one or more devices; each block's
//                            pack kernel stores its boundary planes straight
//                            into the neighbour blocks' halo buffers (peer
//                            memory over NVLink when they sit on another GPU)
// Blocks that exchange halos split every stage in two launches: the interior
// elements run on the block's compute stream while the planes move, and the
// boundary shell runs on its comm stream once the neighbours' planes have
// landed, overlapping the interior's tail.  All blocks of a handle share one
// device-resident step control, so they take the same dt and stop together
// (the alpha barrier of run_partitioned, src/partition.cpp:203-217, 253-261).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "ndgx.h"
#include "ndgx_field.cuh"
#include "ndgx_kernels.h"
#include "ndgx_nccl.h"
#include "ndgx_setup.h"

using ndgx::Control;
using ndgx::StageArgs;
using ndgx::StepParams;

namespace {

void set_error(ndgx_error* e, int code, const std::string& msg, long step = 0, int stage = -1,
               const int* cell = nullptr, int worker = -1) {
  if (!e) return;
  std::memset(e, 0, sizeof(*e));
  e->code = code;
  e->step = step;
  e->stage = stage;
  e->worker = worker;
  for (int a = 0; a < 3; ++a) e->cell[a] = cell ? cell[a] : -1;
  std::snprintf(e->message, sizeof(e->message), "%s", msg.c_str());
}

void clear_error(ndgx_error* e) {
  if (!e) return;
  std::memset(e, 0, sizeof(*e));
  e->stage = -1;
  e->worker = -1;
  e->cell[0] = e->cell[1] = e->cell[2] = -1;
}

struct TransportFailure {
  std::string what;
};

struct CudaFailure {
  cudaError_t rc;
  const char* what;
};

inline void ck(cudaError_t rc, const char* what) {
  if (rc != cudaSuccess) throw CudaFailure{rc, what};
}

std::string fmt_double(double v) {  // std::to_string(double) == "%f"
  char b[64];
  std::snprintf(b, sizeof(b), "%f", v);
  return b;
}

struct Box {
  int o[3] = {0, 0, 0};
  int n[3] = {1, 1, 1};
  long long count() const { return (long long)n[0] * n[1] * n[2]; }
};

// One stage-kernel launch over a block: linear element ranges (one grid row
// each) and the region filter (StageArgs::rng / region).
struct Launch {
  int n = 0;
  int rng[ndgx::kMaxRanges][3] = {};  // begin, end, stride
  int region = 0;
  int inner[2][3] = {};
};

enum Mode { kNoExchange = 0, kNccl = 1, kDirect = 2 };

}  // namespace

// One block of the tiling: its state buffers, halo planes and streams.
struct Blk {
  int id = 0;                       // worker / rank
  int dev = 0;
  int cells[3] = {1, 1, 1};
  int goff[3] = {0, 0, 0};
  size_t n = 0;                     // doubles per state array
  ndgx_rank_plan plan{};            // split axes, neighbours, plane sizes
  bool exchange = false;            // some axis takes its halo from a neighbour block
  std::vector<double*> buf;         // u (two parities) and the live K_j
  double* rcv[3][2][2] = {};        // received stage-input planes [axis][side][parity]
  double* snd[3][2] = {};           // NCCL: this block's packed planes
  double* dst[3][2][2] = {};        // peer stores: the neighbours' rcv this block's planes go to
  cudaStream_t st = nullptr;        // compute stream (block 0's is the handle's stream)
  cudaStream_t cs = nullptr;        // comm stream: NCCL and the boundary shell
  cudaEvent_t ev_pack = nullptr, ev_bnd = nullptr, ev_join = nullptr;
  Launch whole, inner, shell;       // the whole block; interior / boundary shell of a split stage

  long long lin(int x, int y, int z) const { return x + (long long)cells[0] * (y + (long long)cells[1] * z); }
  // the elements of box b as one range (begin, end, stride): a contiguous run
  // of the block's element order, or a run of whole x-columns at stride C0
  bool as_range(const Box& b, int r[3]) const {
    int h = 0;
    for (int a = 0; a < 3; ++a)
      if (b.n[a] > 1) h = a;
    bool run = true;
    for (int a = 0; a < h; ++a) run = run && b.n[a] == cells[a];
    const long long f = lin(b.o[0], b.o[1], b.o[2]);
    const long long l = lin(b.o[0] + b.n[0] - 1, b.o[1] + b.n[1] - 1, b.o[2] + b.n[2] - 1);
    if (run) {
      r[0] = (int)f;
      r[1] = (int)l + 1;
      r[2] = 1;
      return true;
    }
    // one x, a contiguous run of (y, z)
    if (b.n[0] == 1 && (b.n[2] == 1 || b.n[1] == cells[1])) {
      r[0] = (int)f;
      r[1] = (int)l + 1;
      r[2] = cells[0];
      return true;
    }
    return false;
  }
  // Launch over a set of boxes: one range each when they all are ranges,
  // else one contiguous span of them all with the region filter against the
  // interior box `in` (the span's elements outside the set are exactly those
  // the filter skips).
  Launch launch_of(const std::vector<Box>& boxes, int region, const Box& in) const {
    Launch L;
    for (int a = 0; a < 3; ++a) {
      L.inner[0][a] = in.o[a];
      L.inner[1][a] = in.o[a] + in.n[a];
    }
    bool ranges = boxes.size() <= (size_t)ndgx::kMaxRanges;
    long long lo = -1, hi = -1;
    for (const Box& b : boxes) {
      int r[3];
      ranges = ranges && as_range(b, r);
      if (ranges) {
        for (int q = 0; q < 3; ++q) L.rng[L.n][q] = r[q];
        ++L.n;
      }
      const long long f = lin(b.o[0], b.o[1], b.o[2]);
      const long long l = lin(b.o[0] + b.n[0] - 1, b.o[1] + b.n[1] - 1, b.o[2] + b.n[2] - 1) + 1;
      lo = lo < 0 ? f : std::min(lo, f);
      hi = std::max(hi, l);
    }
    if (!ranges && !boxes.empty()) {
      L.n = 1;
      L.rng[0][0] = (int)lo;
      L.rng[0][1] = (int)hi;
      L.rng[0][2] = 1;
      L.region = region;
    }
    return L;
  }

  // Interior and boundary shell of the split axes (an onion peel: per split
  // axis the low and high slabs of what is left).
  void make_launches() {
    Box all;
    for (int a = 0; a < 3; ++a) all.n[a] = cells[a];
    whole = launch_of({all}, 0, all);
    Box rest = all;
    std::vector<Box> sh;
    for (int a = 0; a < 3; ++a) {
      if (!plan.split[a] || rest.n[a] <= 0) continue;
      Box lo = rest, hi = rest;
      lo.n[a] = 1;
      hi.o[a] = rest.o[a] + rest.n[a] - 1;
      hi.n[a] = 1;
      if (lo.count() > 0) sh.push_back(lo);
      if (rest.n[a] > 1 && hi.count() > 0) sh.push_back(hi);
      rest.o[a] += 1;
      rest.n[a] = std::max(0, rest.n[a] - 2);
    }
    inner = rest.count() > 0 ? launch_of({rest}, 1, rest) : Launch{};
    // the span of the interior box holds only interior rows when its (y, z)
    // part is one run: then only x needs testing (region 3)
    if (inner.region == 1 && (rest.n[2] == 1 || rest.n[1] == cells[1])) inner.region = 3;
    shell = launch_of(sh, 2, rest);
  }
};

struct ndgx_solver {
  ndgx_problem p{};
  int dim = 0, N = 0, nv = 0, kind = 0, stages = 0, npe = 0;
  int gcells[3] = {1, 1, 1};
  int hcells[3] = {1, 1, 1};        // cells of the field upload/download exchange
  int hoff[3] = {0, 0, 0};          // its offset in the global mesh
  size_t hn = 0;                    // doubles in that field
  int64_t hdof = 0;
  bool exact = true;
  double K[3][64]{}, lift[3]{}, a[7][7]{}, b[7]{};
  double gl_nodes[8]{}, gl_weights[8]{};  // the quadrature rule (device ICs and diagnostics)
  double cflh = 0.0, two_n_minus_1 = 0.0, const_alpha = -1.0;
  ndgx::StageKernel kern;
  ndgx::StageLaunch lcfg[ndgx::kNumSigs];  // per stage signature (ndgx::kSigs)
  std::vector<Blk> blk;
  int mode = kNoExchange;
  bool partitioned = false;         // run_partitioned semantics: errors are RunError("worker w: ...")
  bool multi_device = false;        // blocks on more than one GPU
  bool eager = false;               // launch step by step, no graphs (multi-device, or NDGX_EAGER=1)
  int dead = -1;      // K slot overwritten by u_new at the last stage (-1: none)
  int parity = 0;     // u lives in buf[parity]
  int xpar = 0;       // halo-plane parity of the next stage launch
  Control* ctl = nullptr;
  Control* ctl_warm = nullptr;
  Control* h_ctl = nullptr;  // pinned mirror
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  long long graph_fixed = -2;
  double graph_tend = -1.0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_fork = nullptr;
  ncclComm_t comm = nullptr;
  const ndgx::Nccl* nc = nullptr;
  long long pending_fixed = -1;  // ndgx_launch_steps bookkeeping
  int pending_start_parity = 0;

  Blk& master() { return blk[0]; }
  const Blk& master() const { return blk[0]; }
  cudaStream_t stream() const { return blk[0].st; }
  void on(const Blk& b) const {
    if (multi_device) ck(cudaSetDevice(b.dev), "cudaSetDevice");
  }

  // ------------------------------------------------------------ buffers
  static double* u_buf(const Blk& b, int par) { return b.buf[par]; }
  static double* out_buf(const Blk& b, int par) { return b.buf[1 - par]; }
  double* k_buf(const Blk& b, int j, int par) const {
    if (j == dead) return b.buf[1 - par];
    int rank = j;
    if (dead >= 0 && j > dead) --rank;
    return b.buf[2 + rank];
  }
  double* staging(const Blk& b, int par) const {
    double* r = k_buf(b, 0, par);
    return r != b.buf[1 - par] ? b.buf[1 - par] : b.buf[2];
  }

  StageArgs stage_args(const Blk& bk, int i, int par, Control* c, bool rhs_only, int xp) const {
    StageArgs s;
    std::memset(&s, 0, sizeof(s));
    s.u = u_buf(bk, par);
    s.is_last = (!rhs_only && i == stages - 1) ? 1 : 0;
    // union (ascending j) of the K_j read by the stage input (a_ij != 0,
    // solver.hpp:58) and, at the last stage, by S (b_j != 0, solver.hpp:71)
    s.nu = 0;
    for (int j = 0; j < i; ++j) {
      const bool ua = a[i][j] != 0.0;
      const bool ub = s.is_last && b[j] != 0.0;
      if (!ua && !ub) continue;
      s.ku[s.nu] = k_buf(bk, j, par);
      s.ca[s.nu] = a[i][j];
      s.cb[s.nu] = b[j];
      if (ua) s.amask |= 1 << s.nu;
      if (ub) s.bmask |= 1 << s.nu;
      ++s.nu;
    }
    if (s.is_last) {
      s.b_last = b[i];
      s.out = out_buf(bk, par);
    } else {
      s.out = k_buf(bk, i, par);
    }
    s.ctl = c;
    s.rhs_only = rhs_only ? 1 : 0;
    s.phase = ndgx::kPhaseStage0 + i;
    s.scan_alpha = (s.is_last && kind == NDGX_EULER_ISOTHERMAL) ? 1 : 0;
    for (int d = 0; d < 3; ++d) {
      s.cells[d] = bk.cells[d];
      s.gcells[d] = gcells[d];
      s.goff[d] = bk.goff[d];
      for (int q = 0; q < 2; ++q) s.ext[d][q] = bk.plan.split[d] ? bk.rcv[d][q][xp] : nullptr;
      s.vel[d] = p.velocity[d];
      s.lift[d] = lift[d];
      for (int q = 0; q < 64; ++q) s.K[d][q] = K[d][q];
    }
    s.sound_speed = p.sound_speed;
    s.block_id = bk.id;
    s.sig = sig_of(s);
    s.depth = lcfg[s.sig].depth;
    return s;
  }

  // Per stage: the stage input U_s at this block's boundary face nodes of
  // each split axis, into the planes the neighbours read (pack_face_trace +
  // exchange_halos, src/solver.cpp:166-187, src/partition.cpp:108-129).
  void launch_pack(const Blk& bk, const StageArgs& s, int xp) const {
    ndgx::PackArgs pa;
    std::memset(&pa, 0, sizeof(pa));
    pa.u = s.u;
    for (int t = 0; t < ndgx::kMaxTerms; ++t) {
      pa.ku[t] = s.ku[t];
      pa.ca[t] = s.ca[t];
    }
    pa.nu = s.nu;
    pa.amask = s.amask;
    pa.dim = dim;
    pa.order = N;
    pa.nv = nv;
    pa.npe = npe;
    pa.ctl = s.ctl;
    pa.rhs_only = s.rhs_only;
    long long total = 0;
    for (int d = 0; d < 3; ++d) {
      pa.cells[d] = bk.cells[d];
      pa.split[d] = bk.plan.split[d];
      pa.plane[d] = bk.plan.plane[d];
      for (int q = 0; q < 2; ++q) pa.snd[d][q] = mode == kNccl ? bk.snd[d][q] : bk.dst[d][q][xp];
      if (bk.plan.split[d]) total += 2 * bk.plan.plane[d];
    }
    const int threads = 256;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((total + threads - 1) / threads, 148LL * 8));
    if (exact)
      ndgx::pack_kernel<true><<<blocks, threads, 0, bk.st>>>(pa);
    else
      ndgx::pack_kernel<false><<<blocks, threads, 0, bk.st>>>(pa);
  }

  // NCCL: swap the packed planes with the neighbour ranks on the comm stream
  // (exchange_halos, src/partition.cpp:108-131: per axis send the high plane
  // up and receive the low halo, send the low plane down and receive the
  // high halo -- the same posting order on every rank, so pairs match even
  // when both neighbours are one rank or this rank itself).
  void launch_nccl(const Blk& bk, int xp) const {
    nccl_check(nc->GroupStart(), "ncclGroupStart");
    for (int d = 0; d < dim; ++d) {
      if (!bk.plan.split[d]) continue;
      const size_t n = (size_t)bk.plan.plane[d];
      nccl_check(nc->Send(bk.snd[d][1], n, ncclFloat64, bk.plan.nbr[d][1], comm, bk.cs), "ncclSend");
      nccl_check(nc->Recv(bk.rcv[d][0][xp], n, ncclFloat64, bk.plan.nbr[d][0], comm, bk.cs), "ncclRecv");
      nccl_check(nc->Send(bk.snd[d][0], n, ncclFloat64, bk.plan.nbr[d][0], comm, bk.cs), "ncclSend");
      nccl_check(nc->Recv(bk.rcv[d][1][xp], n, ncclFloat64, bk.plan.nbr[d][1], comm, bk.cs), "ncclRecv");
    }
    nccl_check(nc->GroupEnd(), "ncclGroupEnd");
  }

  // Per step: every rank's dt comes from the global max wavespeed (the
  // alpha barrier of run_partitioned, src/partition.cpp:201-213, 243-252).
  void launch_alpha_reduce(Control* c) const {
    if (!comm) return;
    // {alpha_bits, any_err}: the global wavespeed and whether any rank failed
    nccl_check(nc->AllReduce(&c->alpha_bits, &c->alpha_bits, 2, ncclUint64, ncclMax, comm, stream()),
               "ncclAllReduce");
  }

  // Multi-rank outcome: the earliest error key of all ranks (keys order like
  // the reference's execution), so every rank takes the same decision.
  void launch_err_reduce(Control* c) const {
    if (!comm) return;
    nccl_check(nc->AllReduce(&c->err_key, &c->err_key, 1, ncclUint64, ncclMin, comm, stream()),
               "ncclAllReduce");
  }

  void nccl_check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) throw TransportFailure{std::string(what) + ": " + nc->GetErrorString(r)};
  }

  // The stage kernel over launch L's ranges (one grid row each) on stream `st`.
  void launch_ranges(const StageArgs& s0, const Launch& L, cudaStream_t st) const {
    if (L.n <= 0) return;
    StageArgs s = s0;
    long long most = 0;
    for (int q = 0; q < L.n; ++q) {
      for (int x = 0; x < 3; ++x) s.rng[q][x] = L.rng[q][x];
      most = std::max<long long>(most, (L.rng[q][1] - L.rng[q][0] + L.rng[q][2] - 1) / L.rng[q][2]);
    }
    s.region = L.region;
    std::memcpy(s.inner, L.inner, sizeof(s.inner));
    // a boundary shell spread over the block, or whole x-columns, read HBM
    // directly: a ring would stream the elements it skips / lose its locality
    if (L.region == 2 || (L.n > 0 && L.rng[0][2] != 1)) s.depth = 0;
    for (int q = 0; q < L.n; ++q)
      if (L.rng[q][2] != 1) s.depth = 0;
    // persistent CTAs (one element per warp): as many as are co-resident
    const long long need = (most + kern.warps - 1) / kern.warps;
    const ndgx::StageLaunch& c = lcfg[s.sig];
    const long long grid = std::max<long long>(1, std::min<long long>(need, (long long)c.grid));
    (L.region == 3 ? kern.fnx : kern.fn)[s.sig]<<<dim3((unsigned)grid, (unsigned)L.n), kern.threads, c.smem, st>>>(s);
  }

  void fork() const {
    if (blk.size() < 2) return;
    ck(cudaEventRecord(ev_fork, stream()), "event");
    for (size_t q = 1; q < blk.size(); ++q) {
      on(blk[q]);
      ck(cudaStreamWaitEvent(blk[q].st, ev_fork, 0), "wait");
    }
    on(blk[0]);
  }

  void join() const {
    if (blk.size() < 2) return;
    for (size_t q = 1; q < blk.size(); ++q) {
      on(blk[q]);
      ck(cudaEventRecord(blk[q].ev_join, blk[q].st), "event");
    }
    on(blk[0]);
    for (size_t q = 1; q < blk.size(); ++q) ck(cudaStreamWaitEvent(stream(), blk[q].ev_join, 0), "wait");
  }

  // RK stage i of every block.  Without halo exchange: one launch over the
  // block.  With it: pack the planes (+ NCCL on the comm stream), run the
  // interior on the compute stream, and the boundary shell on the comm
  // stream once the neighbours' planes are in; the compute stream then waits
  // for the shell, so the next stage sees the whole block.
  void launch_stage_all(int i, int par, Control* c, bool rhs_only) {
    const int xp = xpar;
    xpar ^= 1;
    if (mode == kNoExchange) {
      for (const Blk& bk : blk) {
        on(bk);
        launch_ranges(stage_args(bk, i, par, c, rhs_only, xp), bk.whole, bk.st);
      }
      on(blk[0]);
      return;
    }
    for (const Blk& bk : blk) {
      on(bk);
      const StageArgs s = stage_args(bk, i, par, c, rhs_only, xp);
      if (bk.exchange) {
        launch_pack(bk, s, xp);
        ck(cudaEventRecord(bk.ev_pack, bk.st), "event");
        if (mode == kNccl) {
          ck(cudaStreamWaitEvent(bk.cs, bk.ev_pack, 0), "wait");
          launch_nccl(bk, xp);
        }
      }
      launch_ranges(s, bk.exchange ? bk.inner : bk.whole, bk.st);
    }
    for (const Blk& bk : blk) {
      if (!bk.exchange) continue;
      on(bk);
      if (mode == kDirect) {
        // own planes packed (this stream's order) and every neighbour's planes stored
        ck(cudaStreamWaitEvent(bk.cs, bk.ev_pack, 0), "wait");
        for (int d = 0; d < 3; ++d) {
          if (!bk.plan.split[d]) continue;
          for (int q = 0; q < 2; ++q) {
            const int nb = bk.plan.nbr[d][q];
            if (nb != bk.id) ck(cudaStreamWaitEvent(bk.cs, blk[nb].ev_pack, 0), "wait");
          }
        }
      }
      const StageArgs s = stage_args(bk, i, par, c, rhs_only, xp);
      launch_ranges(s, bk.shell, bk.cs);
      ck(cudaEventRecord(bk.ev_bnd, bk.cs), "event");
      ck(cudaStreamWaitEvent(bk.st, bk.ev_bnd, 0), "wait");
    }
    on(blk[0]);
  }

  StepParams step_params(Control* c, long long fixed, int warmup) const {
    StepParams sp;
    sp.ctl = c;
    sp.fixed_steps = fixed;
    sp.t_end = p.t_end;
    sp.cflh = cflh;
    sp.two_n_minus_1 = two_n_minus_1;
    sp.const_alpha = const_alpha;
    sp.warmup = warmup;
    sp.ranked = comm != nullptr ? 1 : 0;
    return sp;
  }

  void launch_step(const StepParams& sp, int par, Control* c) {
    launch_alpha_reduce(c);
    ndgx::step_begin_kernel<<<1, 1, 0, stream()>>>(sp);
    fork();
    for (int i = 0; i < stages; ++i) launch_stage_all(i, par, c, false);
    join();
  }

  void launch_scan(Control* c, int par) const {
    if (kind != NDGX_EULER_ISOTHERMAL) return;
    fork();
    for (const Blk& bk : blk) {
      on(bk);
      const int threads = 256, blocks = 148 * 8;
      const int3 go = make_int3(bk.goff[0], bk.goff[1], bk.goff[2]);
      if (dim == 2)
        ndgx::alpha_scan_kernel<2><<<blocks, threads, 0, bk.st>>>(u_buf(bk, par), bk.cells[0], bk.cells[1],
                                                                  bk.cells[2], N, p.sound_speed, c, 1, go,
                                                                  gcells[1], gcells[2]);
      else
        ndgx::alpha_scan_kernel<3><<<blocks, threads, 0, bk.st>>>(u_buf(bk, par), bk.cells[0], bk.cells[1],
                                                                  bk.cells[2], N, p.sound_speed, c, 1, go,
                                                                  gcells[1], gcells[2]);
    }
    on(blk[0]);
    join();
  }

  void reset_control(Control* c) const {
    Control h;
    std::memset(&h, 0, sizeof(h));
    h.err_key = ndgx::kNoError;
    h.dt_min = std::numeric_limits<double>::infinity();
    h.dt_max = 0.0;
    *h_ctl = h;
    ck(cudaMemcpyAsync(c, h_ctl, sizeof(Control), cudaMemcpyHostToDevice, stream()), "reset control");
  }

  Control read_control(Control* c) const {
    ck(cudaMemcpyAsync(h_ctl, c, sizeof(Control), cudaMemcpyDeviceToHost, stream()), "read control");
    ck(cudaStreamSynchronize(stream()), "sync");
    return *h_ctl;
  }

  void ensure_graphs(long long fixed) {
    if (eager) return;  // step-by-step launches (see launch_run)
    if (graph[0] && graph_fixed == fixed && graph_tend == p.t_end) return;
    for (auto& g : graph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    const StepParams sp = step_params(ctl, fixed, 0);
    for (int par = 0; par < 2; ++par) {
      cudaGraph_t g;
      // two steps = an even number of stage launches, so the halo-plane
      // parity of each captured stage repeats identically on every replay
      ck(cudaStreamBeginCapture(stream(), comm ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal),
         "begin capture");
      xpar = 0;
      launch_step(sp, par, ctl);
      launch_step(sp, 1 - par, ctl);
      ck(cudaStreamEndCapture(stream(), &g), "end capture");
      ck(cudaGraphInstantiate(&graph[par], g, 0), "graph instantiate");
      cudaGraphDestroy(g);
    }
    graph_fixed = fixed;
    graph_tend = p.t_end;
  }

  // `steps` steps from parity `start_par` (graph pairs, or eager launches
  // when the blocks span several devices).  A trailing odd step of a graph
  // pair is skipped on the device by step_begin (steps >= fixed_steps).
  void launch_run(long long steps, int start_par, long long fixed) {
    if (eager) {
      const StepParams sp = step_params(ctl, fixed, 0);
      for (long long q = 0; q < steps; ++q) launch_step(sp, start_par ^ (int)(q & 1), ctl);
      return;
    }
    for (long long q = 0; q < (steps + 1) / 2; ++q) ck(cudaGraphLaunch(graph[start_par], stream()), "graph");
  }

  static int sig_of(const StageArgs& s) {
    for (int q = 0; q < ndgx::kNumSigs; ++q)
      if (ndgx::kSigs[q].nu == s.nu && ndgx::kSigs[q].am == s.amask && ndgx::kSigs[q].bm == s.bmask) return q;
    return -1;
  }

  // Per stage signature: the per-warp ring depth (0 = direct loads) giving the
  // most resident warps (the element pipeline is issue-bound), then the most
  // elements in flight.
  int configure_launches(const cudaDeviceProp& prop, ndgx_error* err) {
    const int limit = (int)prop.sharedMemPerBlockOptin;
    for (int i = 0; i < stages; ++i) {
      StageArgs t;
      std::memset(&t, 0, sizeof(t));
      for (int j = 0; j < i; ++j) {
        const bool ua = a[i][j] != 0.0, ub = i == stages - 1 && b[j] != 0.0;
        if (!ua && !ub) continue;
        if (ua) t.amask |= 1 << t.nu;
        if (ub) t.bmask |= 1 << t.nu;
        ++t.nu;
      }
      // the kernels take "last stage" from the signature (b-terms present)
      if (sig_of(t) < 0 || (i == stages - 1) != (t.bmask != 0)) {
        set_error(err, NDGX_ERR_CONFIG, "Runge-Kutta tableau without a compiled stage signature");
        return NDGX_ERR_CONFIG;
      }
    }
    // NDGX_DEPTH=<d> forces one ring depth (0 = direct loads) where it fits (tuning)
    const char* env = std::getenv("NDGX_DEPTH");
    const int forced = env ? std::atoi(env) : -1;
    for (int q = 0; q < ndgx::kNumSigs; ++q) {
      const void* fn = reinterpret_cast<const void*>(kern.fn[q]);
      ndgx::StageLaunch best;
      long long best_score = -1;
      for (int d = (kern.tma_ok && (!kern.prefer_direct || forced > 0)) ? 4 : 0; d >= 0; --d) {
        if (d == 1) continue;  // a ring needs one slot ahead
        if (forced >= 0 && d != forced && !(d == 0 && !kern.tma_ok)) continue;
        const int bytes = kern.smem(q, d);
        if (bytes > limit) continue;
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "smem attribute");
        int per_sm = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kern.threads, bytes), "occupancy");
        if (per_sm < 1) continue;
        const long long score = (long long)per_sm * kern.warps * 16 + std::max(1, d - 1);
        if (score > best_score) {
          best_score = score;
          best.depth = d;
          best.smem = bytes;
          best.grid = per_sm * prop.multiProcessorCount;
        }
      }
      if (best_score < 0) {
        set_error(err, NDGX_ERR_CONFIG, "stage kernel does not fit in shared memory");
        return NDGX_ERR_CONFIG;
      }
      ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, best.smem), "smem attribute");
      if (kern.fnx[q] != kern.fn[q])
        ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern.fnx[q]),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, best.smem),
           "smem attribute");
      lcfg[q] = best;
    }
    return NDGX_OK;
  }

  // global AoS cell index -> global cell coordinates
  void global_cell(long long aos_cell, int g[3]) const {
    g[2] = (int)(aos_cell % gcells[2]);
    g[1] = (int)((aos_cell / gcells[2]) % gcells[1]);
    g[0] = (int)(aos_cell / ((long long)gcells[2] * gcells[1]));
  }

  // the block holding a global cell (nullptr: not in this handle)
  const Blk* owner(const int g[3]) const {
    for (const Blk& bk : blk) {
      bool in = true;
      for (int a = 0; a < 3; ++a) in = in && g[a] >= bk.goff[a] && g[a] < bk.goff[a] + bk.cells[a];
      if (in) return &bk;
    }
    return nullptr;
  }

  size_t device_index(const Blk& bk, const int lc[3], int aos_node, int var) const {
    int i = 0, j = 0, k = 0;
    if (dim == 1) i = aos_node;
    if (dim == 2) { i = aos_node / N; j = aos_node % N; }
    if (dim == 3) { i = aos_node / (N * N); j = (aos_node / N) % N; k = aos_node % N; }
    const size_t e = (size_t)lc[0] + (size_t)bk.cells[0] * ((size_t)lc[1] + (size_t)bk.cells[1] * lc[2]);
    const size_t nn = (size_t)i + (size_t)N * ((size_t)j + (size_t)N * k);
    return (e * nv + var) * npe + nn;
  }

  double fetch(const Blk& bk, const double* dev, size_t idx) const {
    double v = 0.0;
    on(bk);
    ck(cudaMemcpy(&v, dev + idx, sizeof(double), cudaMemcpyDeviceToHost), "fetch");
    on(blk[0]);
    return v;
  }

  // Map a device error key onto the reference's exception (message text
  // follows src/solver.cpp:258-261, 325-328, 364-365, 411-413).  A
  // partitioned handle wraps it as run_partitioned does: RunError("worker w:
  // <message>", w) (src/partition.cpp:315-326).  A rank solver whose block
  // does not hold the failure reports "stopped by failure elsewhere".
  int report(unsigned long long key, int start_par, ndgx_error* err) const {
    const long step = (long)(key >> 44);
    const int phase = (int)((key >> 40) & 0xF);
    const long long cell = (long long)((key >> 12) & 0xFFFFFFF);
    const int node = (int)(key & 0xFFF);
    const int par = start_par ^ (int)((step > 0 ? step - 1 : 0) & 1);
    int code = NDGX_ERR_CONFIG, stage = -1, worker = 0;
    int lc[3] = {-1, -1, -1};
    std::string msg;
    const Blk* bk = nullptr;
    if (phase == ndgx::kPhaseZeroSpeed) {
      msg = "fixed-step run requires a positive wavespeed";
      worker = blk[0].id;
    } else if (phase == ndgx::kPhaseInstability) {
      code = NDGX_ERR_INSTABILITY;
      msg = "non-finite state after step " + std::to_string(step);
      worker = (int)cell;  // the block id rides in the cell field
      for (const Blk& q : blk)
        if (q.id == worker) bk = &q;
    } else {
      int g[3];
      global_cell(cell, g);
      bk = owner(g);
      if (bk) {
        worker = bk->id;
        for (int x = 0; x < 3; ++x) lc[x] = g[x] - bk->goff[x];
        // scan keys carry the AoS node; operator keys the reference's
        // volume-traversal order (line (j, k) outer, i inner: j N + i in 2D,
        // (j N + k) N + i in 3D) so that the earliest key is its first failure
        int aos = node;
        if (phase != ndgx::kPhaseScan && dim == 2) aos = (node % N) * N + node / N;
        if (phase != ndgx::kPhaseScan && dim == 3)
          aos = ((node % N) * N + node / (N * N)) * N + (node / N) % N;
        const size_t idx = device_index(*bk, lc, aos, 0);
        code = NDGX_ERR_PHYSICS;
        if (phase == ndgx::kPhaseScan) {
          const double rho = fetch(*bk, u_buf(*bk, par), idx);
          msg = "nonpositive density " + fmt_double(rho) + " in time-step estimate";
        } else {
          // operator PhysicsError at stage `stage`: recompute the stage input there
          stage = phase - ndgx::kPhaseStage0;
          double rho = fetch(*bk, u_buf(*bk, par), idx);
          for (int j = 0; j < stage; ++j) {
            if (a[stage][j] == 0.0) continue;
            rho += a[stage][j] * fetch(*bk, k_buf(*bk, j, par), idx);
          }
          // the reference names the cell in the worker's own block (solver.cpp:258-261)
          msg = "nonpositive density " + fmt_double(rho) + " in flux evaluation at cell (" +
                std::to_string(lc[0]) + "," + std::to_string(lc[1]) + "," + std::to_string(lc[2]) + ")";
        }
      }
    }
    if (comm && phase != ndgx::kPhaseZeroSpeed && bk == nullptr) {
      set_error(err, NDGX_ERR_RUN, "rank " + std::to_string(blk[0].id) + ": stopped by failure elsewhere", step,
                -1, nullptr, blk[0].id);
      return NDGX_ERR_RUN;
    }
    if (partitioned) {
      set_error(err, NDGX_ERR_RUN, "worker " + std::to_string(worker) + ": " + msg, step, stage,
                lc[0] >= 0 ? lc : nullptr, worker);
      return NDGX_ERR_RUN;
    }
    set_error(err, code, msg, code == NDGX_ERR_CONFIG ? 0 : step, stage, lc[0] >= 0 ? lc : nullptr);
    return code;
  }

  ~ndgx_solver() {
    // graphs that captured NCCL work go before the communicator; the
    // communicator is torn down with ncclCommAbort (ncclCommDestroy can block
    // on the proxy of a communicator whose graphs were captured)
    for (auto& g : graph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    for (Blk& bk : blk) {
      cudaSetDevice(bk.dev);
      if (bk.st) cudaStreamSynchronize(bk.st);
      if (bk.cs) cudaStreamSynchronize(bk.cs);
    }
    if (comm && nc) nc->CommAbort(comm);
    for (Blk& bk : blk) {
      cudaSetDevice(bk.dev);
      for (int d = 0; d < 3; ++d)
        for (int q = 0; q < 2; ++q) {
          if (bk.snd[d][q]) cudaFree(bk.snd[d][q]);
          for (int x = 0; x < 2; ++x)
            if (bk.rcv[d][q][x]) cudaFree(bk.rcv[d][q][x]);
        }
      for (double* q : bk.buf) cudaFree(q);
      for (cudaEvent_t e : {bk.ev_pack, bk.ev_bnd, bk.ev_join})
        if (e) cudaEventDestroy(e);
      if (bk.cs) cudaStreamDestroy(bk.cs);
      if (bk.st) cudaStreamDestroy(bk.st);
    }
    if (!blk.empty()) cudaSetDevice(blk[0].dev);
    if (ctl) cudaFree(ctl);
    if (ctl_warm) cudaFree(ctl_warm);
    if (h_ctl) cudaFreeHost(h_ctl);
    for (cudaEvent_t e : {ev0, ev1, ev_fork})
      if (e) cudaEventDestroy(e);
  }
};

namespace {

int cuda_error(ndgx_error* err, const CudaFailure& f) {
  set_error(err, NDGX_ERR_CUDA, std::string(f.what) + ": " + cudaGetErrorString(f.rc));
  return NDGX_ERR_CUDA;
}

int validate_problem(const ndgx_problem* p, ndgx_error* err) {
  auto cfg = [&](const std::string& m) {
    set_error(err, NDGX_ERR_CONFIG, m);
    return (int)NDGX_ERR_CONFIG;
  };
  // Mesh ctor (src/grid.cpp:52-64)
  if (p->dim < 1 || p->dim > 3) return cfg("mesh dimension must be 1..3");
  if (p->order < 2 || p->order > 16) return cfg("mesh order must lie in 2..16");
  for (int a = 0; a < p->dim; ++a) {
    if (p->cells[a] < 1) return cfg("cell count must be >= 1 on every axis");
    if (!(p->length[a] > 0.0)) return cfg("domain length must be positive");
  }
  // EquationModel factories (src/models.cpp:14-33)
  if (p->equation == NDGX_ADVECTION) {
  } else if (p->equation == NDGX_EULER_ISOTHERMAL) {
    if (p->dim < 2) return cfg("isothermal_euler: spatial_dim must be 2 or 3");
    if (!(p->sound_speed > 0.0)) return cfg("isothermal_euler: sound speed must be positive");
  } else {
    return cfg("unknown equation kind");
  }
  if (p->rk < NDGX_RK3 || p->rk > NDGX_RK6)
    return cfg("unknown Runge-Kutta scheme (expected rk3, rk4 or rk6)");
  // validate (src/solver.cpp:349-357)
  if (!(p->cfl > 0.0) || p->cfl > 1.0) return cfg("cfl must lie in (0, 1]");
  if (!(p->t_end > 0.0)) return cfg("t_end must be positive");
  if (p->order > ndgx::kMaxOrder)
    return cfg("the GPU path supports orders 2..8 (got " + std::to_string(p->order) + ")");
  return NDGX_OK;
}

// One worker's plan in decompose()'s tiling (host only).
int plan_of(const ndgx_problem* global, int nranks, int rank, int force_exchange, const std::vector<int>& lo,
            const std::vector<int>& hi, const std::vector<int>& nbr, const int grid[3], ndgx_rank_plan* plan) {
  ndgx_rank_plan pl;
  std::memset(&pl, 0, sizeof(pl));
  pl.rank = rank;
  pl.nranks = nranks;
  const int nv = global->equation == NDGX_ADVECTION ? 1 : global->dim + 1;
  const int N = global->order;
  const long long L = global->dim == 1 ? 1 : (global->dim == 2 ? N : (long long)N * N);
  for (int a = 0; a < 3; ++a) {
    pl.grid[a] = grid[a];
    pl.lo[a] = lo[3 * rank + a];
    pl.hi[a] = hi[3 * rank + a];
    pl.nbr[a][0] = nbr[6 * rank + 2 * a];
    pl.nbr[a][1] = nbr[6 * rank + 2 * a + 1];
    pl.split[a] = a < global->dim && (pl.grid[a] > 1 || force_exchange) ? 1 : 0;
  }
  for (int a = 0; a < 3; ++a) {
    long long cross = 1;
    for (int b = 0; b < 3; ++b)
      if (b != a) cross *= pl.hi[b] - pl.lo[b];
    pl.plane[a] = a < global->dim ? cross * L * nv : 0;
  }
  *plan = pl;
  return NDGX_OK;
}

int decompose_all(const ndgx_problem* global, int workers, std::vector<int>& lo, std::vector<int>& hi,
                  std::vector<int>& nbr, int grid[3], ndgx_error* err) {
  lo.assign(3 * workers, 0);
  hi.assign(3 * workers, 0);
  nbr.assign(6 * workers, 0);
  return ndgx_decompose(global->dim, global->cells, workers, grid, lo.data(), hi.data(), nbr.data(), err);
}

}  // namespace

// A handle over `plans` (nullptr: one block = the whole mesh) on `devices`
// (block q on devices[q % ndev]).  The operator, dt numerator and wavespeed
// use the global mesh, so every block computes with the reference's exact
// coefficients.
static int create_blocks(const ndgx_problem* prob, const std::vector<ndgx_rank_plan>* plans,
                         const std::vector<int>& devices, int mode, ndgx_solver** out, ndgx_error* err) {
  clear_error(err);
  if (!prob || !out) {
    set_error(err, NDGX_ERR_CONFIG, "null argument");
    return NDGX_ERR_CONFIG;
  }
  *out = nullptr;
  if (int rc = validate_problem(prob, err)) return rc;
  ndgx_solver* s = new (std::nothrow) ndgx_solver();
  if (!s) {
    set_error(err, NDGX_ERR_CUDA, "host allocation failed");
    return NDGX_ERR_CUDA;
  }
  try {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      delete s;
      set_error(err, NDGX_ERR_CUDA, "no CUDA device: the ndgx path has no CPU fallback");
      return NDGX_ERR_CUDA;
    }
    for (int d : devices) {
      if (d < 0 || d >= ndev) {
        delete s;
        set_error(err, NDGX_ERR_CONFIG, "device ordinal " + std::to_string(d) + " out of range");
        return NDGX_ERR_CONFIG;
      }
      cudaDeviceProp prop;
      ck(cudaGetDeviceProperties(&prop, d), "cudaGetDeviceProperties");
      if (prop.major != 10) {
        delete s;
        set_error(err, NDGX_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100 (B200)");
        return NDGX_ERR_CUDA;
      }
    }
    ck(cudaSetDevice(devices[0]), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, devices[0]), "cudaGetDeviceProperties");
    s->p = *prob;
    s->p.nodes = s->p.weights = s->p.diff = nullptr;
    s->p.device = devices[0];
    s->dim = prob->dim;
    s->N = prob->order;
    s->kind = prob->equation;
    s->nv = s->kind == NDGX_ADVECTION ? 1 : s->dim + 1;
    s->exact = prob->arith != NDGX_ARITH_FAST;
    s->mode = mode;
    s->npe = 1;
    for (int a = 0; a < s->dim; ++a) s->npe *= s->N;
    for (int a = 0; a < 3; ++a) s->gcells[a] = a < s->dim ? prob->cells[a] : 1;

    const int nblk = plans ? (int)plans->size() : 1;
    s->blk.resize(nblk);
    for (int q = 0; q < nblk; ++q) {
      Blk& bk = s->blk[q];
      bk.dev = devices[q % devices.size()];
      if (bk.dev != devices[0]) s->multi_device = true;
      if (plans) {
        bk.plan = (*plans)[q];
        bk.id = bk.plan.rank;
        for (int a = 0; a < 3; ++a) {
          bk.goff[a] = bk.plan.lo[a];
          bk.cells[a] = bk.plan.hi[a] - bk.plan.lo[a];
          bk.exchange = bk.exchange || bk.plan.split[a] != 0;
        }
      } else {
        bk.plan.nranks = 1;
        for (int a = 0; a < 3; ++a) {
          bk.cells[a] = s->gcells[a];
          bk.plan.grid[a] = 1;
          bk.plan.hi[a] = bk.cells[a];
        }
      }
      if (!bk.exchange) {
        for (int a = 0; a < 3; ++a) bk.plan.split[a] = 0;
      }
      bk.n = (size_t)s->nv * s->npe * bk.cells[0] * bk.cells[1] * bk.cells[2];
      bk.make_launches();
    }
    bool any_exchange = false;
    for (const Blk& bk : s->blk) any_exchange = any_exchange || bk.exchange;
    if (!any_exchange) s->mode = kNoExchange;
    // graphs hold one device's work; NDGX_EAGER=1 takes the multi-device
    // launch sequence on one device (test hook)
    const char* eg = std::getenv("NDGX_EAGER");
    s->eager = s->multi_device || (eg && std::atoi(eg) != 0);
    // the field upload/download exchange: the global mesh for a handle of
    // every block, the block's own for a rank solver
    if (mode == kNccl) {
      for (int a = 0; a < 3; ++a) {
        s->hcells[a] = s->blk[0].cells[a];
        s->hoff[a] = s->blk[0].goff[a];
      }
    } else {
      for (int a = 0; a < 3; ++a) s->hcells[a] = s->gcells[a];
    }
    s->hn = (size_t)s->nv * s->npe * s->hcells[0] * s->hcells[1] * s->hcells[2];
    s->hdof = (int64_t)s->hn;

    // basis: caller's (reference) or our own restatement
    double nodes[16], weights[16], diff[256];
    if (prob->nodes && prob->weights && prob->diff) {
      std::memcpy(nodes, prob->nodes, sizeof(double) * s->N);
      std::memcpy(weights, prob->weights, sizeof(double) * s->N);
      std::memcpy(diff, prob->diff, sizeof(double) * s->N * s->N);
    } else {
      ndgx_gauss_lobatto(s->N, nodes, weights);
      ndgx_differentiation_matrix(s->N, nodes, diff);
    }
    ndgx::build_operator(&s->p, nodes, weights, diff, s->K, s->lift);
    std::memcpy(s->gl_nodes, nodes, sizeof(double) * s->N);
    std::memcpy(s->gl_weights, weights, sizeof(double) * s->N);
    ndgx::rk_tableau(prob->rk, &s->stages, s->a, s->b);
    s->cflh = ndgx::dt_numerator(&s->p);
    s->two_n_minus_1 = (double)(2 * s->N - 1);
    if (s->kind == NDGX_ADVECTION) {
      double alpha = 0.0;  // max_wavespeed_bound, advection (src/solver.cpp:312-317)
      for (int d = 0; d < s->dim; ++d) {
        const double v = std::abs(prob->velocity[d]);
        alpha = (alpha < v) ? v : alpha;
      }
      s->const_alpha = alpha;
    }
    const int last = s->stages - 1;
    s->dead = -1;
    for (int j = 0; j < last; ++j)
      if (s->a[last][j] == 0.0) {
        s->dead = j;
        break;
      }

    s->kern = ndgx::find_stage_kernel(s->dim, s->N, s->kind, s->exact);
    if (!s->kern.fn[0]) {
      delete s;
      set_error(err, NDGX_ERR_CONFIG, "no GPU kernel for this (dim, order, equation)");
      return NDGX_ERR_CONFIG;
    }
    // launch attributes are per device: configure on every device used
    for (size_t q = s->blk.size(); q-- > 0;) {
      ck(cudaSetDevice(s->blk[q].dev), "cudaSetDevice");
      if (int rc = s->configure_launches(prop, err)) {
        delete s;
        return rc;
      }
    }
    ck(cudaSetDevice(devices[0]), "cudaSetDevice");
    if (s->multi_device) {
      // peer stores of the halo planes and the shared step control
      std::vector<int> used;
      for (const Blk& bk : s->blk)
        if (std::find(used.begin(), used.end(), bk.dev) == used.end()) used.push_back(bk.dev);
      for (int x : used)
        for (int y : used) {
          if (x == y) continue;
          int ok = 0;
          ck(cudaDeviceCanAccessPeer(&ok, x, y), "cudaDeviceCanAccessPeer");
          if (!ok) {
            delete s;
            set_error(err, NDGX_ERR_TRANSPORT,
                      "devices " + std::to_string(x) + " and " + std::to_string(y) + " have no peer access");
            return NDGX_ERR_TRANSPORT;
          }
          ck(cudaSetDevice(x), "cudaSetDevice");
          const cudaError_t r = cudaDeviceEnablePeerAccess(y, 0);
          if (r != cudaSuccess && r != cudaErrorPeerAccessAlreadyEnabled) ck(r, "cudaDeviceEnablePeerAccess");
          cudaGetLastError();
        }
      ck(cudaSetDevice(devices[0]), "cudaSetDevice");
    }
    const int nbuf = s->dead >= 0 ? s->stages : s->stages + 1;
    for (Blk& bk : s->blk) {
      ck(cudaSetDevice(bk.dev), "cudaSetDevice");
      ck(cudaStreamCreateWithFlags(&bk.st, cudaStreamNonBlocking), "stream");
      if (bk.exchange) ck(cudaStreamCreateWithFlags(&bk.cs, cudaStreamNonBlocking), "stream");
      ck(cudaEventCreateWithFlags(&bk.ev_pack, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&bk.ev_bnd, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&bk.ev_join, cudaEventDisableTiming), "event");
      for (int q = 0; q < nbuf; ++q) {
        double* d = nullptr;
        ck(cudaMalloc(&d, bk.n * sizeof(double)), "cudaMalloc state");
        bk.buf.push_back(d);
      }
      ck(cudaMemsetAsync(bk.buf[0], 0, bk.n * sizeof(double), bk.st), "memset");
      for (int d = 0; d < 3; ++d)
        if (bk.plan.split[d])
          for (int q = 0; q < 2; ++q) {
            if (s->mode == kNccl) ck(cudaMalloc(&bk.snd[d][q], bk.plan.plane[d] * sizeof(double)), "cudaMalloc plane");
            for (int x = 0; x < 2; ++x) {
              ck(cudaMalloc(&bk.rcv[d][q][x], bk.plan.plane[d] * sizeof(double)), "cudaMalloc plane");
              ck(cudaMemsetAsync(bk.rcv[d][q][x], 0, bk.plan.plane[d] * sizeof(double), bk.st), "memset");
            }
          }
    }
    // peer stores: this block's high plane is the high neighbour's low halo, and vice versa
    if (s->mode == kDirect)
      for (Blk& bk : s->blk)
        for (int d = 0; d < 3; ++d)
          if (bk.plan.split[d])
            for (int x = 0; x < 2; ++x) {
              bk.dst[d][1][x] = s->blk[bk.plan.nbr[d][1]].rcv[d][0][x];
              bk.dst[d][0][x] = s->blk[bk.plan.nbr[d][0]].rcv[d][1][x];
            }
    ck(cudaSetDevice(devices[0]), "cudaSetDevice");
    ck(cudaEventCreate(&s->ev0), "event");
    ck(cudaEventCreate(&s->ev1), "event");
    ck(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming), "event");
    ck(cudaMalloc(&s->ctl, sizeof(Control)), "cudaMalloc control");
    ck(cudaMalloc(&s->ctl_warm, sizeof(Control)), "cudaMalloc control");
    ck(cudaMallocHost(&s->h_ctl, sizeof(Control)), "cudaMallocHost");
    for (Blk& bk : s->blk) {
      ck(cudaSetDevice(bk.dev), "cudaSetDevice");
      ck(cudaStreamSynchronize(bk.st), "sync");
    }
    ck(cudaSetDevice(devices[0]), "cudaSetDevice");
  } catch (const CudaFailure& f) {
    delete s;
    return cuda_error(err, f);
  }
  *out = s;
  return NDGX_OK;
}

extern "C" {

const char* ndgx_version(void) { return "ndgx 0.1.0 sm_100a"; }

int ndgx_create(const ndgx_problem* prob, ndgx_solver** out, ndgx_error* err) {
  if (!prob) {
    clear_error(err);
    set_error(err, NDGX_ERR_CONFIG, "null argument");
    return NDGX_ERR_CONFIG;
  }
  return create_blocks(prob, nullptr, std::vector<int>{prob->device}, kNoExchange, out, err);
}

int ndgx_plan_rank(const ndgx_problem* global, int nranks, int rank, int force_exchange, ndgx_rank_plan* plan,
                   ndgx_error* err) {
  clear_error(err);
  if (!global || !plan) {
    set_error(err, NDGX_ERR_CONFIG, "null argument");
    return NDGX_ERR_CONFIG;
  }
  if (int rc = validate_problem(global, err)) return rc;
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    set_error(err, NDGX_ERR_CONFIG, "rank " + std::to_string(rank) + " outside 0.." + std::to_string(nranks - 1));
    return NDGX_ERR_CONFIG;
  }
  std::vector<int> lo, hi, nbr;
  int grid[3];
  if (int rc = decompose_all(global, nranks, lo, hi, nbr, grid, err)) return rc;
  return plan_of(global, nranks, rank, force_exchange, lo, hi, nbr, grid, plan);
}

int ndgx_create_partitioned(const ndgx_problem* global, int workers, int n_devices, const int* device_ids,
                            int force_exchange, ndgx_solver** out, ndgx_error* err) {
  clear_error(err);
  if (!global || !out) {
    set_error(err, NDGX_ERR_CONFIG, "null argument");
    return NDGX_ERR_CONFIG;
  }
  if (int rc = validate_problem(global, err)) return rc;
  std::vector<int> lo, hi, nbr;
  int grid[3];
  if (int rc = decompose_all(global, workers, lo, hi, nbr, grid, err)) return rc;
  std::vector<ndgx_rank_plan> plans(workers);
  for (int w = 0; w < workers; ++w) plan_of(global, workers, w, force_exchange, lo, hi, nbr, grid, &plans[w]);
  std::vector<int> devs;
  if (n_devices > 0 && device_ids)
    devs.assign(device_ids, device_ids + n_devices);
  else
    devs.push_back(global->device);
  if (int rc = create_blocks(global, &plans, devs, kDirect, out, err)) return rc;
  (*out)->partitioned = true;
  return NDGX_OK;
}

int ndgx_nccl_unique_id(unsigned char id[128], ndgx_error* err) {
  clear_error(err);
  std::string why;
  const ndgx::Nccl* nc = ndgx::nccl(&why);
  if (!nc) {
    set_error(err, NDGX_ERR_TRANSPORT, why);
    return NDGX_ERR_TRANSPORT;
  }
  ncclUniqueId uid;
  const ncclResult_t r = nc->GetUniqueId(&uid);
  if (r != ncclSuccess) {
    set_error(err, NDGX_ERR_TRANSPORT, std::string("ncclGetUniqueId: ") + nc->GetErrorString(r));
    return NDGX_ERR_TRANSPORT;
  }
  std::memcpy(id, uid.internal, sizeof(uid.internal));
  return NDGX_OK;
}

int ndgx_create_rank(const ndgx_problem* global, int nranks, int rank, const unsigned char nccl_id[128],
                     int force_exchange, ndgx_solver** out, ndgx_error* err) {
  ndgx_rank_plan plan;
  if (int rc = ndgx_plan_rank(global, nranks, rank, force_exchange, &plan, err)) return rc;
  std::string why;
  const ndgx::Nccl* nc = ndgx::nccl(&why);
  if (!nc) {
    set_error(err, NDGX_ERR_TRANSPORT, why);
    return NDGX_ERR_TRANSPORT;
  }
  const std::vector<ndgx_rank_plan> plans{plan};
  if (int rc = create_blocks(global, &plans, std::vector<int>{global->device}, kNccl, out, err)) return rc;
  ndgx_solver* s = *out;
  ncclUniqueId uid;
  std::memcpy(uid.internal, nccl_id, sizeof(uid.internal));
  cudaSetDevice(global->device);
  const ncclResult_t r = nc->CommInitRank(&s->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    ndgx_destroy(s);
    *out = nullptr;
    set_error(err, NDGX_ERR_TRANSPORT, std::string("ncclCommInitRank: ") + nc->GetErrorString(r));
    return NDGX_ERR_TRANSPORT;
  }
  s->nc = nc;
  return NDGX_OK;
}

// the extent written in a dump header for `cells` cells of the mesh along `a`
static double field_length(const ndgx_solver* s, int a) {
  return s->hcells[a] == s->gcells[a] ? s->p.length[a] : s->hcells[a] * (s->p.length[a] / s->gcells[a]);
}

static std::string fmt_len(double v) {  // std::ostream << double (precision 6, %g)
  std::ostringstream o;
  o << v;
  return o.str();
}

// ------------------------------------------------------------ f4: device ICs and diagnostics
static ndgx::FieldArgs field_args(const ndgx_solver* s, const Blk& bk) {
  ndgx::FieldArgs a;
  std::memset(&a, 0, sizeof(a));
  a.u = ndgx_solver::u_buf(bk, s->parity);
  a.dim = s->dim;
  a.N = s->N;
  a.nv = s->nv;
  a.npe = s->npe;
  a.jac = 1.0;
  for (int d = 0; d < 3; ++d) {
    a.cells[d] = bk.cells[d];
    a.goff[d] = bk.goff[d];
    a.dx[d] = s->p.length[d] / s->gcells[d];  // Mesh::cell_size (grid.hpp:27)
    if (d < s->dim) a.jac *= 0.5 * a.dx[d];   // src/grid.cpp:33-34
  }
  for (int q = 0; q < s->N; ++q) {
    a.nodes[q] = s->gl_nodes[q];
    a.weights[q] = s->gl_weights[q];
  }
  a.sound_speed = s->p.sound_speed;
  a.ic = -1;
  return a;
}

// the reference's init_* ConfigErrors (src/grid.cpp:135-170)
static int check_ic(const ndgx_solver* s, int ic, const double* amps, int n_modes, ndgx_error* err) {
  if (ic == NDGX_IC_MULTISINE) {
    if (s->kind != NDGX_ADVECTION) {
      set_error(err, NDGX_ERR_CONFIG, "init_multisine applies to the advection scalar only");
      return NDGX_ERR_CONFIG;
    }
    if (n_modes < 1 || !amps) {
      set_error(err, NDGX_ERR_CONFIG, "multisine: need at least one mode");
      return NDGX_ERR_CONFIG;
    }
    if (n_modes > ndgx::kMaxModes) {
      set_error(err, NDGX_ERR_CONFIG, "multisine: more than 256 modes on the device path");
      return NDGX_ERR_CONFIG;
    }
  } else if (ic == NDGX_IC_EULER_SUBSONIC) {
    if (s->kind != NDGX_EULER_ISOTHERMAL) {
      set_error(err, NDGX_ERR_CONFIG, "init_euler_subsonic requires an isothermal Euler model");
      return NDGX_ERR_CONFIG;
    }
    if (s->dim < 2) {
      set_error(err, NDGX_ERR_CONFIG, "init_euler_subsonic is defined for 2D/3D meshes");
      return NDGX_ERR_CONFIG;
    }
  } else {
    set_error(err, NDGX_ERR_CONFIG, "unknown initial condition");
    return NDGX_ERR_CONFIG;
  }
  return NDGX_OK;
}

// the amplitudes on the block's device (freed by the caller)
static double* device_amps(const double* amps, int n_modes) {
  if (!amps || n_modes <= 0) return nullptr;
  double* d = nullptr;
  ck(cudaMalloc(&d, sizeof(double) * n_modes), "cudaMalloc amplitudes");
  ck(cudaMemcpy(d, amps, sizeof(double) * n_modes, cudaMemcpyHostToDevice), "copy amplitudes");
  return d;
}

static unsigned field_grid(const Blk& bk, int npe) {
  const long long nodes = (long long)bk.cells[0] * bk.cells[1] * bk.cells[2] * npe;
  return (unsigned)std::max<long long>(1, std::min<long long>((nodes + 255) / 256, 148LL * 8));
}

// Weighted sums of the handle's blocks (what: 0 totals, 1 l2 vs the IC, 2
// l1), CTA partials summed in index order, blocks in worker order.
static void device_sums(ndgx_solver* s, int what, int var, int ic, const double* amps, int n_modes, double* out) {
  const int nout = what == 0 ? s->nv : 1;
  for (int k = 0; k < nout; ++k) out[k] = 0.0;
  for (const Blk& bk : s->blk) {
    s->on(bk);
    ndgx::FieldArgs a = field_args(s, bk);
    a.what = what;
    a.var = var;
    a.ic = ic;
    a.n_modes = n_modes;
    double* damps = device_amps(amps, n_modes);
    a.amps = damps;
    const unsigned grid = field_grid(bk, s->npe);
    double* part = nullptr;
    ck(cudaMalloc(&part, sizeof(double) * grid * nout), "cudaMalloc partials");
    ndgx::diag_kernel<<<grid, 256, 0, bk.st>>>(a, part);
    ck(cudaGetLastError(), "diag launch");
    std::vector<double> h((size_t)grid * nout);
    ck(cudaMemcpyAsync(h.data(), part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, bk.st), "partials");
    ck(cudaStreamSynchronize(bk.st), "diag sync");
    cudaFree(part);
    if (damps) cudaFree(damps);
    for (unsigned q = 0; q < grid; ++q)
      for (int k = 0; k < nout; ++k) out[k] += h[(size_t)q * nout + k];
  }
  s->on(s->blk[0]);
}

extern "C" {

int ndgx_init_device(ndgx_solver* s, int ic, const double* amplitudes, int n_modes, ndgx_error* err) {
  clear_error(err);
  if (!s) return NDGX_ERR_CONFIG;
  if (int rc = check_ic(s, ic, amplitudes, n_modes, err)) return rc;
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    for (const Blk& bk : s->blk) {
      s->on(bk);
      ndgx::FieldArgs a = field_args(s, bk);
      a.ic = ic;
      a.n_modes = ic == NDGX_IC_MULTISINE ? n_modes : 0;
      double* damps = device_amps(ic == NDGX_IC_MULTISINE ? amplitudes : nullptr, a.n_modes);
      a.amps = damps;
      ndgx::init_field_kernel<<<field_grid(bk, s->npe), 256, 0, bk.st>>>(a);
      ck(cudaGetLastError(), "init launch");
      ck(cudaStreamSynchronize(bk.st), "init sync");
      if (damps) cudaFree(damps);
    }
    s->on(s->blk[0]);
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  }
  return NDGX_OK;
}

int ndgx_conserved_totals_device(ndgx_solver* s, double* out, ndgx_error* err) {
  clear_error(err);
  if (!s || !out) return NDGX_ERR_CONFIG;
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    device_sums(s, 0, 0, -1, nullptr, 0, out);
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  }
  return NDGX_OK;
}

int ndgx_l2_error_ic_device(ndgx_solver* s, int ic, const double* amplitudes, int n_modes, int var, double* out,
                            ndgx_error* err) {
  clear_error(err);
  if (!s || !out) return NDGX_ERR_CONFIG;
  if (int rc = check_ic(s, ic, amplitudes, n_modes, err)) return rc;
  if (var < 0 || var >= s->nv) {
    set_error(err, NDGX_ERR_CONFIG, "l2_error: bad variable");
    return NDGX_ERR_CONFIG;
  }
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    device_sums(s, 1, var, ic, ic == NDGX_IC_MULTISINE ? amplitudes : nullptr,
                ic == NDGX_IC_MULTISINE ? n_modes : 0, out);
    *out = std::sqrt(*out);
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  }
  return NDGX_OK;
}

int ndgx_l1_norm_device(ndgx_solver* s, int var, double* out, ndgx_error* err) {
  clear_error(err);
  if (!s || !out) return NDGX_ERR_CONFIG;
  if (var < 0 || var >= s->nv) {
    set_error(err, NDGX_ERR_CONFIG, "l1_norm: bad variable");
    return NDGX_ERR_CONFIG;
  }
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    device_sums(s, 2, var, -1, nullptr, 0, out);
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  }
  return NDGX_OK;
}

}  // extern "C"

int ndgx_dump_field(ndgx_solver* s, const char* path, ndgx_error* err) {
  clear_error(err);
  if (!s || !path) {
    set_error(err, NDGX_ERR_CONFIG, "null argument");
    return NDGX_ERR_CONFIG;
  }
  std::vector<double> host(s->hn);
  if (int rc = ndgx_download(s, host.data(), err)) return rc;
  std::ofstream out(path, std::ios::binary);
  if (!out) {
    set_error(err, NDGX_ERR_RUN, std::string("cannot open ") + path + " for writing");
    return NDGX_ERR_RUN;
  }
  // the header exactly as dump_field writes it (src/field_io.cpp:18-34)
  std::ostringstream h;
  h << "ndgfield 1\n";
  h << "dim " << s->dim << "\n";
  h << "cells";
  for (int a = 0; a < s->dim; ++a) h << " " << s->hcells[a];
  h << "\norder " << s->N << "\n";
  h << "nvar " << s->nv << "\n";
  h << "length";
  for (int a = 0; a < s->dim; ++a) h << " " << field_length(s, a);  // a block's extent for a rank solver
  h << "\ndata\n";
  const std::string hs = h.str();
  out.write(hs.data(), (std::streamsize)hs.size());
  out.write(reinterpret_cast<const char*>(host.data()), (std::streamsize)(host.size() * sizeof(double)));
  if (!out) {
    set_error(err, NDGX_ERR_RUN, std::string("short write to ") + path);
    return NDGX_ERR_RUN;
  }
  return NDGX_OK;
}

int ndgx_load_field(ndgx_solver* s, const char* path, ndgx_error* err) {
  clear_error(err);
  if (!s || !path) {
    set_error(err, NDGX_ERR_CONFIG, "null argument");
    return NDGX_ERR_CONFIG;
  }
  auto fail = [&](int code, const std::string& m) {
    set_error(err, code, m);
    return code;
  };
  std::ifstream in(path, std::ios::binary);
  if (!in) return fail(NDGX_ERR_RUN, std::string("cannot open ") + path);
  std::string line;
  if (!std::getline(in, line) || line != "ndgfield 1")
    return fail(NDGX_ERR_RUN, std::string(path) + ": not an ndgfield dump");
  int dim = 0, order = 0, nvar = 0, cells[3] = {1, 1, 1};
  std::string lens[3];
  while (std::getline(in, line)) {  // load_field (src/field_io.cpp:36-72)
    if (line == "data") break;
    std::istringstream ls(line);
    std::string key;
    ls >> key;
    if (key == "dim") ls >> dim;
    else if (key == "cells") for (int a = 0; a < dim && a < 3; ++a) ls >> cells[a];
    else if (key == "order") ls >> order;
    else if (key == "nvar") ls >> nvar;
    else if (key == "length") for (int a = 0; a < dim && a < 3; ++a) ls >> lens[a];
    else return fail(NDGX_ERR_RUN, std::string(path) + ": unknown header key '" + key + "'");
    if (!ls) return fail(NDGX_ERR_RUN, std::string(path) + ": malformed header line '" + line + "'");
  }
  if (line != "data") return fail(NDGX_ERR_RUN, std::string(path) + ": missing data section");
  bool same = dim == s->dim && order == s->N && nvar == s->nv;
  for (int a = 0; a < s->dim; ++a) same = same && cells[a] == s->hcells[a];
  if (!same) return fail(NDGX_ERR_CONFIG, std::string(path) + ": field shape does not match the solver's mesh");
  // the extent too: a dump of another domain (or of another rank's block with
  // the same cell counts) would restart with the wrong dt and operator scaling
  for (int a = 0; a < s->dim; ++a)
    if (lens[a] != fmt_len(field_length(s, a)))
      return fail(NDGX_ERR_CONFIG, std::string(path) + ": domain length " + lens[a] + " on axis " +
                                       std::to_string(a) + " does not match the solver's " +
                                       fmt_len(field_length(s, a)));
  std::vector<double> host(s->hn);
  in.read(reinterpret_cast<char*>(host.data()), (std::streamsize)(host.size() * sizeof(double)));
  if (in.gcount() != (std::streamsize)(host.size() * sizeof(double)))
    return fail(NDGX_ERR_RUN, std::string(path) + ": truncated payload");
  return ndgx_upload(s, host.data(), err);
}

int ndgx_get_plan(const ndgx_solver* s, ndgx_rank_plan* plan) {
  if (!s || !plan) return NDGX_ERR_CONFIG;
  *plan = s->blk[0].plan;
  return NDGX_OK;
}

int ndgx_workers(const ndgx_solver* s) { return s ? (int)s->blk.size() : 0; }

int ndgx_get_block(const ndgx_solver* s, int worker, ndgx_rank_plan* plan) {
  if (!s || !plan || worker < 0 || worker >= (int)s->blk.size()) return NDGX_ERR_CONFIG;
  *plan = s->blk[worker].plan;
  return NDGX_OK;
}

void ndgx_destroy(ndgx_solver* s) {
  if (!s) return;
  delete s;
}

int64_t ndgx_dof(const ndgx_solver* s) { return s ? s->hdof : 0; }
size_t ndgx_state_size(const ndgx_solver* s) { return s ? s->hn : 0; }
int ndgx_stages(const ndgx_solver* s) { return s ? s->stages : 0; }
void* ndgx_stream(ndgx_solver* s) { return s ? (void*)s->stream() : nullptr; }

}  // extern "C"

static void permute(const ndgx_solver* s, const Blk& bk, const double* src, double* dst, bool to_device) {
  const long long total = (long long)bk.n;
  const int threads = 256;
  const int blocks = (int)std::min<long long>((total + threads - 1) / threads, 148LL * 16);
  if (to_device)
    ndgx::permute_kernel<true><<<blocks, threads, 0, bk.st>>>(src, dst, s->dim, bk.cells[0], bk.cells[1],
                                                              bk.cells[2], s->N, s->nv, total);
  else
    ndgx::permute_kernel<false><<<blocks, threads, 0, bk.st>>>(src, dst, s->dim, bk.cells[0], bk.cells[1],
                                                               bk.cells[2], s->N, s->nv, total);
}

// Block bk's cells of the handle's AoS field (host) <-> the block's own AoS
// field (device), one strided copy: a block is hcells-strided runs of whole
// cells in the reference layout (copy_block, src/partition.cpp:141-163).
static void copy_block(const ndgx_solver* s, const Blk& bk, double* host, double* dev, bool to_device) {
  const size_t chunk = (size_t)s->nv * s->npe * sizeof(double);
  cudaMemcpy3DParms m;
  std::memset(&m, 0, sizeof(m));
  int off[3];
  for (int a = 0; a < 3; ++a) off[a] = bk.goff[a] - s->hoff[a];
  cudaPitchedPtr h = make_cudaPitchedPtr(host, s->hcells[2] * chunk, s->hcells[2] * chunk, s->hcells[1]);
  cudaPitchedPtr d = make_cudaPitchedPtr(dev, bk.cells[2] * chunk, bk.cells[2] * chunk, bk.cells[1]);
  m.extent = make_cudaExtent(bk.cells[2] * chunk, bk.cells[1], bk.cells[0]);
  if (to_device) {
    m.srcPtr = h;
    m.srcPos = make_cudaPos(off[2] * chunk, off[1], off[0]);
    m.dstPtr = d;
    m.kind = cudaMemcpyHostToDevice;
  } else {
    m.srcPtr = d;
    m.dstPtr = h;
    m.dstPos = make_cudaPos(off[2] * chunk, off[1], off[0]);
    m.kind = cudaMemcpyDeviceToHost;
  }
  ck(cudaMemcpy3DAsync(&m, bk.st), to_device ? "upload" : "download");
}

static bool whole_field(const ndgx_solver* s, const Blk& bk) {
  for (int a = 0; a < 3; ++a)
    if (bk.cells[a] != s->hcells[a]) return false;
  return true;
}

static void upload_blocks(ndgx_solver* s, const double* u_aos) {
  for (const Blk& bk : s->blk) {
    s->on(bk);
    double* st = s->staging(bk, s->parity);
    if (whole_field(s, bk))
      ck(cudaMemcpyAsync(st, u_aos, bk.n * sizeof(double), cudaMemcpyHostToDevice, bk.st), "upload");
    else
      copy_block(s, bk, const_cast<double*>(u_aos), st, true);
    permute(s, bk, st, ndgx_solver::u_buf(bk, s->parity), true);
    ck(cudaGetLastError(), "permute launch");
  }
  for (const Blk& bk : s->blk) {
    s->on(bk);
    ck(cudaStreamSynchronize(bk.st), "upload sync");
  }
  s->on(s->blk[0]);
}

// src(bk) -> handle AoS field on the host
template <class Src>
static void download_blocks(ndgx_solver* s, double* u_aos, Src src) {
  for (const Blk& bk : s->blk) {
    s->on(bk);
    double* st = s->staging(bk, s->parity);
    permute(s, bk, src(bk), st, false);
    ck(cudaGetLastError(), "permute launch");
    if (whole_field(s, bk))
      ck(cudaMemcpyAsync(u_aos, st, bk.n * sizeof(double), cudaMemcpyDeviceToHost, bk.st), "download");
    else
      copy_block(s, bk, u_aos, st, false);
  }
  for (const Blk& bk : s->blk) {
    s->on(bk);
    ck(cudaStreamSynchronize(bk.st), "download sync");
  }
  s->on(s->blk[0]);
}

extern "C" {

int ndgx_upload(ndgx_solver* s, const double* u_aos, ndgx_error* err) {
  clear_error(err);
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    upload_blocks(s, u_aos);
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  }
  return NDGX_OK;
}

int ndgx_download(ndgx_solver* s, double* u_aos, ndgx_error* err) {
  clear_error(err);
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    const int par = s->parity;
    download_blocks(s, u_aos, [&](const Blk& bk) { return ndgx_solver::u_buf(bk, par); });
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  }
  return NDGX_OK;
}

int ndgx_rhs(ndgx_solver* s, double* dudt_aos, ndgx_error* err) {
  clear_error(err);
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    s->reset_control(s->ctl_warm);
    s->fork();
    s->launch_stage_all(0, s->parity, s->ctl_warm, true);
    s->join();
    ck(cudaGetLastError(), "rhs launch");
    const Control c = s->read_control(s->ctl_warm);
    if (c.err_key != ndgx::kNoError) return s->report(c.err_key, s->parity, err);
    const int par = s->parity;
    download_blocks(s, dudt_aos, [&](const Blk& bk) { return s->k_buf(bk, 0, par); });
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  } catch (const TransportFailure& t) {
    set_error(err, NDGX_ERR_TRANSPORT, t.what);
    return NDGX_ERR_TRANSPORT;
  }
  return NDGX_OK;
}

}  // extern "C"

// true when an error key stands for a real failure of a run of `fixed` steps
// (t_end mode: fixed < 0, with the run's final control state c)
static bool real_error(const ndgx_solver* s, unsigned long long key, long long fixed, const Control& c) {
  const long step = (long)(key >> 44);
  const int phase = (int)((key >> 40) & 0xF);
  if (phase == ndgx::kPhaseScan && step > 1) {
    // scan of the state after step-1: only real if that step was followed by another
    if (fixed >= 0) return step <= fixed;
    return !c.done && c.t < s->p.t_end;
  }
  return true;
}

static int run_warmup(ndgx_solver* s, ndgx_error* err) {
  // one untimed step on a scratch copy (src/solver.cpp:397-403): u itself is
  // never written by a step (u_new goes to the other parity buffer)
  s->reset_control(s->ctl_warm);
  s->launch_scan(s->ctl_warm, s->parity);
  s->launch_step(s->step_params(s->ctl_warm, 1, 1), s->parity, s->ctl_warm);
  // every rank takes the same decision from the earliest key of all ranks
  s->launch_err_reduce(s->ctl_warm);
  ck(cudaGetLastError(), "warmup launch");
  const Control c = s->read_control(s->ctl_warm);
  if (c.err_key != ndgx::kNoError) {
    const int phase = (int)((c.err_key >> 40) & 0xF);
    const long step = (long)(c.err_key >> 44);
    // the warm-up has no finite check and no trailing scan
    if (phase != ndgx::kPhaseInstability && !(phase == ndgx::kPhaseScan && step > 1))
      return s->report(c.err_key, s->parity, err);
  }
  return NDGX_OK;
}

static int finish_run(ndgx_solver* s, long long fixed, int start_par, ndgx_stats* stats, ndgx_error* err) {
  ck(cudaEventRecord(s->ev1, s->stream()), "event");
  s->launch_err_reduce(s->ctl);
  const Control c = s->read_control(s->ctl);
  float ms = 0.0f;
  ck(cudaEventElapsedTime(&ms, s->ev0, s->ev1), "elapsed");
  if (c.err_key != ndgx::kNoError && real_error(s, c.err_key, fixed, c)) {
    s->parity = start_par;  // state undefined after an exception; keep the input
    return s->report(c.err_key, start_par, err);
  }
  if (c.aborted) {
    // an error key that is not real for this run (a scan past the last step)
    // never aborts a rank: step_begin completes the run before it looks at errors
    s->parity = start_par;
    set_error(err, NDGX_ERR_RUN, "rank " + std::to_string(s->blk[0].id) + ": stopped by failure elsewhere", 0, -1,
              nullptr, s->blk[0].id);
    return NDGX_ERR_RUN;
  }
  s->parity = start_par ^ (int)(c.steps & 1);
  if (stats) {
    stats->steps = (long)c.steps;
    stats->dt_min = c.dt_min;
    stats->dt_max = c.dt_max;
    stats->wall_seconds = ms * 1e-3;
  }
  return NDGX_OK;
}

extern "C" {

int ndgx_advance(ndgx_solver* s, long fixed_steps, int warmup, ndgx_stats* stats, ndgx_error* err) {
  clear_error(err);
  if (stats) {
    stats->steps = 0;
    stats->dt_min = std::numeric_limits<double>::infinity();
    stats->dt_max = 0.0;
    stats->wall_seconds = 0.0;
  }
  if (!(s->p.cfl > 0.0) || s->p.cfl > 1.0) {
    set_error(err, NDGX_ERR_CONFIG, "cfl must lie in (0, 1]");
    return NDGX_ERR_CONFIG;
  }
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    if (warmup) {
      if (int rc = run_warmup(s, err)) return rc;
    }
    const long long fixed = fixed_steps >= 0 ? fixed_steps : -1;
    s->ensure_graphs(fixed);
    const int start_par = s->parity;
    s->reset_control(s->ctl);
    ck(cudaEventRecord(s->ev0, s->stream()), "event");
    s->launch_scan(s->ctl, start_par);
    if (fixed >= 0) {
      s->launch_run(fixed, start_par, fixed);
    } else {
      // t_end: the device decides when to stop; poll every chunk of steps
      const int chunk = 16;
      for (;;) {
        s->launch_run(chunk, start_par, fixed);
        const Control c = s->read_control(s->ctl);
        // a rank solver stops only when every rank does (done, or aborted after
        // the all-reduced error flag), so no rank leaves collectives unmatched
        if (c.done || (s->comm ? c.aborted != 0 : c.err_key != ndgx::kNoError)) break;
      }
    }
    return finish_run(s, fixed, start_par, stats, err);
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  } catch (const TransportFailure& t) {
    set_error(err, NDGX_ERR_TRANSPORT, t.what);
    return NDGX_ERR_TRANSPORT;
  }
}

int ndgx_launch_steps(ndgx_solver* s, long steps, ndgx_error* err) {
  clear_error(err);
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    const long long fixed = steps;
    s->ensure_graphs(fixed);
    s->pending_start_parity = s->parity;
    s->pending_fixed = fixed;
    s->reset_control(s->ctl);
    ck(cudaEventRecord(s->ev0, s->stream()), "event");
    s->launch_scan(s->ctl, s->parity);
    s->launch_run(fixed, s->parity, fixed);
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  } catch (const TransportFailure& t) {
    set_error(err, NDGX_ERR_TRANSPORT, t.what);
    return NDGX_ERR_TRANSPORT;
  }
  return NDGX_OK;
}

int ndgx_sync(ndgx_solver* s, ndgx_stats* stats, ndgx_error* err) {
  clear_error(err);
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    if (s->pending_fixed < 0) {
      ck(cudaStreamSynchronize(s->stream()), "sync");
      return NDGX_OK;
    }
    const long long fixed = s->pending_fixed;
    s->pending_fixed = -1;
    return finish_run(s, fixed, s->pending_start_parity, stats, err);
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  } catch (const TransportFailure& t) {
    set_error(err, NDGX_ERR_TRANSPORT, t.what);
    return NDGX_ERR_TRANSPORT;
  }
}

// Per-kernel timing in the steady state: two steps (the timed graph's unit)
// are captured with a 1-thread %globaltimer stamp kernel before the step
// control and after every stage, and the graph is replayed `reps` times back
// to back.  ms[i] = mean time of stage i over all but the first replay (a
// split stage's interior and boundary shell end to end, plus one stamp
// launch); ms[stages] = the step control (and a rank solver's wavespeed
// all-reduce).  Every step starts from the current state and writes the
// scratch buffers, so the state is left unchanged.
int ndgx_profile_step(ndgx_solver* s, float* ms, int n, ndgx_error* err) {
  clear_error(err);
  const int reps = 6, per = 2 * (s->stages + 1) + 1;  // stamps per replay
  cudaGraphExec_t exec = nullptr;
  unsigned long long* stamps = nullptr;
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    if (s->multi_device) {
      set_error(err, NDGX_ERR_CONFIG, "profile_step needs the blocks on one device");
      return NDGX_ERR_CONFIG;
    }
    ck(cudaMalloc(&stamps, reps * per * sizeof(unsigned long long) + 16), "cudaMalloc stamps");
    unsigned int* count = reinterpret_cast<unsigned int*>(stamps + reps * per);
    ck(cudaMemsetAsync(count, 0, sizeof(unsigned int), s->stream()), "memset");
    cudaGraph_t g;
    ck(cudaStreamBeginCapture(s->stream(), s->comm ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal),
       "begin capture");
    const StepParams sp = s->step_params(s->ctl_warm, 2LL * reps, 0);
    s->xpar = 0;
    for (int k = 0; k < 2; ++k) {
      ndgx::stamp_kernel<<<1, 1, 0, s->stream()>>>(stamps, count);
      s->launch_alpha_reduce(s->ctl_warm);
      ndgx::step_begin_kernel<<<1, 1, 0, s->stream()>>>(sp);
      for (int i = 0; i < s->stages; ++i) {
        ndgx::stamp_kernel<<<1, 1, 0, s->stream()>>>(stamps, count);
        s->fork();
        s->launch_stage_all(i, s->parity, s->ctl_warm, false);  // both steps from u: u is never written
        s->join();
      }
    }
    ndgx::stamp_kernel<<<1, 1, 0, s->stream()>>>(stamps, count);  // the end of the second step's last stage
    ck(cudaStreamEndCapture(s->stream(), &g), "end capture");
    ck(cudaGraphInstantiate(&exec, g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    s->reset_control(s->ctl_warm);
    s->launch_scan(s->ctl_warm, s->parity);
    for (int r = 0; r < reps; ++r) ck(cudaGraphLaunch(exec, s->stream()), "graph");
    std::vector<unsigned long long> h((size_t)reps * per);
    ck(cudaMemcpyAsync(h.data(), stamps, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s->stream()),
       "stamps");
    ck(cudaStreamSynchronize(s->stream()), "sync");
    // per replay: [before ctl, before stage 0 .. before stage S-1] x 2 steps, then a closing stamp
    const int w = s->stages + 1;
    std::vector<double> acc(w, 0.0);
    int cnt = 0;
    for (int r = 1; r < reps; ++r)
      for (int k = 0; k < 2; ++k) {
        const size_t b0 = (size_t)r * per + (size_t)k * w;
        for (int i = 0; i < s->stages; ++i) acc[i] += (double)(h[b0 + 2 + i] - h[b0 + 1 + i]) * 1e-6;
        acc[s->stages] += (double)(h[b0 + 1] - h[b0]) * 1e-6;
        ++cnt;
      }
    for (int i = 0; i <= s->stages && i < n; ++i) ms[i] = (float)(acc[i] / cnt);
    cudaGraphExecDestroy(exec);
    cudaFree(stamps);
  } catch (const CudaFailure& f) {
    if (exec) cudaGraphExecDestroy(exec);
    if (stamps) cudaFree(stamps);
    return cuda_error(err, f);
  } catch (const TransportFailure& t) {
    set_error(err, NDGX_ERR_TRANSPORT, t.what);
    return NDGX_ERR_TRANSPORT;
  }
  return NDGX_OK;
}

}  // extern "C"
