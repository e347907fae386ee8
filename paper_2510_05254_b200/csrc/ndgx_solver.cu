// ndgx_solver.cu -- the C ABI (include/ndgx.h): device state, step loop,
// CUDA-graph capture, error mapping onto the reference's exception taxonomy.
//
// Reference (paths relative to /root/reference/proj):
//   advance            src/solver.cpp:372-440     -> ndgx_advance
//   serial_rhs         src/solver.cpp:442-456     -> ndgx_rhs
//   RKIntegrator       include/ndg/solver.hpp:39-82 (buffers :41-44)
//   errors             include/ndg/errors.hpp:13-56
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <limits>
#include <new>
#include <string>
#include <vector>

#include "ndgx.h"
#include "ndgx_kernels.h"
#include "ndgx_nccl.h"
#include "ndgx_setup.h"

using ndgx::Control;
using ndgx::StageArgs;
using ndgx::StepParams;

namespace {

void set_error(ndgx_error* e, int code, const std::string& msg, long step = 0, int stage = -1,
               const int* cell = nullptr) {
  if (!e) return;
  std::memset(e, 0, sizeof(*e));
  e->code = code;
  e->step = step;
  e->stage = stage;
  e->worker = -1;
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

}  // namespace

struct ndgx_solver {
  ndgx_problem p{};
  int dim = 0, N = 0, nv = 0, kind = 0, stages = 0, npe = 0;
  int cells[3] = {1, 1, 1};
  size_t n = 0;
  int64_t dof = 0;
  bool exact = true;
  double K[3][64]{}, lift[3]{}, a[7][7]{}, b[7]{};
  double cflh = 0.0, two_n_minus_1 = 0.0, const_alpha = -1.0;
  ndgx::StageKernel kern;
  ndgx::StageLaunch lcfg[ndgx::kNumSigs];  // per stage signature (ndgx::kSigs)
  cudaStream_t stream = nullptr;
  std::vector<double*> buf;
  int dead = -1;      // K slot overwritten by u_new at the last stage (-1: none)
  int parity = 0;     // u lives in buf[parity]
  Control* ctl = nullptr;
  Control* ctl_warm = nullptr;
  Control* h_ctl = nullptr;  // pinned mirror
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  long long graph_fixed = -2;
  double graph_tend = -1.0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // block of a decomposed mesh (defaults: the whole mesh, no exchange)
  ndgx_rank_plan plan{};
  int gcells[3] = {1, 1, 1};
  int goff[3] = {0, 0, 0};
  bool exchange = false;            // some axis takes its halo from the transport
  ncclComm_t comm = nullptr;
  const ndgx::Nccl* nc = nullptr;
  double* snd[3][2] = {};           // packed boundary planes (ours)
  double* rcv[3][2] = {};           // received planes (neighbours')
  long long pending_fixed = -1;  // ndgx_launch_steps bookkeeping
  int pending_start_parity = 0;

  // ------------------------------------------------------------ buffers
  double* u_buf(int par) const { return buf[par]; }
  double* out_buf(int par) const { return buf[1 - par]; }
  double* k_buf(int j, int par) const {
    if (j == dead) return buf[1 - par];
    int rank = j;
    if (dead >= 0 && j > dead) --rank;
    return buf[2 + rank];
  }
  double* staging(int par) const {
    double* r = k_buf(0, par);
    return r != buf[1 - par] ? buf[1 - par] : buf[2];
  }

  StageArgs stage_args(int i, int par, Control* c, bool rhs_only) const {
    StageArgs s;
    std::memset(&s, 0, sizeof(s));
    s.u = u_buf(par);
    s.is_last = (!rhs_only && i == stages - 1) ? 1 : 0;
    // union (ascending j) of the K_j read by the stage input (a_ij != 0,
    // solver.hpp:58) and, at the last stage, by S (b_j != 0, solver.hpp:71)
    s.nu = 0;
    for (int j = 0; j < i; ++j) {
      const bool ua = a[i][j] != 0.0;
      const bool ub = s.is_last && b[j] != 0.0;
      if (!ua && !ub) continue;
      s.ku[s.nu] = k_buf(j, par);
      s.ca[s.nu] = a[i][j];
      s.cb[s.nu] = b[j];
      if (ua) s.amask |= 1 << s.nu;
      if (ub) s.bmask |= 1 << s.nu;
      ++s.nu;
    }
    if (s.is_last) {
      s.b_last = b[i];
      s.out = out_buf(par);
    } else {
      s.out = k_buf(i, par);
    }
    s.ctl = c;
    s.rhs_only = rhs_only ? 1 : 0;
    s.phase = ndgx::kPhaseStage0 + i;
    s.scan_alpha = (s.is_last && kind == NDGX_EULER_ISOTHERMAL) ? 1 : 0;
    for (int d = 0; d < 3; ++d) {
      s.cells[d] = cells[d];
      s.gcells[d] = gcells[d];
      s.goff[d] = goff[d];
      for (int q = 0; q < 2; ++q) s.ext[d][q] = plan.split[d] ? rcv[d][q] : nullptr;
      s.vel[d] = p.velocity[d];
      s.lift[d] = lift[d];
      for (int q = 0; q < 64; ++q) s.K[d][q] = K[d][q];
    }
    s.sound_speed = p.sound_speed;
    s.sig = sig_of(s);
    s.depth = lcfg[s.sig].depth;
    return s;
  }

  // Per stage: pack our boundary planes, swap them with the neighbours
  // (exchange_halos, src/partition.cpp:108-131: per axis send the high plane
  // up and receive the low halo, send the low plane down and receive the
  // high halo -- the same posting order on every rank, so pairs match even
  // when both neighbours are one rank or this rank itself).
  void launch_exchange(const StageArgs& s) const {
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
      pa.cells[d] = cells[d];
      pa.split[d] = plan.split[d];
      pa.plane[d] = plan.plane[d];
      pa.snd[d][0] = snd[d][0];
      pa.snd[d][1] = snd[d][1];
      if (plan.split[d]) total += 2 * plan.plane[d];
    }
    const int threads = 256;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((total + threads - 1) / threads, 148LL * 8));
    if (exact)
      ndgx::pack_kernel<true><<<blocks, threads, 0, stream>>>(pa);
    else
      ndgx::pack_kernel<false><<<blocks, threads, 0, stream>>>(pa);
    nccl_check(nc->GroupStart(), "ncclGroupStart");
    for (int d = 0; d < dim; ++d) {
      if (!plan.split[d]) continue;
      const size_t n = (size_t)plan.plane[d];
      nccl_check(nc->Send(snd[d][1], n, ncclFloat64, plan.nbr[d][1], comm, stream), "ncclSend");
      nccl_check(nc->Recv(rcv[d][0], n, ncclFloat64, plan.nbr[d][0], comm, stream), "ncclRecv");
      nccl_check(nc->Send(snd[d][0], n, ncclFloat64, plan.nbr[d][0], comm, stream), "ncclSend");
      nccl_check(nc->Recv(rcv[d][1], n, ncclFloat64, plan.nbr[d][1], comm, stream), "ncclRecv");
    }
    nccl_check(nc->GroupEnd(), "ncclGroupEnd");
  }

  // Per step: every rank's dt comes from the global max wavespeed (the
  // alpha barrier of run_partitioned, src/partition.cpp:201-213, 243-252).
  void launch_alpha_reduce(Control* c) const {
    if (!comm) return;
    // {alpha_bits, any_err}: the global wavespeed and whether any rank failed
    nccl_check(nc->AllReduce(&c->alpha_bits, &c->alpha_bits, 2, ncclUint64, ncclMax, comm, stream),
               "ncclAllReduce");
  }

  void nccl_check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) throw TransportFailure{std::string(what) + ": " + nc->GetErrorString(r)};
  }

  void launch_stage(const StageArgs& s) const {
    if (exchange) launch_exchange(s);
    // persistent CTAs (one element per warp): as many as are co-resident
    const long long warps = (long long)cells[0] * cells[1] * cells[2];
    const long long need = (warps + kern.warps - 1) / kern.warps;
    const ndgx::StageLaunch& c = lcfg[s.sig];
    const long long grid = std::max<long long>(1, std::min<long long>(need, (long long)c.grid));
    kern.fn[s.sig]<<<(unsigned)grid, kern.threads, c.smem, stream>>>(s);
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

  void launch_step(const StepParams& sp, int par, Control* c) const {
    launch_alpha_reduce(c);
    ndgx::step_begin_kernel<<<1, 1, 0, stream>>>(sp);
    for (int i = 0; i < stages; ++i) launch_stage(stage_args(i, par, c, false));
  }

  void launch_scan(Control* c, int par) const {
    if (kind != NDGX_EULER_ISOTHERMAL) return;
    const int threads = 256, blocks = 148 * 8;
    if (dim == 2)
      ndgx::alpha_scan_kernel<2><<<blocks, threads, 0, stream>>>(u_buf(par), cells[0], cells[1], cells[2], N,
                                                                 p.sound_speed, c, 1);
    else
      ndgx::alpha_scan_kernel<3><<<blocks, threads, 0, stream>>>(u_buf(par), cells[0], cells[1], cells[2], N,
                                                                 p.sound_speed, c, 1);
  }

  void reset_control(Control* c) const {
    Control h;
    std::memset(&h, 0, sizeof(h));
    h.err_key = ndgx::kNoError;
    h.dt_min = std::numeric_limits<double>::infinity();
    h.dt_max = 0.0;
    *h_ctl = h;
    ck(cudaMemcpyAsync(c, h_ctl, sizeof(Control), cudaMemcpyHostToDevice, stream), "reset control");
  }

  Control read_control(Control* c) const {
    ck(cudaMemcpyAsync(h_ctl, c, sizeof(Control), cudaMemcpyDeviceToHost, stream), "read control");
    ck(cudaStreamSynchronize(stream), "sync");
    return *h_ctl;
  }

  void ensure_graphs(long long fixed) {
    if (graph[0] && graph_fixed == fixed && graph_tend == p.t_end) return;
    for (auto& g : graph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    const StepParams sp = step_params(ctl, fixed, 0);
    for (int par = 0; par < 2; ++par) {
      cudaGraph_t g;
      ck(cudaStreamBeginCapture(stream, comm ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal),
         "begin capture");
      launch_step(sp, par, ctl);
      launch_step(sp, 1 - par, ctl);
      ck(cudaStreamEndCapture(stream, &g), "end capture");
      ck(cudaGraphInstantiate(&graph[par], g, 0), "graph instantiate");
      cudaGraphDestroy(g);
    }
    graph_fixed = fixed;
    graph_tend = p.t_end;
  }

  // Co-resident CTAs of the stage kernel (grid of the persistent launch).
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
      const int nu = ndgx::kSigs[q].nu;
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
      lcfg[q] = best;
    }
    return NDGX_OK;
  }

  // device index of (AoS cell index, AoS node key, var)
  // block-local cell of a global AoS cell index (the kernels name cells globally)
  void local_cell(long long aos_cell, int c[3]) const {
    const int g2 = gcells[2], g1 = gcells[1];
    c[2] = (int)(aos_cell % g2) - goff[2];
    c[1] = (int)((aos_cell / g2) % g1) - goff[1];
    c[0] = (int)(aos_cell / ((long long)g2 * g1)) - goff[0];
  }

  size_t device_index(long long aos_cell, int aos_node, int var) const {
    const int c1 = cells[1];
    int lc[3];
    local_cell(aos_cell, lc);
    const int cx = lc[0], cy = lc[1], cz = lc[2];
    int i = 0, j = 0, k = 0;
    if (dim == 1) i = aos_node;
    if (dim == 2) { i = aos_node / N; j = aos_node % N; }
    if (dim == 3) { i = aos_node / (N * N); j = (aos_node / N) % N; k = aos_node % N; }
    const size_t e = (size_t)cx + (size_t)cells[0] * ((size_t)cy + (size_t)c1 * cz);
    const size_t nn = (size_t)i + (size_t)N * ((size_t)j + (size_t)N * k);
    return (e * nv + var) * npe + nn;
  }

  double fetch(const double* dev, size_t idx) const {
    double v = 0.0;
    ck(cudaMemcpy(&v, dev + idx, sizeof(double), cudaMemcpyDeviceToHost), "fetch");
    return v;
  }

  // Map a device error key onto the reference's exception (message text
  // follows src/solver.cpp:258-261, 325-328, 364-365, 411-413).
  int report(unsigned long long key, int start_par, ndgx_error* err) const {
    const long step = (long)(key >> 44);
    const int phase = (int)((key >> 40) & 0xF);
    const long long cell = (long long)((key >> 12) & 0xFFFFFFF);
    const int node = (int)(key & 0xFFF);
    const int par = start_par ^ (int)((step > 0 ? step - 1 : 0) & 1);
    if (phase == ndgx::kPhaseZeroSpeed) {
      set_error(err, NDGX_ERR_CONFIG, "fixed-step run requires a positive wavespeed", step);
      return NDGX_ERR_CONFIG;
    }
    if (phase == ndgx::kPhaseInstability) {
      set_error(err, NDGX_ERR_INSTABILITY, "non-finite state after step " + std::to_string(step), step);
      return NDGX_ERR_INSTABILITY;
    }
    const size_t idx = device_index(cell, node, 0);
    if (phase == ndgx::kPhaseScan) {
      const double rho = fetch(u_buf(par), idx);
      set_error(err, NDGX_ERR_PHYSICS, "nonpositive density " + fmt_double(rho) + " in time-step estimate",
                step);
      return NDGX_ERR_PHYSICS;
    }
    // operator PhysicsError at stage `stage`: recompute the stage input there
    const int stage = phase - ndgx::kPhaseStage0;
    double rho = fetch(u_buf(par), idx);
    for (int j = 0; j < stage; ++j) {
      if (a[stage][j] == 0.0) continue;
      rho += a[stage][j] * fetch(k_buf(j, par), idx);
    }
    int c[3];
    local_cell(cell, c);
    const std::string where = "(" + std::to_string(c[0]) + "," + std::to_string(c[1]) + "," +
                              std::to_string(c[2]) + ")";
    set_error(err, NDGX_ERR_PHYSICS,
              "nonpositive density " + fmt_double(rho) + " in flux evaluation at cell " + where, step,
              stage, c);
    return NDGX_ERR_PHYSICS;
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
    if (stream) cudaStreamSynchronize(stream);
    if (comm && nc) nc->CommAbort(comm);
    for (int d = 0; d < 3; ++d)
      for (int q = 0; q < 2; ++q) {
        if (snd[d][q]) cudaFree(snd[d][q]);
        if (rcv[d][q]) cudaFree(rcv[d][q]);
      }
    for (auto& g : graph)
      if (g) cudaGraphExecDestroy(g);
    for (double* q : buf) cudaFree(q);
    if (ctl) cudaFree(ctl);
    if (ctl_warm) cudaFree(ctl_warm);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
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

}  // namespace

static int create_block(const ndgx_problem* prob, const ndgx_rank_plan* plan, ndgx_solver** out, ndgx_error* err);

extern "C" {

const char* ndgx_version(void) { return "ndgx 0.1.0 sm_100a"; }

int ndgx_create(const ndgx_problem* prob, ndgx_solver** out, ndgx_error* err) {
  return create_block(prob, nullptr, out, err);
}

}  // extern "C"

// A solver for `plan`'s block of the global mesh `prob` (nullptr: the whole
// mesh).  The operator, dt numerator and wavespeed use the global mesh, so
// every block computes with the reference's exact coefficients.
static int create_block(const ndgx_problem* prob, const ndgx_rank_plan* plan, ndgx_solver** out, ndgx_error* err) {
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
    ck(cudaSetDevice(prob->device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, prob->device), "cudaGetDeviceProperties");
    if (prop.major != 10) {
      delete s;
      set_error(err, NDGX_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100 (B200)");
      return NDGX_ERR_CUDA;
    }
    s->p = *prob;
    s->p.nodes = s->p.weights = s->p.diff = nullptr;
    s->dim = prob->dim;
    s->N = prob->order;
    s->kind = prob->equation;
    s->nv = s->kind == NDGX_ADVECTION ? 1 : s->dim + 1;
    s->exact = prob->arith != NDGX_ARITH_FAST;
    for (int a = 0; a < 3; ++a) {
      s->gcells[a] = a < s->dim ? prob->cells[a] : 1;
      s->goff[a] = plan ? plan->lo[a] : 0;
      s->cells[a] = plan ? plan->hi[a] - plan->lo[a] : s->gcells[a];
    }
    if (plan) {
      s->plan = *plan;
      for (int a = 0; a < 3; ++a) s->exchange = s->exchange || plan->split[a] != 0;
    } else {
      s->plan.nranks = 1;
      for (int a = 0; a < 3; ++a) {
        s->plan.grid[a] = 1;
        s->plan.hi[a] = s->cells[a];
      }
    }
    s->npe = 1;
    for (int a = 0; a < s->dim; ++a) s->npe *= s->N;
    s->n = (size_t)s->nv * s->npe * s->cells[0] * s->cells[1] * s->cells[2];
    s->dof = (int64_t)s->n;

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
    if (int rc = s->configure_launches(prop, err)) {
      delete s;
      return rc;
    }
    ck(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&s->ev0), "event");
    ck(cudaEventCreate(&s->ev1), "event");
    const int nbuf = s->dead >= 0 ? s->stages : s->stages + 1;
    for (int q = 0; q < nbuf; ++q) {
      double* d = nullptr;
      ck(cudaMalloc(&d, s->n * sizeof(double)), "cudaMalloc state");
      s->buf.push_back(d);
    }
    ck(cudaMemsetAsync(s->buf[0], 0, s->n * sizeof(double), s->stream), "memset");
    ck(cudaMalloc(&s->ctl, sizeof(Control)), "cudaMalloc control");
    ck(cudaMalloc(&s->ctl_warm, sizeof(Control)), "cudaMalloc control");
    ck(cudaMallocHost(&s->h_ctl, sizeof(Control)), "cudaMallocHost");
    for (int d = 0; d < 3; ++d)
      if (s->plan.split[d])
        for (int q = 0; q < 2; ++q) {
          ck(cudaMalloc(&s->snd[d][q], s->plan.plane[d] * sizeof(double)), "cudaMalloc plane");
          ck(cudaMalloc(&s->rcv[d][q], s->plan.plane[d] * sizeof(double)), "cudaMalloc plane");
          ck(cudaMemsetAsync(s->rcv[d][q], 0, s->plan.plane[d] * sizeof(double), s->stream), "memset");
        }
    ck(cudaStreamSynchronize(s->stream), "sync");
  } catch (const CudaFailure& f) {
    delete s;
    return cuda_error(err, f);
  }
  *out = s;
  return NDGX_OK;
}

extern "C" {

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
  std::vector<int> lo(3 * nranks), hi(3 * nranks), nbr(6 * nranks);
  ndgx_rank_plan pl;
  std::memset(&pl, 0, sizeof(pl));
  if (int rc = ndgx_decompose(global->dim, global->cells, nranks, pl.grid, lo.data(), hi.data(), nbr.data(), err))
    return rc;
  pl.rank = rank;
  pl.nranks = nranks;
  const int nv = global->equation == NDGX_ADVECTION ? 1 : global->dim + 1;
  const int N = global->order;
  const long long L = global->dim == 1 ? 1 : (global->dim == 2 ? N : (long long)N * N);
  for (int a = 0; a < 3; ++a) {
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
  if (int rc = create_block(global, &plan, out, err)) return rc;
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

int ndgx_dump_field(ndgx_solver* s, const char* path, ndgx_error* err) {
  clear_error(err);
  if (!s || !path) {
    set_error(err, NDGX_ERR_CONFIG, "null argument");
    return NDGX_ERR_CONFIG;
  }
  std::vector<double> host(s->n);
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
  for (int a = 0; a < s->dim; ++a) h << " " << s->cells[a];
  h << "\norder " << s->N << "\n";
  h << "nvar " << s->nv << "\n";
  h << "length";
  for (int a = 0; a < s->dim; ++a) {
    // a block's extent: its cells times the global cell size
    const double len = s->cells[a] == s->gcells[a] ? s->p.length[a]
                                                   : s->cells[a] * (s->p.length[a] / s->gcells[a]);
    h << " " << len;
  }
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
  while (std::getline(in, line)) {  // load_field (src/field_io.cpp:36-72)
    if (line == "data") break;
    std::istringstream ls(line);
    std::string key;
    ls >> key;
    double len;
    if (key == "dim") ls >> dim;
    else if (key == "cells") for (int a = 0; a < dim && a < 3; ++a) ls >> cells[a];
    else if (key == "order") ls >> order;
    else if (key == "nvar") ls >> nvar;
    else if (key == "length") for (int a = 0; a < dim && a < 3; ++a) ls >> len;
    else return fail(NDGX_ERR_RUN, std::string(path) + ": unknown header key '" + key + "'");
    if (!ls) return fail(NDGX_ERR_RUN, std::string(path) + ": malformed header line '" + line + "'");
  }
  if (line != "data") return fail(NDGX_ERR_RUN, std::string(path) + ": missing data section");
  bool same = dim == s->dim && order == s->N && nvar == s->nv;
  for (int a = 0; a < s->dim; ++a) same = same && cells[a] == s->cells[a];
  if (!same) return fail(NDGX_ERR_CONFIG, std::string(path) + ": field shape does not match the solver's mesh");
  std::vector<double> host(s->n);
  in.read(reinterpret_cast<char*>(host.data()), (std::streamsize)(host.size() * sizeof(double)));
  if (in.gcount() != (std::streamsize)(host.size() * sizeof(double)))
    return fail(NDGX_ERR_RUN, std::string(path) + ": truncated payload");
  return ndgx_upload(s, host.data(), err);
}

int ndgx_get_plan(const ndgx_solver* s, ndgx_rank_plan* plan) {
  if (!s || !plan) return NDGX_ERR_CONFIG;
  *plan = s->plan;
  return NDGX_OK;
}

void ndgx_destroy(ndgx_solver* s) {
  if (!s) return;
  cudaSetDevice(s->p.device);
  cudaStreamSynchronize(s->stream);
  delete s;
}

int64_t ndgx_dof(const ndgx_solver* s) { return s ? s->dof : 0; }
size_t ndgx_state_size(const ndgx_solver* s) { return s ? s->n : 0; }
int ndgx_stages(const ndgx_solver* s) { return s ? s->stages : 0; }
void* ndgx_stream(ndgx_solver* s) { return s ? (void*)s->stream : nullptr; }

static void permute(const ndgx_solver* s, const double* src, double* dst, bool to_device) {
  const long long total = (long long)s->n;
  const int threads = 256;
  const int blocks = (int)std::min<long long>((total + threads - 1) / threads, 148LL * 16);
  if (to_device)
    ndgx::permute_kernel<true><<<blocks, threads, 0, s->stream>>>(src, dst, s->dim, s->cells[0], s->cells[1],
                                                                  s->cells[2], s->N, s->nv, total);
  else
    ndgx::permute_kernel<false><<<blocks, threads, 0, s->stream>>>(src, dst, s->dim, s->cells[0], s->cells[1],
                                                                   s->cells[2], s->N, s->nv, total);
}

int ndgx_upload(ndgx_solver* s, const double* u_aos, ndgx_error* err) {
  clear_error(err);
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    double* st = s->staging(s->parity);
    ck(cudaMemcpyAsync(st, u_aos, s->n * sizeof(double), cudaMemcpyHostToDevice, s->stream), "upload");
    permute(s, st, s->u_buf(s->parity), true);
    ck(cudaGetLastError(), "permute launch");
    ck(cudaStreamSynchronize(s->stream), "upload sync");
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  } catch (const TransportFailure& t) {
    set_error(err, NDGX_ERR_TRANSPORT, t.what);
    return NDGX_ERR_TRANSPORT;
  }
  return NDGX_OK;
}

int ndgx_download(ndgx_solver* s, double* u_aos, ndgx_error* err) {
  clear_error(err);
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    double* st = s->staging(s->parity);
    permute(s, s->u_buf(s->parity), st, false);
    ck(cudaGetLastError(), "permute launch");
    ck(cudaMemcpyAsync(u_aos, st, s->n * sizeof(double), cudaMemcpyDeviceToHost, s->stream), "download");
    ck(cudaStreamSynchronize(s->stream), "download sync");
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  } catch (const TransportFailure& t) {
    set_error(err, NDGX_ERR_TRANSPORT, t.what);
    return NDGX_ERR_TRANSPORT;
  }
  return NDGX_OK;
}

int ndgx_rhs(ndgx_solver* s, double* dudt_aos, ndgx_error* err) {
  clear_error(err);
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    s->reset_control(s->ctl_warm);
    const StageArgs a = s->stage_args(0, s->parity, s->ctl_warm, true);
    s->launch_stage(a);
    ck(cudaGetLastError(), "rhs launch");
    const Control c = s->read_control(s->ctl_warm);
    if (c.err_key != ndgx::kNoError) return s->report(c.err_key, s->parity, err);
    double* st = s->staging(s->parity);
    permute(s, a.out, st, false);
    ck(cudaMemcpyAsync(dudt_aos, st, s->n * sizeof(double), cudaMemcpyDeviceToHost, s->stream), "download");
    ck(cudaStreamSynchronize(s->stream), "rhs sync");
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  } catch (const TransportFailure& t) {
    set_error(err, NDGX_ERR_TRANSPORT, t.what);
    return NDGX_ERR_TRANSPORT;
  }
  return NDGX_OK;
}

static int run_warmup(ndgx_solver* s, ndgx_error* err) {
  // one untimed step on a scratch copy (src/solver.cpp:397-403): u itself is
  // never written by a step (u_new goes to the other parity buffer)
  s->reset_control(s->ctl_warm);
  s->launch_scan(s->ctl_warm, s->parity);
  s->launch_step(s->step_params(s->ctl_warm, 1, 1), s->parity, s->ctl_warm);
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
  ck(cudaEventRecord(s->ev1, s->stream), "event");
  const Control c = s->read_control(s->ctl);
  float ms = 0.0f;
  ck(cudaEventElapsedTime(&ms, s->ev0, s->ev1), "elapsed");
  if (c.err_key != ndgx::kNoError) {
    const long step = (long)(c.err_key >> 44);
    const int phase = (int)((c.err_key >> 40) & 0xF);
    bool real = true;
    if (phase == ndgx::kPhaseScan && step > 1) {
      // scan of the state after step-1: only real if that step was followed by another
      if (fixed >= 0) real = step <= fixed;
      else real = !c.done && c.t < s->p.t_end;
    }
    if (real) {
      s->parity = start_par;  // state undefined after an exception; keep the input
      return s->report(c.err_key, start_par, err);
    }
  }
  if (c.aborted && c.err_key == ndgx::kNoError) {
    s->parity = start_par;
    set_error(err, NDGX_ERR_RUN, "rank " + std::to_string(s->plan.rank) + ": stopped by failure elsewhere");
    if (err) err->worker = s->plan.rank;
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
    ck(cudaEventRecord(s->ev0, s->stream), "event");
    s->launch_scan(s->ctl, start_par);
    if (fixed >= 0) {
      // pairs of steps alternate the parity; a trailing odd step is skipped
      // on the device by step_begin (steps >= fixed_steps)
      for (long long q = 0; q < (fixed + 1) / 2; ++q) ck(cudaGraphLaunch(s->graph[start_par], s->stream), "graph");
    } else {
      // t_end: the device decides when to stop; poll every chunk of steps
      const int chunk = 8;  // graph launches (2 steps each) between polls
      for (;;) {
        for (int q = 0; q < chunk; ++q) ck(cudaGraphLaunch(s->graph[start_par], s->stream), "graph");
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
    ck(cudaEventRecord(s->ev0, s->stream), "event");
    s->launch_scan(s->ctl, s->parity);
    for (long long q = 0; q < (fixed + 1) / 2; ++q) ck(cudaGraphLaunch(s->graph[s->parity], s->stream), "graph");
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
      ck(cudaStreamSynchronize(s->stream), "sync");
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

int ndgx_profile_step(ndgx_solver* s, float* ms, int n, ndgx_error* err) {
  clear_error(err);
  try {
    ck(cudaSetDevice(s->p.device), "cudaSetDevice");
    std::vector<cudaEvent_t> ev(s->stages + 3);
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    s->reset_control(s->ctl_warm);
    s->launch_scan(s->ctl_warm, s->parity);
    ck(cudaEventRecord(ev[0], s->stream), "event");
    ndgx::step_begin_kernel<<<1, 1, 0, s->stream>>>(s->step_params(s->ctl_warm, 1, 0));
    ck(cudaEventRecord(ev[1], s->stream), "event");
    for (int i = 0; i < s->stages; ++i) {
      s->launch_stage(s->stage_args(i, s->parity, s->ctl_warm, false));
      ck(cudaEventRecord(ev[2 + i], s->stream), "event");
    }
    ck(cudaStreamSynchronize(s->stream), "sync");
    for (int i = 0; i < s->stages && i < n; ++i) ck(cudaEventElapsedTime(&ms[i], ev[1 + i], ev[2 + i]), "elapsed");
    if (s->stages < n) ck(cudaEventElapsedTime(&ms[s->stages], ev[0], ev[1]), "elapsed");
    for (auto& e : ev) cudaEventDestroy(e);
  } catch (const CudaFailure& f) {
    return cuda_error(err, f);
  } catch (const TransportFailure& t) {
    set_error(err, NDGX_ERR_TRANSPORT, t.what);
    return NDGX_ERR_TRANSPORT;
  }
  return NDGX_OK;
}

}  // extern "C"
