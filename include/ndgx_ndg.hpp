// ndgx_ndg.hpp -- header-only adapter that plugs the ndgx C ABI into the
// reference solver's own C++ types (/root/reference/proj/include/ndg/*).
//
// Include it from a translation unit that already has the reference's
// include directory on its path and link libndgx.so.  It provides
//
//   ndgx::advance(config, initial, plan)        == ndg::advance        (src/solver.cpp:372-440)
//   ndgx::serial_rhs(mesh, basis, model, field) == ndg::serial_rhs     (src/solver.cpp:442-456)
//   ndgx::run_partitioned(config, initial, P, plan, devices)
//                                               == ndg::run_partitioned (src/partition.cpp:186-333)
//        P blocks of the reference's own decompose() tiling in one ndgx handle
//        (block w on devices[w % devices.size()]), halos by peer stores, the
//        reference's RunError("worker w: ...") contract
//
// Arithmetic: every entry takes `arith` last.  The default NDGX_ARITH_EXACT
// is bit-identical to the reference (the reference's unfused operation
// order: 1.03e11 DOF*stage/s on C3).  NDGX_ARITH_FAST (FMA contraction, FP64
// tensor cores; <= 1e-12 relative L2 vs the reference) is the headline
// throughput, 2.12e11 -- pass it explicitly.
//
// with the same argument meaning, return types and exceptions
// (include/ndg/errors.hpp:13-56).  The operator coefficients are built from
// the caller's own gauss_lobatto/differentiation_matrix, so they are bitwise
// the reference's.  The one-line switch at the reference's call site is
// shown in INTEGRATION.md (experiments.cpp:82-90, timed_run).
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "ndg/basis.hpp"
#include "ndg/errors.hpp"
#include "ndg/grid.hpp"
#include "ndg/models.hpp"
#include "ndg/partition.hpp"
#include "ndg/solver.hpp"
#include "ndgx.h"

namespace ndgx {

/// Throw the reference exception that matches an ndgx status.
[[noreturn]] inline void rethrow(const ndgx_error& e) {
  const std::string msg = e.message;
  switch (e.code) {
    case NDGX_ERR_CONFIG: throw ndg::ConfigError(msg);
    case NDGX_ERR_PHYSICS: throw ndg::PhysicsError(msg);
    case NDGX_ERR_INSTABILITY: throw ndg::InstabilityError(msg, e.step);
    case NDGX_ERR_DECOMPOSITION: throw ndg::DecompositionError(msg);
    case NDGX_ERR_TRANSPORT: throw ndg::TransportError(msg);
    case NDGX_ERR_RUN: throw ndg::RunError(msg, e.worker);
    default: throw std::runtime_error("ndgx: " + msg);
  }
}

inline void check(int rc, const ndgx_error& e) {
  if (rc != NDGX_OK) rethrow(e);
}

/// ndgx_problem from the reference's configuration objects.
inline ndgx_problem make_problem(const ndg::Mesh& mesh, const ndg::EquationModel& model,
                                 const ndg::NodalBasis& basis, ndg::RKMethod rk, double cfl,
                                 double t_end, int device, int arith) {
  ndgx_problem p{};
  p.dim = mesh.dim;
  for (int a = 0; a < 3; ++a) {
    p.cells[a] = mesh.cells[a];
    p.length[a] = mesh.length[a];
    p.velocity[a] = model.velocity()[a];
  }
  p.order = mesh.order;
  p.equation = model.kind() == ndg::EquationKind::advection ? NDGX_ADVECTION : NDGX_EULER_ISOTHERMAL;
  p.sound_speed = model.sound_speed();
  p.rk = rk == ndg::RKMethod::rk3 ? NDGX_RK3 : (rk == ndg::RKMethod::rk4 ? NDGX_RK4 : NDGX_RK6);
  p.cfl = cfl;
  p.t_end = t_end;
  p.nodes = basis.rule.nodes.data();
  p.weights = basis.rule.weights.data();
  p.diff = basis.diff_matrix.data();
  p.device = device;
  p.arith = arith;
  return p;
}

/// RAII handle.
class Solver {
public:
  explicit Solver(const ndgx_problem& p) {
    ndgx_error e{};
    check(ndgx_create(&p, &h_, &e), e);
  }
  /// run_partitioned's workers in one handle (ndgx_create_partitioned).
  Solver(const ndgx_problem& p, int workers, const std::vector<int>& devices) {
    ndgx_error e{};
    check(ndgx_create_partitioned(&p, workers, (int)devices.size(), devices.empty() ? nullptr : devices.data(), 0,
                                  &h_, &e),
          e);
  }
  ~Solver() { ndgx_destroy(h_); }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;
  ndgx_solver* get() const { return h_; }

private:
  ndgx_solver* h_ = nullptr;
};

/// Drop-in for ndg::advance (src/solver.cpp:372-440) on one B200.
inline ndg::AdvanceResult advance(const ndg::SolverConfig& config, const ndg::StateField& initial,
                                  ndg::StepPlan plan = {}, int device = 0,
                                  int arith = NDGX_ARITH_EXACT) {
  ndg::validate(config);
  const ndg::NodalBasis basis =
      ndg::differentiation_matrix(ndg::gauss_lobatto(config.mesh.order));
  Solver s(make_problem(config.mesh, config.model, basis, config.rk, config.cfl, config.t_end,
                        device, arith));
  ndgx_error e{};
  check(ndgx_upload(s.get(), initial.data(), &e), e);
  ndgx_stats st{};
  check(ndgx_advance(s.get(), plan.fixed_steps, plan.warmup ? 1 : 0, &st, &e), e);
  ndg::AdvanceResult r;
  r.state = initial;
  check(ndgx_download(s.get(), r.state.data(), &e), e);
  r.stats.steps = st.steps;
  r.stats.dt_min = st.dt_min;
  r.stats.dt_max = st.dt_max;
  r.stats.wall_seconds = st.wall_seconds;
  return r;
}

/// Drop-in for ndg::run_partitioned (src/partition.cpp:186-333;
/// include/ndg/partition.hpp:66-67): the same PartitionedResult (state gathered
/// in the global AoS layout, worker 0's step statistics, the reference's own
/// BlockDecomposition), failures as ndg::RunError("worker w: <what>", w).
/// The halo exchange overlaps the interior elements on the device, so each
/// worker's timing is reported as compute time.  States are bit-identical to
/// ndg::run_partitioned in NDGX_ARITH_EXACT.
inline ndg::PartitionedResult run_partitioned(const ndg::SolverConfig& config, const ndg::StateField& initial,
                                              int worker_count, ndg::StepPlan plan = {},
                                              const std::vector<int>& devices = {0},
                                              int arith = NDGX_ARITH_EXACT) {
  ndg::validate(config);
  ndg::PartitionedResult r;
  r.decomposition = ndg::decompose(config.mesh, worker_count);
  const ndg::NodalBasis basis =
      ndg::differentiation_matrix(ndg::gauss_lobatto(config.mesh.order));
  Solver s(make_problem(config.mesh, config.model, basis, config.rk, config.cfl, config.t_end,
                        devices.empty() ? 0 : devices[0], arith),
           worker_count, devices);
  ndgx_error e{};
  check(ndgx_upload(s.get(), initial.data(), &e), e);
  ndgx_stats st{};
  check(ndgx_advance(s.get(), plan.fixed_steps, plan.warmup ? 1 : 0, &st, &e), e);
  r.state = initial;
  check(ndgx_download(s.get(), r.state.data(), &e), e);
  r.stats.steps = st.steps;
  r.stats.dt_min = st.dt_min;
  r.stats.dt_max = st.dt_max;
  r.stats.wall_seconds = st.wall_seconds;
  r.worker_timings.assign(worker_count, ndg::WorkerTiming{st.wall_seconds, 0.0});
  return r;
}

/// Drop-in for ndg::serial_rhs (src/solver.cpp:442-456).
inline ndg::StateField serial_rhs(const ndg::Mesh& mesh, const ndg::NodalBasis& basis,
                                  const ndg::EquationModel& model, const ndg::StateField& field,
                                  int device = 0, int arith = NDGX_ARITH_EXACT) {
  if (basis.rule.order != mesh.order) throw ndg::ConfigError("basis order does not match mesh order");
  if (model.spatial_dim() != mesh.dim)
    throw ndg::ConfigError("model dimension does not match mesh dimension");
  Solver s(make_problem(mesh, model, basis, ndg::RKMethod::rk4, 0.4, 1.0, device, arith));
  ndgx_error e{};
  check(ndgx_upload(s.get(), field.data(), &e), e);
  ndg::StateField out(field.shape());
  check(ndgx_rhs(s.get(), out.data(), &e), e);
  return out;
}

}  // namespace ndgx
