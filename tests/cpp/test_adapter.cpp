// GPU integration test of the C++ drop-in (include/ndgx_ndg.hpp) against the
// UNMODIFIED reference library (oracle/_ref/libndg_ref.so): the reference's
// own test scenarios (proj/tests/test_solver.cpp) are replayed through
// ndgx::advance / ndgx::serial_rhs and compared with ndg::advance /
// ndg::serial_rhs by memcmp.  Built by tests/cpp/Makefile; run by
// tests/test_cpp_adapter.py (-m gpu).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>

#include "ndgx_ndg.hpp"

static int g_fail = 0, g_checks = 0;
#define CHECK(...)                                                           \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(__VA_ARGS__)) {                                                    \
      ++g_fail;                                                              \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__);    \
    }                                                                        \
  } while (0)

using namespace ndg;

static bool same(const StateField& a, const StateField& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

static void case_advance(const char* name, const Mesh& mesh, const EquationModel& model, RKMethod rk,
                         const StateField& init, StepPlan plan, double t_end = 1.0) {
  SolverConfig config{mesh, model, rk, 0.4, t_end};
  const AdvanceResult want = ndg::advance(config, init, plan);
  const AdvanceResult got = ndgx::advance(config, init, plan);
  const bool ok = same(want.state, got.state) && want.stats.steps == got.stats.steps &&
                  want.stats.dt_min == got.stats.dt_min && want.stats.dt_max == got.stats.dt_max;
  std::printf("%s %s (steps %ld)\n", ok ? "ok  " : "FAIL", name, got.stats.steps);
  CHECK(ok);
}

int main() {
  const EquationModel adv1 = EquationModel::advection(1, {1, 0, 0});
  const EquationModel adv2 = EquationModel::advection(2, {1, 0.5, 0});
  const EquationModel eu2 = EquationModel::isothermal_euler(2, 1.0);
  const EquationModel eu3 = EquationModel::isothermal_euler(3, 1.0);
  {
    const Mesh m(1, {1024, 1, 1}, 4);
    case_advance("1D adv o4 RK4 1024 (100 steps)", m, adv1, RKMethod::rk4,
                 init_multisine(m, adv1, gauss_lobatto(4), {1.0}), StepPlan{100, false});
  }
  {
    const Mesh m(2, {24, 20, 1}, 8);
    case_advance("2D adv o8 RK3 24x20 (t_end 0.05)", m, adv2, RKMethod::rk3,
                 init_multisine(m, adv2, gauss_lobatto(8), 6, 3), StepPlan{-1, true}, 0.05);
  }
  {
    const Mesh m(2, {48, 48, 1}, 8);
    case_advance("2D Euler o8 RK4 48^2 (100 steps, warm-up)", m, eu2, RKMethod::rk4,
                 init_euler_subsonic(m, eu2, gauss_lobatto(8)), StepPlan{100, true});
  }
  {
    const Mesh m(3, {12, 12, 12}, 4);
    case_advance("3D Euler o4 RK6 12^3 (20 steps)", m, eu3, RKMethod::rk6,
                 init_euler_subsonic(m, eu3, gauss_lobatto(4)), StepPlan{20, false});
  }
  {  // serial_rhs equality (solver.cpp:442-456)
    const Mesh m(2, {16, 16, 1}, 6);
    const NodalBasis basis = differentiation_matrix(gauss_lobatto(6));
    const StateField f = init_euler_subsonic(m, eu2, basis.rule);
    CHECK(same(ndg::serial_rhs(m, basis, eu2, f), ndgx::serial_rhs(m, basis, eu2, f)));
  }
  {  // test_solver.cpp:239-255
    const Mesh mesh(2, {4, 4, 1}, 3);
    const NodalBasis basis = differentiation_matrix(gauss_lobatto(3));
    StateField f = init_euler_subsonic(mesh, eu2, basis.rule, 0);
    f.at({2, 1, 0}, {1, 1, 0}, 0) = -0.5;
    std::string want, got;
    try { ndg::serial_rhs(mesh, basis, eu2, f); } catch (const PhysicsError& e) { want = e.what(); }
    try {
      ndgx::serial_rhs(mesh, basis, eu2, f);
    } catch (const PhysicsError& e) {
      got = e.what();
    }
    CHECK(!got.empty() && got == want);
    CHECK(got.find("density") != std::string::npos && got.find("cell") != std::string::npos);
  }
  {  // test_solver.cpp:380-394
    const Mesh mesh(1, {8, 1, 1}, 3);
    StateField f = init_multisine(mesh, adv1, gauss_lobatto(3), {1.0});
    f.values()[3] = std::numeric_limits<double>::quiet_NaN();
    SolverConfig config{mesh, adv1, RKMethod::rk4, 0.4, 1.0};
    long step = -1;
    std::string what;
    try {
      ndgx::advance(config, f);
    } catch (const InstabilityError& e) {
      step = e.step();
      what = e.what();
    }
    CHECK(step == 1);
    CHECK(what.find("step 1") != std::string::npos);
  }
  {  // test_solver.cpp:277-300
    const EquationModel still = EquationModel::advection(1, {0, 0, 0});
    const Mesh mesh(1, {8, 1, 1}, 3);
    const StateField f = init_multisine(mesh, still, gauss_lobatto(3), {0.5});
    const AdvanceResult r = ndgx::advance(SolverConfig{mesh, still, RKMethod::rk4, 0.4, 0.7}, f);
    CHECK(r.stats.steps == 1);
    CHECK(r.stats.dt_max == 0.7);
    CHECK(same(r.state, f));
    const StateField g = init_multisine(mesh, adv1, gauss_lobatto(3), {1.0});
    const AdvanceResult s = ndgx::advance(SolverConfig{mesh, adv1, RKMethod::rk4, 0.4, 0.004}, g);
    CHECK(s.stats.steps == 1);
    CHECK(s.stats.dt_max == 0.004);
    bool threw = false;
    try {
      ndgx::advance(SolverConfig{mesh, still, RKMethod::rk4, 0.4, 1.0}, f, StepPlan{3, false});
    } catch (const ConfigError&) {
      threw = true;
    }
    CHECK(threw);
  }
  // ---- run_partitioned (proj/tests/test_partition.cpp:267-349) against the reference's own
  {
    const Mesh mesh(2, {8, 8, 1}, 3);
    const EquationModel model = EquationModel::advection(2, {1, 0, 0});
    const StateField init = init_multisine(mesh, model, gauss_lobatto(3), 4, 2026);
    const SolverConfig config{mesh, model, RKMethod::rk4, 0.4, 1.0};
    for (int workers : {1, 2, 4}) {
      const PartitionedResult want = ndg::run_partitioned(config, init, workers, StepPlan{10, false});
      const PartitionedResult got = ndgx::run_partitioned(config, init, workers, StepPlan{10, false});
      const bool ok = same(want.state, got.state) && want.stats.steps == got.stats.steps &&
                      got.worker_timings.size() == (size_t)workers &&
                      got.decomposition.grid == want.decomposition.grid;
      std::printf("%s run_partitioned 2D adv o3 RK4 8x8 P=%d\n", ok ? "ok  " : "FAIL", workers);
      CHECK(ok);
    }
  }
  {
    const Mesh mesh(3, {4, 4, 4}, 2);
    const EquationModel model = EquationModel::advection(3, {1, 0, 0});
    const StateField init = init_multisine(mesh, model, gauss_lobatto(2), 2, 5);
    const SolverConfig config{mesh, model, RKMethod::rk3, 0.4, 1.0};
    const PartitionedResult want = ndg::run_partitioned(config, init, 2, StepPlan{6, false});
    const PartitionedResult got = ndgx::run_partitioned(config, init, 2, StepPlan{6, false});
    std::printf("%s run_partitioned 3D adv o2 RK3 4^3 P=2\n", same(want.state, got.state) ? "ok  " : "FAIL");
    CHECK(same(want.state, got.state));
  }
  {
    const Mesh mesh(2, {8, 8, 1}, 3);
    const EquationModel model = EquationModel::isothermal_euler(2, 1.0);
    const StateField init = init_euler_subsonic(mesh, model, gauss_lobatto(3), 0);
    const SolverConfig config{mesh, model, RKMethod::rk4, 0.4, 1.0};
    const PartitionedResult want = ndg::run_partitioned(config, init, 4, StepPlan{8, false});
    const PartitionedResult got = ndgx::run_partitioned(config, init, 4, StepPlan{8, false});
    const bool ok = same(want.state, got.state) && want.stats.dt_min == got.stats.dt_min;
    std::printf("%s run_partitioned 2D Euler o3 RK4 8x8 P=4\n", ok ? "ok  " : "FAIL");
    CHECK(ok);
  }
  {
    const Mesh mesh(2, {6, 6, 1}, 3);
    const EquationModel model = EquationModel::advection(2, {1, 0, 0});
    const StateField init = init_multisine(mesh, model, gauss_lobatto(3), 3, 7);
    const SolverConfig config{mesh, model, RKMethod::rk4, 0.4, 0.03};
    const PartitionedResult want = ndg::run_partitioned(config, init, 2);
    const PartitionedResult got = ndgx::run_partitioned(config, init, 2);
    const bool ok = same(want.state, got.state) && want.stats.steps == got.stats.steps &&
                    want.stats.dt_max == got.stats.dt_max;
    std::printf("%s run_partitioned t_end 6x6 P=2 (steps %ld)\n", ok ? "ok  " : "FAIL", got.stats.steps);
    CHECK(ok);
  }
  {
    const Mesh mesh(3, {4, 4, 16}, 4);
    const EquationModel model = EquationModel::isothermal_euler(3, 1.0);
    const StateField init = init_euler_subsonic(mesh, model, gauss_lobatto(4));
    const SolverConfig config{mesh, model, RKMethod::rk6, 0.4, 1.0};
    const PartitionedResult want = ndg::run_partitioned(config, init, 4, StepPlan{5, true});
    const PartitionedResult got = ndgx::run_partitioned(config, init, 4, StepPlan{5, true});
    const bool ok = same(want.state, got.state) && want.decomposition.grid == got.decomposition.grid &&
                    want.stats.dt_max == got.stats.dt_max;
    std::printf("%s run_partitioned 3D Euler o4 RK6 4x4x16 P=4 z-slabs\n", ok ? "ok  " : "FAIL");
    CHECK(ok);
  }
  {  // a failing worker surfaces as RunError naming it (test_partition.cpp:330-349)
    const Mesh mesh(2, {8, 8, 1}, 3);
    const EquationModel model = EquationModel::isothermal_euler(2, 1.0);
    StateField init = init_euler_subsonic(mesh, model, gauss_lobatto(3), 0);
    init.at({6, 6, 0}, {1, 1, 0}, 0) = -2.0;
    const SolverConfig config{mesh, model, RKMethod::rk4, 0.4, 1.0};
    std::string want, got;
    int want_w = -1, got_w = -1;
    try { ndg::run_partitioned(config, init, 2, StepPlan{4, false}); } catch (const RunError& e) {
      want = e.what();
      want_w = e.worker();
    }
    try { ndgx::run_partitioned(config, init, 2, StepPlan{4, false}); } catch (const RunError& e) {
      got = e.what();
      got_w = e.worker();
    }
    std::printf("%s RunError: '%s' (reference '%s')\n", got == want && got_w == 1 ? "ok  " : "FAIL", got.c_str(),
                want.c_str());
    CHECK(got == want && got_w == want_w && got_w == 1);
  }
  std::printf("%d/%d checks passed\n", g_checks - g_fail, g_checks);
  return g_fail == 0 ? 0 : 1;
}
