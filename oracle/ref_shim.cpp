// TEST INFRASTRUCTURE ONLY -- a C-ABI shim over the UNMODIFIED reference
// solver, compiled from its own sources under /root/reference/proj by
// oracle/Makefile into oracle/_ref/libndg_ref.so.  Used (a) to pin the plain-C
// oracle (ndg_oracle.c) bit-for-bit and to generate tests/golden/, and (b) as
// the reference CPU arm of bench.py (`--impl reference`, cpu_baseline kind
// "reference").  Never linked by the product.
//
// The exported signatures reuse ndgo_config / ndgo_stats / ndgo_error from
// ndg_oracle.h so tests can swap the two implementations.

#include <cstring>
#include <exception>
#include <string>

#include "ndg/basis.hpp"
#include "ndg/errors.hpp"
#include "ndg/field_io.hpp"
#include "ndg/grid.hpp"
#include "ndg/models.hpp"
#include "ndg/partition.hpp"
#include "ndg/solver.hpp"
#include "ndg_oracle.h"

namespace {

ndg::Mesh mesh_of(const ndgo_config* c) {
  return ndg::Mesh(c->dim, {c->cells[0], c->cells[1], c->cells[2]}, c->order,
                   {c->length[0], c->length[1], c->length[2]});
}

ndg::EquationModel model_of(const ndgo_config* c) {
  if (c->kind == 0)
    return ndg::EquationModel::advection(c->dim,
                                         {c->velocity[0], c->velocity[1], c->velocity[2]});
  return ndg::EquationModel::isothermal_euler(c->dim, c->sound_speed);
}

ndg::RKMethod rk_of(const ndgo_config* c) {
  return c->rk == 0 ? ndg::RKMethod::rk3 : (c->rk == 1 ? ndg::RKMethod::rk4 : ndg::RKMethod::rk6);
}

ndg::SolverConfig config_of(const ndgo_config* c) {
  return ndg::SolverConfig{mesh_of(c), model_of(c), rk_of(c), c->cfl, c->t_end};
}

ndg::StateField field_of(const ndgo_config* c, const double* u) {
  ndg::StateField f(mesh_of(c), model_of(c));
  std::memcpy(f.data(), u, f.size() * sizeof(double));
  return f;
}

void put(ndgo_error* e, int code, long step, int worker, const std::string& msg) {
  if (!e) return;
  e->code = code;
  e->step = step;
  e->worker = worker;
  std::snprintf(e->message, sizeof(e->message), "%s", msg.c_str());
}

template <typename Fn>
int guarded(ndgo_error* err, Fn&& fn) {
  try {
    fn();
    if (err) err->code = 0;
    return 0;
  } catch (const ndg::ConfigError& e) {
    put(err, 1, 0, -1, e.what());
    return 1;
  } catch (const ndg::PhysicsError& e) {
    put(err, 2, 0, -1, e.what());
    return 2;
  } catch (const ndg::InstabilityError& e) {
    put(err, 3, e.step(), -1, e.what());
    return 3;
  } catch (const ndg::DecompositionError& e) {
    put(err, 4, 0, -1, e.what());
    return 4;
  } catch (const ndg::RunError& e) {
    put(err, 6, 0, e.worker(), e.what());
    return 6;
  } catch (const std::exception& e) {
    put(err, 9, 0, -1, e.what());
    return 9;
  }
}

}  // namespace

extern "C" {

int ref_gauss_lobatto(int order, double* nodes, double* weights, double* diff) {
  const ndg::NodalBasis b = ndg::differentiation_matrix(ndg::gauss_lobatto(order));
  for (int k = 0; k < order; ++k) {
    nodes[k] = b.rule.nodes[k];
    weights[k] = b.rule.weights[k];
  }
  for (int k = 0; k < order * order; ++k) diff[k] = b.diff_matrix[k];
  return 0;
}

int ref_init_multisine(const ndgo_config* c, const double* amps, int n, double* out) {
  ndg::StateField f = ndg::init_multisine(mesh_of(c), model_of(c), ndg::gauss_lobatto(c->order),
                                          std::vector<double>(amps, amps + n));
  std::memcpy(out, f.data(), f.size() * sizeof(double));
  return 0;
}

int ref_init_multisine_seed(const ndgo_config* c, int n_modes, unsigned long long seed,
                            double* out) {
  ndg::StateField f =
      ndg::init_multisine(mesh_of(c), model_of(c), ndg::gauss_lobatto(c->order), n_modes, seed);
  std::memcpy(out, f.data(), f.size() * sizeof(double));
  return 0;
}

int ref_init_euler_subsonic(const ndgo_config* c, double* out) {
  ndg::StateField f =
      ndg::init_euler_subsonic(mesh_of(c), model_of(c), ndg::gauss_lobatto(c->order), 0);
  std::memcpy(out, f.data(), f.size() * sizeof(double));
  return 0;
}

// dump_field (src/field_io.cpp:18-34) of a host field in FieldShape order
int ref_dump_field(const ndgo_config* c, const double* u, const char* path) {
  const ndg::Mesh mesh = mesh_of(c);
  ndg::StateField f(mesh, model_of(c));
  std::memcpy(f.data(), u, f.size() * sizeof(double));
  ndg::dump_field(path, mesh, f);
  return 0;
}

double ref_l2_error(const ndgo_config* c, const double* a, const double* b, int var) {
  return ndg::l2_error(mesh_of(c), ndg::gauss_lobatto(c->order), field_of(c, a),
                       field_of(c, b), var);
}

int ref_conserved_totals(const ndgo_config* c, const double* u, double* out) {
  const std::vector<double> t =
      ndg::conserved_totals(mesh_of(c), ndg::gauss_lobatto(c->order), field_of(c, u));
  std::memcpy(out, t.data(), t.size() * sizeof(double));
  return 0;
}

int ref_serial_rhs(const ndgo_config* c, const double* u, double* dudt, ndgo_error* err) {
  return guarded(err, [&] {
    const ndg::Mesh mesh = mesh_of(c);
    const ndg::NodalBasis basis = ndg::differentiation_matrix(ndg::gauss_lobatto(c->order));
    ndg::StateField d = ndg::serial_rhs(mesh, basis, model_of(c), field_of(c, u));
    std::memcpy(dudt, d.data(), d.size() * sizeof(double));
  });
}

int ref_advance(const ndgo_config* c, double* u, long fixed_steps, int warmup,
                ndgo_stats* stats, ndgo_error* err) {
  return guarded(err, [&] {
    ndg::AdvanceResult r = ndg::advance(config_of(c), field_of(c, u),
                                        ndg::StepPlan{fixed_steps, warmup != 0});
    std::memcpy(u, r.state.data(), r.state.size() * sizeof(double));
    stats->steps = r.stats.steps;
    stats->dt_min = r.stats.dt_min;
    stats->dt_max = r.stats.dt_max;
    stats->wall_seconds = r.stats.wall_seconds;
  });
}

int ref_run_partitioned(const ndgo_config* c, double* u, int workers, long fixed_steps,
                        int warmup, ndgo_stats* stats, ndgo_error* err) {
  return guarded(err, [&] {
    ndg::PartitionedResult r = ndg::run_partitioned(
        config_of(c), field_of(c, u), workers, ndg::StepPlan{fixed_steps, warmup != 0});
    std::memcpy(u, r.state.data(), r.state.size() * sizeof(double));
    stats->steps = r.stats.steps;
    stats->dt_min = r.stats.dt_min;
    stats->dt_max = r.stats.dt_max;
    stats->wall_seconds = r.stats.wall_seconds;
  });
}

int ref_decompose(const ndgo_config* c, int workers, int grid[3], int* lo, int* hi, int* nbr,
                  ndgo_error* err) {
  return guarded(err, [&] {
    const ndg::BlockDecomposition d = ndg::decompose(mesh_of(c), workers);
    for (int a = 0; a < 3; ++a) grid[a] = d.grid[a];
    for (int w = 0; w < workers; ++w)
      for (int a = 0; a < 3; ++a) {
        lo[w * 3 + a] = d.blocks[w].lo[a];
        hi[w * 3 + a] = d.blocks[w].hi[a];
        nbr[(w * 3 + a) * 2 + 0] = d.blocks[w].neighbor[a][0];
        nbr[(w * 3 + a) * 2 + 1] = d.blocks[w].neighbor[a][1];
      }
  });
}

int ref_pack_face_trace(const ndgo_config* c, const int cells[3], const double* u, int axis,
                        int cell_d, int node_d, double* out) {
  ndg::FieldShape s;
  s.dim = c->dim;
  s.cells = {cells[0], cells[1], cells[2]};
  s.order = c->order;
  s.n_var = c->kind == 0 ? 1 : c->dim + 1;
  std::vector<double> uu(u, u + s.size()), o;
  ndg::pack_face_trace(s, uu, axis, cell_d, node_d, o);
  std::memcpy(out, o.data(), o.size() * sizeof(double));
  return static_cast<int>(o.size());
}

double ref_max_wavespeed_bound(const ndgo_config* c, const double* u, ndgo_error* err) {
  double a = -1.0;
  guarded(err, [&] {
    ndg::StateField f = field_of(c, u);
    a = ndg::max_wavespeed_bound(f.shape(), model_of(c), f.values());
  });
  return a;
}

}  // extern "C"
