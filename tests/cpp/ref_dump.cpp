// TEST INFRASTRUCTURE ONLY: dump a raw field with the reference's own
// dump_field (src/field_io.cpp:18-34), via oracle/_ref/libndg_ref.so.
//   ref_dump <dim> <c0> <c1> <c2> <order> <kind> <l0> <l1> <l2> <raw.f64> <out.ndgf>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ndg_oracle.h"

extern "C" int ref_dump_field(const ndgo_config* c, const double* u, const char* path);

int main(int argc, char** argv) {
  if (argc != 12) {
    std::fprintf(stderr, "usage: ref_dump dim c0 c1 c2 order kind l0 l1 l2 raw out\n");
    return 2;
  }
  ndgo_config c{};
  c.dim = std::atoi(argv[1]);
  for (int a = 0; a < 3; ++a) c.cells[a] = std::atoi(argv[2 + a]);
  c.order = std::atoi(argv[5]);
  c.kind = std::atoi(argv[6]);
  for (int a = 0; a < 3; ++a) c.length[a] = std::strtod(argv[7 + a], nullptr);
  c.velocity[0] = 1.0;
  c.sound_speed = 1.0;
  c.rk = 1;
  c.cfl = 0.4;
  c.t_end = 1.0;
  std::FILE* f = std::fopen(argv[10], "rb");
  if (!f) return 3;
  std::vector<double> u;
  double v;
  while (std::fread(&v, sizeof v, 1, f) == 1) u.push_back(v);
  std::fclose(f);
  return ref_dump_field(&c, u.data(), argv[11]);
}
