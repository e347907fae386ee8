// TEST INFRASTRUCTURE ONLY: run one of the reference's experiment sweeps
// (run_experiment, src/experiments.cpp) on the CPU and print its CSV report.
//   ref_experiments <experiment> <equation> <dim> <orders,..> <rk> <cells,..>
//                   <nk> <seed> <workers,..> <cfl> <t_end> <steps> <compare_equations>
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "ndg/experiments.hpp"
#include "ndg/report.hpp"

static std::vector<int> ints(const std::string& s) {
  std::vector<int> v;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) v.push_back(std::atoi(tok.c_str()));
  return v;
}

int main(int argc, char** argv) {
  if (argc != 14) return 2;
  ndg::ExperimentSpec s;
  s.experiment = argv[1];
  s.equation = argv[2];
  s.dim = std::atoi(argv[3]);
  s.orders = ints(argv[4]);
  s.rk = argv[5];
  s.cells = ints(argv[6]);
  s.nk = std::atoi(argv[7]);
  s.seed = std::strtoull(argv[8], nullptr, 10);
  s.workers = ints(argv[9]);
  s.cfl = std::strtod(argv[10], nullptr);
  s.t_end = std::strtod(argv[11], nullptr);
  s.steps = std::atol(argv[12]);
  s.compare_equations = std::atoi(argv[13]) != 0;
  try {
    std::cout << ndg::report_to_csv(ndg::run_experiment(s));
  } catch (const std::exception& e) {
    std::cerr << e.what() << "\n";
    return 1;
  }
  return 0;
}
