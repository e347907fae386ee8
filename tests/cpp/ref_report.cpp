// TEST INFRASTRUCTURE ONLY: round-trip a CSV report through the reference's
// own reader and writer (read_report_csv + report_to_csv, src/report.cpp).
//   ref_report <in.csv>   -> the reference's CSV bytes on stdout
#include <cstdio>
#include <iostream>

#include "ndg/report.hpp"

int main(int argc, char** argv) {
  if (argc != 2) return 2;
  const ndg::BenchReport r = ndg::read_report_csv(argv[1]);
  std::cout << ndg::report_to_csv(r);
  return 0;
}
