// ndgx_setup.h -- host setup helpers shared by the C-ABI implementation.
#pragma once

#include "ndgx.h"

namespace ndgx {

void legendre(int n, double x, double* p, double* dp);
void rk_tableau(int rk, int* stages, double a[7][7], double b[7]);
// K_d[k*N+l] = 2 D[l][k] w_l / (dx_d w_k), lift_d = 2 / (dx_d w_0)
void build_operator(const ndgx_problem* p, const double* nodes, const double* weights,
                    const double* diff, double K[3][64], double lift[3]);
double dt_numerator(const ndgx_problem* p);  // cfl * min_d dx_d

}  // namespace ndgx
