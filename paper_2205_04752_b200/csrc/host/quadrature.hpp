// Symmetric triangle rules handed to the device kernels.
// Same tables and orbit expansion as the reference's gauss_rule
// (proj/src/quadrature.cpp:11-95): weights sum to 1/2, points are
// reference coordinates (l1, l2) of barycentric (l0, l1, l2).
#pragma once

#include <vector>

namespace hmb {

struct TriangleRule {
  std::vector<double> a, b, w;
  int order = 0;
};

TriangleRule gauss_rule(int order);  // orders 1..6, throws otherwise

// QuadratureConfig (proj/include/hmbem/kernels.hpp:44-52) restricted to what
// collocation uses: point_order tiers (kernels.cpp:87-93)
struct QuadratureConfig {
  int disjoint_order = 4;
  double far_ratio = 4.0;
  double mid_ratio = 1.5;
  // rule orders of the far / mid / near tiers
  int tier_order(int tier) const;
};

// n-point Gauss-Legendre on [0, 1] (quadrature.cpp:97-125)
void gauss_legendre_01(int n, std::vector<double>& x, std::vector<double>& w);

// Sauter-Schwab pair rule of a touching pair (PairCase 1 vertex, 2 edge,
// 3 identical; quadrature.cpp:168-338): `order` Gauss-Legendre points per
// dimension of [0,1]^4 on each subdomain simplex
struct PairRuleTable {
  std::vector<double> xr1, xr2, yr1, yr2, w;
};
PairRuleTable singular_pair_rule(int pair_case, int order);

// GalerkinKernels' QuadratureConfig defaults (kernels.hpp:44-52)
struct GalerkinQuadrature {
  int singular_order = 7;
  int identical_bump = 2;
};

}  // namespace hmb
