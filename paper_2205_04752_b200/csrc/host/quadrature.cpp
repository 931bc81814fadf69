#include "quadrature.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <string>

#include "errors.hpp"

namespace hmb {

namespace {

// symmetric orbit of the barycentric triple (x, y, z) with weight w; a
// permutation is dropped when its first two coordinates repeat one of the
// last six points (the reference's de-duplication window)
struct OrbitBuilder {
  std::vector<std::array<double, 3>> pts;
  std::vector<double> wts;
  void orbit(double x, double y, double z, double w) {
    const std::array<std::array<double, 3>, 6> perms = {
        {{x, y, z}, {x, z, y}, {y, x, z}, {y, z, x}, {z, x, y}, {z, y, x}}};
    for (const auto& p : perms) {
      const std::size_t from = pts.size() >= 6 ? pts.size() - 6 : 0;
      const bool dup = std::any_of(pts.begin() + from, pts.end(), [&](const auto& q) {
        return std::abs(q[0] - p[0]) < 1e-15 && std::abs(q[1] - p[1]) < 1e-15;
      });
      if (!dup) {
        pts.push_back(p);
        wts.push_back(w);
      }
    }
  }
  TriangleRule finish(int order) const {
    TriangleRule r;
    r.order = order;
    for (std::size_t i = 0; i < pts.size(); ++i) {
      r.a.push_back(pts[i][1]);
      r.b.push_back(pts[i][2]);
      r.w.push_back(0.5 * wts[i]);
    }
    return r;
  }
};

}  // namespace

TriangleRule gauss_rule(int order) {
  OrbitBuilder ob;
  const double third = 1.0 / 3.0;
  if (order == 1) {
    ob.orbit(third, third, third, 1.0);
  } else if (order == 2) {
    ob.orbit(2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0, third);
  } else if (order == 3 || order == 4) {  // Dunavant degree 4
    ob.orbit(0.816847572980459, 0.091576213509771, 0.091576213509771,
             0.109951743655322);
    ob.orbit(0.108103018168070, 0.445948490915965, 0.445948490915965,
             0.223381589678011);
  } else if (order == 5) {  // Radon 7-point rule
    const double s15 = std::sqrt(15.0);
    ob.orbit(third, third, third, 9.0 / 40.0);
    ob.orbit((9.0 - 2.0 * s15) / 21.0, (6.0 + s15) / 21.0, (6.0 + s15) / 21.0,
             (155.0 + s15) / 1200.0);
    ob.orbit((9.0 + 2.0 * s15) / 21.0, (6.0 - s15) / 21.0, (6.0 - s15) / 21.0,
             (155.0 - s15) / 1200.0);
  } else if (order == 6) {
    ob.orbit(0.873821971016996, 0.063089014491502, 0.063089014491502,
             0.050844906370207);
    ob.orbit(0.501426509658179, 0.249286745170910, 0.249286745170910,
             0.116786275726379);
    ob.orbit(0.636502499121399, 0.310352451033785, 0.053145049844816,
             0.082851075618374);
  } else {
    throw Error("gauss_rule: unsupported order " + std::to_string(order));
  }
  return ob.finish(order);
}

void gauss_legendre_01(int n, std::vector<double>& x, std::vector<double>& w) {
  if (n < 1) throw Error("gauss_legendre_01: n must be positive");
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  // Newton on P_n from the Chebyshev-like guess, symmetric pairs mapped to [0,1]
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p_cur = 1.0, p_prev = 0.0;
      for (int j = 0; j < n; ++j) {
        const double p_old = p_prev;
        p_prev = p_cur;
        p_cur = ((2.0 * j + 1.0) * z * p_prev - j * p_old) / (j + 1.0);
      }
      dp = n * (z * p_cur - p_prev) / (z * z - 1.0);
      const double step = p_cur / dp;
      z -= step;
      if (std::abs(step) < 1e-16) break;
    }
    const double wi = 1.0 / ((1.0 - z * z) * dp * dp);
    x[i] = 0.5 * (1.0 - z);
    x[n - 1 - i] = 0.5 * (1.0 + z);
    w[i] = w[n - 1 - i] = wi;
  }
}

namespace {

// the subdomain maps [0,1]^4 -> (x1, x2, y1, y2) and the Jacobian; each
// expression as the reference writes it (the rounding is the rule)
void ss_point(int pc, int s, double xi, double e1, double e2, double e3, double* p) {
  double& x1 = p[0];
  double& x2 = p[1];
  double& y1 = p[2];
  double& y2 = p[3];
  double& jac = p[4];
  if (pc == 3) {  // identical, 6 simplices
    jac = xi * xi * xi * e1 * e1 * e2;
    if (s == 0) { x1 = xi * e1 * (1 - e2); x2 = xi * (1 - e1 * (1 - e2)); y1 = xi * e1 * (1 - e2 * e3); y2 = xi * (1 - e1); }
    if (s == 1) { x1 = xi * e1 * (1 - e2 * e3); x2 = xi * (1 - e1); y1 = xi * e1 * (1 - e2); y2 = xi * (1 - e1 * (1 - e2)); }
    if (s == 2) { x1 = xi * (1 - e1 * (1 - e2 * (1 - e3))); x2 = xi * e1 * (1 - e2 * (1 - e3)); y1 = xi * (1 - e1); y2 = xi * e1 * (1 - e2); }
    if (s == 3) { x1 = xi * (1 - e1); x2 = xi * e1 * (1 - e2); y1 = xi * (1 - e1 * (1 - e2 * (1 - e3))); y2 = xi * e1 * (1 - e2 * (1 - e3)); }
    if (s == 4) { x1 = xi * (1 - e1); x2 = xi * e1 * (1 - e2 * e3); y1 = xi * (1 - e1 * (1 - e2)); y2 = xi * e1 * (1 - e2); }
    if (s == 5) { x1 = xi * (1 - e1 * (1 - e2)); x2 = xi * e1 * (1 - e2); y1 = xi * (1 - e1); y2 = xi * e1 * (1 - e2 * e3); }
  } else if (pc == 2) {  // shared edge, 5 simplices
    jac = xi * xi * xi * e1 * e1;
    if (s == 0) { x1 = xi * (1 - e1 * e3); x2 = xi * e1 * e3; y1 = xi * (1 - e1); y2 = xi * e1 * (1 - e2); }
    if (s == 1) { x1 = xi * (1 - e1); x2 = xi * e1; y1 = xi * (1 - e1 * e2); y2 = xi * e1 * e2 * (1 - e3); }
    if (s == 2) { x1 = xi * (1 - e1); x2 = xi * e1 * (1 - e2); y1 = xi * (1 - e1 * e2 * e3); y2 = xi * e1 * e2 * e3; }
    if (s == 3) { x1 = xi * (1 - e1 * e2); x2 = xi * e1 * e2 * (1 - e3); y1 = xi * (1 - e1); y2 = xi * e1; }
    if (s == 4) { x1 = xi * (1 - e1); x2 = xi * e1 * (1 - e2 * e3); y1 = xi * (1 - e1 * e2); y2 = xi * e1 * e2; }
    if (s > 0) jac *= e2;
  } else {  // shared vertex, 2 simplices
    jac = xi * xi * xi * e2;
    if (s == 0) { x1 = xi * (1 - e1); x2 = xi * e1; y1 = xi * e2 * (1 - e3); y2 = xi * e2 * e3; }
    else { x1 = xi * e2 * (1 - e3); x2 = xi * e2 * e3; y1 = xi * (1 - e1); y2 = xi * e1; }
  }
}

}  // namespace

PairRuleTable singular_pair_rule(int pair_case, int order) {
  if (pair_case < 1 || pair_case > 3) throw Error("singular_pair_rule: bad pair case");
  std::vector<double> gx, gw;
  gauss_legendre_01(order, gx, gw);
  const int simplices = pair_case == 3 ? 6 : pair_case == 2 ? 5 : 2;
  PairRuleTable r;
  double p[5];
  for (int s = 0; s < simplices; ++s)
    for (int a = 0; a < order; ++a)
      for (int b = 0; b < order; ++b)
        for (int c = 0; c < order; ++c)
          for (int d = 0; d < order; ++d) {
            ss_point(pair_case, s, gx[a], gx[b], gx[c], gx[d], p);
            r.xr1.push_back(p[0]);
            r.xr2.push_back(p[1]);
            r.yr1.push_back(p[2]);
            r.yr2.push_back(p[3]);
            r.w.push_back(p[4] * gw[a] * gw[b] * gw[c] * gw[d]);
          }
  return r;
}

int QuadratureConfig::tier_order(int tier) const {
  if (tier == 0) return std::min(disjoint_order, 2);
  if (tier == 1) return disjoint_order;
  return std::min(disjoint_order + 1, 6);
}

}  // namespace hmb
