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

int QuadratureConfig::tier_order(int tier) const {
  if (tier == 0) return std::min(disjoint_order, 2);
  if (tier == 1) return disjoint_order;
  return std::min(disjoint_order + 1, 6);
}

}  // namespace hmb
