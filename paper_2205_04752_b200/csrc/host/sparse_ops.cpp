#include "sparse_ops.hpp"

#include "errors.hpp"

namespace hmb {

namespace {

V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}

}  // namespace

Ell3 build_t_matrix(const Mesh& mesh, int k, int l) {
  if (k < 0 || l < 0 || k > 2 || l > 2 || k == l) throw Error("T(k,l): bad components");
  if (mesh.normals.size() != mesh.triangles.size())
    throw MeshError("mesh geometry caches missing (call finish())");
  Ell3 e;
  e.rows = mesh.nt();
  e.cols = mesh.nv();
  e.col.resize(3 * e.rows);
  e.val.resize(3 * e.rows);
  for (int t = 0; t < e.rows; ++t) {
    // hat-function gradients n x (opposite edge) / (2 area) (operators.cpp:8-14)
    const V3& n = mesh.normals[t];
    const Real inv2a = 1.0 / (2.0 * mesh.areas[t]);
    for (int a = 0; a < 3; ++a) {
      const V3& p = mesh.corner(t, (a + 1) % 3);
      const V3& q = mesh.corner(t, (a + 2) % 3);
      const V3 g = cross(n, V3{q[0] - p[0], q[1] - p[1], q[2] - p[2]});
      const Real gk = g[k] * inv2a, gl = g[l] * inv2a;
      e.col[3 * t + a] = mesh.triangles[t][a];
      e.val[3 * t + a] = n[l] * gk - n[k] * gl;
    }
  }
  return e;
}

Ell3 build_mass_matrix(const Mesh& mesh) {
  Ell3 e;
  e.rows = mesh.nt();
  e.cols = mesh.nv();
  e.col.resize(3 * e.rows);
  e.val.resize(3 * e.rows);
  for (int t = 0; t < e.rows; ++t)
    for (int a = 0; a < 3; ++a) {
      e.col[3 * t + a] = mesh.triangles[t][a];
      e.val[3 * t + a] = mesh.areas[t] / 3.0;
    }
  return e;
}

}  // namespace hmb
