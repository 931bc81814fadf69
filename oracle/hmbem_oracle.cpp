// hmbem_oracle.cpp -- CPU ORACLE (test infrastructure only).
//
// A plain-C++ restatement of the reference library's hot path
// (/root/reference/proj, "hmbem"; Bauer & Bebendorf, arXiv 2205.04752) used
// as the parity checker for the B200 implementation and as the timed CPU
// baseline ("kind": "port").  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
// The product path never links or calls it.
//
// The reference itself cannot be compiled here (Eigen3 and vendor/ are
// absent), so every function below restates the
// reference semantics with std::vector and explicit loops and cites the
// reference file:line it follows.  Compile with -O3 -DNDEBUG
// -ffp-contract=off (reference Release flags, proj/CMakeLists.txt:7-9).
//
// Parity status: pinned against the reference's own known-answer tests
// (Kelvin KAT, gauss_rule exactness, cube(9) mesh counts, cluster KATs,
// storage KAT, ACA/H-matrix/AMVM property tests) -- see tests/test_oracle_*.
// Bit-level agreement with an Eigen build is unpinned (reduction orders of
// Eigen's norm/dot/GEMV are not recoverable without Eigen).
//
// Builder-defined extension (not in the reference): the self-collocation
// term (point = centroid of its own triangle) is the exact closed-form
// integral of the Kelvin tensor over the flat triangle, see self_term().

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace oracle {

using Real = double;
using Vec3 = std::array<Real, 3>;

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// small vector helpers; norm() sums (x0^2 + x1^2) + x2^2 like Eigen's
// unrolled Vector3d redux (types.hpp:14 Vec3; used at cluster.hpp:26,
// cluster.cpp:18, kernels.cpp:22)
static inline Vec3 sub(const Vec3& a, const Vec3& b) {
  return {a[0] - b[0], a[1] - b[1], a[2] - b[2]};
}
static inline Real sqnorm(const Vec3& a) {
  return (a[0] * a[0] + a[1] * a[1]) + a[2] * a[2];
}
static inline Real norm3(const Vec3& a) { return std::sqrt(sqnorm(a)); }
static inline Real dot3(const Vec3& a, const Vec3& b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
static inline Vec3 cross3(const Vec3& a, const Vec3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2],
          a[0] * b[1] - a[1] * b[0]};
}

// ---------------------------------------------------------------------------
// parallel_for: atomic work counter over hardware_concurrency workers, first
// exception rethrown (proj/include/hmbem/parallel.hpp:12-48)
static int g_thread_cap = 0;

static void parallel_for(long n, const std::function<void(long)>& body) {
  int workers = g_thread_cap > 0
                    ? g_thread_cap
                    : static_cast<int>(std::thread::hardware_concurrency());
  if (workers < 1) workers = 1;
  if (workers == 1 || n < 2) {
    for (long i = 0; i < n; ++i) body(i);
    return;
  }
  std::atomic<long> next{0};
  std::exception_ptr error;
  std::atomic<bool> failed{false};
  auto work = [&]() {
    for (;;) {
      const long i = next.fetch_add(1);
      if (i >= n || failed.load()) return;
      try {
        body(i);
      } catch (...) {
        if (!failed.exchange(true)) error = std::current_exception();
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < workers; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  if (failed.load() && error) std::rethrow_exception(error);
}

// ---------------------------------------------------------------------------
// Quadrature (proj/src/quadrature.cpp:11-95, 97-125)
struct Rule {
  std::vector<Real> a, b, w;  // reference coordinates (l1, l2), weights
};

// orbit expansion with de-duplication over the last six points
// (quadrature.cpp:13-31)
static void add_orbit(std::vector<std::array<Real, 3>>& pts,
                      std::vector<Real>& ws, Real a, Real b, Real c, Real w) {
  const Real perms[6][3] = {{a, b, c}, {a, c, b}, {b, a, c},
                            {b, c, a}, {c, a, b}, {c, b, a}};
  for (const auto& p : perms) {
    bool seen = false;
    const std::size_t lo = pts.size() >= 6 ? pts.size() - 6 : 0;
    for (std::size_t i = lo; i < pts.size(); ++i)
      if (std::abs(pts[i][0] - p[0]) < 1e-15 &&
          std::abs(pts[i][1] - p[1]) < 1e-15) {
        seen = true;
        break;
      }
    if (!seen) {
      pts.push_back({p[0], p[1], p[2]});
      ws.push_back(w);
    }
  }
}

// barycentric (l0,l1,l2) -> reference (l1,l2), weight/2 (quadrature.cpp:33-46)
static Rule from_orbits(const std::vector<std::array<Real, 3>>& pts,
                        const std::vector<Real>& ws) {
  Rule r;
  for (std::size_t i = 0; i < pts.size(); ++i) {
    r.a.push_back(pts[i][1]);
    r.b.push_back(pts[i][2]);
    r.w.push_back(0.5 * ws[i]);
  }
  return r;
}

// symmetric triangle rules of orders 1..6 (quadrature.cpp:52-95)
static Rule gauss_rule(int order) {
  std::vector<std::array<Real, 3>> pts;
  std::vector<Real> ws;
  const Real third = 1.0 / 3.0;
  switch (order) {
    case 1:
      add_orbit(pts, ws, third, third, third, 1.0);
      break;
    case 2:
      add_orbit(pts, ws, 2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0, third);
      break;
    case 3:
    case 4:
      add_orbit(pts, ws, 0.816847572980459, 0.091576213509771,
                0.091576213509771, 0.109951743655322);
      add_orbit(pts, ws, 0.108103018168070, 0.445948490915965,
                0.445948490915965, 0.223381589678011);
      break;
    case 5: {
      const Real s15 = std::sqrt(15.0);
      add_orbit(pts, ws, third, third, third, 9.0 / 40.0);
      add_orbit(pts, ws, (9.0 - 2.0 * s15) / 21.0, (6.0 + s15) / 21.0,
                (6.0 + s15) / 21.0, (155.0 + s15) / 1200.0);
      add_orbit(pts, ws, (9.0 + 2.0 * s15) / 21.0, (6.0 - s15) / 21.0,
                (6.0 - s15) / 21.0, (155.0 - s15) / 1200.0);
      break;
    }
    case 6:
      add_orbit(pts, ws, 0.873821971016996, 0.063089014491502,
                0.063089014491502, 0.050844906370207);
      add_orbit(pts, ws, 0.501426509658179, 0.249286745170910,
                0.249286745170910, 0.116786275726379);
      add_orbit(pts, ws, 0.636502499121399, 0.310352451033785,
                0.053145049844816, 0.082851075618374);
      break;
    default:
      throw Error("gauss_rule: unsupported order " + std::to_string(order));
  }
  return from_orbits(pts, ws);
}

// Gauss-Legendre on [0,1] by Newton on P_n (quadrature.cpp:97-125)
static void gauss_legendre_01(int n, std::vector<Real>& x,
                              std::vector<Real>& w) {
  if (n < 1) throw Error("gauss_legendre_01: n must be positive");
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  const int m = (n + 1) / 2;
  for (int i = 0; i < m; ++i) {
    Real z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    Real pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      Real p0 = 1.0, p1 = 0.0;
      for (int j = 0; j < n; ++j) {
        const Real p2 = p1;
        p1 = p0;
        p0 = ((2.0 * j + 1.0) * z * p1 - j * p2) / (j + 1.0);
      }
      pp = n * (z * p0 - p1) / (z * z - 1.0);
      const Real dz = p0 / pp;
      z -= dz;
      if (std::abs(dz) < 1e-16) break;
    }
    x[i] = 0.5 * (1.0 - z);
    x[n - 1 - i] = 0.5 * (1.0 + z);
    const Real wi = 1.0 / ((1.0 - z * z) * pp * pp);
    w[i] = wi;
    w[n - 1 - i] = wi;
  }
}

// ---------------------------------------------------------------------------
// Mesh geometry caches as computed by load_mesh (proj/src/mesh.cpp:229-247)
// and triangle_diameter (mesh.cpp:105-109).
struct Mesh {
  std::vector<Vec3> vertices;
  std::vector<std::array<int, 3>> triangles;
  std::vector<Vec3> normals, centroids;
  std::vector<Real> areas, diam;

  int nt() const { return static_cast<int>(triangles.size()); }
  Vec3 corner(int t, int k) const { return vertices[triangles[t][k]]; }
};

static void finish_geometry(Mesh& m) {
  const int nt = m.nt();
  m.normals.resize(nt);
  m.centroids.resize(nt);
  m.areas.resize(nt);
  m.diam.resize(nt);
  Real scale = 0.0;
  for (const Vec3& v : m.vertices) scale = std::max(scale, norm3(v));
  for (int t = 0; t < nt; ++t) {
    const Vec3 c0 = m.corner(t, 0), c1 = m.corner(t, 1), c2 = m.corner(t, 2);
    const Vec3 n = cross3(sub(c1, c0), sub(c2, c0));
    const Real area = 0.5 * norm3(n);
    if (area <= 1e-14 * scale * scale)
      throw Error("degenerate triangle " + std::to_string(t));
    m.areas[t] = area;
    for (int d = 0; d < 3; ++d) {
      m.normals[t][d] = n[d] / (2.0 * area);
      m.centroids[t][d] = ((c0[d] + c1[d]) + c2[d]) / 3.0;
    }
    m.diam[t] = std::max({norm3(sub(c0, c1)), norm3(sub(c1, c2)),
                          norm3(sub(c0, c2))});
  }
}

// voxel_surface(n, lo, hi, inside): outward-oriented voxel boundary with two
// triangles per face, diagonal c00-c11 (proj/tools/meshgen.cpp:27-83;
// test variant proj/tests/oracles.cpp:45-98 with lo=-1, hi=1).  Restated
// here (independently of the product generator) so the product mesh can
// be checked against it.  `inside` == nullptr means the full cube.
static void voxel_surface(int n, Real lo, Real hi, Mesh& mesh) {
  auto coord = [&](int i) { return (lo * (n - i) + hi * i) / n; };
  std::map<std::array<int, 3>, int> ids;
  auto vertex = [&](int i, int j, int k) {
    const std::array<int, 3> key = {i, j, k};
    auto it = ids.find(key);
    if (it != ids.end()) return it->second;
    const int id = static_cast<int>(mesh.vertices.size());
    mesh.vertices.push_back({coord(i), coord(j), coord(k)});
    ids[key] = id;
    return id;
  };
  auto cell_inside = [&](int i, int j, int k) {
    return !(i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n);
  };
  const int tang[3][2] = {{1, 2}, {2, 0}, {0, 1}};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        const int cell[3] = {i, j, k};
        for (int d = 0; d < 3; ++d)
          for (int s = -1; s <= 1; s += 2) {
            int nb[3] = {i, j, k};
            nb[d] += s;
            if (cell_inside(nb[0], nb[1], nb[2])) continue;
            int base[3] = {cell[0], cell[1], cell[2]};
            if (s > 0) base[d] += 1;
            int du[3] = {0, 0, 0}, dv[3] = {0, 0, 0};
            du[tang[d][0]] = 1;
            dv[tang[d][1]] = 1;
            auto corner = [&](int a, int b) {
              return vertex(base[0] + a * du[0] + b * dv[0],
                            base[1] + a * du[1] + b * dv[1],
                            base[2] + a * du[2] + b * dv[2]);
            };
            const int c00 = corner(0, 0), c10 = corner(1, 0);
            const int c11 = corner(1, 1), c01 = corner(0, 1);
            if (s > 0) {
              mesh.triangles.push_back({c00, c10, c11});
              mesh.triangles.push_back({c00, c11, c01});
            } else {
              mesh.triangles.push_back({c00, c11, c10});
              mesh.triangles.push_back({c00, c01, c11});
            }
          }
      }
}

// ---------------------------------------------------------------------------
// 1/sqrt(x), x > 0: bit-level seed 0x5fe6eb50c7b537a9 - (bits(x) >> 1) and
// four Newton steps y <- y * fma(-(x/2 * y), y, 1.5).  Part of the canonical
// evaluation order shared with the device (rsqrt_canon in
// paper_2205_04752_b200/csrc/gpu/hmgpu_device.cuh): deterministic, ~1 ulp.
static inline Real rsqrt_canon(Real x) {
  long long i;
  std::memcpy(&i, &x, sizeof(i));
  i = 0x5fe6eb50c7b537a9LL - (i >> 1);
  Real y;
  std::memcpy(&y, &i, sizeof(y));
  const Real h = 0.5 * x;
  for (int it = 0; it < 4; ++it) y = y * std::fma(-(h * y), y, 1.5);
  return y;
}

// ---------------------------------------------------------------------------
// Kelvin tensor and collocation entries
struct Material {
  Real E = 1.0, nu = 0.3;
};

// (proj/src/kernels.cpp:7-14)
static void lame_constants(Real E, Real nu, Real& lambda, Real& mu) {
  if (E <= 0.0) throw Error("lame_constants: E must be positive");
  if (nu <= 0.0 || nu >= 0.5)
    throw Error("lame_constants: nu must lie in (0, 1/2)");
  lambda = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  mu = E / (2.0 * (1.0 + nu));
}

// S(x) = c[(3-4nu) delta/|x| + x x^T/|x|^3], c = (1+nu)/(8 pi E (1-nu))
// (proj/src/kernels.cpp:21-28); row-major 3x3 out
static void kelvin_tensor(const Vec3& x, const Material& m, Real* s) {
  const Real r = norm3(x);
  if (r == 0.0) throw Error("kelvin_tensor: singular point x = 0");
  const Real c = (1.0 + m.nu) / (8.0 * M_PI * m.E * (1.0 - m.nu));
  const Real d = c * (3.0 - 4.0 * m.nu) / r;
  const Real k3 = c / (r * r * r);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      s[3 * i + j] = (i == j ? d : 0.0) + k3 * (x[i] * x[j]);
}

struct Kelvin {
  const Mesh* mesh = nullptr;
  Material mat;
  Rule rules[7];  // index = order
  Kelvin(const Mesh* m, Material mt) : mesh(m), mat(mt) {
    for (int o = 1; o <= 6; ++o) rules[o] = gauss_rule(o);
  }

  // point_order with QuadratureConfig defaults disjoint_order = 4,
  // far_ratio = 4, mid_ratio = 1.5 (kernels.cpp:87-93, kernels.hpp:44-52)
  int disjoint_order = 4;
  void set_disjoint_order(int o) { disjoint_order = o; }
  int point_order(const Vec3& p, int tj) const {
    const Real dj = mesh->diam[tj];
    const Real gap = norm3(sub(p, mesh->centroids[tj])) - 0.5 * dj;
    if (gap >= 4.0 * dj) return std::min(disjoint_order, 2);
    if (gap >= 1.5 * dj) return disjoint_order;
    return std::min(disjoint_order + 1, 6);
  }

  // colloc_single: 2 area_j sum_q w_q S(p - y_q)_rc (kernels.cpp:176-187)
  // with S(x)_rc = c [(3-4nu) delta_rc / |x| + x_r x_c / |x|^3]
  // (kelvin_tensor, kernels.cpp:21-28).  Canonical evaluation order, shared
  // bit for bit with the device kernels: the constant c is factored out of
  // the quadrature sum, 1/|x| is rsqrt_canon (bit-seeded Newton, ~1 ulp),
  // and every fused multiply-add is written explicitly (std::fma); Eigen's
  // own association is not recoverable here, so this order
  // is the parity contract.  Agrees with the literal kelvin_tensor form to
  // rounding (tests/test_oracle_kats.py::test_canonical_entry_matches_literal).
  Real colloc_single(const Vec3& p, int r, int c, int tj) const {
    const Rule& rule = rules[point_order(p, tj)];
    const Vec3 y0 = mesh->corner(tj, 0), y1 = mesh->corner(tj, 1),
               y2 = mesh->corner(tj, 2);
    const Vec3 e1 = sub(y1, y0), e2 = sub(y2, y0);
    Real acc_d = 0.0, acc_x = 0.0;
    for (std::size_t q = 0; q < rule.w.size(); ++q) {
      const Real a = rule.a[q], b = rule.b[q], w = rule.w[q];
      const Real dx = p[0] - std::fma(b, e2[0], std::fma(a, e1[0], y0[0]));
      const Real dy = p[1] - std::fma(b, e2[1], std::fma(a, e1[1], y0[1]));
      const Real dz = p[2] - std::fma(b, e2[2], std::fma(a, e1[2], y0[2]));
      const Real r2 = std::fma(dz, dz, std::fma(dy, dy, dx * dx));
      const Real ri = rsqrt_canon(r2);
      const Real wr = w * ri;
      const Real d[3] = {dx, dy, dz};
      acc_d = acc_d + wr;
      acc_x = std::fma(wr * ri * ri, d[r] * d[c], acc_x);
    }
    const Real s = r == c ? std::fma(c34(), acc_d, acc_x) : acc_x;
    return 2.0 * mesh->areas[tj] * cst() * s;
  }

  // the literal reference form (kelvin_tensor per point, one component
  // kept) -- used only to check the canonical order above
  Real colloc_single_literal(const Vec3& p, int r, int c, int tj) const {
    const Rule& rule = rules[point_order(p, tj)];
    const Vec3 y0 = mesh->corner(tj, 0), y1 = mesh->corner(tj, 1),
               y2 = mesh->corner(tj, 2);
    const Vec3 e1 = sub(y1, y0), e2 = sub(y2, y0);
    Real acc = 0.0;
    Real s[9];
    for (std::size_t q = 0; q < rule.w.size(); ++q) {
      Vec3 y;
      for (int d = 0; d < 3; ++d)
        y[d] = (y0[d] + rule.a[q] * e1[d]) + rule.b[q] * e2[d];
      kelvin_tensor(sub(p, y), mat, s);
      acc += rule.w[q] * s[3 * r + c];
    }
    return 2.0 * mesh->areas[tj] * acc;
  }

  Real cst() const { return (1.0 + mat.nu) / (8.0 * M_PI * mat.E * (1.0 - mat.nu)); }
  Real c34() const { return 3.0 - 4.0 * mat.nu; }

  // BUILDER-DEFINED self term (reference undefined):
  // exact integral over triangle t of S(p - y) dA for p in the plane of t
  // (p = centroid).  Polar coordinates about p over the three sub-triangles
  // (p, a, b): per edge with in-plane outward normal m, tangent t, signed
  // height h = (a-p).m, s_i = (v_i-p).t, r_i = |v_i-p|:
  //   I1  += h ln((r2+s2)/(r1+s1))                      (= analytic potential,
  //          proj/tests/oracles.cpp:209-232 with d = 0)
  //   Irc += h [ m_r m_c dsin + (m_r t_c + t_r m_c) h (1/r1 - 1/r2)
  //              + t_r t_c (ln((r2+s2)/(r1+s1)) - dsin) ],  dsin = s2/r2-s1/r1
  //   S_self_rc = c [ (3-4nu) delta_rc I1 + Irc ]
  void self_term(const Vec3& p, int t, Real* out6) const {
    const Vec3 v[3] = {mesh->corner(t, 0), mesh->corner(t, 1),
                       mesh->corner(t, 2)};
    Vec3 nrm = cross3(sub(v[1], v[0]), sub(v[2], v[0]));
    const Real nn = norm3(nrm);
    for (int d = 0; d < 3; ++d) nrm[d] /= nn;
    Real i1 = 0.0;
    Real irc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int e = 0; e < 3; ++e) {
      const Vec3& a = v[e];
      const Vec3& b = v[(e + 1) % 3];
      Vec3 tt = sub(b, a);
      const Real len = norm3(tt);
      for (int d = 0; d < 3; ++d) tt[d] /= len;
      const Vec3 mm = cross3(tt, nrm);
      const Vec3 pa = sub(a, p), pb = sub(b, p);
      const Real h = dot3(pa, mm);
      const Real s1 = dot3(pa, tt), s2 = dot3(pb, tt);
      const Real r1 = norm3(pa), r2 = norm3(pb);
      const Real lg = std::log((r2 + s2) / (r1 + s1));
      const Real dsin = s2 / r2 - s1 / r1;
      const Real dcos = h / r1 - h / r2;
      i1 += h * lg;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          irc[r][c] += h * (mm[r] * mm[c] * dsin +
                            (mm[r] * tt[c] + tt[r] * mm[c]) * dcos +
                            tt[r] * tt[c] * (lg - dsin));
    }
    const Real cst = (1.0 + mat.nu) / (8.0 * M_PI * mat.E * (1.0 - mat.nu));
    const Real c34 = 3.0 - 4.0 * mat.nu;
    const int rr[6] = {0, 0, 0, 1, 1, 2}, cc[6] = {0, 1, 2, 1, 2, 2};
    for (int k = 0; k < 6; ++k)
      out6[k] = cst * ((rr[k] == cc[k] ? c34 * i1 : 0.0) + irc[rr[k]][cc[k]]);
  }

  // ---- double layer (colloc_double, kernels.cpp:189-210) ----------------
  // kelvin_traction (kernels.cpp:30-55) in closed form: with x = y - p,
  // n . x = nx, r = |x|:
  //   T_ij = c [ ((2mu - 2 lambda (1-2nu)) n_i x_j + mu (1-k34) n_j x_i
  //             + delta_ij mu (1-k34) nx) / r^3 - 6 mu x_i x_j nx / r^5 ]
  // Canonical order (shared with the device): rsqrt_canon, explicit fma.
  std::vector<std::vector<int>> vtri;  // vertex_triangles (mesh.cpp:245-247)
  Real lam = 0.0, mu = 0.0;
  void prepare_double() {
    lame_constants(mat.E, mat.nu, lam, mu);
    vtri.assign(mesh->vertices.size(), {});
    for (int t = 0; t < mesh->nt(); ++t)
      for (int v : mesh->triangles[t]) vtri[v].push_back(t);
  }
  Real colloc_double(const Vec3& p, int r, int c, int node) const {
    const Real b1 = 2.0 * mu - 2.0 * lam * (1.0 - 2.0 * mat.nu);
    const Real a2 = mu * (1.0 - c34());
    const Real a6 = 6.0 * mu;
    Real acc = 0.0;
    for (int tau : vtri[node]) {
      const Rule& rule = rules[point_order(p, tau)];
      int local = 0;
      while (mesh->triangles[tau][local] != node) ++local;
      const Vec3 y0 = mesh->corner(tau, 0), y1 = mesh->corner(tau, 1),
                 y2 = mesh->corner(tau, 2);
      const Vec3 e1 = sub(y1, y0), e2 = sub(y2, y0);
      const Vec3& n = mesh->normals[tau];
      Real part = 0.0;
      for (std::size_t q = 0; q < rule.w.size(); ++q) {
        const Real a = rule.a[q], b = rule.b[q];
        Real x[3];
        for (int d = 0; d < 3; ++d) x[d] = std::fma(b, e2[d], std::fma(a, e1[d], y0[d])) - p[d];
        const Real ri = rsqrt_canon(std::fma(x[2], x[2], std::fma(x[1], x[1], x[0] * x[0])));
        const Real ri2 = ri * ri, ri3 = ri2 * ri, ri5 = ri3 * ri2;
        const Real nx = std::fma(x[2], n[2], std::fma(x[1], n[1], x[0] * n[0]));
        Real sv = std::fma(b1, n[r] * x[c], a2 * (n[c] * x[r]));
        if (r == c) sv = std::fma(a2, nx, sv);
        const Real v = std::fma(-(a6 * ri5), (x[r] * x[c]) * nx, ri3 * sv);
        const Real psi = local == 0 ? (1.0 - a) - b : (local == 1 ? a : b);
        part = std::fma(rule.w[q] * psi, v, part);
      }
      acc = acc + (2.0 * mesh->areas[tau] * cst()) * part;
    }
    return acc;
  }
  // the literal reference form (kelvin_traction per point) -- checks the
  // canonical order only
  Real colloc_double_literal(const Vec3& p, int r, int c, int node) const {
    const Real cc = cst(), k34 = c34();
    Real acc = 0.0;
    for (int tau : vtri[node]) {
      const Rule& rule = rules[point_order(p, tau)];
      int local = 0;
      while (mesh->triangles[tau][local] != node) ++local;
      const Vec3 y0 = mesh->corner(tau, 0), y1 = mesh->corner(tau, 1),
                 y2 = mesh->corner(tau, 2);
      const Vec3& n = mesh->normals[tau];
      Real part = 0.0;
      for (std::size_t q = 0; q < rule.w.size(); ++q) {
        const Real b1 = rule.a[q], b2 = rule.b[q];
        Vec3 x;
        for (int d = 0; d < 3; ++d)
          x[d] = (y0[d] + b1 * (y1[d] - y0[d]) + b2 * (y2[d] - y0[d])) - p[d];
        const Real rr = norm3(x), r3 = rr * rr * rr, r5 = r3 * rr * rr;
        auto dU = [&](int k, int i, int j) {
          Real v = -k34 * (i == j ? x[k] / r3 : 0.0);
          v += ((i == k ? x[j] : 0.0) + (j == k ? x[i] : 0.0)) / r3;
          v -= 3.0 * x[i] * x[j] * x[k] / r5;
          return cc * v;
        };
        const Real div_j = -2.0 * cc * (1.0 - 2.0 * mat.nu) * x[c] / r3;
        Real t = lam * n[r] * div_j;
        for (int k = 0; k < 3; ++k) t += mu * n[k] * (dU(k, r, c) + dU(r, k, c));
        const Real psi = local == 0 ? 1.0 - b1 - b2 : local == 1 ? b1 : b2;
        part += rule.w[q] * t * psi;
      }
      acc += 2.0 * mesh->areas[tau] * part;
    }
    return acc;
  }

  // north-star entry: centroid collocation, A_rc[i,j]
  Real entry(int i, int j, int r, int c) const {
    if (i == j) {
      Real s6[6];
      self_term(mesh->centroids[i], i, s6);
      const int lo = std::min(r, c), hi = std::max(r, c);
      static const int idx[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
      return s6[idx[lo][hi]];
    }
    return colloc_single(mesh->centroids[i], r, c, j);
  }
};

// ---------------------------------------------------------------------------
// Galerkin pair quadrature (proj/src/quadrature.cpp:127-338) and the scalar
// Galerkin kernels V_Delta, V_kl (proj/src/kernels.cpp:75-149), SURVEY.md 8f
// rank 2.  PairCase numbering as quadrature.hpp:28.
// component (r,c) of the symmetric 3x3 grids, row-major upper triangle
static const int kCompR[6] = {0, 0, 0, 1, 1, 2};
static const int kCompC[6] = {0, 1, 2, 1, 2, 2};
enum PairCase { kDisjoint = 0, kVertex = 1, kEdge = 2, kIdentical = 3 };

// classify_pair (quadrature.cpp:127-156): identical, shared edge traversed
// in opposite directions, shared vertex, disjoint; rotations put the shared
// simplex first.
static int classify_pair(const std::array<int, 3>& a, const std::array<int, 3>& b,
                         int& rot_a, int& rot_b) {
  rot_a = rot_b = 0;
  if (a == b) return kIdentical;
  for (int rt = 0; rt < 3; ++rt)
    for (int rs = 0; rs < 3; ++rs)
      if (b[rs] == a[(rt + 1) % 3] && b[(rs + 1) % 3] == a[rt]) {
        rot_a = rt;
        rot_b = rs;
        return kEdge;
      }
  for (int rt = 0; rt < 3; ++rt)
    for (int rs = 0; rs < 3; ++rs)
      if (a[rt] == b[rs]) {
        rot_a = rt;
        rot_b = rs;
        return kVertex;
      }
  return kDisjoint;
}
// test_vertex_perm / trial_vertex_perm (quadrature.cpp:158-166)
static std::array<int, 3> test_vertex_perm(int rot) {
  return {rot, (rot + 1) % 3, (rot + 2) % 3};
}
static std::array<int, 3> trial_vertex_perm(int c, int rot) {
  std::array<int, 3> p = {rot, (rot + 1) % 3, (rot + 2) % 3};
  if (c == kEdge) std::swap(p[0], p[1]);
  return p;
}

struct PairRule {
  std::vector<Real> xr1, xr2, yr1, yr2, w;
};

// 32 partial sums combined by the xor butterfly (the device's warp_sum)
static Real butterfly32(const Real* p0) {
  Real p[32];
  std::copy(p0, p0 + 32, p);
  for (int o = 16; o > 0; o >>= 1) {
    Real q[32];
    for (int l = 0; l < 32; ++l) q[l] = p[l] + p[l ^ o];
    std::copy(q, q + 32, p);
  }
  return p[0];
}

// Sauter-Schwab maps [0,1]^4 -> pairs of reference coordinates
// (quadrature.cpp:177-286), same expressions and association
static void ss_map(int c, Real xi, Real e1, Real e2, Real e3, int s, Real* p) {
  Real& x1 = p[0];
  Real& x2 = p[1];
  Real& y1 = p[2];
  Real& y2 = p[3];
  Real& jac = p[4];
  if (c == kIdentical) {
    jac = xi * xi * xi * e1 * e1 * e2;
    switch (s) {
      case 0: x1 = xi * e1 * (1 - e2); x2 = xi * (1 - e1 * (1 - e2));
              y1 = xi * e1 * (1 - e2 * e3); y2 = xi * (1 - e1); break;
      case 1: x1 = xi * e1 * (1 - e2 * e3); x2 = xi * (1 - e1);
              y1 = xi * e1 * (1 - e2); y2 = xi * (1 - e1 * (1 - e2)); break;
      case 2: x1 = xi * (1 - e1 * (1 - e2 * (1 - e3))); x2 = xi * e1 * (1 - e2 * (1 - e3));
              y1 = xi * (1 - e1); y2 = xi * e1 * (1 - e2); break;
      case 3: x1 = xi * (1 - e1); x2 = xi * e1 * (1 - e2);
              y1 = xi * (1 - e1 * (1 - e2 * (1 - e3))); y2 = xi * e1 * (1 - e2 * (1 - e3)); break;
      case 4: x1 = xi * (1 - e1); x2 = xi * e1 * (1 - e2 * e3);
              y1 = xi * (1 - e1 * (1 - e2)); y2 = xi * e1 * (1 - e2); break;
      default: x1 = xi * (1 - e1 * (1 - e2)); x2 = xi * e1 * (1 - e2);
               y1 = xi * (1 - e1); y2 = xi * e1 * (1 - e2 * e3); break;
    }
  } else if (c == kEdge) {
    jac = xi * xi * xi * e1 * e1;
    switch (s) {
      case 0: x1 = xi * (1 - e1 * e3); x2 = xi * e1 * e3;
              y1 = xi * (1 - e1); y2 = xi * e1 * (1 - e2); break;
      case 1: x1 = xi * (1 - e1); x2 = xi * e1;
              y1 = xi * (1 - e1 * e2); y2 = xi * e1 * e2 * (1 - e3); jac *= e2; break;
      case 2: x1 = xi * (1 - e1); x2 = xi * e1 * (1 - e2);
              y1 = xi * (1 - e1 * e2 * e3); y2 = xi * e1 * e2 * e3; jac *= e2; break;
      case 3: x1 = xi * (1 - e1 * e2); x2 = xi * e1 * e2 * (1 - e3);
              y1 = xi * (1 - e1); y2 = xi * e1; jac *= e2; break;
      default: x1 = xi * (1 - e1); x2 = xi * e1 * (1 - e2 * e3);
               y1 = xi * (1 - e1 * e2); y2 = xi * e1 * e2; jac *= e2; break;
    }
  } else {
    jac = xi * xi * xi * e2;
    if (s == 0) {
      x1 = xi * (1 - e1); x2 = xi * e1; y1 = xi * e2 * (1 - e3); y2 = xi * e2 * e3;
    } else {
      x1 = xi * e2 * (1 - e3); x2 = xi * e2 * e3; y1 = xi * (1 - e1); y2 = xi * e1;
    }
  }
}

// build_pair_rule (quadrature.cpp:290-336): disjoint = tensor product of
// two triangle rules (test point outer); singular = simplices x n^4
// Gauss-Legendre with the weight jac * w0 * w1 * w2 * w3 (left to right)
static PairRule build_pair_rule(int c, int order) {
  PairRule r;
  if (c == kDisjoint) {
    const Rule t = gauss_rule(order);
    const size_t n = t.w.size();
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < n; ++j) {
        r.xr1.push_back(t.a[i]);
        r.xr2.push_back(t.b[i]);
        r.yr1.push_back(t.a[j]);
        r.yr2.push_back(t.b[j]);
        r.w.push_back(t.w[i] * t.w[j]);
      }
    return r;
  }
  const int ns = c == kIdentical ? 6 : c == kEdge ? 5 : 2;
  std::vector<Real> gx, gw;
  gauss_legendre_01(order, gx, gw);
  const int n = order;
  Real p[5];
  for (int s = 0; s < ns; ++s)
    for (int i0 = 0; i0 < n; ++i0)
      for (int i1 = 0; i1 < n; ++i1)
        for (int i2 = 0; i2 < n; ++i2)
          for (int i3 = 0; i3 < n; ++i3) {
            ss_map(c, gx[i0], gx[i1], gx[i2], gx[i3], s, p);
            r.xr1.push_back(p[0]);
            r.xr2.push_back(p[1]);
            r.yr1.push_back(p[2]);
            r.yr2.push_back(p[3]);
            r.w.push_back(p[4] * gw[i0] * gw[i1] * gw[i2] * gw[i3]);
          }
  return r;
}

// Galerkin V_Delta / V_kl entries with QuadratureConfig defaults
// (kernels.hpp:44-52: disjoint_order 4, singular_order 7, identical_bump 2,
// far 4, mid 1.5, near 0.75).  Canonical evaluation order (parity contract
// with the device, as for colloc_single): points by explicit fma from the
// rotated corners, 1/|x-y| by rsqrt_canon, 1/(4 pi) and 4 area_i area_j
// factored out of the pair sum.
//   comp 0..5: V_kl for (k,l) = kCompR/kCompC (V_lk aliases V_kl,
//              operators.cpp:226-233); comp 6: V_Delta
struct Galerkin {
  const Mesh* mesh = nullptr;
  PairRule disjoint[7];  // by triangle-rule order (2, 4, 5 used)
  PairRule singular[4];  // by PairCase (orders 7, 7, 9)
  explicit Galerkin(const Mesh* m) : mesh(m) {
    for (int o : {2, 4, 5}) disjoint[o] = build_pair_rule(kDisjoint, o);
    singular[kVertex] = build_pair_rule(kVertex, 7);
    singular[kEdge] = build_pair_rule(kEdge, 7);
    singular[kIdentical] = build_pair_rule(kIdentical, 9);
  }

  // disjoint_order (kernels.cpp:75-85)
  int disjoint_order(int ti, int tj) const {
    const Real di = mesh->diam[ti], dj = mesh->diam[tj];
    const Real dmax = std::max(di, dj);
    const Real gap = norm3(sub(mesh->centroids[ti], mesh->centroids[tj])) - 0.5 * (di + dj);
    if (gap >= 4.0 * dmax) return 2;
    if (gap >= 1.5 * dmax) return 4;
    if (gap >= 0.75 * dmax) return 4;
    return 5;
  }

  const PairRule& rule_for(int ti, int tj, int& pc, int& rt, int& rs) const {
    pc = classify_pair(mesh->triangles[ti], mesh->triangles[tj], rt, rs);
    return pc == kDisjoint ? disjoint[disjoint_order(ti, tj)] : singular[pc];
  }

  // all seven components of one pair (integrate_pair, kernels.cpp:95-128):
  // out7[0..5] = V_kl, out7[6] = V_Delta
  void entry7(int i, int j, Real* out7) const {
    if (i > j) std::swap(i, j);  // kernels.cpp:132-133, 141 (exact symmetry)
    int pc, rt, rs;
    const PairRule& r = rule_for(i, j, pc, rt, rs);
    const auto xp = test_vertex_perm(rt);
    const auto yp = trial_vertex_perm(pc, rs);
    const Vec3 x0 = mesh->corner(i, xp[0]), x1 = mesh->corner(i, xp[1]),
               x2 = mesh->corner(i, xp[2]);
    const Vec3 y0 = mesh->corner(j, yp[0]), y1 = mesh->corner(j, yp[1]),
               y2 = mesh->corner(j, yp[2]);
    const Vec3 ex1 = sub(x1, x0), ex2 = sub(x2, x0), ey1 = sub(y1, y0), ey2 = sub(y2, y0);
    // disjoint pairs: one sequential sum in rule order; touching pairs (the
    // Sauter-Schwab tables, up to 39366 points): warp order, i.e. 32
    // lane-strided partial sums (point q into partial q % 32, in order)
    // combined by the xor butterfly, so that a warp shares one pair
    const int nl = pc == kDisjoint ? 1 : 32;
    Real ad[32] = {0}, akl[32][6] = {{0}};
    for (size_t q = 0; q < r.w.size(); ++q) {
      const int l = static_cast<int>(q % nl);
      const Real a1 = r.xr1[q], a2 = r.xr2[q], b1 = r.yr1[q], b2 = r.yr2[q];
      Real d[3];
      for (int c = 0; c < 3; ++c)
        d[c] = std::fma(a2, ex2[c], std::fma(a1, ex1[c], x0[c])) -
               std::fma(b2, ey2[c], std::fma(b1, ey1[c], y0[c]));
      const Real ri = rsqrt_canon(std::fma(d[2], d[2], std::fma(d[1], d[1], d[0] * d[0])));
      const Real wr = r.w[q] * ri;
      const Real w3 = wr * ri * ri;
      ad[l] = ad[l] + wr;
      for (int k = 0; k < 6; ++k)
        akl[l][k] = std::fma(w3, d[kCompR[k]] * d[kCompC[k]], akl[l][k]);
    }
    if (nl == 32) {
      Real t[32];
      ad[0] = butterfly32(ad);
      for (int k = 0; k < 6; ++k) {
        for (int l = 0; l < 32; ++l) t[l] = akl[l][k];
        akl[0][k] = butterfly32(t);
      }
    }
    const Real f = 4.0 * mesh->areas[i] * mesh->areas[j] * (1.0 / (4.0 * M_PI));
    for (int k = 0; k < 6; ++k) out7[k] = f * akl[0][k];
    out7[6] = f * ad[0];
  }
  Real entry(int i, int j, int comp) const {
    Real o[7];
    entry7(i, j, o);
    return o[comp];
  }

  // K_Delta(i, node) = sum over the triangles tau of the node (ascending ids,
  // load_mesh's vertex_triangles, mesh.cpp:245-247), tau != i, of
  // integrate_pair(i, tau) of (x-y).n(tau) / (4 pi |x-y|^3) psi_node(y)
  // (kernels.cpp:151-167; no orientation swap).  Canonical order: per pair
  // sum_q fma(w / r^3, ((x-y).n) * bary_local, .) (warp order for touching
  // pairs, as entry7), the 4 area area / (4 pi) scale per pair, pairs summed
  // in tau order.
  std::vector<std::vector<int>> vtri;
  void build_vtri() {
    vtri.assign(mesh->vertices.size(), {});
    for (int t = 0; t < mesh->nt(); ++t)
      for (int v : mesh->triangles[t]) vtri[v].push_back(t);
  }
  Real kdelta(int i, int node) const {
    Real total = 0.0;
    for (int tau : vtri[node]) {
      if (tau == i) continue;
      int local = 0;
      while (mesh->triangles[tau][local] != node) ++local;
      const Vec3& nrm = mesh->normals[tau];
      int pc, rt, rs;
      const PairRule& r = rule_for(i, tau, pc, rt, rs);
      const auto xp = test_vertex_perm(rt);
      const auto yp = trial_vertex_perm(pc, rs);
      const Vec3 x0 = mesh->corner(i, xp[0]), x1 = mesh->corner(i, xp[1]),
                 x2 = mesh->corner(i, xp[2]);
      const Vec3 y0 = mesh->corner(tau, yp[0]), y1 = mesh->corner(tau, yp[1]),
                 y2 = mesh->corner(tau, yp[2]);
      const Vec3 ex1 = sub(x1, x0), ex2 = sub(x2, x0), ey1 = sub(y1, y0), ey2 = sub(y2, y0);
      const int nl = pc == kDisjoint ? 1 : 32;  // warp order for touching pairs
      Real part[32] = {0};
      for (size_t q = 0; q < r.w.size(); ++q) {
        const Real a1 = r.xr1[q], a2 = r.xr2[q], b1 = r.yr1[q], b2 = r.yr2[q];
        Real d[3];
        for (int c = 0; c < 3; ++c)
          d[c] = std::fma(a2, ex2[c], std::fma(a1, ex1[c], x0[c])) -
                 std::fma(b2, ey2[c], std::fma(b1, ey1[c], y0[c]));
        const Real ri = rsqrt_canon(std::fma(d[2], d[2], std::fma(d[1], d[1], d[0] * d[0])));
        const Real w3 = r.w[q] * ri * ri * ri;
        const Real dn = std::fma(d[2], nrm[2], std::fma(d[1], nrm[1], d[0] * nrm[0]));
        // barycentric of y w.r.t. the original vertex order (kernels.cpp:119-123)
        const Real bv = local == yp[0] ? (1.0 - b1) - b2 : local == yp[1] ? b1 : b2;
        const int l = static_cast<int>(q % nl);
        part[l] = std::fma(w3, dn * bv, part[l]);
      }
      const Real acc = nl == 32 ? butterfly32(part) : part[0];
      total += 4.0 * mesh->areas[i] * mesh->areas[tau] * (1.0 / (4.0 * M_PI)) * acc;
    }
    return total;
  }
  // literal form (kernels.cpp:151-167 with integrate_pair's loop)
  Real kdelta_literal(int i, int node) const {
    Real total = 0.0;
    for (int tau : vtri[node]) {
      if (tau == i) continue;
      int local = 0;
      while (mesh->triangles[tau][local] != node) ++local;
      int pc, rt, rs;
      const PairRule& r = rule_for(i, tau, pc, rt, rs);
      const auto xp = test_vertex_perm(rt);
      const auto yp = trial_vertex_perm(pc, rs);
      Vec3 X[3], Y[3];
      for (int v = 0; v < 3; ++v) {
        X[v] = mesh->corner(i, xp[v]);
        Y[v] = mesh->corner(tau, yp[v]);
      }
      Real acc = 0.0;
      for (size_t q = 0; q < r.w.size(); ++q) {
        Vec3 x, y;
        for (int c = 0; c < 3; ++c) {
          x[c] = X[0][c] + r.xr1[q] * (X[1][c] - X[0][c]) + r.xr2[q] * (X[2][c] - X[0][c]);
          y[c] = Y[0][c] + r.yr1[q] * (Y[1][c] - Y[0][c]) + r.yr2[q] * (Y[2][c] - Y[0][c]);
        }
        Real bary[3];
        bary[yp[0]] = 1.0 - r.yr1[q] - r.yr2[q];
        bary[yp[1]] = r.yr1[q];
        bary[yp[2]] = r.yr2[q];
        const Vec3 d = sub(x, y);
        const Real rr = norm3(d);
        acc += r.w[q] * (dot3(d, mesh->normals[tau]) / (4.0 * M_PI * rr * rr * rr) * bary[local]);
      }
      total += 4.0 * mesh->areas[i] * mesh->areas[tau] * acc;
    }
    return total;
  }
  // the literal form of integrate_pair with the reference's integrand
  // (acc += w f(x, y), 4 area area acc) -- checks the canonical order only
  Real entry_literal(int i, int j, int comp) const {
    if (i > j) std::swap(i, j);
    int pc, rt, rs;
    const PairRule& r = rule_for(i, j, pc, rt, rs);
    const auto xp = test_vertex_perm(rt);
    const auto yp = trial_vertex_perm(pc, rs);
    Vec3 X[3], Y[3];
    for (int v = 0; v < 3; ++v) {
      X[v] = mesh->corner(i, xp[v]);
      Y[v] = mesh->corner(j, yp[v]);
    }
    Real acc = 0.0;
    for (size_t q = 0; q < r.w.size(); ++q) {
      Vec3 x, y;
      for (int c = 0; c < 3; ++c) {
        x[c] = X[0][c] + r.xr1[q] * (X[1][c] - X[0][c]) + r.xr2[q] * (X[2][c] - X[0][c]);
        y[c] = Y[0][c] + r.yr1[q] * (Y[1][c] - Y[0][c]) + r.yr2[q] * (Y[2][c] - Y[0][c]);
      }
      const Vec3 d = sub(x, y);
      const Real rr = norm3(d);
      const Real f = comp == 6 ? 1.0 / (4.0 * M_PI * rr)
                               : d[kCompR[comp]] * d[kCompC[comp]] / (4.0 * M_PI * rr * rr * rr);
      acc += r.w[q] * f;
    }
    return 4.0 * mesh->areas[i] * mesh->areas[j] * acc;
  }
};

// ---------------------------------------------------------------------------
// Entry oracles (proj/include/hmbem/aca.hpp:15-44)
struct EntryOracle {
  virtual ~EntryOracle() = default;
  virtual long rows() const = 0;
  virtual long cols() const = 0;
  virtual Real entry(long i, long j) const = 0;
  // entries evaluated through row()/col() (ACA rows, columns, dense fill)
  mutable std::atomic<long> evaluated{0};
  void row(long i, const int* col_ids, long n, Real* out) const {
    for (long k = 0; k < n; ++k) out[k] = entry(i, col_ids[k]);
    evaluated += n;
  }
  void col(long j, const int* row_ids, long m, Real* out) const {
    for (long k = 0; k < m; ++k) out[k] = entry(row_ids[k], j);
    evaluated += m;
  }
};

struct DenseOracle : EntryOracle {  // column-major m x n (aca.hpp:34-44)
  long m, n;
  std::vector<Real> a;
  long rows() const override { return m; }
  long cols() const override { return n; }
  Real entry(long i, long j) const override { return a[j * m + i]; }
};

// CollocSingleOracle(r, c) with evaluation points = triangle centroids
// (kernels.hpp:107-126)
struct KelvinComponentOracle : EntryOracle {
  const Kelvin* k;
  int r, c;
  long rows() const override { return k->mesh->nt(); }
  long cols() const override { return k->mesh->nt(); }
  Real entry(long i, long j) const override {
    return k->entry(static_cast<int>(i), static_cast<int>(j), r, c);
  }
};

// KernelOracle over V_kl (comp 0..5) or V_Delta (comp 6) (kernels.hpp:95-105)
struct GalerkinComponentOracle : EntryOracle {
  const Galerkin* g;
  int comp;
  long rows() const override { return g->mesh->nt(); }
  long cols() const override { return g->mesh->nt(); }
  Real entry(long i, long j) const override {
    return g->entry(static_cast<int>(i), static_cast<int>(j), comp);
  }
};

// KernelOracle over K_Delta: triangles x nodes (kernels.hpp:95-105, 120)
struct KDeltaOracle : EntryOracle {
  const Galerkin* g;
  long rows() const override { return g->mesh->nt(); }
  long cols() const override { return static_cast<long>(g->mesh->vertices.size()); }
  Real entry(long i, long j) const override {
    return g->kdelta(static_cast<int>(i), static_cast<int>(j));
  }
};

// CollocSingleOracle(r, c) at arbitrary evaluation points (kernels.hpp:107-126
// as evaluate_interior uses it, baca.cpp:657-668)
struct KelvinPointOracle : EntryOracle {
  const Kelvin* k;
  const std::vector<Vec3>* pts;
  int r, c;
  long rows() const override { return static_cast<long>(pts->size()); }
  long cols() const override { return k->mesh->nt(); }
  Real entry(long i, long j) const override {
    return k->colloc_single((*pts)[i], r, c, static_cast<int>(j));
  }
};

// CollocDoubleOracle(r, c) at arbitrary points (kernels.hpp:128-147):
// points x nodes
struct KelvinDoubleOracle : EntryOracle {
  const Kelvin* k;
  const std::vector<Vec3>* pts;
  int r, c;
  long rows() const override { return static_cast<long>(pts->size()); }
  long cols() const override { return static_cast<long>(k->mesh->vertices.size()); }
  Real entry(long i, long j) const override {
    return k->colloc_double((*pts)[i], r, c, static_cast<int>(j));
  }
};

// Newton kernel over points with a bounded diagonal: CentroidKernelOracle /
// PointKernelOracle fixtures (proj/tests/test_hmatrix.cpp:12-28,
// proj/tests/test_amvm.cpp:9-22)
struct NewtonOracle : EntryOracle {
  std::vector<Vec3> pts;
  Real diag = 2.0;
  long rows() const override { return static_cast<long>(pts.size()); }
  long cols() const override { return static_cast<long>(pts.size()); }
  Real entry(long i, long j) const override {
    const Real r = norm3(sub(pts[i], pts[j]));
    return r == 0.0 ? diag : 1.0 / r;
  }
};

// ---------------------------------------------------------------------------
// Clustering (proj/include/hmbem/cluster.hpp:13-99, proj/src/cluster.cpp)
struct Box {
  Vec3 lo = {std::numeric_limits<Real>::max(), std::numeric_limits<Real>::max(),
             std::numeric_limits<Real>::max()};
  Vec3 hi = {std::numeric_limits<Real>::lowest(),
             std::numeric_limits<Real>::lowest(),
             std::numeric_limits<Real>::lowest()};
  void absorb(const Box& o) {
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], o.lo[d]);
      hi[d] = std::max(hi[d], o.hi[d]);
    }
  }
  void absorb(const Vec3& p) {
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], p[d]);
      hi[d] = std::max(hi[d], p[d]);
    }
  }
  Real mid(int d) const { return 0.5 * (lo[d] + hi[d]); }
  Real diameter() const { return norm3(sub(hi, lo)); }
};

// (cluster.cpp:12-24)
static Real box_distance(const Box& a, const Box& b) {
  Vec3 gap = {0, 0, 0};
  for (int d = 0; d < 3; ++d) {
    const Real g = std::max(a.lo[d] - b.hi[d], b.lo[d] - a.hi[d]);
    gap[d] = std::max(g, 0.0);
  }
  return norm3(gap);
}

static bool admissible(const Box& t, const Box& s, Real eta) {
  if (eta <= 0.0) throw Error("admissible: beta must be positive");
  return std::min(t.diameter(), s.diameter()) < eta * box_distance(t, s);
}

struct Node {
  int begin = 0, end = 0;
  Box box;
  int child[2] = {-1, -1};
  int level = 0;
  int size() const { return end - begin; }
  bool leaf() const { return child[0] < 0; }
};

struct Tree {
  std::vector<Node> nodes;
  std::vector<int> perm, inv_perm;
  int b_min = 1, depth = 0;
  int size() const { return static_cast<int>(perm.size()); }
};

// geometric bisection: longest axis (first max), stable sort by support
// midpoint, lower half takes the extra element (cluster.cpp:28-78)
static int tree_build(const std::vector<Box>& sup, Tree& tree, int begin,
                      int end, int level) {
  const int id = static_cast<int>(tree.nodes.size());
  tree.nodes.emplace_back();
  tree.nodes[id].begin = begin;
  tree.nodes[id].end = end;
  tree.nodes[id].level = level;
  tree.depth = std::max(tree.depth, level);
  Box box;
  for (int p = begin; p < end; ++p) box.absorb(sup[tree.perm[p]]);
  tree.nodes[id].box = box;
  if (end - begin <= tree.b_min) return id;
  int axis = 0;
  Real best = box.hi[0] - box.lo[0];
  for (int d = 1; d < 3; ++d)
    if (box.hi[d] - box.lo[d] > best) {
      best = box.hi[d] - box.lo[d];
      axis = d;
    }
  std::stable_sort(tree.perm.begin() + begin, tree.perm.begin() + end,
                   [&](int a, int b) {
                     return sup[a].mid(axis) < sup[b].mid(axis);
                   });
  const int mid = begin + (end - begin + 1) / 2;
  const int left = tree_build(sup, tree, begin, mid, level + 1);
  const int right = tree_build(sup, tree, mid, end, level + 1);
  tree.nodes[id].child[0] = left;
  tree.nodes[id].child[1] = right;
  return id;
}

static Tree build_cluster_tree(const std::vector<Box>& sup, int b_min) {
  if (sup.empty()) throw Error("build_cluster_tree: empty support set");
  if (b_min < 1) throw Error("build_cluster_tree: b_min must be >= 1");
  Tree tree;
  tree.b_min = b_min;
  tree.perm.resize(sup.size());
  std::iota(tree.perm.begin(), tree.perm.end(), 0);
  tree_build(sup, tree, 0, static_cast<int>(sup.size()), 0);
  tree.inv_perm.resize(sup.size());
  for (std::size_t p = 0; p < tree.perm.size(); ++p)
    tree.inv_perm[tree.perm[p]] = static_cast<int>(p);
  return tree;
}

struct Block {
  int row_node = 0, col_node = 0;
  bool admissible = false;
  int level = 0;
};

struct Partition {
  const Tree* rows = nullptr;
  const Tree* cols = nullptr;
  std::vector<Block> blocks;
  Real eta = 0.0;
  int depth() const { return std::max(rows->depth, cols->depth); }
};

// admissibility-first quad-tree recursion (cluster.cpp:82-116)
static void subdivide(const Tree& rows, const Tree& cols, int t, int s,
                      int level, Real eta, std::vector<Block>& out) {
  const Node& rn = rows.nodes[t];
  const Node& cn = cols.nodes[s];
  if (admissible(rn.box, cn.box, eta)) {
    out.push_back({t, s, true, level});
    return;
  }
  if (rn.leaf() || cn.leaf()) {
    out.push_back({t, s, false, level});
    return;
  }
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      subdivide(rows, cols, rn.child[a], cn.child[b], level + 1, eta, out);
}

static Partition build_block_partition(const Tree* rows, const Tree* cols,
                                       Real eta) {
  Partition p;
  p.rows = rows;
  p.cols = cols;
  p.eta = eta;
  subdivide(*rows, *cols, 0, 0, 0, eta, p.blocks);
  return p;
}

// (cluster.cpp:118-128)
static int sparsity_constant(const Partition& p) {
  std::map<int, int> rc, cc;
  for (const auto& b : p.blocks) {
    ++rc[b.row_node];
    ++cc[b.col_node];
  }
  int c_sp = 0;
  for (const auto& kv : rc) c_sp = std::max(c_sp, kv.second);
  for (const auto& kv : cc) c_sp = std::max(c_sp, kv.second);
  return c_sp;
}

// nlohmann::json::dump(2) layout of partition_to_json (cluster.cpp:130-148):
// object keys in lexicographic order, shortest round-trip doubles.
static std::string fmt_double(Real v) {
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

static std::string partition_to_json(const Partition& p) {
  std::string o = "{\n";
  o += "  \"beta\": " + fmt_double(p.eta) + ",\n";
  o += "  \"blocks\": [";
  for (std::size_t i = 0; i < p.blocks.size(); ++i) {
    const Block& b = p.blocks[i];
    o += i ? ",\n" : "\n";
    o += "    {\n";
    o += std::string("      \"admissible\": ") +
         (b.admissible ? "true" : "false") + ",\n";
    o += "      \"col_node\": " + std::to_string(b.col_node) + ",\n";
    o += "      \"cols\": " + std::to_string(p.cols->nodes[b.col_node].size()) +
         ",\n";
    o += "      \"level\": " + std::to_string(b.level) + ",\n";
    o += "      \"row_node\": " + std::to_string(b.row_node) + ",\n";
    o += "      \"rows\": " + std::to_string(p.rows->nodes[b.row_node].size()) +
         "\n";
    o += "    }";
  }
  o += p.blocks.empty() ? "]" : "\n  ]";
  o += ",\n  \"c_sp\": " + std::to_string(sparsity_constant(p)) + ",\n";
  o += "  \"cols\": " + std::to_string(p.cols->size()) + ",\n";
  o += "  \"depth\": " + std::to_string(p.depth()) + ",\n";
  o += "  \"rows\": " + std::to_string(p.rows->size()) + "\n}";
  return o;
}

// ---------------------------------------------------------------------------
// ACA with partial pivoting (proj/include/hmbem/aca.hpp:47-117,
// proj/src/aca.cpp:7-150)
enum AcaStop { STOP_NONE = 0, STOP_INEQ = 1, STOP_EXHAUSTED = 2,
               STOP_RANKCAP = 3, STOP_STEPS = 4 };

struct BlockView {
  const EntryOracle* oracle = nullptr;
  const int* row_ids = nullptr;
  const int* col_ids = nullptr;
  long m = 0, n = 0;
};

// resumable state: U (m x k) and V (n x k) column-major, pivots, consumed
// mask Z, running Frobenius norm (aca.hpp:76-94)
struct Factor {
  long m = 0, n = 0;
  std::vector<Real> U, V;
  std::vector<std::pair<int, int>> pivots;
  std::vector<char> consumed;
  int num_consumed = 0;
  Real frob_sq = 0.0;
  int last_stop = STOP_NONE;
  int rank() const { return static_cast<int>(pivots.size()); }
  bool exhausted() const { return num_consumed == static_cast<int>(m); }
  Real frob() const { return std::sqrt(std::max(frob_sq, 0.0)); }
  const Real* Ucol(int l) const { return U.data() + static_cast<long>(l) * m; }
  const Real* Vcol(int l) const { return V.data() + static_cast<long>(l) * n; }
  // S x over pivot range [k_lo, k_hi): U_r (V_r^T x) (aca.cpp:7-11)
  // tail products in the device order (z_l by warp_dot, y += U(:,l) z_l
  // with fma), the parity contract of gamma_contributions
  void apply_range_device_order(int k_lo, int k_hi, const Real* x, Real* y) const;

  void apply_range(int k_lo, int k_hi, const Real* x, Real* y_add,
                   Real coeff = 1.0) const {
    if (k_hi <= k_lo) return;
    std::vector<Real> z(k_hi - k_lo, 0.0);
    for (int l = k_lo; l < k_hi; ++l) {
      Real s = 0.0;
      const Real* v = Vcol(l);
      for (long j = 0; j < n; ++j) s += v[j] * x[j];
      z[l - k_lo] = s;
    }
    for (int l = k_lo; l < k_hi; ++l) {
      const Real* u = Ucol(l);
      const Real zl = coeff * z[l - k_lo];
      for (long i = 0; i < m; ++i) y_add[i] += u[i] * zl;
    }
  }
};

template <class A, class B>
static Real warp_dot(long n, A a, B b);

void Factor::apply_range_device_order(int k_lo, int k_hi, const Real* x,
                                      Real* y) const {
  for (int l = k_lo; l < k_hi; ++l) {
    const Real* v = Vcol(l);
    const Real* u = Ucol(l);
    const Real z = warp_dot(n, [&](long j) { return v[j]; }, [&](long j) { return x[j]; });
    for (long i = 0; i < m; ++i) y[i] = std::fma(u[i], z, y[i]);
  }
}

static Factor empty_factor(long m, long n) {
  Factor f;
  f.m = m;
  f.n = n;
  f.consumed.assign(static_cast<std::size_t>(m), 0);
  return f;
}

static Real vnorm(const std::vector<Real>& v) {
  Real s = 0.0;
  for (Real x : v) s += x * x;
  return std::sqrt(s);
}

// Sum of a_j * b_j in the device's warp order: 32 lane-strided partial sums
// accumulated with fma, combined by an xor butterfly.  This is the parity
// contract for every reduction inside the ACA (the reference's Eigen
// reduction order is unpinned).
template <class A, class B>
static Real warp_dot(long n, A a, B b) {
  Real p[32] = {0};
  for (long j = 0; j < n; ++j) p[j & 31] = std::fma(a(j), b(j), p[j & 31]);
  for (int o = 16; o > 0; o >>= 1) {
    Real q[32];
    for (int l = 0; l < 32; ++l) q[l] = p[l] + p[l ^ o];
    std::copy(q, q + 32, p);
  }
  return p[0];
}

// one ACA step (aca.cpp:41-102); stop_factor < 0 disables the accuracy test
static int aca_step(Factor& f, const BlockView& blk, Real stop_factor) {
  const long m = blk.m, n = blk.n;
  std::vector<Real> v(n), u(m);
  for (;;) {
    if (f.exhausted()) return STOP_EXHAUSTED;
    int i = -1;
    if (f.rank() == 0) {
      for (long r = 0; r < m; ++r)
        if (!f.consumed[r]) {
          i = static_cast<int>(r);
          break;
        }
    } else {
      Real best = -1.0;
      const Real* ul = f.Ucol(f.rank() - 1);
      for (long r = 0; r < m; ++r) {
        if (f.consumed[r]) continue;
        const Real mag = std::abs(ul[r]);
        if (mag > best) {
          best = mag;
          i = static_cast<int>(r);
        }
      }
    }
    blk.oracle->row(blk.row_ids[i], blk.col_ids, n, v.data());
    Real row_scale = 0.0;
    for (long c = 0; c < n; ++c) row_scale = std::max(row_scale, std::abs(v[c]));
    for (long c = 0; c < n; ++c)  // v -= U(i,l) V(:,l), l ascending
      for (int l = 0; l < f.rank(); ++l)
        v[c] = std::fma(-f.Ucol(l)[i], f.Vcol(l)[c], v[c]);
    f.consumed[i] = 1;
    ++f.num_consumed;
    int j = 0;
    Real pivot_mag = n > 0 ? std::abs(v[0]) : 0.0;
    for (long c = 1; c < n; ++c)
      if (std::abs(v[c]) > pivot_mag) {
        pivot_mag = std::abs(v[c]);
        j = static_cast<int>(c);
      }
    if (pivot_mag <= 1e-14 * row_scale || row_scale == 0.0) continue;
    const Real piv = v[j];
    for (long c = 0; c < n; ++c) v[c] /= piv;
    blk.oracle->col(blk.col_ids[j], blk.row_ids, m, u.data());
    for (long r = 0; r < m; ++r)  // u -= V(j,l) U(:,l), l ascending
      for (int l = 0; l < f.rank(); ++l)
        u[r] = std::fma(-f.Vcol(l)[j], f.Ucol(l)[r], u[r]);
    const Real uu = warp_dot(m, [&](long r) { return u[r]; }, [&](long r) { return u[r]; });
    const Real vv = warp_dot(n, [&](long c) { return v[c]; }, [&](long c) { return v[c]; });
    if (stop_factor >= 0.0 &&
        std::sqrt(uu) * std::sqrt(vv) <= stop_factor * f.frob())
      return STOP_INEQ;
    // ||S_k||^2 = ||S_{k-1}||^2 + 2 sum_l (u.u_l)(v.v_l) + ||u||^2 ||v||^2
    Real cross = 0.0;
    for (int l = 0; l < f.rank(); ++l) {
      const Real* ul = f.Ucol(l);
      const Real* vl = f.Vcol(l);
      const Real du = warp_dot(m, [&](long r) { return u[r]; }, [&](long r) { return ul[r]; });
      const Real dv = warp_dot(n, [&](long c) { return v[c]; }, [&](long c) { return vl[c]; });
      cross = std::fma(du, dv, cross);
    }
    f.frob_sq += 2.0 * cross + uu * vv;
    f.U.insert(f.U.end(), u.begin(), u.end());
    f.V.insert(f.V.end(), v.begin(), v.end());
    f.pivots.emplace_back(i, j);
    return STOP_NONE;
  }
}

// (aca.cpp:106-124)
static Factor aca_run(const BlockView& blk, Real eps, Real beta, long max_rank,
                      const Factor* start = nullptr) {
  if (eps <= 0.0) throw Error("aca_run: eps must be positive");
  if (beta <= 0.0 || beta >= 1.0) throw Error("aca_run: beta must be in (0,1)");
  const long cap = std::min(max_rank, std::min(blk.m, blk.n));
  Factor f = start ? *start : empty_factor(blk.m, blk.n);
  const Real stop_factor = eps * (1.0 - beta) / (1.0 + eps);
  while (f.rank() < cap) {
    const int s = aca_step(f, blk, stop_factor);
    if (s != STOP_NONE) {
      f.last_stop = s;
      return f;
    }
  }
  f.last_stop = f.exhausted() ? STOP_EXHAUSTED : STOP_RANKCAP;
  return f;
}

// (aca.cpp:126-143)
static Factor aca_extend(Factor f, int steps, const BlockView& blk,
                         long max_rank) {
  const long cap = std::min(max_rank, std::min(blk.m, blk.n));
  int done = 0;
  while (done < steps && f.rank() < cap) {
    const int s = aca_step(f, blk, -1.0);
    if (s != STOP_NONE) {
      f.last_stop = s;
      return f;
    }
    ++done;
  }
  f.last_stop = f.exhausted()                    ? STOP_EXHAUSTED
                : f.rank() >= cap && done < steps ? STOP_RANKCAP
                                                  : STOP_STEPS;
  return f;
}

// ---------------------------------------------------------------------------
// H-matrix (proj/include/hmbem/hmatrix.hpp, proj/src/hmatrix.cpp)
struct AssemblyConfig {
  Real eps = 1e-6, beta = 0.8;
  int initial_rank = -1, lookahead = 2;
  long max_rank = 1L << 30;
};

struct HBlock {
  Factor factor;
  int current_rank = 0;
  std::vector<Real> dense;  // column-major m x n; empty => low rank
  bool lowrank() const { return dense.empty(); }
};

struct HMatrix {
  const Partition* part = nullptr;
  const EntryOracle* oracle = nullptr;
  AssemblyConfig cfg;
  std::vector<HBlock> blocks;
  long total_pivots = 0;
  long entries = 0;  // kernel entries evaluated (ACA rows/cols + dense)

  BlockView view(int b) const {
    const Block& blk = part->blocks[b];
    const Node& rn = part->rows->nodes[blk.row_node];
    const Node& cn = part->cols->nodes[blk.col_node];
    return {oracle, part->rows->perm.data() + rn.begin,
            part->cols->perm.data() + cn.begin, rn.size(), cn.size()};
  }

  // serial matvec with permutation gather/scatter (hmatrix.cpp:22-45)
  void matvec(const Real* x, Real* y, int mode) const {
    const auto& rperm = part->rows->perm;
    const auto& cperm = part->cols->perm;
    const int nc = part->cols->size(), nr = part->rows->size();
    std::vector<Real> xi(nc), yi(nr, 0.0);
    for (int p = 0; p < nc; ++p) xi[p] = x[cperm[p]];
    for (std::size_t b = 0; b < blocks.size(); ++b) {
      const Block& blk = part->blocks[b];
      const Node& rn = part->rows->nodes[blk.row_node];
      const Node& cn = part->cols->nodes[blk.col_node];
      const Real* seg = xi.data() + cn.begin;
      Real* out = yi.data() + rn.begin;
      const HBlock& hb = blocks[b];
      if (hb.lowrank()) {
        const int k = mode == 0 ? hb.current_rank : hb.factor.rank();
        hb.factor.apply_range(0, k, seg, out);
      } else {
        const long m = rn.size(), n = cn.size();
        for (long j = 0; j < n; ++j) {
          const Real xj = seg[j];
          const Real* col = hb.dense.data() + j * m;
          for (long i = 0; i < m; ++i) out[i] += col[i] * xj;
        }
      }
    }
    for (int p = 0; p < nr; ++p) y[rperm[p]] = yi[p];
  }

  // (hmatrix.cpp:47-72)
  void matvec_transposed(const Real* x, Real* y, int mode) const {
    const auto& rperm = part->rows->perm;
    const auto& cperm = part->cols->perm;
    const int nc = part->cols->size(), nr = part->rows->size();
    std::vector<Real> xi(nr), yi(nc, 0.0);
    for (int p = 0; p < nr; ++p) xi[p] = x[rperm[p]];
    for (std::size_t b = 0; b < blocks.size(); ++b) {
      const Block& blk = part->blocks[b];
      const Node& rn = part->rows->nodes[blk.row_node];
      const Node& cn = part->cols->nodes[blk.col_node];
      const Real* seg = xi.data() + rn.begin;
      Real* out = yi.data() + cn.begin;
      const HBlock& hb = blocks[b];
      const long m = rn.size(), n = cn.size();
      if (hb.lowrank()) {
        const int k = mode == 0 ? hb.current_rank : hb.factor.rank();
        for (int l = 0; l < k; ++l) {
          Real s = 0.0;
          for (long i = 0; i < m; ++i) s += hb.factor.Ucol(l)[i] * seg[i];
          for (long j = 0; j < n; ++j) out[j] += hb.factor.Vcol(l)[j] * s;
        }
      } else {
        for (long j = 0; j < n; ++j) {
          Real s = 0.0;
          for (long i = 0; i < m; ++i) s += hb.dense[j * m + i] * seg[i];
          out[j] += s;
        }
      }
    }
    for (int p = 0; p < nc; ++p) y[cperm[p]] = yi[p];
  }

  void promote(int b) { blocks[b].current_rank = blocks[b].factor.rank(); }

  // (hmatrix.cpp:104-111)
  long extend_lookahead(int b, int steps) {
    HBlock& hb = blocks[b];
    if (!hb.lowrank() || hb.factor.exhausted()) return 0;
    const int before = hb.factor.rank();
    hb.factor = aca_extend(std::move(hb.factor), steps, view(b), cfg.max_rank);
    return hb.factor.rank() - before;
  }

  // storage accounting in MB (hmatrix.cpp:113-138)
  Real storage_mb_current() const {
    Real units = 0;
    for (std::size_t b = 0; b < blocks.size(); ++b) {
      const HBlock& hb = blocks[b];
      if (hb.lowrank())
        units += static_cast<Real>(hb.current_rank) * (hb.factor.m + hb.factor.n);
      else
        units += static_cast<Real>(hb.dense.size());
    }
    return units * 8.0 / (1 << 20);
  }
  Real storage_mb_tail() const {
    Real units = 0;
    for (const auto& hb : blocks)
      if (hb.lowrank())
        units += static_cast<Real>(hb.factor.rank() - hb.current_rank) *
                 (hb.factor.m + hb.factor.n);
    return units * 8.0 / (1 << 20);
  }
};

// assemble: parallel over blocks, full mode (aca_run at eps) or coarse mode
// (aca_extend initial_rank), then look-ahead extension; dense rows for
// non-admissible blocks (hmatrix.cpp:147-186)
static std::unique_ptr<HMatrix> assemble(const Partition* p,
                                         const EntryOracle* oracle,
                                         const AssemblyConfig& cfg) {
  auto h = std::make_unique<HMatrix>();
  h->part = p;
  h->oracle = oracle;
  h->cfg = cfg;
  if (oracle->rows() != p->rows->size() || oracle->cols() != p->cols->size())
    throw Error("HMatrix: oracle does not cover the index range");
  const int nb = static_cast<int>(p->blocks.size());
  std::vector<HBlock> built(nb);
  std::atomic<long> pivots{0};
  parallel_for(nb, [&](long b) {
    const Block& blk = p->blocks[b];
    const BlockView v = h->view(static_cast<int>(b));
    HBlock hb;
    if (blk.admissible) {
      Factor f;
      if (cfg.initial_rank >= 0)
        f = aca_extend(empty_factor(v.m, v.n), cfg.initial_rank, v,
                       cfg.max_rank);
      else
        f = aca_run(v, cfg.eps, cfg.beta, cfg.max_rank);
      hb.current_rank = f.rank();
      f = aca_extend(std::move(f), cfg.lookahead, v, cfg.max_rank);
      pivots += f.rank();
      hb.factor = std::move(f);
    } else {
      hb.dense.assign(static_cast<std::size_t>(v.m * v.n), 0.0);
      std::vector<Real> r(v.n);
      for (long i = 0; i < v.m; ++i) {
        oracle->row(v.row_ids[i], v.col_ids, v.n, r.data());
        for (long j = 0; j < v.n; ++j) hb.dense[j * v.m + i] = r[j];
      }
      hb.current_rank = 0;
    }
    built[b] = std::move(hb);
  });
  h->blocks = std::move(built);  // install serially (hmatrix.cpp:183)
  h->total_pivots = pivots.load();
  return h;
}

// ---------------------------------------------------------------------------
// 3x3 Kelvin block grid: six component H-matrices over one partition, the
// (c,r) cell aliasing (r,c) (proj/src/baca.cpp:669-687), matvec through the
// BlockGrid case of matvec (proj/src/expr.cpp:197-215).
static int comp_index(int r, int c) {
  const int lo = std::min(r, c), hi = std::max(r, c);
  static const int idx[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  return idx[lo][hi];
}

struct Grid {
  int ncomp = 1;           // 1 (scalar H-matrix) or 6 (Kelvin 3x3 grid)
  long nblk = 0;           // rows per grid cell
  long ncol = 0;           // columns per grid cell (0: square, = nblk)
  std::vector<std::unique_ptr<HMatrix>> h;
  long rows() const { return ncomp == 6 ? 3 * nblk : nblk; }

  void matvec(const Real* x, Real* y, int mode) const {
    if (ncomp == 1) {
      h[0]->matvec(x, y, mode);
      return;
    }
    const long nc = ncol > 0 ? ncol : nblk;
    std::vector<Real> tmp(nblk);
    std::fill(y, y + 3 * nblk, 0.0);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        h[comp_index(i, j)]->matvec(x + j * nc, tmp.data(), mode);
        for (long p = 0; p < nblk; ++p) y[i * nblk + p] += tmp[p];
      }
  }
};

// ---------------------------------------------------------------------------
// AMVM (proj/src/amvm.cpp).  Occurrences of the 3x3 grid flatten to the nine
// cells (i,j) in row-major order with prefix = embedding of row block i and
// suffix = selection of x block j (expr.cpp:474-498); grouping by H-matrix
// in first-appearance order gives the component order 0..5.
struct Term {
  int comp = 0, block = 0;
  std::vector<long> idx;
  std::vector<Real> val;
  Real norm_sq = 0.0;
};

struct Gamma {
  Real gamma = 0.0;
  std::vector<Real> difference;
  std::vector<Term> terms;
};

// (amvm.cpp:46-125)
static Gamma gamma_contributions(const Grid& g, const Real* x) {
  Gamma out;
  const long N = g.nblk, M = g.rows();
  out.difference.assign(M, 0.0);
  std::vector<Real> scratch(M, 0.0);
  std::vector<char> hit(M, 0);
  std::vector<long> touched;
  auto add = [&](long i, Real v) {
    if (!hit[i]) {
      hit[i] = 1;
      touched.push_back(i);
    }
    scratch[i] += v;
  };
  for (int comp = 0; comp < g.ncomp; ++comp) {
    const HMatrix& h = *g.h[comp];
    // occurrence list of this H-matrix, in occurrence order
    std::vector<std::pair<int, int>> occ;  // (row block i, col block j)
    if (g.ncomp == 1) {
      occ.push_back({0, 0});
    } else {
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          if (comp_index(i, j) == comp) occ.push_back({i, j});
    }
    const Partition& part = *h.part;
    for (int b = 0; b < static_cast<int>(h.blocks.size()); ++b) {
      const HBlock& hb = h.blocks[b];
      if (!hb.lowrank() || hb.factor.rank() - hb.current_rank == 0) continue;
      const Block& blk = part.blocks[b];
      const Node& rn = part.rows->nodes[blk.row_node];
      const Node& cn = part.cols->nodes[blk.col_node];
      const int* rids = part.rows->perm.data() + rn.begin;
      const int* cids = part.cols->perm.data() + cn.begin;
      const int k0 = hb.current_rank, k1 = hb.factor.rank();
      for (const auto& o : occ) {
        const Real* xi = x + o.second * N;
        std::vector<Real> seg(cn.size()), y(rn.size(), 0.0);
        for (int c = 0; c < cn.size(); ++c) seg[c] = xi[cids[c]];
        hb.factor.apply_range_device_order(k0, k1, seg.data(), y.data());
        for (int r = 0; r < rn.size(); ++r) {
          const Real v = 1.0 * y[r];
          if (g.ncomp == 1) {
            add(rids[r], v);
          } else {
            if (v == 0.0) continue;
            add(o.first * N + rids[r], 1.0 * v);
          }
        }
      }
      Term term;
      term.comp = comp;
      term.block = b;
      std::sort(touched.begin(), touched.end());
      for (long i : touched) {
        term.idx.push_back(i);
        term.val.push_back(scratch[i]);
        scratch[i] = 0.0;
        hit[i] = 0;
      }
      touched.clear();
      if (term.idx.empty()) continue;
      for (std::size_t i = 0; i < term.idx.size(); ++i) {
        out.difference[term.idx[i]] += term.val[i];
        term.norm_sq += term.val[i] * term.val[i];
      }
      out.terms.push_back(std::move(term));
    }
  }
  out.gamma = vnorm(out.difference);
  return out;
}

// row-sorted greedy marking (amvm.cpp:131-184)
static std::vector<int> mark_blocks(const Gamma& g, Real theta, int c_sp,
                                    long m_rows, long n_cols, Real* gamma_pk) {
  std::vector<int> marked;
  if (g.gamma <= 0.0) {
    if (gamma_pk) *gamma_pk = 0.0;
    return marked;
  }
  const Real threshold =
      (1.0 - theta) * g.gamma /
      std::sqrt(static_cast<Real>(c_sp) * static_cast<Real>(m_rows) *
                static_cast<Real>(n_cols));
  const Real target = (1.0 - theta) * g.gamma;
  std::vector<std::vector<int>> row_blocks(m_rows);
  for (std::size_t t = 0; t < g.terms.size(); ++t)
    for (std::size_t i = 0; i < g.terms[t].idx.size(); ++i)
      if (std::abs(g.terms[t].val[i]) >= threshold)
        row_blocks[g.terms[t].idx[i]].push_back(static_cast<int>(t));
  std::vector<long> order(m_rows);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](long a, long b) {
    return std::abs(g.difference[a]) > std::abs(g.difference[b]);
  });
  std::vector<Real> residual = g.difference;
  Real res_sq = 0.0;
  for (Real v : residual) res_sq += v * v;
  std::vector<char> in_set(g.terms.size(), 0);
  const Real target_sq = target * target;
  for (long row : order) {
    if (res_sq <= target_sq) break;
    for (int t : row_blocks[row]) {
      if (in_set[t]) continue;
      in_set[t] = 1;
      marked.push_back(t);
      const Term& term = g.terms[t];
      Real dot = 0.0;
      for (std::size_t i = 0; i < term.idx.size(); ++i)
        dot += residual[term.idx[i]] * term.val[i];
      res_sq += term.norm_sq - 2.0 * dot;
      for (std::size_t i = 0; i < term.idx.size(); ++i)
        residual[term.idx[i]] -= term.val[i];
      if (res_sq <= target_sq) break;
    }
  }
  if (gamma_pk) *gamma_pk = vnorm(residual);
  return marked;
}

struct AmvmIter {
  int k = 0;
  Real gamma = 0.0, gamma_pk = 0.0;
  int marked = 0;
  long cumulative_pivots = 0;
  Real storage_mb = 0.0;
  Real e_hat = -1.0;
};

// Algorithm 2 (amvm.cpp:199-268)
static std::vector<Real> amvm_multiply(Grid& g, const Real* x, Real theta,
                                       Real eps_amvm, int lookahead_steps,
                                       int max_iterations, int c_sp,
                                       std::vector<AmvmIter>& iters,
                                       int& converged) {
  if (theta <= 0.0 || theta >= 1.0)
    throw Error("amvm_multiply: theta must lie in (0,1)");
  if (eps_amvm <= 0.0) throw Error("amvm_multiply: eps_amvm must be positive");
  const long M = g.rows();
  auto pivots = [&]() {
    long p = 0;
    for (auto& h : g.h) p += h->total_pivots;
    return p;
  };
  auto storage = [&]() {
    Real s = 0;
    for (auto& h : g.h) s += h->storage_mb_current();
    return s;
  };
  std::vector<Real> b(M), b_hat_prev;
  g.matvec(x, b.data(), 0);
  iters.clear();
  for (int k = 0;; ++k) {
    Gamma gc = gamma_contributions(g, x);
    if (!b_hat_prev.empty()) {
      Real s = 0.0;
      for (long i = 0; i < M; ++i) {
        const Real d = b[i] + gc.difference[i] - b_hat_prev[i];
        s += d * d;
      }
      iters.back().e_hat = std::sqrt(s);
    }
    AmvmIter it;
    it.k = k;
    it.gamma = gc.gamma;
    it.cumulative_pivots = pivots();
    it.storage_mb = storage();
    if (gc.gamma <= eps_amvm) {
      iters.push_back(it);
      converged = 1;
      return b;
    }
    if (k >= max_iterations) {
      iters.push_back(it);
      converged = 0;
      return b;
    }
    Real gpk = 0.0;
    const auto marked = mark_blocks(gc, theta, c_sp, M, M, &gpk);
    it.gamma_pk = gpk;
    it.marked = static_cast<int>(marked.size());
    iters.push_back(it);
    b_hat_prev.resize(M);
    for (long i = 0; i < M; ++i) b_hat_prev[i] = b[i] + gc.difference[i];
    for (int t : marked) g.h[gc.terms[t].comp]->promote(gc.terms[t].block);
    std::vector<long> added(marked.size(), 0);
    parallel_for(static_cast<long>(marked.size()), [&](long i) {
      const Term& term = gc.terms[marked[i]];
      added[i] = g.h[term.comp]->extend_lookahead(term.block, lookahead_steps);
    });
    for (std::size_t i = 0; i < marked.size(); ++i)
      g.h[gc.terms[marked[i]].comp]->total_pivots += added[i];
    g.matvec(x, b.data(), 0);
  }
}

// ---------------------------------------------------------------------------
// random_vector: mt19937_64 + uniform_real_distribution(-1,1)
// (proj/tests/oracles.cpp:415-421)
static void random_vector(long n, unsigned seed, Real* out) {
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<Real> dist(-1.0, 1.0);
  for (long i = 0; i < n; ++i) out[i] = dist(gen);
}

static void normal_vector(long n, unsigned long seed, Real* out) {
  std::mt19937_64 gen(seed);
  std::normal_distribution<Real> dist(0.0, 1.0);
  for (long i = 0; i < n; ++i) out[i] = dist(gen);
}

}  // namespace oracle

// ===========================================================================
// C ABI for the Python test harness (ctypes).  Every function returns 0 on
// success and nonzero on error; or_last_error() returns the message.
using namespace oracle;

namespace {
thread_local std::string g_err;

// built with -mfma (explicit std::fma in the canonical order): refuse to run
// on a CPU without FMA instead of faulting
const bool g_cpu_ok = __builtin_cpu_supports("fma");

template <class F>
int guard(F&& f) {
  if (!g_cpu_ok) {
    g_err = "oracle built with -mfma but this CPU has no FMA";
    return 1;
  }
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// A self-contained problem: mesh (for Kelvin) or points (Newton) or a dense
// matrix, its tree and partition, and the assembled grid.
struct Problem {
  Mesh mesh;
  Material mat;
  std::unique_ptr<Kelvin> kelvin;
  std::unique_ptr<Galerkin> galerkin;
  std::vector<Vec3> eval_pts;
  std::vector<std::unique_ptr<EntryOracle>> oracles;
  Tree rows_tree, cols_tree;
  std::unique_ptr<Partition> part;
  Grid grid;
  int kind = 0;  // 0 Kelvin centroid collocation, 1 Newton points, 2 dense,
                 // 3 Galerkin V_kl grid, 4 Galerkin V_Delta
  long n = 0;
  double t_assemble = 0.0;
  long entries_counted = 0;
};

double now_s() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

void or_set_threads(int n) { g_thread_cap = n; }

int or_gauss_rule(int order, int* npts, double* a, double* b, double* w) {
  return guard([&] {
    const Rule r = gauss_rule(order);
    *npts = static_cast<int>(r.w.size());
    if (a)
      for (std::size_t i = 0; i < r.w.size(); ++i) {
        a[i] = r.a[i];
        b[i] = r.b[i];
        w[i] = r.w[i];
      }
  });
}

int or_gauss_legendre_01(int n, double* x, double* w) {
  return guard([&] {
    std::vector<Real> xs, ws;
    gauss_legendre_01(n, xs, ws);
    std::copy(xs.begin(), xs.end(), x);
    std::copy(ws.begin(), ws.end(), w);
  });
}

int or_lame_constants(double E, double nu, double* lambda, double* mu) {
  return guard([&] { lame_constants(E, nu, *lambda, *mu); });
}

int or_kelvin_tensor(const double* x, double E, double nu, double* out9) {
  return guard([&] {
    Material m{E, nu};
    kelvin_tensor({x[0], x[1], x[2]}, m, out9);
  });
}

// voxel cube surface; call with verts == nullptr to query sizes
int or_voxel_surface(int n, double lo, double hi, int* nv, int* nt,
                     double* verts, int* tris) {
  return guard([&] {
    Mesh m;
    voxel_surface(n, lo, hi, m);
    *nv = static_cast<int>(m.vertices.size());
    *nt = m.nt();
    if (verts) {
      for (int v = 0; v < *nv; ++v)
        for (int d = 0; d < 3; ++d) verts[3 * v + d] = m.vertices[v][d];
      for (int t = 0; t < *nt; ++t)
        for (int d = 0; d < 3; ++d) tris[3 * t + d] = m.triangles[t][d];
    }
  });
}

// Synthetic BASELINE meshes (the reference ships none):
// unit icosphere -- the icosahedron refined `level` times by edge midpoints
// projected to the sphere (20 * 4^level triangles, outward winding) -- and
// the ellipsoid (icosphere scaled by the semi-axes).  Stated here so the
// reference arm of bench.py and the tests build the inputs without the
// product package; tests/test_host.py checks they equal the product's
// generators bit for bit.
static void icosphere_mesh(int level, Mesh& m) {
  if (level < 0 || level > 10) throw std::runtime_error("icosphere level out of range");
  const Real g = (1.0 + std::sqrt(5.0)) / 2.0;
  std::vector<Vec3> v = {{-1, g, 0}, {1, g, 0},  {-1, -g, 0}, {1, -g, 0},
                         {0, -1, g}, {0, 1, g},  {0, -1, -g}, {0, 1, -g},
                         {g, 0, -1}, {g, 0, 1},  {-g, 0, -1}, {-g, 0, 1}};
  auto unit = [](Vec3 p) {
    const Real r = std::sqrt((p[0] * p[0] + p[1] * p[1]) + p[2] * p[2]);
    for (int d = 0; d < 3; ++d) p[d] /= r;
    return p;
  };
  for (Vec3& p : v) p = unit(p);
  std::vector<std::array<int, 3>> f = {
      {0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
      {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
      {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
      {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
  for (int l = 0; l < level; ++l) {
    std::map<std::pair<int, int>, int> cache;
    auto mid = [&](int a, int b) {
      const auto key = std::make_pair(std::min(a, b), std::max(a, b));
      const auto it = cache.find(key);
      if (it != cache.end()) return it->second;
      Vec3 q;
      for (int d = 0; d < 3; ++d) q[d] = 0.5 * (v[a][d] + v[b][d]);
      v.push_back(unit(q));
      cache[key] = static_cast<int>(v.size()) - 1;
      return static_cast<int>(v.size()) - 1;
    };
    std::vector<std::array<int, 3>> nf;
    nf.reserve(4 * f.size());
    for (const auto& t : f) {
      const int ab = mid(t[0], t[1]), bc = mid(t[1], t[2]), ca = mid(t[2], t[0]);
      nf.push_back({t[0], ab, ca});
      nf.push_back({t[1], bc, ab});
      nf.push_back({t[2], ca, bc});
      nf.push_back({ab, bc, ca});
    }
    f.swap(nf);
  }
  m.vertices = std::move(v);
  m.triangles = std::move(f);
}

// icosphere (ax = ay = az = 1) or ellipsoid; verts == nullptr queries sizes
int or_ellipsoid(int level, double ax, double ay, double az, int* nv, int* nt,
                 double* verts, int* tris) {
  return guard([&] {
    Mesh m;
    icosphere_mesh(level, m);
    *nv = static_cast<int>(m.vertices.size());
    *nt = m.nt();
    if (verts) {
      const double s[3] = {ax, ay, az};
      for (int v = 0; v < *nv; ++v)
        for (int d = 0; d < 3; ++d) verts[3 * v + d] = m.vertices[v][d] * s[d];
      for (int t = 0; t < *nt; ++t)
        for (int d = 0; d < 3; ++d) tris[3 * t + d] = m.triangles[t][d];
    }
  });
}

// geometry caches: centroids, areas, normals, diameters (mesh.cpp:229-247)
int or_mesh_geometry(int nv, const double* verts, int nt, const int* tris,
                     double* centroids, double* areas, double* normals,
                     double* diam) {
  return guard([&] {
    Mesh m;
    m.vertices.resize(nv);
    for (int v = 0; v < nv; ++v)
      m.vertices[v] = {verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]};
    m.triangles.resize(nt);
    for (int t = 0; t < nt; ++t)
      m.triangles[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    finish_geometry(m);
    for (int t = 0; t < nt; ++t) {
      for (int d = 0; d < 3; ++d) {
        centroids[3 * t + d] = m.centroids[t][d];
        normals[3 * t + d] = m.normals[t][d];
      }
      areas[t] = m.areas[t];
      diam[t] = m.diam[t];
    }
  });
}

int or_random_vector(long n, unsigned seed, double* out) {
  return guard([&] { random_vector(n, seed, out); });
}

int or_normal_vector(long n, unsigned long seed, double* out) {
  return guard([&] { normal_vector(n, seed, out); });
}

int or_analytic_potential_self(const double* v9, const double* p,
                               double* i1) {
  // I1 of the self term for a single triangle (E,nu irrelevant): used by the
  // KAT against the analytic flat-triangle potential.
  return guard([&] {
    Mesh m;
    m.vertices = {{v9[0], v9[1], v9[2]}, {v9[3], v9[4], v9[5]},
                  {v9[6], v9[7], v9[8]}};
    m.triangles = {{0, 1, 2}};
    finish_geometry(m);
    // with E = (1+nu)/(8 pi (1-nu)) the prefactor c is 1; read I1 from the
    // trace: sum_r S_rr = c (3 (3-4nu) + 1) I1
    Material mt{1.0, 0.25};
    mt.E = (1.0 + mt.nu) / (8.0 * M_PI * (1.0 - mt.nu));
    Kelvin k(&m, mt);
    Real s6[6];
    k.self_term({p[0], p[1], p[2]}, 0, s6);
    const Real tr = s6[0] + s6[3] + s6[5];
    *i1 = tr / (3.0 * (3.0 - 4.0 * mt.nu) + 1.0);
  });
}

// ---- problems -------------------------------------------------------------
// kind 0: Kelvin collocation on a mesh (6 components), supports = triangle
// corner boxes (operators.cpp:190-192), one tree for rows and columns.
int or_problem_kelvin(int nv, const double* verts, int nt, const int* tris,
                      double E, double nu, int b_min, double eta,
                      void** out) {
  return guard([&] {
    auto p = std::make_unique<Problem>();
    p->kind = 0;
    p->mesh.vertices.resize(nv);
    for (int v = 0; v < nv; ++v)
      p->mesh.vertices[v] = {verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]};
    p->mesh.triangles.resize(nt);
    for (int t = 0; t < nt; ++t)
      p->mesh.triangles[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    finish_geometry(p->mesh);
    Real lam, mu;
    lame_constants(E, nu, lam, mu);
    p->mat = {E, nu};
    p->kelvin = std::make_unique<Kelvin>(&p->mesh, p->mat);
    p->n = nt;
    std::vector<Box> boxes(nt);
    for (int t = 0; t < nt; ++t)
      for (int k = 0; k < 3; ++k) boxes[t].absorb(p->mesh.corner(t, k));
    p->rows_tree = build_cluster_tree(boxes, b_min);
    p->part = std::make_unique<Partition>(
        build_block_partition(&p->rows_tree, &p->rows_tree, eta));
    for (int c = 0; c < 6; ++c) {
      auto o = std::make_unique<KelvinComponentOracle>();
      o->k = p->kelvin.get();
      o->r = kCompR[c];
      o->c = kCompC[c];
      p->oracles.push_back(std::move(o));
    }
    p->grid.ncomp = 6;
    p->grid.nblk = nt;
    *out = p.release();
  });
}

// kind 6: the single-layer grid of evaluate_interior -- Kelvin collocation at
// arbitrary points (rows: point-box tree; columns: the triangle tree),
// partition (point tree, triangle tree, eta) (baca.cpp:645-653)
int or_problem_kelvin_points(int nv, const double* verts, int nt, const int* tris, int npts,
                             const double* pts, double E, double nu, int b_min, double eta,
                             void** out) {
  return guard([&] {
    auto p = std::make_unique<Problem>();
    p->kind = 6;
    p->mesh.vertices.resize(nv);
    for (int v = 0; v < nv; ++v)
      p->mesh.vertices[v] = {verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]};
    p->mesh.triangles.resize(nt);
    for (int t = 0; t < nt; ++t)
      p->mesh.triangles[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    finish_geometry(p->mesh);
    p->mat = {E, nu};
    p->kelvin = std::make_unique<Kelvin>(&p->mesh, p->mat);
    p->eval_pts.resize(npts);
    std::vector<Box> pb(npts), tb(nt);
    for (int i = 0; i < npts; ++i) {
      p->eval_pts[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
      pb[i].absorb(p->eval_pts[i]);
    }
    for (int t = 0; t < nt; ++t)
      for (int k = 0; k < 3; ++k) tb[t].absorb(p->mesh.corner(t, k));
    p->n = npts;
    p->rows_tree = build_cluster_tree(pb, b_min);
    p->cols_tree = build_cluster_tree(tb, b_min);
    p->part = std::make_unique<Partition>(
        build_block_partition(&p->rows_tree, &p->cols_tree, eta));
    for (int c = 0; c < 6; ++c) {
      auto o = std::make_unique<KelvinPointOracle>();
      o->k = p->kelvin.get();
      o->pts = &p->eval_pts;
      o->r = kCompR[c];
      o->c = kCompC[c];
      p->oracles.push_back(std::move(o));
    }
    p->grid.ncomp = 6;
    p->grid.nblk = npts;
    p->grid.ncol = nt;
    *out = p.release();
  });
}

// kind 7: one cell (r, c) of evaluate_interior's double-layer grid W~
// (CollocDoubleOracle, points x nodes; partition point tree x node tree,
// baca.cpp:650-651, 674-677); disjoint_order as QuadratureConfig
int or_problem_kelvin_double(int nv, const double* verts, int nt, const int* tris, int npts,
                             const double* pts, int r, int c, double E, double nu, int b_min,
                             double eta, int disjoint_order, void** out) {
  return guard([&] {
    auto p = std::make_unique<Problem>();
    p->kind = 7;
    p->mesh.vertices.resize(nv);
    for (int v = 0; v < nv; ++v)
      p->mesh.vertices[v] = {verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]};
    p->mesh.triangles.resize(nt);
    for (int t = 0; t < nt; ++t)
      p->mesh.triangles[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    finish_geometry(p->mesh);
    p->mat = {E, nu};
    p->kelvin = std::make_unique<Kelvin>(&p->mesh, p->mat);
    p->kelvin->set_disjoint_order(disjoint_order);
    p->kelvin->prepare_double();
    p->eval_pts.resize(npts);
    std::vector<Box> pb(npts), tb(nt), nb(nv);
    for (int i = 0; i < npts; ++i) {
      p->eval_pts[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
      pb[i].absorb(p->eval_pts[i]);
    }
    for (int t = 0; t < nt; ++t)
      for (int k = 0; k < 3; ++k) tb[t].absorb(p->mesh.corner(t, k));
    for (int v = 0; v < nv; ++v)
      for (int t : p->kelvin->vtri[v]) nb[v].absorb(tb[t]);
    p->n = npts;
    p->rows_tree = build_cluster_tree(pb, b_min);
    p->cols_tree = build_cluster_tree(nb, b_min);
    p->part = std::make_unique<Partition>(
        build_block_partition(&p->rows_tree, &p->cols_tree, eta));
    auto o = std::make_unique<KelvinDoubleOracle>();
    o->k = p->kelvin.get();
    o->pts = &p->eval_pts;
    o->r = r;
    o->c = c;
    p->oracles.push_back(std::move(o));
    p->grid.ncomp = 1;
    p->grid.nblk = npts;
    *out = p.release();
  });
}

// kinds 3 / 4: Galerkin scalar kernels on the triangle partition of
// assemble_operators (operators.cpp:186-200, corner boxes, one tree):
// which = 0 -> the six V_kl as a symmetric 3x3 grid, 1 -> V_Delta alone.
int or_problem_galerkin(int nv, const double* verts, int nt, const int* tris, int which,
                        int b_min, double eta, void** out) {
  return guard([&] {
    auto p = std::make_unique<Problem>();
    p->kind = which == 0 ? 3 : 4;
    p->mesh.vertices.resize(nv);
    for (int v = 0; v < nv; ++v)
      p->mesh.vertices[v] = {verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]};
    p->mesh.triangles.resize(nt);
    for (int t = 0; t < nt; ++t)
      p->mesh.triangles[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    finish_geometry(p->mesh);
    p->galerkin = std::make_unique<Galerkin>(&p->mesh);
    p->n = nt;
    std::vector<Box> boxes(nt);
    for (int t = 0; t < nt; ++t)
      for (int k = 0; k < 3; ++k) boxes[t].absorb(p->mesh.corner(t, k));
    p->rows_tree = build_cluster_tree(boxes, b_min);
    p->part = std::make_unique<Partition>(
        build_block_partition(&p->rows_tree, &p->rows_tree, eta));
    const int nc = which == 0 ? 6 : 1;
    for (int c = 0; c < nc; ++c) {
      auto o = std::make_unique<GalerkinComponentOracle>();
      o->g = p->galerkin.get();
      o->comp = which == 0 ? c : 6;
      p->oracles.push_back(std::move(o));
    }
    p->grid.ncomp = nc;
    p->grid.nblk = nt;
    *out = p.release();
  });
}

// kind 5: K_Delta on the triangle x node partition of assemble_operators
// (operators.cpp:186-200): node boxes = union of the incident triangles'
// corner boxes, separate row (triangle) and column (node) trees.
int or_problem_kdelta(int nv, const double* verts, int nt, const int* tris, int b_min,
                      double eta, void** out) {
  return guard([&] {
    auto p = std::make_unique<Problem>();
    p->kind = 5;
    p->mesh.vertices.resize(nv);
    for (int v = 0; v < nv; ++v)
      p->mesh.vertices[v] = {verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]};
    p->mesh.triangles.resize(nt);
    for (int t = 0; t < nt; ++t)
      p->mesh.triangles[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    finish_geometry(p->mesh);
    p->galerkin = std::make_unique<Galerkin>(&p->mesh);
    p->galerkin->build_vtri();
    p->n = nt;
    std::vector<Box> tb(nt), nb(nv);
    for (int t = 0; t < nt; ++t)
      for (int k = 0; k < 3; ++k) tb[t].absorb(p->mesh.corner(t, k));
    for (int v = 0; v < nv; ++v)
      for (int t : p->galerkin->vtri[v]) nb[v].absorb(tb[t]);
    p->rows_tree = build_cluster_tree(tb, b_min);
    p->cols_tree = build_cluster_tree(nb, b_min);
    p->part = std::make_unique<Partition>(
        build_block_partition(&p->rows_tree, &p->cols_tree, eta));
    auto o = std::make_unique<KDeltaOracle>();
    o->g = p->galerkin.get();
    p->oracles.push_back(std::move(o));
    p->grid.ncomp = 1;
    p->grid.nblk = nt;
    *out = p.release();
  });
}

// build_t_matrix (operators.cpp:8-33) / mass (operators.cpp:82-88) as a
// dense row-major n_tri x n_vert array; which 0 T12, 1 T13, 2 T23, 3 mass
int or_sparse_op(int nv, const double* verts, int nt, const int* tris, int which,
                 double* dense) {
  return guard([&] {
    Mesh m;
    m.vertices.resize(nv);
    for (int v = 0; v < nv; ++v) m.vertices[v] = {verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]};
    m.triangles.resize(nt);
    for (int t = 0; t < nt; ++t) m.triangles[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    finish_geometry(m);
    std::fill(dense, dense + static_cast<long>(nt) * nv, 0.0);
    const int kk[3] = {0, 0, 1}, ll[3] = {1, 2, 2};
    for (int t = 0; t < nt; ++t) {
      if (which == 3) {
        for (int a = 0; a < 3; ++a)
          dense[static_cast<long>(t) * nv + m.triangles[t][a]] += m.areas[t] / 3.0;
        continue;
      }
      const int k = kk[which], l = ll[which];
      const Vec3& n = m.normals[t];
      const Real inv2a = 1.0 / (2.0 * m.areas[t]);
      const Vec3 c[3] = {m.corner(t, 0), m.corner(t, 1), m.corner(t, 2)};
      Vec3 g[3] = {cross3(n, sub(c[2], c[1])), cross3(n, sub(c[0], c[2])),
                   cross3(n, sub(c[1], c[0]))};
      for (int a = 0; a < 3; ++a) {
        for (int d = 0; d < 3; ++d) g[a][d] *= inv2a;
        const Real v = n[l] * g[a][k] - n[k] * g[a][l];
        if (v != 0.0) dense[static_cast<long>(t) * nv + m.triangles[t][a]] += v;
      }
    }
  });
}

// pair_rule(case, order) tables (quadrature.cpp:290-338); NULL arrays query n
int or_pair_rule(int pc, int order, int* n, double* xr1, double* xr2, double* yr1,
                 double* yr2, double* w) {
  return guard([&] {
    const PairRule r = build_pair_rule(pc, order);
    *n = static_cast<int>(r.w.size());
    if (!w) return;
    for (size_t q = 0; q < r.w.size(); ++q) {
      xr1[q] = r.xr1[q];
      xr2[q] = r.xr2[q];
      yr1[q] = r.yr1[q];
      yr2[q] = r.yr2[q];
      w[q] = r.w[q];
    }
  });
}

// classify_pair + vertex permutations (quadrature.cpp:127-166)
int or_classify_pair(const int* a3, const int* b3, int* rot_a, int* rot_b, int* perm_a,
                     int* perm_b) {
  return guard([&] {
    const std::array<int, 3> a = {a3[0], a3[1], a3[2]}, b = {b3[0], b3[1], b3[2]};
    const int c = classify_pair(a, b, *rot_a, *rot_b);
    const auto pa = test_vertex_perm(*rot_a), pb = trial_vertex_perm(c, *rot_b);
    for (int k = 0; k < 3; ++k) {
      perm_a[k] = pa[k];
      perm_b[k] = pb[k];
    }
    *rot_a = c * 16 + *rot_a;  // case in the high bits
  });
}

// kind 1: Newton kernel over points with point boxes or explicit boxes.
// boxes6 == nullptr => point boxes.
int or_problem_newton(int n, const double* pts, const double* boxes6,
                      double diag, int b_min, double eta, void** out) {
  return guard([&] {
    auto p = std::make_unique<Problem>();
    p->kind = 1;
    auto o = std::make_unique<NewtonOracle>();
    o->diag = diag;
    o->pts.resize(n);
    std::vector<Box> boxes(n);
    for (int i = 0; i < n; ++i) {
      o->pts[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
      if (boxes6) {
        boxes[i].absorb(Vec3{boxes6[6 * i], boxes6[6 * i + 1], boxes6[6 * i + 2]});
        boxes[i].absorb(Vec3{boxes6[6 * i + 3], boxes6[6 * i + 4], boxes6[6 * i + 5]});
      } else {
        boxes[i].absorb(o->pts[i]);
      }
    }
    p->oracles.push_back(std::move(o));
    p->n = n;
    p->rows_tree = build_cluster_tree(boxes, b_min);
    p->part = std::make_unique<Partition>(
        build_block_partition(&p->rows_tree, &p->rows_tree, eta));
    p->grid.ncomp = 1;
    p->grid.nblk = n;
    *out = p.release();
  });
}

// kind 2: explicit column-major dense matrix (m x n) with point boxes for
// rows and columns (separate trees).
int or_problem_dense(int m, int n, const double* a, const double* row_pts,
                     const double* col_pts, int b_min, double eta,
                     void** out) {
  return guard([&] {
    auto p = std::make_unique<Problem>();
    p->kind = 2;
    auto o = std::make_unique<DenseOracle>();
    o->m = m;
    o->n = n;
    o->a.assign(a, a + static_cast<long>(m) * n);
    p->oracles.push_back(std::move(o));
    std::vector<Box> rb(m), cb(n);
    for (int i = 0; i < m; ++i)
      rb[i].absorb(Vec3{row_pts[3 * i], row_pts[3 * i + 1], row_pts[3 * i + 2]});
    for (int j = 0; j < n; ++j)
      cb[j].absorb(Vec3{col_pts[3 * j], col_pts[3 * j + 1], col_pts[3 * j + 2]});
    p->rows_tree = build_cluster_tree(rb, b_min);
    p->cols_tree = build_cluster_tree(cb, b_min);
    p->part = std::make_unique<Partition>(
        build_block_partition(&p->rows_tree, &p->cols_tree, eta));
    p->grid.ncomp = 1;
    p->grid.nblk = m;
    p->n = m;
    *out = p.release();
  });
}

void or_problem_free(void* h) { delete static_cast<Problem*>(h); }

static Problem* P(void* h) { return static_cast<Problem*>(h); }
static const Tree& cols_tree(const Problem* p) {
  return p->part->cols == &p->rows_tree ? p->rows_tree : p->cols_tree;
}

int or_tree_info(void* h, int which, int* n_nodes, int* depth, int* size) {
  return guard([&] {
    const Tree& t = which == 0 ? P(h)->rows_tree : cols_tree(P(h));
    *n_nodes = static_cast<int>(t.nodes.size());
    *depth = t.depth;
    *size = t.size();
  });
}

// nodes as int rows [begin, end, child0, child1, level] and boxes [lo, hi]
int or_tree_nodes(void* h, int which, int* nodes5, double* boxes6, int* perm) {
  return guard([&] {
    const Tree& t = which == 0 ? P(h)->rows_tree : cols_tree(P(h));
    for (std::size_t i = 0; i < t.nodes.size(); ++i) {
      const Node& nd = t.nodes[i];
      nodes5[5 * i] = nd.begin;
      nodes5[5 * i + 1] = nd.end;
      nodes5[5 * i + 2] = nd.child[0];
      nodes5[5 * i + 3] = nd.child[1];
      nodes5[5 * i + 4] = nd.level;
      for (int d = 0; d < 3; ++d) {
        boxes6[6 * i + d] = nd.box.lo[d];
        boxes6[6 * i + 3 + d] = nd.box.hi[d];
      }
    }
    std::copy(t.perm.begin(), t.perm.end(), perm);
  });
}

int or_partition_info(void* h, int* n_blocks, int* n_adm, int* c_sp) {
  return guard([&] {
    const Partition& p = *P(h)->part;
    *n_blocks = static_cast<int>(p.blocks.size());
    int na = 0;
    for (const auto& b : p.blocks) na += b.admissible;
    *n_adm = na;
    *c_sp = sparsity_constant(p);
  });
}

// blocks as rows [row_node, col_node, admissible, level]
int or_partition_blocks(void* h, int* blocks4) {
  return guard([&] {
    const Partition& p = *P(h)->part;
    for (std::size_t i = 0; i < p.blocks.size(); ++i) {
      blocks4[4 * i] = p.blocks[i].row_node;
      blocks4[4 * i + 1] = p.blocks[i].col_node;
      blocks4[4 * i + 2] = p.blocks[i].admissible;
      blocks4[4 * i + 3] = p.blocks[i].level;
    }
  });
}

// JSON dump; call with buf == nullptr to get the length (incl. NUL)
int or_partition_json(void* h, char* buf, long* len) {
  return guard([&] {
    const std::string s = partition_to_json(*P(h)->part);
    if (!buf) {
      *len = static_cast<long>(s.size()) + 1;
      return;
    }
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

// literal kelvin_tensor-based collocation entry (canonical-order check)
int or_entry_literal(void* h, int comp, long i, long j, double* out) {
  return guard([&] {
    Problem* p = P(h);
    if (p->kind == 5) {
      *out = p->galerkin->kdelta_literal(static_cast<int>(i), static_cast<int>(j));
      return;
    }
    if (p->kind == 7) {
      const auto* o = static_cast<const KelvinDoubleOracle*>(p->oracles[0].get());
      *out = p->kelvin->colloc_double_literal(p->eval_pts[i], o->r, o->c, static_cast<int>(j));
      return;
    }
    if (p->kind == 3 || p->kind == 4) {
      *out = p->galerkin->entry_literal(static_cast<int>(i), static_cast<int>(j),
                                        p->kind == 4 ? 6 : comp);
      return;
    }
    if (p->kind != 0) throw Error("kelvin or galerkin only");
    *out = p->kelvin->colloc_single_literal(p->mesh.centroids[i], kCompR[comp],
                                            kCompC[comp], static_cast<int>(j));
  });
}

// single entry A_comp[i, j] in external ids
int or_entry(void* h, int comp, long i, long j, double* out) {
  return guard([&] { *out = P(h)->oracles[comp]->entry(i, j); });
}

// rows of the exact product A x from oracle entries (Kelvin grid): for each
// requested output dof r*N + i, exact = sum_c sum_j A_rc(i, j) x[c*N + j]
// and mag = sum |A_rc(i, j) x[c*N + j]| -- the checker of the H-matvec at
// sizes where no dense matrix fits (config 5); rows x 64 column chunks in
// parallel, the chunk sums added in order
int or_rows_dot(void* h, int n, const long* out_dofs, const double* x, double* exact,
                double* mag) {
  return guard([&] {
    Problem* p = P(h);
    if (p->oracles.size() != 6) throw Error("or_rows_dot: Kelvin problems only");
    const long N = p->oracles[0]->cols();
    const int kChunks = 64;
    const int comp_of[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
    std::vector<double> pe(static_cast<size_t>(n) * kChunks), pm(pe.size());
    parallel_for(static_cast<long>(n) * kChunks, [&](long w) {
      const long q = w / kChunks, ch = w % kChunks;
      const long r = out_dofs[q] / N, i = out_dofs[q] % N;
      const long j0 = N * ch / kChunks, j1 = N * (ch + 1) / kChunks;
      double e = 0.0, a = 0.0;
      for (int c = 0; c < 3; ++c) {
        const EntryOracle& o = *p->oracles[comp_of[r][c]];
        for (long j = j0; j < j1; ++j) {
          const double t = o.entry(i, j) * x[c * N + j];
          e += t;
          a += std::abs(t);
        }
      }
      pe[w] = e;
      pm[w] = a;
    });
    for (int q = 0; q < n; ++q) {
      double e = 0.0, a = 0.0;
      for (int ch = 0; ch < kChunks; ++ch) {
        e += pe[static_cast<size_t>(q) * kChunks + ch];
        a += pm[static_cast<size_t>(q) * kChunks + ch];
      }
      exact[q] = e;
      mag[q] = a;
    }
  });
}

// dense component matrix (row-major m x n); comp for Kelvin in 0..5
int or_dense(void* h, int comp, double* out) {
  return guard([&] {
    const EntryOracle& o = *P(h)->oracles[comp];
    const long m = o.rows(), n = o.cols();
    parallel_for(m, [&](long i) {
      for (long j = 0; j < n; ++j) out[i * n + j] = o.entry(i, j);
    });
  });
}

// assemble every component; records wall time
int or_assemble(void* h, double eps, double beta, int initial_rank,
                int lookahead, long max_rank) {
  return guard([&] {
    Problem* p = P(h);
    AssemblyConfig cfg;
    cfg.eps = eps;
    cfg.beta = beta;
    cfg.initial_rank = initial_rank;
    cfg.lookahead = lookahead;
    cfg.max_rank = max_rank;
    p->grid.h.clear();
    const double t0 = now_s();
    for (int c = 0; c < p->grid.ncomp; ++c)
      p->grid.h.push_back(assemble(p->part.get(), p->oracles[c].get(), cfg));
    p->t_assemble = now_s() - t0;
  });
}

int or_assemble_time(void* h, double* seconds, long* entries) {
  return guard([&] {
    *seconds = P(h)->t_assemble;
    long e = 0;
    for (const auto& o : P(h)->oracles) e += o->evaluated.load();
    *entries = e;
  });
}

int or_reset_entry_count(void* h) {
  return guard([&] {
    for (const auto& o : P(h)->oracles) o->evaluated = 0;
  });
}

// ranks per (comp, block): current and look-ahead (-1 for dense blocks),
// plus the consumed count and last stop rule
int or_ranks(void* h, int* k_cur, int* k_look, int* consumed, int* stop) {
  return guard([&] {
    const Problem* p = P(h);
    const long nb = static_cast<long>(p->part->blocks.size());
    for (int c = 0; c < p->grid.ncomp; ++c)
      for (long b = 0; b < nb; ++b) {
        const HBlock& hb = p->grid.h[c]->blocks[b];
        const long o = c * nb + b;
        k_cur[o] = hb.lowrank() ? hb.current_rank : -1;
        k_look[o] = hb.lowrank() ? hb.factor.rank() : -1;
        if (consumed) consumed[o] = hb.lowrank() ? hb.factor.num_consumed : -1;
        if (stop) stop[o] = hb.lowrank() ? hb.factor.last_stop : -1;
      }
  });
}

// factor of (comp, block): U (m x K), V (n x K) column-major, pivots (K x 2),
// frob_sq; call with U == nullptr to query m, n, K
int or_factor(void* h, int comp, int b, int* m, int* n, int* K, double* U,
              double* V, int* piv, double* frob_sq) {
  return guard([&] {
    const HBlock& hb = P(h)->grid.h[comp]->blocks[b];
    if (!hb.lowrank()) throw Error("or_factor: dense block");
    *m = static_cast<int>(hb.factor.m);
    *n = static_cast<int>(hb.factor.n);
    *K = hb.factor.rank();
    if (U) {
      std::copy(hb.factor.U.begin(), hb.factor.U.end(), U);
      std::copy(hb.factor.V.begin(), hb.factor.V.end(), V);
      for (int l = 0; l < *K; ++l) {
        piv[2 * l] = hb.factor.pivots[l].first;
        piv[2 * l + 1] = hb.factor.pivots[l].second;
      }
      *frob_sq = hb.factor.frob_sq;
    }
  });
}

// dense payload of a non-admissible block (column-major m x n)
int or_dense_block(void* h, int comp, int b, double* out) {
  return guard([&] {
    const HBlock& hb = P(h)->grid.h[comp]->blocks[b];
    std::copy(hb.dense.begin(), hb.dense.end(), out);
  });
}

int or_matvec(void* h, const double* x, double* y, int mode) {
  return guard([&] { P(h)->grid.matvec(x, y, mode); });
}

int or_matvec_transposed(void* h, const double* x, double* y, int mode) {
  return guard([&] {
    if (P(h)->grid.ncomp != 1) throw Error("transposed: scalar only");
    P(h)->grid.h[0]->matvec_transposed(x, y, mode);
  });
}

// best-of-`reps` single-threaded matvec wall time
int or_matvec_time(void* h, const double* x, double* y, int reps,
                   double* best) {
  return guard([&] {
    *best = 1e300;
    for (int r = 0; r < reps; ++r) {
      const double t0 = now_s();
      P(h)->grid.matvec(x, y, 0);
      *best = std::min(*best, now_s() - t0);
    }
  });
}

int or_storage(void* h, double* mb_current, double* mb_tail, long* pivots) {
  return guard([&] {
    *mb_current = 0;
    *mb_tail = 0;
    *pivots = 0;
    for (auto& hm : P(h)->grid.h) {
      *mb_current += hm->storage_mb_current();
      *mb_tail += hm->storage_mb_tail();
      *pivots += hm->total_pivots;
    }
  });
}

int or_promote(void* h, int comp, int b) {
  return guard([&] { P(h)->grid.h[comp]->promote(b); });
}

int or_extend(void* h, int comp, int b, int steps) {
  return guard([&] {
    P(h)->grid.h[comp]->total_pivots +=
        P(h)->grid.h[comp]->extend_lookahead(b, steps);
  });
}

// gamma contributions: returns gamma, difference (rows), number of terms;
// term arrays via or_gamma_terms after this call (kept in the problem)
static thread_local Gamma g_last_gamma;

int or_gamma(void* h, const double* x, double* gamma, double* difference,
             int* n_terms) {
  return guard([&] {
    g_last_gamma = gamma_contributions(P(h)->grid, x);
    *gamma = g_last_gamma.gamma;
    std::copy(g_last_gamma.difference.begin(), g_last_gamma.difference.end(),
              difference);
    *n_terms = static_cast<int>(g_last_gamma.terms.size());
  });
}

// per term: comp, block, nnz, norm_sq
int or_gamma_terms(int* comp, int* block, int* nnz, double* norm_sq) {
  return guard([&] {
    for (std::size_t t = 0; t < g_last_gamma.terms.size(); ++t) {
      comp[t] = g_last_gamma.terms[t].comp;
      block[t] = g_last_gamma.terms[t].block;
      nnz[t] = static_cast<int>(g_last_gamma.terms[t].idx.size());
      norm_sq[t] = g_last_gamma.terms[t].norm_sq;
    }
  });
}

int or_gamma_term_data(int t, long* idx, double* val) {
  return guard([&] {
    const Term& term = g_last_gamma.terms.at(t);
    std::copy(term.idx.begin(), term.idx.end(), idx);
    std::copy(term.val.begin(), term.val.end(), val);
  });
}

int or_mark(double theta, int c_sp, long m_rows, long n_cols, int* marked,
            int* n_marked, double* gamma_pk) {
  return guard([&] {
    const auto mk =
        mark_blocks(g_last_gamma, theta, c_sp, m_rows, n_cols, gamma_pk);
    *n_marked = static_cast<int>(mk.size());
    std::copy(mk.begin(), mk.end(), marked);
  });
}

// full AMVM; iteration records as rows of 7 doubles
// [k, gamma, gamma_pk, marked, cumulative_pivots, storage_mb, e_hat]
int or_amvm(void* h, const double* x, double theta, double eps_amvm,
            int lookahead_steps, int max_iterations, double* b,
            double* iters7, int* n_iters, int* converged) {
  return guard([&] {
    Problem* p = P(h);
    std::vector<AmvmIter> it;
    const int c_sp = std::max(1, sparsity_constant(*p->part));
    auto res = amvm_multiply(p->grid, x, theta, eps_amvm, lookahead_steps,
                             max_iterations, c_sp, it, *converged);
    std::copy(res.begin(), res.end(), b);
    *n_iters = static_cast<int>(it.size());
    for (std::size_t i = 0; i < it.size(); ++i) {
      double* r = iters7 + 7 * i;
      r[0] = it[i].k;
      r[1] = it[i].gamma;
      r[2] = it[i].gamma_pk;
      r[3] = it[i].marked;
      r[4] = static_cast<double>(it[i].cumulative_pivots);
      r[5] = it[i].storage_mb;
      r[6] = it[i].e_hat;
    }
  });
}

// admissibility of two boxes [lo, hi] (cluster.cpp:21-24)
int or_admissible(const double* a6, const double* b6, double eta, int* out) {
  return guard([&] {
    Box a, b;
    a.absorb(Vec3{a6[0], a6[1], a6[2]});
    a.absorb(Vec3{a6[3], a6[4], a6[5]});
    b.absorb(Vec3{b6[0], b6[1], b6[2]});
    b.absorb(Vec3{b6[3], b6[4], b6[5]});
    *out = admissible(a, b, eta) ? 1 : 0;
  });
}

// ACA of one admissible block of the problem's partition without
// assembling the rest (sampled parity at full problem size):
// full mode run + look-ahead extension as in assemble (hmatrix.cpp:160-168)
int or_aca_block(void* h, int comp, int b, double eps, double beta,
                 int initial_rank, int lookahead, int* k_cur, int* K,
                 double* frob_sq, long* entries) {
  return guard([&] {
    Problem* p = P(h);
    HMatrix tmp;
    tmp.part = p->part.get();
    tmp.oracle = p->oracles.at(comp).get();
    const BlockView v = tmp.view(b);
    if (!p->part->blocks.at(b).admissible) throw Error("block is not admissible");
    const long before = tmp.oracle->evaluated.load();
    Factor f = initial_rank >= 0
                   ? aca_extend(empty_factor(v.m, v.n), initial_rank, v, 1L << 30)
                   : aca_run(v, eps, beta, 1L << 30);
    *k_cur = f.rank();
    f = aca_extend(std::move(f), lookahead, v, 1L << 30);
    *K = f.rank();
    *frob_sq = f.frob_sq;
    if (entries) *entries = tmp.oracle->evaluated.load() - before;
  });
}

// ---- single-block ACA on a dense column-major matrix (test_aca ports) -----
struct AcaHandle {
  DenseOracle o;
  std::vector<int> rows, cols;
  Factor f;
};

int or_aca_dense_new(int m, int n, const double* a, void** out) {
  return guard([&] {
    auto h = std::make_unique<AcaHandle>();
    h->o.m = m;
    h->o.n = n;
    h->o.a.assign(a, a + static_cast<long>(m) * n);
    h->rows.resize(m);
    h->cols.resize(n);
    std::iota(h->rows.begin(), h->rows.end(), 0);
    std::iota(h->cols.begin(), h->cols.end(), 0);
    h->f = empty_factor(m, n);
    *out = h.release();
  });
}

void or_aca_dense_free(void* h) { delete static_cast<AcaHandle*>(h); }

// mode 0: aca_run(eps, beta, max_rank) resuming from the current state;
// mode 1: aca_extend(steps, max_rank)
int or_aca_dense_step(void* hh, int mode, double eps, double beta, int steps,
                      long max_rank) {
  return guard([&] {
    AcaHandle* h = static_cast<AcaHandle*>(hh);
    BlockView v{&h->o, h->rows.data(), h->cols.data(), h->o.m, h->o.n};
    if (mode == 0)
      h->f = aca_run(v, eps, beta, max_rank, &h->f);
    else
      h->f = aca_extend(std::move(h->f), steps, v, max_rank);
  });
}

int or_aca_dense_state(void* hh, int* K, int* num_consumed, int* last_stop,
                       double* frob_sq, double* U, double* V, int* piv) {
  return guard([&] {
    const Factor& f = static_cast<AcaHandle*>(hh)->f;
    *K = f.rank();
    *num_consumed = f.num_consumed;
    *last_stop = f.last_stop;
    *frob_sq = f.frob_sq;
    if (U) {
      std::copy(f.U.begin(), f.U.end(), U);
      std::copy(f.V.begin(), f.V.end(), V);
      for (int l = 0; l < f.rank(); ++l) {
        piv[2 * l] = f.pivots[l].first;
        piv[2 * l + 1] = f.pivots[l].second;
      }
    }
  });
}

}  // extern "C"
