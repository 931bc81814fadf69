#include "geometry.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <unordered_map>

#include "errors.hpp"

namespace hmb {

namespace {

inline V3 vsub(const V3& a, const V3& b) {
  return {a[0] - b[0], a[1] - b[1], a[2] - b[2]};
}
// (x0^2 + x1^2) + x2^2: the Vector3d::norm order assumed throughout
inline Real vnorm(const V3& a) {
  return std::sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]);
}
inline V3 vcross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2],
          a[0] * b[1] - a[1] * b[0]};
}

}  // namespace

void Mesh::finish() {
  const int n = nt();
  centroids.assign(n, V3{0, 0, 0});
  normals.assign(n, V3{0, 0, 0});
  areas.assign(n, 0.0);
  diam.assign(n, 0.0);
  Real scale = 0.0;
  for (const V3& v : vertices) scale = std::max(scale, vnorm(v));
  for (int t = 0; t < n; ++t) {
    for (int k = 0; k < 3; ++k)
      if (triangles[t][k] < 0 || triangles[t][k] >= nv())
        throw MeshError("vertex index out of range in triangle " +
                        std::to_string(t));
    const V3& a = corner(t, 0);
    const V3& b = corner(t, 1);
    const V3& c = corner(t, 2);
    const V3 cr = vcross(vsub(b, a), vsub(c, a));
    const Real area = 0.5 * vnorm(cr);
    if (area <= 1e-14 * scale * scale)
      throw MeshError("degenerate triangle " + std::to_string(t));
    areas[t] = area;
    for (int d = 0; d < 3; ++d) {
      normals[t][d] = cr[d] / (2.0 * area);
      centroids[t][d] = ((a[d] + b[d]) + c[d]) / 3.0;
    }
    diam[t] = std::max({vnorm(vsub(a, b)), vnorm(vsub(b, c)), vnorm(vsub(a, c))});
  }
}

void Mesh::validate_admissible() const {
  std::map<std::pair<int, int>, int> edges;
  for (const auto& tri : triangles)
    for (int e = 0; e < 3; ++e)
      if (++edges[{tri[e], tri[(e + 1) % 3]}] > 1)
        throw MeshError("non-admissible triangulation: repeated directed edge");
  for (const auto& kv : edges)
    if (!edges.count({kv.first.second, kv.first.first}))
      throw MeshError("non-admissible triangulation: open edge " +
                      std::to_string(kv.first.first) + "-" +
                      std::to_string(kv.first.second));
  std::vector<std::vector<int>> vt(nv());
  for (int t = 0; t < nt(); ++t)
    for (int v : triangles[t]) vt[v].push_back(t);
  for (int v = 0; v < nv(); ++v)
    for (std::size_t a = 0; a < vt[v].size(); ++a)
      for (std::size_t b = a + 1; b < vt[v].size(); ++b) {
        int shared = 0;
        for (int i : triangles[vt[v][a]])
          for (int j : triangles[vt[v][b]]) shared += i == j;
        if (shared > 2)
          throw MeshError("non-admissible triangulation: triangles share a face");
      }
}

void Mesh::label_dirichlet(const std::string& text) {
  struct Clause {
    int axis, op;
    Real value;
  };
  std::vector<Clause> clauses;
  std::stringstream ss(text);
  std::string term;
  while (std::getline(ss, term, '|')) {
    term.erase(std::remove_if(term.begin(), term.end(), ::isspace), term.end());
    if (term.empty()) continue;
    if (term.size() < 4 || term[0] != 'x' || term[1] < '1' || term[1] > '3')
      throw MeshError("labeling predicate: bad clause '" + term + "'");
    Clause c{term[1] - '1', 0, 0.0};
    std::size_t pos = 2;
    if (term.compare(pos, 2, "<=") == 0) {
      c.op = 2;
      pos += 2;
    } else if (term.compare(pos, 2, ">=") == 0) {
      c.op = 3;
      pos += 2;
    } else if (term[pos] == '<') {
      c.op = 0;
      pos += 1;
    } else if (term[pos] == '>') {
      c.op = 1;
      pos += 1;
    } else {
      throw MeshError("labeling predicate: bad operator in '" + term + "'");
    }
    try {
      c.value = std::stod(term.substr(pos));
    } catch (const std::exception&) {
      throw MeshError("labeling predicate: bad value in '" + term + "'");
    }
    clauses.push_back(c);
  }
  if (clauses.empty())
    throw MeshError("labeling predicate: no clauses in '" + text + "'");
  if (centroids.size() != triangles.size()) finish();
  dirichlet.assign(nt(), 0);
  for (int t = 0; t < nt(); ++t)
    for (const Clause& c : clauses) {
      const Real x = centroids[t][c.axis];
      const bool hit = c.op == 0   ? x < c.value
                       : c.op == 1 ? x > c.value
                       : c.op == 2 ? x <= c.value
                                   : x >= c.value;
      if (hit) {
        dirichlet[t] = 1;
        break;
      }
    }
}

Mesh make_icosphere(int level) {
  if (level < 0 || level > 10) throw ConfigError("icosphere level out of range");
  const Real g = (1.0 + std::sqrt(5.0)) / 2.0;
  std::vector<V3> v = {{-1, g, 0}, {1, g, 0},  {-1, -g, 0}, {1, -g, 0},
                       {0, -1, g}, {0, 1, g},  {0, -1, -g}, {0, 1, -g},
                       {g, 0, -1}, {g, 0, 1},  {-g, 0, -1}, {-g, 0, 1}};
  for (V3& p : v) {
    const Real r = vnorm(p);
    for (int d = 0; d < 3; ++d) p[d] /= r;
  }
  std::vector<std::array<int, 3>> f = {
      {0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
      {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
      {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
      {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
  for (int l = 0; l < level; ++l) {
    std::unordered_map<long long, int> mid;
    mid.reserve(f.size() * 2);
    auto midpoint = [&](int a, int b) {
      const long long key = static_cast<long long>(std::min(a, b)) << 32 |
                            static_cast<unsigned>(std::max(a, b));
      auto it = mid.find(key);
      if (it != mid.end()) return it->second;
      V3 m;
      for (int d = 0; d < 3; ++d) m[d] = 0.5 * (v[a][d] + v[b][d]);
      const Real r = vnorm(m);
      for (int d = 0; d < 3; ++d) m[d] /= r;
      const int id = static_cast<int>(v.size());
      v.push_back(m);
      mid.emplace(key, id);
      return id;
    };
    std::vector<std::array<int, 3>> nf;
    nf.reserve(f.size() * 4);
    for (const auto& t : f) {
      const int ab = midpoint(t[0], t[1]);
      const int bc = midpoint(t[1], t[2]);
      const int ca = midpoint(t[2], t[0]);
      nf.push_back({t[0], ab, ca});
      nf.push_back({t[1], bc, ab});
      nf.push_back({t[2], ca, bc});
      nf.push_back({ab, bc, ca});
    }
    f.swap(nf);
  }
  Mesh m;
  m.vertices = std::move(v);
  m.triangles = std::move(f);
  m.finish();
  return m;
}

Mesh make_ellipsoid(int level, Real ax, Real ay, Real az) {
  Mesh m = make_icosphere(level);
  for (V3& p : m.vertices) {
    p[0] *= ax;
    p[1] *= ay;
    p[2] *= az;
  }
  m.finish();
  return m;
}

Mesh make_voxel_cube(int n, Real lo, Real hi) {
  if (n < 1) throw ConfigError("voxel cube: n must be >= 1");
  Mesh m;
  auto coord = [&](int i) { return (lo * (n - i) + hi * i) / n; };
  const long long s = n + 1;
  std::unordered_map<long long, int> ids;
  auto vertex = [&](int i, int j, int k) {
    const long long key = (static_cast<long long>(i) * s + j) * s + k;
    auto it = ids.find(key);
    if (it != ids.end()) return it->second;
    const int id = m.nv();
    m.vertices.push_back({coord(i), coord(j), coord(k)});
    ids.emplace(key, id);
    return id;
  };
  // lattice tangents (u, v) with u x v = +d (meshgen.cpp:50-80)
  static const int tang[3][2] = {{1, 2}, {2, 0}, {0, 1}};
  auto outside = [&](int i) { return i < 0 || i >= n; };
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        const int cell[3] = {i, j, k};
        for (int d = 0; d < 3; ++d)
          for (int sg = -1; sg <= 1; sg += 2) {
            if (!outside(cell[d] + sg)) continue;  // neighbour inside the cube
            int base[3] = {i, j, k};
            if (sg > 0) base[d] += 1;
            int du[3] = {0, 0, 0}, dv[3] = {0, 0, 0};
            du[tang[d][0]] = 1;
            dv[tang[d][1]] = 1;
            auto c = [&](int a, int b) {
              return vertex(base[0] + a * du[0] + b * dv[0],
                            base[1] + a * du[1] + b * dv[1],
                            base[2] + a * du[2] + b * dv[2]);
            };
            const int c00 = c(0, 0), c10 = c(1, 0), c11 = c(1, 1), c01 = c(0, 1);
            if (sg > 0) {
              m.triangles.push_back({c00, c10, c11});
              m.triangles.push_back({c00, c11, c01});
            } else {
              m.triangles.push_back({c00, c11, c10});
              m.triangles.push_back({c00, c01, c11});
            }
          }
      }
  m.finish();
  return m;
}

Mesh load_off(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw MeshError("cannot open mesh file " + path);
  auto next = [&]() {
    std::string line;
    while (std::getline(in, line)) {
      const auto pos = line.find('#');
      if (pos != std::string::npos) line.erase(pos);
      if (line.find_first_not_of(" \t\r\n") != std::string::npos) return line;
    }
    throw MeshError("unexpected end of mesh file " + path);
  };
  {
    std::stringstream ss(next());
    std::string tag;
    ss >> tag;
    if (tag != "OFF") throw MeshError("mesh file " + path + ": missing OFF header");
  }
  int nv = 0, nt = 0, ne = 0;
  {
    std::stringstream ss(next());
    if (!(ss >> nv >> nt >> ne) || nv <= 0 || nt <= 0)
      throw MeshError("mesh file " + path + ": bad counts line");
  }
  Mesh m;
  m.vertices.resize(nv);
  for (int v = 0; v < nv; ++v) {
    std::stringstream ss(next());
    if (!(ss >> m.vertices[v][0] >> m.vertices[v][1] >> m.vertices[v][2]))
      throw MeshError("mesh file " + path + ": bad vertex line");
  }
  m.triangles.resize(nt);
  for (int t = 0; t < nt; ++t) {
    std::stringstream ss(next());
    int k = 0;
    auto& tri = m.triangles[t];
    if (!(ss >> k >> tri[0] >> tri[1] >> tri[2]) || k != 3)
      throw MeshError("mesh file " + path + ": bad triangle line");
    for (int i : tri)
      if (i < 0 || i >= nv)
        throw MeshError("mesh file " + path + ": vertex index out of range");
  }
  m.finish();
  m.validate_admissible();
  return m;
}

void save_off(const Mesh& m, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw MeshError("cannot write mesh file " + path);
  out << "OFF\n" << m.nv() << " " << m.nt() << " 0\n";
  char buf[128];
  for (const V3& v : m.vertices) {
    std::snprintf(buf, sizeof(buf), "%.17g %.17g %.17g\n", v[0], v[1], v[2]);
    out << buf;
  }
  for (const auto& t : m.triangles)
    out << "3 " << t[0] << " " << t[1] << " " << t[2] << "\n";
}

}  // namespace hmb
