#include "geometry.hpp"

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <fstream>
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

namespace {

// directed edge a -> b packed into one sortable key
inline std::uint64_t edge_key(int a, int b) {
  return (static_cast<std::uint64_t>(static_cast<std::uint32_t>(a)) << 32) |
         static_cast<std::uint32_t>(b);
}

}  // namespace

// Same acceptance rule as the reference's check (proj/src/mesh.cpp:68-101):
// every directed edge occurs once and its reverse exists (closed and
// consistently oriented), and no two triangles span the same vertex set.
// Implemented on sorted key arrays instead of ordered maps.
void Mesh::validate_admissible() const {
  std::vector<std::uint64_t> dir;
  dir.reserve(3 * triangles.size());
  for (const auto& tri : triangles) {
    dir.push_back(edge_key(tri[0], tri[1]));
    dir.push_back(edge_key(tri[1], tri[2]));
    dir.push_back(edge_key(tri[2], tri[0]));
  }
  std::sort(dir.begin(), dir.end());
  const auto dup = std::adjacent_find(dir.begin(), dir.end());
  if (dup != dir.end())
    throw MeshError("mesh is not admissible: directed edge " +
                    std::to_string(*dup >> 32) + "->" +
                    std::to_string(*dup & 0xffffffffu) + " used twice");
  for (const std::uint64_t k : dir) {
    const int a = static_cast<int>(k >> 32), b = static_cast<int>(k & 0xffffffffu);
    if (!std::binary_search(dir.begin(), dir.end(), edge_key(b, a)))
      throw MeshError("mesh is not admissible: boundary edge " + std::to_string(a) +
                      "->" + std::to_string(b) + " has no twin");
  }
  // duplicated faces: equal sorted vertex triples
  std::vector<std::pair<std::array<int, 3>, int>> faces(triangles.size());
  for (std::size_t t = 0; t < triangles.size(); ++t) {
    faces[t].first = triangles[t];
    std::sort(faces[t].first.begin(), faces[t].first.end());
    faces[t].second = static_cast<int>(t);
  }
  std::sort(faces.begin(), faces.end());
  for (std::size_t t = 1; t < faces.size(); ++t)
    if (faces[t].first == faces[t - 1].first)
      throw MeshError("mesh is not admissible: triangles " +
                      std::to_string(faces[t - 1].second) + " and " +
                      std::to_string(faces[t].second) + " span the same face");
}

namespace {

// One clause of a centroid predicate, e.g. "x3<=0": axis 0..2, comparison,
// threshold.  Grammar as documented by the reference (mesh.hpp:42-48): a
// '|'-separated disjunction of x<axis><op><value>, op in {<, >, <=, >=},
// whitespace ignored.
struct Clause {
  int axis = 0;
  char op = '<';      // '<' '>' 'l' (<=) 'g' (>=)
  Real value = 0.0;
  bool test(Real x) const {
    switch (op) {
      case '<': return x < value;
      case '>': return x > value;
      case 'l': return x <= value;
      default: return x >= value;
    }
  }
};

Clause parse_clause(const std::string& raw) {
  std::string t;
  for (char ch : raw)
    if (!std::isspace(static_cast<unsigned char>(ch))) t.push_back(ch);
  const auto bad = [&](const char* why) {
    return MeshError(std::string("dirichlet predicate: ") + why + " in clause '" + t + "'");
  };
  if (t.size() < 3 || t[0] != 'x' || t[1] < '1' || t[1] > '3')
    throw bad("expected x1, x2 or x3");
  Clause c;
  c.axis = t[1] - '1';
  std::size_t at = 2;
  const bool eq = at + 1 < t.size() && t[at + 1] == '=';
  if (t[at] == '<') c.op = eq ? 'l' : '<';
  else if (t[at] == '>') c.op = eq ? 'g' : '>';
  else throw bad("expected <, >, <= or >=");
  at += eq ? 2 : 1;
  const std::string num = t.substr(at);
  char* end = nullptr;
  errno = 0;
  c.value = num.empty() ? 0.0 : std::strtod(num.c_str(), &end);
  if (num.empty() || errno != 0 || end != num.c_str() + num.size())
    throw bad("expected a number");
  return c;
}

}  // namespace

void Mesh::label_dirichlet(const std::string& text) {
  std::vector<Clause> clauses;
  std::size_t from = 0;
  while (from <= text.size()) {
    const std::size_t bar = std::min(text.find('|', from), text.size());
    const std::string piece = text.substr(from, bar - from);
    if (piece.find_first_not_of(" \t\r\n") != std::string::npos)
      clauses.push_back(parse_clause(piece));
    from = bar + 1;
  }
  if (clauses.empty()) throw MeshError("dirichlet predicate '" + text + "' has no clauses");
  if (centroids.size() != triangles.size()) finish();
  dirichlet.assign(nt(), 0);
  for (int t = 0; t < nt(); ++t)
    dirichlet[t] = std::any_of(clauses.begin(), clauses.end(), [&](const Clause& c) {
      return c.test(centroids[t][c.axis]);
    });
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

// OFF reader (the format of the reference's load_mesh, mesh.cpp:180-219):
// "OFF", then "nv nt ne", nv vertex lines, nt lines "3 a b c"; '#' starts a
// comment.  The file is read as a stream of non-comment lines, each record on
// its own line.
Mesh load_off(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw MeshError("load_off: cannot read " + path);
  std::vector<std::string> lines;
  for (std::string raw; std::getline(in, raw);) {
    raw = raw.substr(0, raw.find('#'));
    if (raw.find_first_not_of(" \t\r\n") != std::string::npos) lines.push_back(raw);
  }
  std::size_t cur = 0;
  const auto record = [&](const char* what) -> std::istringstream {
    if (cur >= lines.size())
      throw MeshError("load_off: " + path + " ends before the " + what);
    return std::istringstream(lines[cur++]);
  };
  std::string magic;
  record("header") >> magic;
  if (magic != "OFF") throw MeshError("load_off: " + path + " is not an OFF file");
  long long nv = 0, nt = 0, ne = 0;
  if (!(record("size line") >> nv >> nt >> ne) || nv < 1 || nt < 1 || nv > INT32_MAX ||
      nt > INT32_MAX)
    throw MeshError("load_off: " + path + ": invalid size line");
  Mesh m;
  m.vertices.resize(static_cast<std::size_t>(nv));
  for (V3& v : m.vertices)
    if (!(record("vertex list") >> v[0] >> v[1] >> v[2]))
      throw MeshError("load_off: " + path + ": unreadable vertex record");
  m.triangles.resize(static_cast<std::size_t>(nt));
  for (auto& tri : m.triangles) {
    int corners = 0;
    if (!(record("face list") >> corners >> tri[0] >> tri[1] >> tri[2]) || corners != 3)
      throw MeshError("load_off: " + path + ": unreadable face record (triangles only)");
    if (*std::min_element(tri.begin(), tri.end()) < 0 ||
        *std::max_element(tri.begin(), tri.end()) >= nv)
      throw MeshError("load_off: " + path + ": face refers to a missing vertex");
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
