#include "cluster.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <numeric>
#include <unordered_map>

#include "errors.hpp"

namespace hmb {

namespace {
inline Real norm_ordered(Real x, Real y, Real z) {
  return std::sqrt((x * x + y * y) + z * z);
}
}  // namespace

Box::Box() {
  lo.fill(std::numeric_limits<Real>::max());
  hi.fill(std::numeric_limits<Real>::lowest());
}
void Box::absorb(const Box& o) {
  for (int d = 0; d < 3; ++d) {
    lo[d] = std::min(lo[d], o.lo[d]);
    hi[d] = std::max(hi[d], o.hi[d]);
  }
}
void Box::absorb(const V3& p) {
  for (int d = 0; d < 3; ++d) {
    lo[d] = std::min(lo[d], p[d]);
    hi[d] = std::max(hi[d], p[d]);
  }
}
Real Box::diameter() const {
  return norm_ordered(hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]);
}

Real box_distance(const Box& a, const Box& b) {
  Real g[3];
  for (int d = 0; d < 3; ++d)
    g[d] = std::max(std::max(a.lo[d] - b.hi[d], b.lo[d] - a.hi[d]), 0.0);
  return norm_ordered(g[0], g[1], g[2]);
}

bool admissible(const Box& t, const Box& s, Real eta) {
  if (eta <= 0.0) throw Error("admissible: eta must be positive");
  return std::min(t.diameter(), s.diameter()) < eta * box_distance(t, s);
}

std::vector<int> ClusterTree::leaves() const {
  std::vector<int> out;
  // DFS pre-order visits leaves left to right, i.e. in index order
  for (std::size_t i = 0; i < nodes.size(); ++i)
    if (nodes[i].is_leaf()) out.push_back(static_cast<int>(i));
  return out;
}

namespace {

// Explicit-stack construction producing the same DFS pre-order ids as the
// reference's recursion (cluster.cpp:33-60): a node's id is assigned when it
// is popped, left child is processed before the right one.
struct Pending {
  int begin, end, level, parent, slot;
};

}  // namespace

ClusterTree build_cluster_tree(const std::vector<Box>& sup, int b_min) {
  if (sup.empty()) throw Error("build_cluster_tree: empty support set");
  if (b_min < 1) throw Error("build_cluster_tree: b_min must be >= 1");
  const int n = static_cast<int>(sup.size());
  // support midpoints per axis, precomputed (0.5 * (lo + hi) per component)
  std::vector<Real> mid[3];
  for (int d = 0; d < 3; ++d) {
    mid[d].resize(n);
    for (int i = 0; i < n; ++i) mid[d][i] = 0.5 * (sup[i].lo[d] + sup[i].hi[d]);
  }
  ClusterTree tree;
  tree.b_min = b_min;
  tree.perm.resize(n);
  std::iota(tree.perm.begin(), tree.perm.end(), 0);
  std::vector<Pending> stack = {{0, n, 0, -1, 0}};
  while (!stack.empty()) {
    const Pending job = stack.back();
    stack.pop_back();
    const int id = static_cast<int>(tree.nodes.size());
    tree.nodes.emplace_back();
    if (job.parent >= 0) tree.nodes[job.parent].child[job.slot] = id;
    ClusterNode& node = tree.nodes.back();
    node.begin = job.begin;
    node.end = job.end;
    node.level = job.level;
    tree.depth = std::max(tree.depth, job.level);
    Box box;
    for (int p = job.begin; p < job.end; ++p) box.absorb(sup[tree.perm[p]]);
    node.box = box;
    if (job.end - job.begin <= b_min) continue;
    int axis = 0;
    for (int d = 1; d < 3; ++d)
      if (box.hi[d] - box.lo[d] > box.hi[axis] - box.lo[axis]) axis = d;
    const std::vector<Real>& key = mid[axis];
    std::stable_sort(tree.perm.begin() + job.begin, tree.perm.begin() + job.end,
                     [&key](int a, int b) { return key[a] < key[b]; });
    const int m = job.begin + (job.end - job.begin + 1) / 2;
    // push right first so the left subtree is numbered first
    stack.push_back({m, job.end, job.level + 1, id, 1});
    stack.push_back({job.begin, m, job.level + 1, id, 0});
  }
  tree.inv_perm.resize(n);
  for (int p = 0; p < n; ++p) tree.inv_perm[tree.perm[p]] = p;
  return tree;
}

std::vector<Box> triangle_supports(const Mesh& m) {
  std::vector<Box> boxes(m.nt());
  for (int t = 0; t < m.nt(); ++t)
    for (int k = 0; k < 3; ++k) boxes[t].absorb(m.corner(t, k));
  return boxes;
}

int BlockPartition::num_admissible() const {
  int n = 0;
  for (const auto& b : blocks) n += b.admissible;
  return n;
}
int BlockPartition::tree_depth() const {
  return std::max(rows->depth, cols->depth);
}

BlockPartition build_block_partition(const ClusterTree& rows,
                                     const ClusterTree& cols, Real eta) {
  if (eta <= 0.0) throw Error("admissible: eta must be positive");
  BlockPartition p;
  p.rows = &rows;
  p.cols = &cols;
  p.eta = eta;
  // explicit stack, children pushed in reverse so that (0,0),(0,1),(1,0),
  // (1,1) come out in the reference's recursion order (cluster.cpp:82-97)
  struct Job {
    int t, s, level;
  };
  std::vector<Job> stack = {{0, 0, 0}};
  while (!stack.empty()) {
    const Job j = stack.back();
    stack.pop_back();
    const ClusterNode& rn = rows.nodes[j.t];
    const ClusterNode& cn = cols.nodes[j.s];
    if (admissible(rn.box, cn.box, eta)) {
      p.blocks.push_back({j.t, j.s, true, j.level});
    } else if (rn.is_leaf() || cn.is_leaf()) {
      p.blocks.push_back({j.t, j.s, false, j.level});
    } else {
      for (int a = 1; a >= 0; --a)
        for (int b = 1; b >= 0; --b)
          stack.push_back({rn.child[a], cn.child[b], j.level + 1});
    }
  }
  return p;
}

int sparsity_constant(const BlockPartition& p) {
  std::vector<int> rc(p.rows->nodes.size(), 0), cc(p.cols->nodes.size(), 0);
  int c_sp = 0;
  for (const auto& b : p.blocks) {
    c_sp = std::max(c_sp, ++rc[b.row_node]);
    c_sp = std::max(c_sp, ++cc[b.col_node]);
  }
  return c_sp;
}

namespace {
std::string shortest_double(Real v) {
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}
}  // namespace

std::string partition_to_json(const BlockPartition& p) {
  std::string o;
  o.reserve(p.blocks.size() * 140 + 256);
  o += "{\n  \"beta\": " + shortest_double(p.eta) + ",\n  \"blocks\": [";
  bool first = true;
  for (const BlockInfo& b : p.blocks) {
    o += first ? "\n" : ",\n";
    first = false;
    o += "    {\n      \"admissible\": ";
    o += b.admissible ? "true" : "false";
    o += ",\n      \"col_node\": " + std::to_string(b.col_node);
    o += ",\n      \"cols\": " + std::to_string(p.cols->nodes[b.col_node].size());
    o += ",\n      \"level\": " + std::to_string(b.level);
    o += ",\n      \"row_node\": " + std::to_string(b.row_node);
    o += ",\n      \"rows\": " + std::to_string(p.rows->nodes[b.row_node].size());
    o += "\n    }";
  }
  o += p.blocks.empty() ? "]" : "\n  ]";
  o += ",\n  \"c_sp\": " + std::to_string(sparsity_constant(p));
  o += ",\n  \"cols\": " + std::to_string(p.cols->size());
  o += ",\n  \"depth\": " + std::to_string(p.tree_depth());
  o += ",\n  \"rows\": " + std::to_string(p.rows->size()) + "\n}";
  return o;
}

}  // namespace hmb
