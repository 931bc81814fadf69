// Cluster tree and admissible block partition (host side of the hot path).
//
// Same contract as the reference (proj/include/hmbem/cluster.hpp:13-99,
// proj/src/cluster.cpp:12-148) and bit-exact with it: AABB supports,
// longest-axis (first max) geometric bisection with a stable sort on support
// midpoints and the lower half taking the odd element, DFS pre-order node
// ids; admissibility-first quad-tree recursion in child order (0,0),(0,1),
// (1,0),(1,1).  Compiled with -ffp-contract=off.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "geometry.hpp"

namespace hmb {

struct Box {
  V3 lo, hi;
  Box();
  void absorb(const Box& o);
  void absorb(const V3& p);
  Real diameter() const;
};

Real box_distance(const Box& a, const Box& b);
// min(diam t, diam s) < eta * dist(t, s)   (cluster.cpp:21-24)
bool admissible(const Box& t, const Box& s, Real eta);

struct ClusterNode {
  int begin = 0, end = 0;  // [begin, end) in permuted (internal) order
  Box box;
  int child[2] = {-1, -1};
  int level = 0;
  int size() const { return end - begin; }
  bool is_leaf() const { return child[0] < 0; }
};

struct ClusterTree {
  std::vector<ClusterNode> nodes;  // nodes[0] = root, DFS pre-order
  std::vector<int> perm;           // internal position -> external id
  std::vector<int> inv_perm;       // external id -> internal position
  int b_min = 1;
  int depth = 0;
  int size() const { return static_cast<int>(perm.size()); }
  std::vector<int> leaves() const;  // leaf node ids in index order
};

ClusterTree build_cluster_tree(const std::vector<Box>& supports, int b_min);

// one support box per triangle from its three corners (operators.cpp:190-192)
std::vector<Box> triangle_supports(const Mesh& m);

struct BlockInfo {
  int row_node = 0, col_node = 0;
  bool admissible = false;
  int level = 0;
};

struct BlockPartition {
  const ClusterTree* rows = nullptr;
  const ClusterTree* cols = nullptr;
  std::vector<BlockInfo> blocks;
  Real eta = 0.0;
  int num_admissible() const;
  int tree_depth() const;
};

BlockPartition build_block_partition(const ClusterTree& rows,
                                     const ClusterTree& cols, Real eta);
int sparsity_constant(const BlockPartition& p);
// byte layout of nlohmann::json::dump(2) of partition_to_json
// (cluster.cpp:130-148): sorted keys, shortest round-trip doubles
std::string partition_to_json(const BlockPartition& p);

}  // namespace hmb
