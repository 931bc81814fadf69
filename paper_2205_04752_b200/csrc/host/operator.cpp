#include "operator.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>

#include "errors.hpp"
#include "hmgpu.h"

namespace hmb {

namespace {

const int kCompR[6] = {0, 0, 0, 1, 1, 2};
const int kCompC[6] = {0, 1, 2, 1, 2, 2};

int check_status(hmgpu_ctx* ctx, int st, const char* what) {
  if (st == HMGPU_OK) return st;
  const std::string msg =
      std::string(what) + ": " + (ctx ? hmgpu_last_error(ctx) : "no context");
  if (st == HMGPU_ERR_DIMENSION) throw DimensionError(msg);
  if (st == HMGPU_ERR_INVALID) throw Error(msg);
  throw DeviceError(st, msg);
}

std::vector<int> nodes4(const ClusterTree& t) {
  std::vector<int> out(4 * t.nodes.size());
  for (std::size_t i = 0; i < t.nodes.size(); ++i) {
    out[4 * i] = t.nodes[i].begin;
    out[4 * i + 1] = t.nodes[i].end;
    out[4 * i + 2] = t.nodes[i].child[0];
    out[4 * i + 3] = t.nodes[i].child[1];
  }
  return out;
}

}  // namespace

void HOperator::check(int status, const char* what) const {
  check_status(ctx_, status, what);
}

HOperator::~HOperator() {
  if (ctx_) hmgpu_destroy(ctx_);
}

long long HOperator::rows() const {
  return static_cast<long long>(n_rows_) * (ncomp_ == 6 ? 3 : 1);
}
long long HOperator::cols() const {
  return static_cast<long long>(n_cols_) * (ncomp_ == 6 ? 3 : 1);
}

// Block-row shard: the first tree level with >= count nodes (plus shallower
// leaves) is split into `count` contiguous runs; every block's row cluster
// must fall inside one run (true for the eta = 1 partitions, whose blocks
// start below the top levels).
void HOperator::init_partition(Real eta, Shard shard) {
  part_ = build_block_partition(*rows_, col_tree(), eta);
  if (shard.count < 1 || shard.rank < 0 || shard.rank >= shard.count)
    throw ConfigError("bad shard (rank, count)");
  row_begin_ = 0;
  row_end_ = n_rows_;
  if (shard.count == 1) return;
  const ClusterTree& t = *rows_;
  int level = 0;
  std::vector<int> frontier;
  for (;; ++level) {
    frontier.clear();
    for (std::size_t i = 0; i < t.nodes.size(); ++i) {
      const ClusterNode& nd = t.nodes[i];
      if (nd.level == level || (nd.is_leaf() && nd.level < level))
        frontier.push_back(static_cast<int>(i));
    }
    if (static_cast<int>(frontier.size()) >= shard.count || level > t.depth) break;
  }
  if (static_cast<int>(frontier.size()) < shard.count)
    throw ConfigError("more shards than row clusters");
  std::sort(frontier.begin(), frontier.end(), [&](int a, int b) {
    return t.nodes[a].begin < t.nodes[b].begin;
  });
  const int nf = static_cast<int>(frontier.size());
  std::vector<int> owner(n_rows_, 0);
  for (int f = 0; f < nf; ++f) {
    const int r = static_cast<int>(static_cast<long long>(f) * shard.count / nf);
    const ClusterNode& nd = t.nodes[frontier[f]];
    for (int p = nd.begin; p < nd.end; ++p) owner[p] = r;
    if (r == shard.rank) {
      if (row_end_ == n_rows_ && row_begin_ == 0) row_begin_ = nd.begin;
      row_end_ = nd.end;
    }
  }
  // first frontier node of this rank gives the begin (reset above)
  for (int f = 0; f < nf; ++f)
    if (static_cast<int>(static_cast<long long>(f) * shard.count / nf) == shard.rank) {
      row_begin_ = t.nodes[frontier[f]].begin;
      break;
    }
  for (const BlockInfo& b : part_.blocks) {
    const ClusterNode& rn = t.nodes[b.row_node];
    if (owner[rn.begin] != owner[rn.end - 1])
      throw ConfigError("a partition block spans two shards; use fewer GPUs");
  }
}

std::unique_ptr<HOperator> HOperator::kelvin(const Mesh& mesh, Real E, Real nu,
                                             int b_min, Real eta, int device,
                                             Shard shard, QuadratureConfig qc) {
  if (mesh.centroids.size() != mesh.triangles.size())
    throw MeshError("mesh geometry caches missing (call finish())");
  if (E <= 0.0) throw Error("lame_constants: E must be positive");
  if (nu <= 0.0 || nu >= 0.5) throw Error("lame_constants: nu must lie in (0, 1/2)");
  std::unique_ptr<HOperator> op(new HOperator());
  op->kind_ = Kelvin;
  op->ncomp_ = 6;
  op->n_rows_ = op->n_cols_ = mesh.nt();
  op->rows_ = std::make_unique<ClusterTree>(
      build_cluster_tree(triangle_supports(mesh), b_min));
  op->init_partition(eta, shard);
  if (device < 0) return op;  // host-only: tree and partition
  op->check(hmgpu_create(device, &op->ctx_), "hmgpu_create");
  std::vector<double> verts(3 * mesh.nv()), cen(3 * mesh.nt());
  std::vector<int> tris(3 * mesh.nt());
  for (int v = 0; v < mesh.nv(); ++v)
    for (int d = 0; d < 3; ++d) verts[3 * v + d] = mesh.vertices[v][d];
  for (int t = 0; t < mesh.nt(); ++t)
    for (int d = 0; d < 3; ++d) {
      tris[3 * t + d] = mesh.triangles[t][d];
      cen[3 * t + d] = mesh.centroids[t][d];
    }
  op->check(hmgpu_set_kelvin_geometry(op->ctx_, mesh.nv(), verts.data(), mesh.nt(),
                                      tris.data(), cen.data(), mesh.areas.data(),
                                      mesh.diam.data(), E, nu),
            "hmgpu_set_kelvin_geometry");
  for (int tier = 0; tier < 3; ++tier) {
    const TriangleRule r = gauss_rule(qc.tier_order(tier));
    op->check(hmgpu_set_rule(op->ctx_, tier, static_cast<int>(r.w.size()), r.a.data(),
                             r.b.data(), r.w.data()),
              "hmgpu_set_rule");
  }
  op->check(hmgpu_set_tier_ratios(op->ctx_, qc.far_ratio, qc.mid_ratio),
            "hmgpu_set_tier_ratios");
  return op;
}

namespace {
// distance from p to the triangle (a, b, c): the plane projection when it
// falls inside, else the nearest edge point (validation threshold only)
Real point_triangle_distance(const V3& p, const V3& a, const V3& b, const V3& c) {
  auto sub = [](const V3& x, const V3& y) { return V3{x[0] - y[0], x[1] - y[1], x[2] - y[2]}; };
  auto dot = [](const V3& x, const V3& y) { return x[0] * y[0] + x[1] * y[1] + x[2] * y[2]; };
  auto seg = [&](const V3& u, const V3& v) {
    const V3 d = sub(v, u), w = sub(p, u);
    Real t = dot(w, d) / dot(d, d);
    t = std::min(1.0, std::max(0.0, t));
    const V3 q{u[0] + t * d[0] - p[0], u[1] + t * d[1] - p[1], u[2] + t * d[2] - p[2]};
    return std::sqrt(dot(q, q));
  };
  const V3 e0 = sub(b, a), e1 = sub(c, a), w = sub(p, a);
  const Real a00 = dot(e0, e0), a01 = dot(e0, e1), a11 = dot(e1, e1);
  const Real det = a00 * a11 - a01 * a01;
  const Real s = (a11 * dot(w, e0) - a01 * dot(w, e1)) / det;
  const Real t = (a00 * dot(w, e1) - a01 * dot(w, e0)) / det;
  if (s >= 0 && t >= 0 && s + t <= 1) {
    const V3 q{a[0] + s * e0[0] + t * e1[0] - p[0], a[1] + s * e0[1] + t * e1[1] - p[1],
               a[2] + s * e0[2] + t * e1[2] - p[2]};
    return std::sqrt(dot(q, q));
  }
  return std::min({seg(a, b), seg(b, c), seg(c, a)});
}
}  // namespace

namespace {
void check_interior_points(const Mesh& mesh, const std::vector<V3>& points,
                           Real min_distance_factor) {
  Real max_diam = 0.0;
  for (Real d : mesh.diam) max_diam = std::max(max_diam, d);
  const Real min_dist = min_distance_factor * max_diam;
  for (size_t i = 0; i < points.size(); ++i) {
    Real d = std::numeric_limits<Real>::max();
    for (int t = 0; t < mesh.nt() && d > min_dist; ++t)
      d = std::min(d, point_triangle_distance(points[i], mesh.corner(t, 0), mesh.corner(t, 1),
                                              mesh.corner(t, 2)));
    if (d <= min_dist)
      throw Error("evaluate_interior: point " + std::to_string(i) +
                  " is closer to the surface than the quadrature threshold");
  }
}
}  // namespace

std::unique_ptr<HOperator> HOperator::kelvin_double_points(
    const Mesh& mesh, const std::vector<V3>& points, int r, int c, Real E, Real nu, int b_min,
    Real eta, int device, Shard shard, Real min_distance_factor, QuadratureConfig qc) {
  if (mesh.normals.size() != mesh.triangles.size())
    throw MeshError("mesh geometry caches missing (call finish())");
  if (points.empty()) throw Error("evaluate_interior: no points");
  if (E <= 0.0) throw Error("lame_constants: E must be positive");
  if (nu <= 0.0 || nu >= 0.5) throw Error("lame_constants: nu must lie in (0, 1/2)");
  if (r < 0 || r > 2 || c < 0 || c > 2) throw Error("double layer: cell (r, c) in 0..2");
  check_interior_points(mesh, points, min_distance_factor);
  std::unique_ptr<HOperator> op(new HOperator());
  op->kind_ = Kelvin;
  op->ncomp_ = 1;
  op->n_rows_ = static_cast<int>(points.size());
  op->n_cols_ = mesh.nv();
  std::vector<Box> pb(points.size());
  for (size_t i = 0; i < points.size(); ++i) pb[i].absorb(points[i]);
  const std::vector<Box> tb = triangle_supports(mesh);
  std::vector<Box> nb(mesh.nv());
  for (int t = 0; t < mesh.nt(); ++t)
    for (int k = 0; k < 3; ++k) nb[mesh.triangles[t][k]].absorb(tb[t]);
  op->rows_ = std::make_unique<ClusterTree>(build_cluster_tree(pb, b_min));
  op->cols_ = std::make_unique<ClusterTree>(build_cluster_tree(nb, b_min));
  op->init_partition(eta, shard);
  if (device < 0) return op;
  op->check(hmgpu_create(device, &op->ctx_), "hmgpu_create");
  std::vector<double> verts(3 * mesh.nv()), cen(3 * mesh.nt()), nrm(3 * mesh.nt()),
      ep(3 * points.size());
  std::vector<int> tris(3 * mesh.nt());
  for (int v = 0; v < mesh.nv(); ++v)
    for (int d = 0; d < 3; ++d) verts[3 * v + d] = mesh.vertices[v][d];
  for (int t = 0; t < mesh.nt(); ++t)
    for (int d = 0; d < 3; ++d) {
      tris[3 * t + d] = mesh.triangles[t][d];
      cen[3 * t + d] = mesh.centroids[t][d];
      nrm[3 * t + d] = mesh.normals[t][d];
    }
  for (size_t i = 0; i < points.size(); ++i)
    for (int d = 0; d < 3; ++d) ep[3 * i + d] = points[i][d];
  op->check(hmgpu_set_kdouble_geometry(op->ctx_, mesh.nv(), verts.data(), mesh.nt(),
                                       tris.data(), cen.data(), mesh.areas.data(),
                                       mesh.diam.data(), nrm.data(), E, nu, r, c),
            "hmgpu_set_kdouble_geometry");
  op->check(hmgpu_set_eval_points(op->ctx_, static_cast<int>(points.size()), ep.data()),
            "hmgpu_set_eval_points");
  for (int tier = 0; tier < 3; ++tier) {
    const TriangleRule rr = gauss_rule(qc.tier_order(tier));
    op->check(hmgpu_set_rule(op->ctx_, tier, static_cast<int>(rr.w.size()), rr.a.data(),
                             rr.b.data(), rr.w.data()),
              "hmgpu_set_rule");
  }
  op->check(hmgpu_set_tier_ratios(op->ctx_, qc.far_ratio, qc.mid_ratio),
            "hmgpu_set_tier_ratios");
  return op;
}

std::unique_ptr<HOperator> HOperator::kelvin_points(const Mesh& mesh,
                                                    const std::vector<V3>& points, Real E,
                                                    Real nu, int b_min, Real eta, int device,
                                                    Shard shard, Real min_distance_factor,
                                                    QuadratureConfig qc) {
  if (mesh.centroids.size() != mesh.triangles.size())
    throw MeshError("mesh geometry caches missing (call finish())");
  if (points.empty()) throw Error("evaluate_interior: no points");
  if (E <= 0.0) throw Error("lame_constants: E must be positive");
  if (nu <= 0.0 || nu >= 0.5) throw Error("lame_constants: nu must lie in (0, 1/2)");
  check_interior_points(mesh, points, min_distance_factor);
  std::unique_ptr<HOperator> op(new HOperator());
  op->kind_ = Kelvin;
  op->ncomp_ = 6;
  op->n_rows_ = static_cast<int>(points.size());
  op->n_cols_ = mesh.nt();
  std::vector<Box> pb(points.size());
  for (size_t i = 0; i < points.size(); ++i) pb[i].absorb(points[i]);
  op->rows_ = std::make_unique<ClusterTree>(build_cluster_tree(pb, b_min));
  op->cols_ = std::make_unique<ClusterTree>(
      build_cluster_tree(triangle_supports(mesh), b_min));
  op->init_partition(eta, shard);
  if (device < 0) return op;
  op->check(hmgpu_create(device, &op->ctx_), "hmgpu_create");
  std::vector<double> verts(3 * mesh.nv()), cen(3 * mesh.nt()), ep(3 * points.size());
  std::vector<int> tris(3 * mesh.nt());
  for (int v = 0; v < mesh.nv(); ++v)
    for (int d = 0; d < 3; ++d) verts[3 * v + d] = mesh.vertices[v][d];
  for (int t = 0; t < mesh.nt(); ++t)
    for (int d = 0; d < 3; ++d) {
      tris[3 * t + d] = mesh.triangles[t][d];
      cen[3 * t + d] = mesh.centroids[t][d];
    }
  for (size_t i = 0; i < points.size(); ++i)
    for (int d = 0; d < 3; ++d) ep[3 * i + d] = points[i][d];
  op->check(hmgpu_set_kelvin_geometry(op->ctx_, mesh.nv(), verts.data(), mesh.nt(),
                                      tris.data(), cen.data(), mesh.areas.data(),
                                      mesh.diam.data(), E, nu),
            "hmgpu_set_kelvin_geometry");
  op->check(hmgpu_set_eval_points(op->ctx_, static_cast<int>(points.size()), ep.data()),
            "hmgpu_set_eval_points");
  for (int tier = 0; tier < 3; ++tier) {
    const TriangleRule r = gauss_rule(qc.tier_order(tier));
    op->check(hmgpu_set_rule(op->ctx_, tier, static_cast<int>(r.w.size()), r.a.data(),
                             r.b.data(), r.w.data()),
              "hmgpu_set_rule");
  }
  op->check(hmgpu_set_tier_ratios(op->ctx_, qc.far_ratio, qc.mid_ratio),
            "hmgpu_set_tier_ratios");
  return op;
}

std::unique_ptr<HOperator> HOperator::galerkin(const Mesh& mesh, int which, int b_min,
                                               Real eta, int device, Shard shard,
                                               QuadratureConfig qc, GalerkinQuadrature gq) {
  if (mesh.centroids.size() != mesh.triangles.size())
    throw MeshError("mesh geometry caches missing (call finish())");
  if (which != 0 && which != 1) throw Error("galerkin: which must be 0 (V_kl) or 1 (V_Delta)");
  std::unique_ptr<HOperator> op(new HOperator());
  op->kind_ = Galerkin;
  op->ncomp_ = which == 0 ? 6 : 1;
  op->n_rows_ = op->n_cols_ = mesh.nt();
  op->rows_ = std::make_unique<ClusterTree>(
      build_cluster_tree(triangle_supports(mesh), b_min));
  op->init_partition(eta, shard);
  if (device < 0) return op;
  op->check(hmgpu_create(device, &op->ctx_), "hmgpu_create");
  std::vector<double> verts(3 * mesh.nv()), cen(3 * mesh.nt());
  std::vector<int> tris(3 * mesh.nt());
  for (int v = 0; v < mesh.nv(); ++v)
    for (int d = 0; d < 3; ++d) verts[3 * v + d] = mesh.vertices[v][d];
  for (int t = 0; t < mesh.nt(); ++t)
    for (int d = 0; d < 3; ++d) {
      tris[3 * t + d] = mesh.triangles[t][d];
      cen[3 * t + d] = mesh.centroids[t][d];
    }
  op->check(hmgpu_set_galerkin_geometry(op->ctx_, mesh.nv(), verts.data(), mesh.nt(),
                                        tris.data(), cen.data(), mesh.areas.data(),
                                        mesh.diam.data(), which),
            "hmgpu_set_galerkin_geometry");
  // disjoint pairs: tensor rules of orders 2 / 4 / 5 (disjoint_order,
  // kernels.cpp:75-85 with the default disjoint_order 4)
  for (int tier = 0; tier < 3; ++tier) {
    const TriangleRule r = gauss_rule(qc.tier_order(tier));
    op->check(hmgpu_set_rule(op->ctx_, tier, static_cast<int>(r.w.size()), r.a.data(),
                             r.b.data(), r.w.data()),
              "hmgpu_set_rule");
  }
  // touching pairs: singular_order for vertex / edge, + identical_bump for
  // coincident pairs (GalerkinKernels constructor, kernels.cpp:62-73)
  for (int pc = 1; pc <= 3; ++pc) {
    const PairRuleTable r = singular_pair_rule(
        pc, gq.singular_order + (pc == 3 ? gq.identical_bump : 0));
    op->check(hmgpu_set_pair_rule(op->ctx_, pc, static_cast<int>(r.w.size()), r.xr1.data(),
                                  r.xr2.data(), r.yr1.data(), r.yr2.data(), r.w.data()),
              "hmgpu_set_pair_rule");
  }
  return op;
}

std::unique_ptr<HOperator> HOperator::kdelta(const Mesh& mesh, int b_min, Real eta,
                                             int device, Shard shard, QuadratureConfig qc,
                                             GalerkinQuadrature gq) {
  if (mesh.centroids.size() != mesh.triangles.size())
    throw MeshError("mesh geometry caches missing (call finish())");
  std::unique_ptr<HOperator> op(new HOperator());
  op->kind_ = KDelta;
  op->ncomp_ = 1;
  op->n_rows_ = mesh.nt();
  op->n_cols_ = mesh.nv();
  const std::vector<Box> tb = triangle_supports(mesh);
  std::vector<Box> nb(mesh.nv());
  for (int t = 0; t < mesh.nt(); ++t)
    for (int k = 0; k < 3; ++k) nb[mesh.triangles[t][k]].absorb(tb[t]);
  op->rows_ = std::make_unique<ClusterTree>(build_cluster_tree(tb, b_min));
  op->cols_ = std::make_unique<ClusterTree>(build_cluster_tree(nb, b_min));
  op->init_partition(eta, shard);
  if (device < 0) return op;
  op->check(hmgpu_create(device, &op->ctx_), "hmgpu_create");
  std::vector<double> verts(3 * mesh.nv()), cen(3 * mesh.nt()), nrm(3 * mesh.nt());
  std::vector<int> tris(3 * mesh.nt());
  for (int v = 0; v < mesh.nv(); ++v)
    for (int d = 0; d < 3; ++d) verts[3 * v + d] = mesh.vertices[v][d];
  for (int t = 0; t < mesh.nt(); ++t)
    for (int d = 0; d < 3; ++d) {
      tris[3 * t + d] = mesh.triangles[t][d];
      cen[3 * t + d] = mesh.centroids[t][d];
      nrm[3 * t + d] = mesh.normals[t][d];
    }
  op->check(hmgpu_set_kdelta_geometry(op->ctx_, mesh.nv(), verts.data(), mesh.nt(),
                                      tris.data(), cen.data(), mesh.areas.data(),
                                      mesh.diam.data(), nrm.data()),
            "hmgpu_set_kdelta_geometry");
  for (int tier = 0; tier < 3; ++tier) {
    const TriangleRule r = gauss_rule(qc.tier_order(tier));
    op->check(hmgpu_set_rule(op->ctx_, tier, static_cast<int>(r.w.size()), r.a.data(),
                             r.b.data(), r.w.data()),
              "hmgpu_set_rule");
  }
  for (int pc = 1; pc <= 3; ++pc) {
    const PairRuleTable r = singular_pair_rule(
        pc, gq.singular_order + (pc == 3 ? gq.identical_bump : 0));
    op->check(hmgpu_set_pair_rule(op->ctx_, pc, static_cast<int>(r.w.size()), r.xr1.data(),
                                  r.xr2.data(), r.yr1.data(), r.yr2.data(), r.w.data()),
              "hmgpu_set_pair_rule");
  }
  return op;
}

std::unique_ptr<HOperator> HOperator::newton(const std::vector<V3>& pts,
                                             const std::vector<Box>* boxes,
                                             Real diag, int b_min, Real eta,
                                             int device, Shard shard) {
  std::unique_ptr<HOperator> op(new HOperator());
  op->kind_ = Newton;
  op->ncomp_ = 1;
  op->n_rows_ = op->n_cols_ = static_cast<int>(pts.size());
  std::vector<Box> b;
  if (boxes) {
    b = *boxes;
  } else {
    b.resize(pts.size());
    for (std::size_t i = 0; i < pts.size(); ++i) b[i].absorb(pts[i]);
  }
  op->rows_ = std::make_unique<ClusterTree>(build_cluster_tree(b, b_min));
  op->init_partition(eta, shard);
  if (device < 0) return op;
  op->check(hmgpu_create(device, &op->ctx_), "hmgpu_create");
  std::vector<double> flat(3 * pts.size());
  for (std::size_t i = 0; i < pts.size(); ++i)
    for (int d = 0; d < 3; ++d) flat[3 * i + d] = pts[i][d];
  op->check(hmgpu_set_points(op->ctx_, static_cast<int>(pts.size()), flat.data(), diag),
            "hmgpu_set_points");
  return op;
}

std::unique_ptr<HOperator> HOperator::dense(int m, int n, const double* a,
                                            const std::vector<V3>& row_pts,
                                            const std::vector<V3>& col_pts,
                                            int b_min, Real eta, int device,
                                            Shard shard) {
  if (static_cast<int>(row_pts.size()) != m || static_cast<int>(col_pts.size()) != n)
    throw DimensionError("dense operator: point counts do not match the matrix");
  std::unique_ptr<HOperator> op(new HOperator());
  op->kind_ = Dense;
  op->ncomp_ = 1;
  op->n_rows_ = m;
  op->n_cols_ = n;
  std::vector<Box> rb(m), cb(n);
  for (int i = 0; i < m; ++i) rb[i].absorb(row_pts[i]);
  for (int j = 0; j < n; ++j) cb[j].absorb(col_pts[j]);
  op->rows_ = std::make_unique<ClusterTree>(build_cluster_tree(rb, b_min));
  op->cols_ = std::make_unique<ClusterTree>(build_cluster_tree(cb, b_min));
  op->init_partition(eta, shard);
  if (device < 0) return op;
  op->check(hmgpu_create(device, &op->ctx_), "hmgpu_create");
  op->check(hmgpu_set_dense_matrix(op->ctx_, m, n, a), "hmgpu_set_dense_matrix");
  return op;
}

AssemblyStats HOperator::assemble(const AssemblyConfig& cfg) {
  if (!ctx_) throw DeviceError(HMGPU_ERR_NODEVICE, "assemble: operator has no device");
  const ClusterTree& ct = col_tree();
  const std::vector<int> rn = nodes4(*rows_), cn = nodes4(ct);
  std::vector<int> bl(4 * part_.blocks.size());
  for (std::size_t b = 0; b < part_.blocks.size(); ++b) {
    bl[4 * b] = part_.blocks[b].row_node;
    bl[4 * b + 1] = part_.blocks[b].col_node;
    bl[4 * b + 2] = part_.blocks[b].admissible ? 1 : 0;
    bl[4 * b + 3] = part_.blocks[b].level;
  }
  check(hmgpu_set_partition(ctx_, n_rows_, rows_->perm.data(),
                            static_cast<int>(rows_->nodes.size()), rn.data(), n_cols_,
                            ct.perm.data(), static_cast<int>(ct.nodes.size()), cn.data(),
                            static_cast<int>(part_.blocks.size()), bl.data(),
                            row_begin_, row_end_),
        "hmgpu_set_partition");
  hmgpu_assembly_stats s{};
  check(hmgpu_assemble(ctx_, cfg.eps, cfg.beta, cfg.initial_rank, cfg.lookahead,
                       cfg.max_rank, &s),
        "hmgpu_assemble");
  cfg_ = cfg;
  assembled_ = true;
  AssemblyStats out;
  out.aca_entries = s.aca_entries;
  out.dense_entries = s.dense_entries;
  out.aca_steps = s.aca_steps;
  out.pivots = s.pivots;
  out.ms_total = s.ms_total;
  out.ms_nearfield = s.ms_nearfield;
  out.ms_aca = s.ms_aca;
  out.relaunches = s.aca_relaunches;
  out.counted_flops = s.counted_flops;
  return out;
}

void HOperator::matvec(const double* x, double* y, int nrhs, Mode mode,
                       bool device_ptrs) const {
  if (!assembled_) throw Error("matvec: operator not assembled");
  check(hmgpu_matvec(ctx_, x, y, nrhs, static_cast<int>(mode),
                     device_ptrs ? HMGPU_PTR_DEVICE : HMGPU_PTR_HOST),
        "hmgpu_matvec");
}

void HOperator::matvec_transposed(const double* x, double* y, int nrhs, Mode mode,
                                  bool device_ptrs) const {
  if (!assembled_) throw Error("matvec_transposed: operator not assembled");
  check(hmgpu_matvec_transposed(ctx_, x, y, nrhs, static_cast<int>(mode),
                                device_ptrs ? HMGPU_PTR_DEVICE : HMGPU_PTR_HOST),
        "hmgpu_matvec_transposed");
}

std::vector<double> HOperator::matvec(const std::vector<double>& x, Mode mode) const {
  if (static_cast<long long>(x.size()) != cols())
    throw DimensionError("HMatrix::matvec: size");
  std::vector<double> y(rows());
  matvec(x.data(), y.data(), 1, mode);
  return y;
}

void HOperator::promote(const std::vector<std::pair<int, int>>& cb) {
  std::vector<int> flat;
  for (auto& p : cb) {
    flat.push_back(p.first);
    flat.push_back(p.second);
  }
  check(hmgpu_promote(ctx_, static_cast<int>(cb.size()), flat.data()), "hmgpu_promote");
}

void HOperator::extend_lookahead(const std::vector<std::pair<int, int>>& cb, int steps) {
  std::vector<int> flat;
  for (auto& p : cb) {
    flat.push_back(p.first);
    flat.push_back(p.second);
  }
  check(hmgpu_extend(ctx_, static_cast<int>(cb.size()), flat.data(), steps),
        "hmgpu_extend");
}

void HOperator::ranks(std::vector<int>& k_cur, std::vector<int>& k_look,
                      std::vector<int>* consumed, std::vector<int>* last_stop) const {
  const std::size_t n = static_cast<std::size_t>(ncomp_) * part_.blocks.size();
  k_cur.resize(n);
  k_look.resize(n);
  if (consumed) consumed->resize(n);
  if (last_stop) last_stop->resize(n);
  check(hmgpu_ranks(ctx_, k_cur.data(), k_look.data(),
                    consumed ? consumed->data() : nullptr,
                    last_stop ? last_stop->data() : nullptr),
        "hmgpu_ranks");
}

long long HOperator::total_pivots() const {
  hmgpu_storage_info s{};
  check(hmgpu_storage(ctx_, &s), "hmgpu_storage");
  return s.pivots;
}

double HOperator::storage_mb_current() const {
  hmgpu_storage_info s{};
  check(hmgpu_storage(ctx_, &s), "hmgpu_storage");
  return s.mb_current;
}
double HOperator::storage_mb_tail() const {
  hmgpu_storage_info s{};
  check(hmgpu_storage(ctx_, &s), "hmgpu_storage");
  return s.mb_tail;
}
long long HOperator::matvec_bytes() const {
  hmgpu_storage_info s{};
  check(hmgpu_storage(ctx_, &s), "hmgpu_storage");
  return s.matvec_bytes;
}

// ---------------------------------------------------------------------------
// gamma_contributions (amvm.cpp:46-125): the device returns the tail
// products of every (comp, block) with a look-ahead tail, grouped by
// component (= by H-matrix in first-appearance order); the host turns them
// into sparse terms over the operator's output rows exactly as the
// occurrence scatter does (grid cells carry an embedding prefix, so zero
// values are skipped there, amvm.cpp:112-116).
namespace {
GammaContributions gamma_contributions_rows(const HOperator& op, const double* x);
}

GammaContributions gamma_contributions(const HOperator& op, const double* x) {
  if (op.row_begin() != 0 || op.row_end() != op.row_tree().size())
    throw ConfigError("gamma_contributions: sharded operators are not supported");
  return gamma_contributions_rows(op, x);
}

namespace {
// the estimator terms of the blocks the operator holds: every block for a
// whole operator, the shard's block rows for a shard (difference nonzero on
// its rows only)
GammaContributions gamma_contributions_rows(const HOperator& op, const double* x) {
  GammaContributions g;
  const long long M = op.rows();
  const int N = op.row_tree().size();
  g.difference.assign(M, 0.0);
  int n_terms = 0;
  long long n_vals = 0;
  check_status(op.gpu(), hmgpu_tail_terms(op.gpu(), x, &n_terms, &n_vals, nullptr, nullptr),
               "hmgpu_tail_terms");
  std::vector<long long> meta(4LL * n_terms);
  std::vector<double> vals(n_vals);
  if (n_terms > 0)
    check_status(op.gpu(),
                 hmgpu_tail_terms(op.gpu(), x, &n_terms, &n_vals, meta.data(), vals.data()),
                 "hmgpu_tail_terms");
  const bool grid = op.ncomp() == 6;
  const auto& rperm = op.row_tree().perm;
  std::vector<std::pair<long long, double>> buf;
  for (int t = 0; t < n_terms; ++t) {
    const int comp = static_cast<int>(meta[4 * t]);
    const int b = static_cast<int>(meta[4 * t + 1]);
    const int nocc = static_cast<int>(meta[4 * t + 2]);
    const long long off = meta[4 * t + 3];
    const ClusterNode& rn = op.row_tree().nodes[op.partition().blocks[b].row_node];
    const int m = rn.size();
    buf.clear();
    for (int o = 0; o < nocc; ++o) {
      const int rb = grid ? (o == 0 ? kCompR[comp] : kCompC[comp]) : 0;
      for (int i = 0; i < m; ++i) {
        const double v = vals[off + static_cast<long long>(o) * m + i];
        if (grid && v == 0.0) continue;
        buf.emplace_back(static_cast<long long>(rb) * N + rperm[rn.begin + i], v);
      }
    }
    if (buf.empty()) continue;
    std::sort(buf.begin(), buf.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    BlockTerm term;
    term.comp = comp;
    term.block = b;
    term.idx.reserve(buf.size());
    term.val.reserve(buf.size());
    for (const auto& e : buf) {
      term.idx.push_back(e.first);
      term.val.push_back(e.second);
      g.difference[e.first] += e.second;
      term.norm_sq += e.second * e.second;
    }
    g.terms.push_back(std::move(term));
  }
  double s = 0.0;
  for (double v : g.difference) s += v * v;
  g.gamma = std::sqrt(s);
  return g;
}
}  // namespace

// the transposed occurrences (gamma_contributions with occ.transposed,
// amvm.cpp:100-106): per (comp, block) the tail V[:,k:K](U[:,k:K]^T x) over
// the block columns (external column ids), grid occurrence 0 = cell (R, C)
// transposed (x_R -> component C), 1 = its alias (x_C -> R)
GammaContributions gamma_contributions_transposed(const HOperator& op, const double* x) {
  if (op.row_begin() != 0 || op.row_end() != op.row_tree().size())
    throw ConfigError("gamma_contributions: sharded operators are not supported");
  GammaContributions g;
  const long long NCOLS = op.cols();
  const int N = op.col_tree().size();
  g.difference.assign(NCOLS, 0.0);
  int n_terms = 0;
  long long n_vals = 0;
  check_status(op.gpu(), hmgpu_tail_terms_t(op.gpu(), x, &n_terms, &n_vals, nullptr, nullptr),
               "hmgpu_tail_terms_t");
  std::vector<long long> meta(4LL * n_terms);
  std::vector<double> vals(n_vals);
  if (n_terms > 0)
    check_status(op.gpu(),
                 hmgpu_tail_terms_t(op.gpu(), x, &n_terms, &n_vals, meta.data(), vals.data()),
                 "hmgpu_tail_terms_t");
  const bool grid = op.ncomp() == 6;
  const auto& cperm = op.col_tree().perm;
  std::vector<std::pair<long long, double>> buf;
  for (int t = 0; t < n_terms; ++t) {
    const int comp = static_cast<int>(meta[4 * t]);
    const int b = static_cast<int>(meta[4 * t + 1]);
    const int nocc = static_cast<int>(meta[4 * t + 2]);
    const long long off = meta[4 * t + 3];
    const ClusterNode& cn = op.col_tree().nodes[op.partition().blocks[b].col_node];
    const int n = cn.size();
    buf.clear();
    for (int o = 0; o < nocc; ++o) {
      const int ob = grid ? (o == 0 ? kCompC[comp] : kCompR[comp]) : 0;
      for (int j = 0; j < n; ++j) {
        const double v = vals[off + static_cast<long long>(o) * n + j];
        if (grid && v == 0.0) continue;
        buf.emplace_back(static_cast<long long>(ob) * N + cperm[cn.begin + j], v);
      }
    }
    if (buf.empty()) continue;
    std::sort(buf.begin(), buf.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    BlockTerm term;
    term.comp = comp;
    term.block = b;
    for (const auto& e : buf) {
      term.idx.push_back(e.first);
      term.val.push_back(e.second);
      g.difference[e.first] += e.second;
      term.norm_sq += e.second * e.second;
    }
    g.terms.push_back(std::move(term));
  }
  double s2 = 0.0;
  for (double v : g.difference) s2 += v * v;
  g.gamma = std::sqrt(s2);
  return g;
}

// row-sorted greedy marking (amvm.cpp:131-184)
std::vector<int> mark_blocks(const GammaContributions& g, Real theta, int c_sp,
                             long long m_rows, long long n_cols, Real* gamma_pk_out) {
  std::vector<int> marked;
  if (g.gamma <= 0.0) {
    if (gamma_pk_out) *gamma_pk_out = 0.0;
    return marked;
  }
  const Real threshold = (1.0 - theta) * g.gamma /
                         std::sqrt(static_cast<Real>(c_sp) * static_cast<Real>(m_rows) *
                                   static_cast<Real>(n_cols));
  const Real target = (1.0 - theta) * g.gamma;
  // CSR of (row -> terms reaching the threshold there), terms in order
  std::vector<int> cnt(m_rows + 1, 0);
  for (const BlockTerm& t : g.terms)
    for (std::size_t i = 0; i < t.idx.size(); ++i)
      if (std::abs(t.val[i]) >= threshold) ++cnt[t.idx[i] + 1];
  for (long long r = 0; r < m_rows; ++r) cnt[r + 1] += cnt[r];
  std::vector<int> fill(cnt.begin(), cnt.end() - 1), lists(cnt[m_rows]);
  for (std::size_t t = 0; t < g.terms.size(); ++t)
    for (std::size_t i = 0; i < g.terms[t].idx.size(); ++i)
      if (std::abs(g.terms[t].val[i]) >= threshold)
        lists[fill[g.terms[t].idx[i]]++] = static_cast<int>(t);
  std::vector<long long> order(m_rows);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](long long a, long long b) {
    return std::abs(g.difference[a]) > std::abs(g.difference[b]);
  });
  std::vector<Real> residual = g.difference;
  Real res_sq = 0.0;
  for (Real v : residual) res_sq += v * v;
  std::vector<char> in_set(g.terms.size(), 0);
  const Real target_sq = target * target;
  for (long long row : order) {
    if (res_sq <= target_sq) break;
    bool done = false;
    for (int e = cnt[row]; e < cnt[row + 1]; ++e) {
      const int t = lists[e];
      if (in_set[t]) continue;
      in_set[t] = 1;
      marked.push_back(t);
      const BlockTerm& term = g.terms[t];
      Real dot = 0.0;
      for (std::size_t i = 0; i < term.idx.size(); ++i)
        dot += residual[term.idx[i]] * term.val[i];
      res_sq += term.norm_sq - 2.0 * dot;
      for (std::size_t i = 0; i < term.idx.size(); ++i)
        residual[term.idx[i]] -= term.val[i];
      if (res_sq <= target_sq) {
        done = true;
        break;
      }
    }
    if (done) break;
  }
  Real s = 0.0;
  for (Real v : residual) s += v * v;
  if (gamma_pk_out) *gamma_pk_out = std::sqrt(s);
  return marked;
}

// mark_blocks (amvm.cpp:131-184) over ranks that each hold the terms of
// their own rows (g.difference: the whole difference vector, every rank's
// rows; own: this rank's rows).  The walk visits the rows in ONE global
// order (|diff| descending, stable) and stops once the global residual
// reaches the target; a term lives on the rank owning its block's rows and
// only terms on the same rows change each other's residual contribution, so
// each rank walks its own rows in the global order without stopping and
// records per term Delta = ||term||^2 - 2 <residual, term>; the events of
// all ranks merged by row position are the unsharded walk's res_sq updates
// bit for bit, and the stopping event fixes every rank's marked terms.
// Returns this rank's marked term indices; gamma(P_k) and the marked count
// over all ranks through the out-parameters.
std::vector<int> mark_blocks_sharded(const GammaContributions& g, const std::vector<char>& own,
                                     Real theta, int c_sp, long long m_rows, long long n_cols,
                                     const AllGather& allgather, int nranks, int rank,
                                     Real* gamma_pk_out, int* n_marked_out) {
  const long long M = m_rows;
  std::vector<int> marked;
  std::vector<double> residual = g.difference;
  int n_marked = 0;
  double gamma2 = 0.0;
  for (double v : g.difference) gamma2 += v * v;
  const double gamma = std::sqrt(gamma2);
  if (gamma > 0.0) {
    const double threshold =
        (1.0 - theta) * gamma /
        std::sqrt(static_cast<double>(c_sp) * static_cast<double>(M) *
                  static_cast<double>(n_cols));
    const double target = (1.0 - theta) * gamma;
    const double target_sq = target * target;
    std::vector<int> cnt(M + 1, 0);
    for (const BlockTerm& t : g.terms)
      for (std::size_t i = 0; i < t.idx.size(); ++i)
        if (std::abs(t.val[i]) >= threshold) ++cnt[t.idx[i] + 1];
    for (long long r = 0; r < M; ++r) cnt[r + 1] += cnt[r];
    std::vector<int> fill(cnt.begin(), cnt.end() - 1), lists(cnt[M]);
    for (std::size_t t = 0; t < g.terms.size(); ++t)
      for (std::size_t i = 0; i < g.terms[t].idx.size(); ++i)
        if (std::abs(g.terms[t].val[i]) >= threshold)
          lists[fill[g.terms[t].idx[i]]++] = static_cast<int>(t);
    std::vector<long long> order(M);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](long long a, long long b) {
      return std::abs(g.difference[a]) > std::abs(g.difference[b]);
    });
    double res_sq = 0.0;
    for (double v : residual) res_sq += v * v;
    struct Ev {
      long long pos;
      double delta;
    };
    std::vector<Ev> ev;
    std::vector<int> ev_term;
    {
      std::vector<double> rl = g.difference;
      std::vector<char> in_set(g.terms.size(), 0);
      for (long long p = 0; p < M; ++p) {
        const long long row = order[p];
        for (int e = cnt[row]; e < cnt[row + 1]; ++e) {
          const int t = lists[e];
          if (in_set[t]) continue;
          in_set[t] = 1;
          const BlockTerm& term = g.terms[t];
          double dot = 0.0;
          for (std::size_t i = 0; i < term.idx.size(); ++i) dot += rl[term.idx[i]] * term.val[i];
          ev.push_back(Ev{p, term.norm_sq - 2.0 * dot});
          ev_term.push_back(t);
          for (std::size_t i = 0; i < term.idx.size(); ++i) rl[term.idx[i]] -= term.val[i];
        }
      }
    }
    // every rank's events, merged by row position (a row's events come from
    // one rank, in that rank's walk order)
    long long ne = static_cast<long long>(ev.size());
    std::vector<long long> counts(nranks);
    allgather(&ne, counts.data(), static_cast<long long>(sizeof(long long)));
    long long maxne = 1;
    for (long long q : counts) maxne = std::max(maxne, q);
    std::vector<Ev> send(maxne, Ev{-1, 0.0}), all(static_cast<size_t>(maxne) * nranks);
    std::copy(ev.begin(), ev.end(), send.begin());
    allgather(send.data(), all.data(), maxne * static_cast<long long>(sizeof(Ev)));
    std::vector<long long> cur(nranks, 0);
    if (res_sq > target_sq) {
      for (;;) {
        int best = -1;
        for (int r = 0; r < nranks; ++r)
          if (cur[r] < counts[r] &&
              (best < 0 || all[static_cast<size_t>(r) * maxne + cur[r]].pos <
                               all[static_cast<size_t>(best) * maxne + cur[best]].pos))
            best = r;
        if (best < 0) break;  // every event taken: the walk ran out of terms
        res_sq += all[static_cast<size_t>(best) * maxne + cur[best]].delta;
        ++cur[best];
        ++n_marked;
        if (res_sq <= target_sq) break;
      }
    }
    for (long long e = 0; e < cur[rank]; ++e) {
      const BlockTerm& term = g.terms[ev_term[e]];
      marked.push_back(ev_term[e]);
      for (std::size_t i = 0; i < term.idx.size(); ++i) residual[term.idx[i]] -= term.val[i];
    }
  }
  // gamma(P_k): the residual rows of every rank, summed in row order
  for (long long i = 0; i < M; ++i)
    if (!own[i]) residual[i] = 0.0;
  std::vector<double> all(static_cast<size_t>(M) * nranks);
  allgather(residual.data(), all.data(), M * static_cast<long long>(sizeof(double)));
  double rs = 0.0;
  for (long long i = 0; i < M; ++i) {
    double v = 0.0;
    for (int r = 0; r < nranks; ++r) v += all[static_cast<size_t>(r) * M + i];
    rs += v * v;
  }
  if (gamma_pk_out) *gamma_pk_out = std::sqrt(rs);
  if (n_marked_out) *n_marked_out = n_marked;
  return marked;
}

// Algorithm 2 over a block-row shard: every rank holds the
// blocks of its rows; the ranks exchange (hmgpu_comm_allgather, collective)
// the estimator's difference vector (disjoint rows: their sum is exact), the
// storage figures, and the marking events.  The marking walk of
// mark_blocks (amvm.cpp:131-184) visits the rows in ONE global order (|diff|
// descending, stable) and stops once the global residual reaches the
// target; a term lives on the rank owning its block's rows, and only terms
// on the same rows change each other's residual contribution, so each rank
// walks its own rows in the global order without stopping and records, per
// term, Delta = ||term||^2 - 2 <residual, term>; the merged event stream
// (by global row position) is the unsharded walk's sequence of res_sq
// updates, bit for bit, and the stopping event picks every rank's marked
// set.  x must be given on every rank (the product is hmgpu_matvec_dist).
std::vector<double> amvm_multiply_sharded(HOperator& op, const double* x,
                                          const AmvmConfig& cfg, AmvmReport& report) {
  hmgpu_ctx* c = op.gpu();
  int nranks = 0, rank = 0, kind = 0;
  check_status(c, hmgpu_comm_info(c, &nranks, &rank, &kind, nullptr, nullptr),
               "hmgpu_comm_info");
  if (!kind)
    throw ConfigError("amvm_multiply: a sharded operator needs a communicator (hmgpu_comm_*)");
  report = AmvmReport{};
  report.c_sp = std::max(1, sparsity_constant(op.partition()));
  const long long M = op.rows();
  const int N = op.row_tree().size();
  const AllGather allgather = [c](const void* send, void* recv, long long bytes) {
    check_status(c, hmgpu_comm_allgather(c, send, recv, bytes), "hmgpu_comm_allgather");
  };
  // rows of this shard (external dof ids)
  std::vector<char> own(M, 0);
  {
    const auto& perm = op.row_tree().perm;
    const int nout = static_cast<int>(M / N);
    for (int p = op.row_begin(); p < op.row_end(); ++p)
      for (int r = 0; r < nout; ++r) own[static_cast<long long>(r) * N + perm[p]] = 1;
  }
  // every rank's rows, one vector: the ranks' rows are disjoint
  auto combine = [&](std::vector<double>& v) {
    std::vector<double> all(static_cast<size_t>(M) * nranks);
    allgather(v.data(), all.data(), M * static_cast<long long>(sizeof(double)));
    for (long long i = 0; i < M; ++i) {
      double s = 0.0;
      for (int r = 0; r < nranks; ++r) s += all[static_cast<size_t>(r) * M + i];
      v[i] = s;
    }
  };
  auto storage = [&](long long& pivots, double& mb) {
    hmgpu_storage_info si{};
    check_status(c, hmgpu_storage(c, &si), "hmgpu_storage");
    struct {
      long long p;
      double mb;
    } mine{si.pivots, si.mb_current};
    std::vector<decltype(mine)> all(nranks);
    allgather(&mine, all.data(), static_cast<long long>(sizeof(mine)));
    pivots = 0;
    mb = 0.0;
    for (const auto& a : all) {
      pivots += a.p;
      mb += a.mb;
    }
  };
  std::vector<double> b(M), b_hat_prev;
  auto matvec = [&] {
    check_status(c, hmgpu_matvec_dist(c, x, b.data(), 1, HMGPU_MODE_CURRENT, HMGPU_PTR_HOST),
                 "hmgpu_matvec_dist");
  };
  matvec();
  for (int k = 0;; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    GammaContributions g = gamma_contributions_rows(op, x);
    combine(g.difference);
    double s2 = 0.0;
    for (double v : g.difference) s2 += v * v;
    const double gamma = std::sqrt(s2);
    if (!b_hat_prev.empty()) {
      double s = 0.0;
      for (long long i = 0; i < M; ++i) {
        const double d = b[i] + g.difference[i] - b_hat_prev[i];
        s += d * d;
      }
      report.iterations.back().e_hat = std::sqrt(s);
    }
    AmvmIteration it;
    it.k = k;
    it.gamma = gamma;
    storage(it.cumulative_pivots, it.storage_mb);
    auto finish = [&](const char* why, bool conv) {
      it.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count();
      report.iterations.push_back(it);
      report.termination = why;
      report.converged = conv;
      return b;
    };
    if (gamma <= cfg.eps_amvm) return finish("tolerance", true);
    if (k >= cfg.max_iterations) return finish("max_iterations", false);
    // ---- marking (mark_blocks, amvm.cpp:131-184) across the ranks
    std::vector<std::pair<int, int>> mine_marked;
    int n_marked = 0;
    double gpk = 0.0;
    for (int t : mark_blocks_sharded(g, own, cfg.theta, report.c_sp, M, op.cols(), allgather,
                                     nranks, rank, &gpk, &n_marked))
      mine_marked.emplace_back(g.terms[t].comp, g.terms[t].block);
    it.gamma_pk = gpk;
    it.marked = n_marked;
    b_hat_prev.resize(M);
    for (long long i = 0; i < M; ++i) b_hat_prev[i] = b[i] + g.difference[i];
    if (!mine_marked.empty()) {
      op.promote(mine_marked);
      op.extend_lookahead(mine_marked, cfg.lookahead_steps);
    }
    matvec();
    it.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                .count();
    report.iterations.push_back(it);
  }
}

// Algorithm 2 (amvm.cpp:199-268).  The estimator, the marking walk and the
// refinement run on the device (hmgpu_amvm_*); the host only sees gamma,
// gamma(P_k), the marked count and the difference vector (for e_hat).
std::vector<double> amvm_multiply(HOperator& op, const double* x,
                                  const AmvmConfig& cfg, AmvmReport& report) {
  if (cfg.theta <= 0.0 || cfg.theta >= 1.0)
    throw Error("amvm_multiply: theta must lie in (0,1)");
  if (cfg.eps_amvm <= 0.0) throw Error("amvm_multiply: eps_amvm must be positive");
  if (op.row_begin() != 0 || op.row_end() != op.row_tree().size())
    return amvm_multiply_sharded(op, x, cfg, report);
  using clk = std::chrono::steady_clock;
  const auto ts = clk::now();
  report = AmvmReport{};
  report.c_sp = std::max(1, sparsity_constant(op.partition()));
  const auto ts1 = clk::now();
  const long long M = op.rows();
  std::vector<double> b(M), b_hat_prev, diff(M);
  // one matvec per rank change: sweep the blocks in place instead of
  // re-packing the stream plan each sweep (hmgpu_set_matvec_policy)
  // the caller's policy is restored on exit
  struct DirectMatvec {
    hmgpu_ctx* c;
    int saved = 0;
    explicit DirectMatvec(hmgpu_ctx* cc) : c(cc) {
      hmgpu_get_matvec_policy(c, &saved);
      hmgpu_set_matvec_policy(c, 1);
    }
    ~DirectMatvec() { hmgpu_set_matvec_policy(c, saved); }
  } direct(op.gpu());
  op.matvec(x, b.data(), 1, Mode::Current);
  static const bool verbose = std::getenv("HMGPU_VERBOSE") != nullptr;
  auto lap = [&](const char* what, clk::time_point& t) {
    if (!verbose) return;
    const auto now = clk::now();
    std::fprintf(stderr, "[amvm] %-10s %9.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  };
  if (verbose)
    std::fprintf(stderr, "[amvm] setup      %9.2f ms (c_sp %.2f ms)\n",
                 std::chrono::duration<double, std::milli>(clk::now() - ts).count(),
                 std::chrono::duration<double, std::milli>(ts1 - ts).count());
  for (int k = 0;; ++k) {
    const auto t0 = clk::now();
    auto tl = t0;
    double gamma = 0.0;
    check_status(op.gpu(), hmgpu_amvm_estimate(op.gpu(), x, &gamma, diff.data()),
                 "hmgpu_amvm_estimate");
    lap("gamma", tl);
    if (!b_hat_prev.empty()) {
      double s = 0.0;
      for (long long i = 0; i < M; ++i) {
        const double d = b[i] + diff[i] - b_hat_prev[i];
        s += d * d;
      }
      report.iterations.back().e_hat = std::sqrt(s);
    }
    AmvmIteration it;
    it.k = k;
    it.gamma = gamma;
    {
      hmgpu_storage_info si{};  // one pass over the items for both figures
      check_status(op.gpu(), hmgpu_storage(op.gpu(), &si), "hmgpu_storage");
      it.cumulative_pivots = si.pivots;
      it.storage_mb = si.mb_current;
    }
    lap("account", tl);
    if (gamma <= cfg.eps_amvm) {
      it.ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
      report.iterations.push_back(it);
      report.termination = "tolerance";
      report.converged = true;
      return b;
    }
    if (k >= cfg.max_iterations) {
      it.ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
      report.iterations.push_back(it);
      report.termination = "max_iterations";
      report.converged = false;
      return b;
    }
    double gpk = 0.0;
    int nm = 0;
    if (gamma > 0.0)
      check_status(op.gpu(),
                   hmgpu_amvm_mark(op.gpu(), cfg.theta, report.c_sp, M, op.cols(), &gpk, &nm),
                   "hmgpu_amvm_mark");
    lap("mark", tl);
    it.gamma_pk = gpk;
    it.marked = nm;
    b_hat_prev.resize(M);
    for (long long i = 0; i < M; ++i) b_hat_prev[i] = b[i] + diff[i];
    if (nm > 0)
      check_status(op.gpu(), hmgpu_amvm_refine(op.gpu(), cfg.lookahead_steps, nullptr),
                   "hmgpu_amvm_refine");
    lap("refine", tl);
    op.matvec(x, b.data(), 1, Mode::Current);
    lap("matvec", tl);
    it.ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    report.iterations.push_back(it);
  }
}

}  // namespace hmb
