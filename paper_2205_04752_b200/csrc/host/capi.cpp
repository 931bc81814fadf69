// Flat C API of the host layer (include/hmbem.h).  Exceptions are mapped
// to status codes here; nothing throws across the ABI.

#include <cstring>
#include <random>
#include <memory>
#include <string>

#include "cluster.hpp"
#include "errors.hpp"
#include "geometry.hpp"
#include "hmbem.h"
#include "hmgpu.h"
#include "operator.hpp"
#include "sparse_ops.hpp"
#include "quadrature.hpp"

struct hmb_mesh {
  hmb::Mesh mesh;
};

struct hmb_op {
  std::unique_ptr<hmb::HOperator> op;
  hmb::GammaContributions gamma;  // last estimator (hmb_gamma)
};

namespace {

thread_local std::string g_err;
thread_local int g_dev_status = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    return HMB_OK;
  } catch (const hmb::MeshError& e) {
    g_err = e.what();
    return HMB_MESH_ERROR;
  } catch (const hmb::ConfigError& e) {
    g_err = e.what();
    return HMB_CONFIG_ERROR;
  } catch (const hmb::DimensionError& e) {
    g_err = e.what();
    return HMB_DIMENSION_ERROR;
  } catch (const hmb::DeviceError& e) {
    g_err = e.what();
    g_dev_status = e.status;
    return HMB_DEVICE_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HMB_ERROR;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw hmb::Error(std::string("null argument: ") + what);
}

const hmb::ClusterTree& tree_of(const hmb_op* op, int which) {
  return which == 0 ? op->op->row_tree() : op->op->col_tree();
}

}  // namespace

extern "C" {

const char* hmb_last_error(void) { return g_err.c_str(); }
int hmb_device_status(void) { return g_dev_status; }

int hmb_mesh_icosphere(int level, hmb_mesh** out) {
  return guard([&] {
    need(out, "out");
    auto m = std::make_unique<hmb_mesh>();
    m->mesh = hmb::make_icosphere(level);
    *out = m.release();
  });
}

int hmb_mesh_ellipsoid(int level, double ax, double ay, double az, hmb_mesh** out) {
  return guard([&] {
    need(out, "out");
    auto m = std::make_unique<hmb_mesh>();
    m->mesh = hmb::make_ellipsoid(level, ax, ay, az);
    *out = m.release();
  });
}

int hmb_mesh_voxel_cube(int n, double lo, double hi, hmb_mesh** out) {
  return guard([&] {
    need(out, "out");
    auto m = std::make_unique<hmb_mesh>();
    m->mesh = hmb::make_voxel_cube(n, lo, hi);
    *out = m.release();
  });
}

int hmb_mesh_from_arrays(int nv, const double* verts, int nt, const int* tris,
                         hmb_mesh** out) {
  return guard([&] {
    need(out, "out");
    need(verts, "verts");
    need(tris, "tris");
    if (nv < 3 || nt < 1) throw hmb::MeshError("mesh needs >= 3 vertices, >= 1 triangle");
    auto m = std::make_unique<hmb_mesh>();
    m->mesh.vertices.resize(nv);
    for (int v = 0; v < nv; ++v)
      for (int d = 0; d < 3; ++d) m->mesh.vertices[v][d] = verts[3 * v + d];
    m->mesh.triangles.resize(nt);
    for (int t = 0; t < nt; ++t)
      for (int d = 0; d < 3; ++d) m->mesh.triangles[t][d] = tris[3 * t + d];
    m->mesh.finish();
    *out = m.release();
  });
}

int hmb_mesh_load_off(const char* path, hmb_mesh** out) {
  return guard([&] {
    need(out, "out");
    need(path, "path");
    auto m = std::make_unique<hmb_mesh>();
    m->mesh = hmb::load_off(path);
    *out = m.release();
  });
}

int hmb_mesh_save_off(const hmb_mesh* m, const char* path) {
  return guard([&] {
    need(m, "mesh");
    need(path, "path");
    hmb::save_off(m->mesh, path);
  });
}

int hmb_mesh_validate(const hmb_mesh* m) {
  return guard([&] {
    need(m, "mesh");
    m->mesh.validate_admissible();
  });
}

int hmb_mesh_label(hmb_mesh* m, const char* pred) {
  return guard([&] {
    need(m, "mesh");
    need(pred, "predicate");
    m->mesh.label_dirichlet(pred);
  });
}

int hmb_mesh_sizes(const hmb_mesh* m, int* nv, int* nt) {
  return guard([&] {
    need(m, "mesh");
    if (nv) *nv = m->mesh.nv();
    if (nt) *nt = m->mesh.nt();
  });
}

int hmb_mesh_get(const hmb_mesh* m, double* verts, int* tris, double* centroids,
                 double* areas, double* normals, double* diam, int* dirichlet) {
  return guard([&] {
    need(m, "mesh");
    const hmb::Mesh& M = m->mesh;
    for (int v = 0; v < M.nv() && verts; ++v)
      for (int d = 0; d < 3; ++d) verts[3 * v + d] = M.vertices[v][d];
    for (int t = 0; t < M.nt(); ++t) {
      for (int d = 0; d < 3; ++d) {
        if (tris) tris[3 * t + d] = M.triangles[t][d];
        if (centroids) centroids[3 * t + d] = M.centroids[t][d];
        if (normals) normals[3 * t + d] = M.normals[t][d];
      }
      if (areas) areas[t] = M.areas[t];
      if (diam) diam[t] = M.diam[t];
      if (dirichlet) dirichlet[t] = M.dirichlet.empty() ? 0 : M.dirichlet[t];
    }
  });
}

void hmb_mesh_free(hmb_mesh* m) { delete m; }

int hmb_pair_rule(int pair_case, int order, int* n, double* xr1, double* xr2, double* yr1,
                  double* yr2, double* w) {
  return guard([&] {
    need(n, "n");
    const hmb::PairRuleTable r = hmb::singular_pair_rule(pair_case, order);
    *n = static_cast<int>(r.w.size());
    if (!w) return;
    std::copy(r.xr1.begin(), r.xr1.end(), xr1);
    std::copy(r.xr2.begin(), r.xr2.end(), xr2);
    std::copy(r.yr1.begin(), r.yr1.end(), yr1);
    std::copy(r.yr2.begin(), r.yr2.end(), yr2);
    std::copy(r.w.begin(), r.w.end(), w);
  });
}

int hmb_sparse_op(const hmb_mesh* m, int which, int* cols3, double* vals3) {
  return guard([&] {
    need(m, "mesh");
    need(cols3, "cols3");
    need(vals3, "vals3");
    const hmb::Ell3 e = which == 0   ? hmb::build_t_matrix(m->mesh, 0, 1)
                        : which == 1 ? hmb::build_t_matrix(m->mesh, 0, 2)
                        : which == 2 ? hmb::build_t_matrix(m->mesh, 1, 2)
                        : which == 3 ? hmb::build_mass_matrix(m->mesh)
                                     : throw hmb::Error("hmb_sparse_op: which in 0..3");
    std::copy(e.col.begin(), e.col.end(), cols3);
    std::copy(e.val.begin(), e.val.end(), vals3);
  });
}

int hmb_random_vector(long long n, unsigned long long seed, int kind, double* out) {
  return guard([&] {
    need(out, "out");
    std::mt19937_64 gen(seed);
    if (kind == 0) {  // uniform [-1, 1) (proj/tests/oracles.cpp:415-421)
      std::uniform_real_distribution<double> dist(-1.0, 1.0);
      for (long long i = 0; i < n; ++i) out[i] = dist(gen);
    } else if (kind == 1) {  // standard normal
      std::normal_distribution<double> dist(0.0, 1.0);
      for (long long i = 0; i < n; ++i) out[i] = dist(gen);
    } else {
      throw hmb::Error("random_vector: kind must be 0 (uniform) or 1 (normal)");
    }
  });
}

int hmb_gauss_rule(int order, int* npts, double* a, double* b, double* w) {
  return guard([&] {
    need(npts, "npts");
    const hmb::TriangleRule r = hmb::gauss_rule(order);
    *npts = static_cast<int>(r.w.size());
    if (a) std::memcpy(a, r.a.data(), r.a.size() * sizeof(double));
    if (b) std::memcpy(b, r.b.data(), r.b.size() * sizeof(double));
    if (w) std::memcpy(w, r.w.data(), r.w.size() * sizeof(double));
  });
}

int hmb_admissible(const double* a6, const double* b6, double eta, int* out) {
  return guard([&] {
    need(a6, "a");
    need(b6, "b");
    need(out, "out");
    hmb::Box a, b;
    a.absorb(hmb::V3{a6[0], a6[1], a6[2]});
    a.absorb(hmb::V3{a6[3], a6[4], a6[5]});
    b.absorb(hmb::V3{b6[0], b6[1], b6[2]});
    b.absorb(hmb::V3{b6[3], b6[4], b6[5]});
    *out = hmb::admissible(a, b, eta) ? 1 : 0;
  });
}

int hmb_op_kelvin(const hmb_mesh* m, double E, double nu, int b_min, double eta,
                  int device, int shard_rank, int shard_count, hmb_op** out) {
  return guard([&] {
    need(m, "mesh");
    need(out, "out");
    auto op = std::make_unique<hmb_op>();
    op->op = hmb::HOperator::kelvin(m->mesh, E, nu, b_min, eta, device,
                                    hmb::Shard{shard_rank, shard_count});
    *out = op.release();
  });
}

int hmb_op_kelvin_points(const hmb_mesh* m, int npts, const double* pts, double E,
                         double nu, int b_min, double eta, double min_distance_factor,
                         int disjoint_order, int device, int shard_rank, int shard_count,
                         hmb_op** out) {
  return guard([&] {
    need(m, "mesh");
    need(pts, "pts");
    need(out, "out");
    std::vector<hmb::V3> p(npts);
    for (int i = 0; i < npts; ++i) p[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    hmb::QuadratureConfig qc;
    qc.disjoint_order = disjoint_order;
    auto op = std::make_unique<hmb_op>();
    op->op = hmb::HOperator::kelvin_points(m->mesh, p, E, nu, b_min, eta, device,
                                           hmb::Shard{shard_rank, shard_count},
                                           min_distance_factor, qc);
    *out = op.release();
  });
}

int hmb_op_kelvin_double(const hmb_mesh* m, int npts, const double* pts, int r, int c,
                         double E, double nu, int b_min, double eta,
                         double min_distance_factor, int disjoint_order, int device,
                         int shard_rank, int shard_count, hmb_op** out) {
  return guard([&] {
    need(m, "mesh");
    need(pts, "pts");
    need(out, "out");
    std::vector<hmb::V3> p(npts);
    for (int i = 0; i < npts; ++i) p[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    hmb::QuadratureConfig qc;
    qc.disjoint_order = disjoint_order;
    auto op = std::make_unique<hmb_op>();
    op->op = hmb::HOperator::kelvin_double_points(m->mesh, p, r, c, E, nu, b_min, eta, device,
                                                  hmb::Shard{shard_rank, shard_count},
                                                  min_distance_factor, qc);
    *out = op.release();
  });
}

int hmb_op_galerkin(const hmb_mesh* m, int which, int b_min, double eta, int device,
                    int shard_rank, int shard_count, hmb_op** out) {
  return guard([&] {
    need(m, "mesh");
    need(out, "out");
    auto op = std::make_unique<hmb_op>();
    op->op = hmb::HOperator::galerkin(m->mesh, which, b_min, eta, device,
                                      hmb::Shard{shard_rank, shard_count});
    *out = op.release();
  });
}

int hmb_op_kdelta(const hmb_mesh* m, int b_min, double eta, int device, int shard_rank,
                  int shard_count, hmb_op** out) {
  return guard([&] {
    need(m, "mesh");
    need(out, "out");
    auto op = std::make_unique<hmb_op>();
    op->op = hmb::HOperator::kdelta(m->mesh, b_min, eta, device,
                                    hmb::Shard{shard_rank, shard_count});
    *out = op.release();
  });
}

int hmb_op_newton(int n, const double* pts, const double* boxes6, double diag,
                  int b_min, double eta, int device, hmb_op** out) {
  return guard([&] {
    need(pts, "pts");
    need(out, "out");
    std::vector<hmb::V3> p(n);
    for (int i = 0; i < n; ++i) p[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    std::vector<hmb::Box> boxes;
    if (boxes6) {
      boxes.resize(n);
      for (int i = 0; i < n; ++i) {
        boxes[i].absorb(hmb::V3{boxes6[6 * i], boxes6[6 * i + 1], boxes6[6 * i + 2]});
        boxes[i].absorb(hmb::V3{boxes6[6 * i + 3], boxes6[6 * i + 4], boxes6[6 * i + 5]});
      }
    }
    auto op = std::make_unique<hmb_op>();
    op->op = hmb::HOperator::newton(p, boxes6 ? &boxes : nullptr, diag, b_min, eta, device);
    *out = op.release();
  });
}

int hmb_op_dense(int m, int n, const double* a, const double* row_pts,
                 const double* col_pts, int b_min, double eta, int device,
                 hmb_op** out) {
  return guard([&] {
    need(a, "matrix");
    need(row_pts, "row_pts");
    need(col_pts, "col_pts");
    need(out, "out");
    std::vector<hmb::V3> rp(m), cp(n);
    for (int i = 0; i < m; ++i) rp[i] = {row_pts[3 * i], row_pts[3 * i + 1], row_pts[3 * i + 2]};
    for (int j = 0; j < n; ++j) cp[j] = {col_pts[3 * j], col_pts[3 * j + 1], col_pts[3 * j + 2]};
    auto op = std::make_unique<hmb_op>();
    op->op = hmb::HOperator::dense(m, n, a, rp, cp, b_min, eta, device);
    *out = op.release();
  });
}

void hmb_op_free(hmb_op* op) { delete op; }

int hmb_op_info(const hmb_op* op, long long* rows, long long* cols, int* ncomp,
                int* row_begin, int* row_end) {
  return guard([&] {
    need(op, "op");
    if (rows) *rows = op->op->rows();
    if (cols) *cols = op->op->cols();
    if (ncomp) *ncomp = op->op->ncomp();
    if (row_begin) *row_begin = op->op->row_begin();
    if (row_end) *row_end = op->op->row_end();
  });
}

void* hmb_op_gpu(const hmb_op* op) { return op ? op->op->gpu() : nullptr; }

int hmb_tree_info(const hmb_op* op, int which, int* n_nodes, int* depth, int* size) {
  return guard([&] {
    need(op, "op");
    const hmb::ClusterTree& t = tree_of(op, which);
    if (n_nodes) *n_nodes = static_cast<int>(t.nodes.size());
    if (depth) *depth = t.depth;
    if (size) *size = t.size();
  });
}

int hmb_tree_nodes(const hmb_op* op, int which, int* nodes5, double* boxes6, int* perm) {
  return guard([&] {
    need(op, "op");
    const hmb::ClusterTree& t = tree_of(op, which);
    for (std::size_t i = 0; i < t.nodes.size(); ++i) {
      const hmb::ClusterNode& nd = t.nodes[i];
      if (nodes5) {
        nodes5[5 * i] = nd.begin;
        nodes5[5 * i + 1] = nd.end;
        nodes5[5 * i + 2] = nd.child[0];
        nodes5[5 * i + 3] = nd.child[1];
        nodes5[5 * i + 4] = nd.level;
      }
      if (boxes6)
        for (int d = 0; d < 3; ++d) {
          boxes6[6 * i + d] = nd.box.lo[d];
          boxes6[6 * i + 3 + d] = nd.box.hi[d];
        }
    }
    if (perm) std::memcpy(perm, t.perm.data(), t.perm.size() * sizeof(int));
  });
}

int hmb_partition_info(const hmb_op* op, int* n_blocks, int* n_adm, int* c_sp) {
  return guard([&] {
    need(op, "op");
    const hmb::BlockPartition& p = op->op->partition();
    if (n_blocks) *n_blocks = static_cast<int>(p.blocks.size());
    if (n_adm) *n_adm = p.num_admissible();
    if (c_sp) *c_sp = hmb::sparsity_constant(p);
  });
}

int hmb_partition_blocks(const hmb_op* op, int* blocks4) {
  return guard([&] {
    need(op, "op");
    need(blocks4, "blocks4");
    const hmb::BlockPartition& p = op->op->partition();
    for (std::size_t i = 0; i < p.blocks.size(); ++i) {
      blocks4[4 * i] = p.blocks[i].row_node;
      blocks4[4 * i + 1] = p.blocks[i].col_node;
      blocks4[4 * i + 2] = p.blocks[i].admissible ? 1 : 0;
      blocks4[4 * i + 3] = p.blocks[i].level;
    }
  });
}

int hmb_partition_json(const hmb_op* op, char* buf, long long* len) {
  return guard([&] {
    need(op, "op");
    need(len, "len");
    const std::string s = hmb::partition_to_json(op->op->partition());
    const long long need_len = static_cast<long long>(s.size()) + 1;
    if (!buf) {
      *len = need_len;
      return;
    }
    if (*len < need_len) {
      *len = need_len;
      throw hmb::DimensionError("partition_json: buffer too small");
    }
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int hmb_assemble(hmb_op* op, double eps, double beta, int initial_rank, int lookahead,
                 long long max_rank, double* stats8) {
  return guard([&] {
    need(op, "op");
    hmb::AssemblyConfig cfg;
    cfg.eps = eps;
    cfg.beta = beta;
    cfg.initial_rank = initial_rank;
    cfg.lookahead = lookahead;
    cfg.max_rank = max_rank;
    const hmb::AssemblyStats s = op->op->assemble(cfg);
    if (stats8) {
      stats8[0] = static_cast<double>(s.aca_entries);
      stats8[1] = static_cast<double>(s.dense_entries);
      stats8[2] = static_cast<double>(s.aca_steps);
      stats8[3] = static_cast<double>(s.pivots);
      stats8[4] = s.ms_total;
      stats8[5] = s.ms_nearfield;
      stats8[6] = s.relaunches;
      stats8[7] = s.counted_flops;
    }
  });
}

int hmb_matvec(const hmb_op* op, const double* x, double* y, int nrhs, int mode,
               int device_ptrs) {
  return guard([&] {
    need(op, "op");
    need(x, "x");
    need(y, "y");
    op->op->matvec(x, y, nrhs, mode ? hmb::Mode::Lookahead : hmb::Mode::Current,
                   device_ptrs != 0);
  });
}

int hmb_matvec_transposed(const hmb_op* op, const double* x, double* y, int nrhs, int mode,
                          int device_ptrs) {
  return guard([&] {
    need(op, "op");
    need(x, "x");
    need(y, "y");
    op->op->matvec_transposed(x, y, nrhs, mode ? hmb::Mode::Lookahead : hmb::Mode::Current,
                              device_ptrs != 0);
  });
}

int hmb_ranks(const hmb_op* op, int* k_cur, int* k_look, int* consumed, int* last_stop) {
  return guard([&] {
    need(op, "op");
    std::vector<int> kc, kl, co, ls;
    op->op->ranks(kc, kl, &co, &ls);
    if (k_cur) std::memcpy(k_cur, kc.data(), kc.size() * sizeof(int));
    if (k_look) std::memcpy(k_look, kl.data(), kl.size() * sizeof(int));
    if (consumed) std::memcpy(consumed, co.data(), co.size() * sizeof(int));
    if (last_stop) std::memcpy(last_stop, ls.data(), ls.size() * sizeof(int));
  });
}

int hmb_promote(hmb_op* op, int n, const int* cb) {
  return guard([&] {
    need(op, "op");
    std::vector<std::pair<int, int>> v;
    for (int i = 0; i < n; ++i) v.emplace_back(cb[2 * i], cb[2 * i + 1]);
    op->op->promote(v);
  });
}

int hmb_extend(hmb_op* op, int n, const int* cb, int steps) {
  return guard([&] {
    need(op, "op");
    std::vector<std::pair<int, int>> v;
    for (int i = 0; i < n; ++i) v.emplace_back(cb[2 * i], cb[2 * i + 1]);
    op->op->extend_lookahead(v, steps);
  });
}

int hmb_storage(const hmb_op* op, double* out7) {
  return guard([&] {
    need(op, "op");
    need(out7, "out");
    hmgpu_storage_info s{};
    const int st = hmgpu_storage(op->op->gpu(), &s);
    if (st != HMGPU_OK)
      throw hmb::DeviceError(st, std::string("hmgpu_storage: ") +
                                     hmgpu_last_error(op->op->gpu()));
    out7[0] = s.mb_current;
    out7[1] = s.mb_tail;
    out7[2] = s.mb_dense;
    out7[3] = s.mb_arena_allocated;
    out7[4] = static_cast<double>(s.matvec_bytes);
    out7[5] = static_cast<double>(s.matvec_flops);
    out7[6] = static_cast<double>(op->op->total_pivots());
  });
}

int hmb_factor(const hmb_op* op, int comp, int block, int* m, int* n, int* K, int* k_cur,
               double* U, double* V, int* piv, double* frob_sq) {
  return guard([&] {
    need(op, "op");
    const int st = hmgpu_download_factor(op->op->gpu(), comp, block, m, n, K, k_cur, U, V,
                                         piv, frob_sq);
    if (st != HMGPU_OK)
      throw hmb::DeviceError(st, std::string("hmgpu_download_factor: ") +
                                     hmgpu_last_error(op->op->gpu()));
  });
}

int hmb_dense_block(const hmb_op* op, int comp, int block, double* out) {
  return guard([&] {
    need(op, "op");
    const int st = hmgpu_download_dense(op->op->gpu(), comp, block, out);
    if (st != HMGPU_OK)
      throw hmb::DeviceError(st, std::string("hmgpu_download_dense: ") +
                                     hmgpu_last_error(op->op->gpu()));
  });
}

int hmb_gamma(hmb_op* op, const double* x, double* gamma, double* difference,
              int* n_terms) {
  return guard([&] {
    need(op, "op");
    need(x, "x");
    op->gamma = hmb::gamma_contributions(*op->op, x);
    if (gamma) *gamma = op->gamma.gamma;
    if (difference)
      std::memcpy(difference, op->gamma.difference.data(),
                  op->gamma.difference.size() * sizeof(double));
    if (n_terms) *n_terms = static_cast<int>(op->gamma.terms.size());
  });
}

int hmb_gamma_t(hmb_op* op, const double* x, double* gamma, double* difference, int* n_terms) {
  return guard([&] {
    need(op, "op");
    need(x, "x");
    op->gamma = hmb::gamma_contributions_transposed(*op->op, x);
    if (gamma) *gamma = op->gamma.gamma;
    if (difference)
      std::memcpy(difference, op->gamma.difference.data(),
                  op->gamma.difference.size() * sizeof(double));
    if (n_terms) *n_terms = static_cast<int>(op->gamma.terms.size());
  });
}

int hmb_gamma_terms(const hmb_op* op, int* comp, int* block, int* nnz, double* norm_sq) {
  return guard([&] {
    need(op, "op");
    const auto& terms = op->gamma.terms;
    for (std::size_t t = 0; t < terms.size(); ++t) {
      if (comp) comp[t] = terms[t].comp;
      if (block) block[t] = terms[t].block;
      if (nnz) nnz[t] = static_cast<int>(terms[t].idx.size());
      if (norm_sq) norm_sq[t] = terms[t].norm_sq;
    }
  });
}

int hmb_gamma_term_data(const hmb_op* op, int t, long long* idx, double* val) {
  return guard([&] {
    need(op, "op");
    const hmb::BlockTerm& term = op->gamma.terms.at(t);
    if (idx) std::memcpy(idx, term.idx.data(), term.idx.size() * sizeof(long long));
    if (val) std::memcpy(val, term.val.data(), term.val.size() * sizeof(double));
  });
}

int hmb_mark(const hmb_op* op, double theta, int c_sp, long long m_rows, long long n_cols,
             int* marked, int* n_marked, double* gamma_pk) {
  return guard([&] {
    need(op, "op");
    const auto mk = hmb::mark_blocks(op->gamma, theta, c_sp, m_rows, n_cols, gamma_pk);
    if (n_marked) *n_marked = static_cast<int>(mk.size());
    if (marked) std::memcpy(marked, mk.data(), mk.size() * sizeof(int));
  });
}

int hmb_mark_sharded(int n_terms, const long long* term_ptr, const long long* idx,
                     const double* val, const double* difference,
                     const unsigned char* own_rows, long long m_rows, long long n_cols,
                     double theta, int c_sp, int nranks, int rank,
                     hmb_allgather_fn allgather, void* user, int* marked, int* n_marked,
                     int* n_marked_total, double* gamma_pk) {
  return guard([&] {
    need(difference, "difference");
    need(own_rows, "own_rows");
    if (!allgather) throw hmb::Error("mark_blocks: no all-gather");
    if (n_terms < 0 || m_rows < 0 || nranks < 1 || rank < 0 || rank >= nranks)
      throw hmb::DimensionError("mark_blocks: bad sizes");
    if (n_terms > 0) {
      need(term_ptr, "term_ptr");
      need(idx, "idx");
      need(val, "val");
    }
    hmb::GammaContributions g;
    g.difference.assign(difference, difference + m_rows);
    g.terms.resize(n_terms);
    for (int t = 0; t < n_terms; ++t) {
      hmb::BlockTerm& term = g.terms[t];
      for (long long e = term_ptr[t]; e < term_ptr[t + 1]; ++e) {
        if (idx[e] < 0 || idx[e] >= m_rows) throw hmb::DimensionError("mark_blocks: row index");
        term.idx.push_back(idx[e]);
        term.val.push_back(val[e]);
        term.norm_sq += val[e] * val[e];
      }
    }
    std::vector<char> own(own_rows, own_rows + m_rows);
    const hmb::AllGather ag = [&](const void* send, void* recv, long long bytes) {
      if (allgather(user, send, recv, bytes)) throw hmb::Error("mark_blocks: all-gather failed");
    };
    int total = 0;
    const auto mk = hmb::mark_blocks_sharded(g, own, theta, c_sp, m_rows, n_cols, ag, nranks,
                                             rank, gamma_pk, &total);
    if (n_marked) *n_marked = static_cast<int>(mk.size());
    if (n_marked_total) *n_marked_total = total;
    if (marked) std::memcpy(marked, mk.data(), mk.size() * sizeof(int));
  });
}

int hmb_amvm(hmb_op* op, const double* x, double theta, double eps_amvm,
             int lookahead_steps, int max_iterations, double* b, double* iters8,
             int* n_iters, int* converged) {
  return guard([&] {
    need(op, "op");
    need(x, "x");
    need(b, "b");
    if (max_iterations < 0) throw hmb::ConfigError("amvm_multiply: max_iterations must be >= 0");
    hmb::AmvmConfig cfg;
    cfg.theta = theta;
    cfg.eps_amvm = eps_amvm;
    cfg.lookahead_steps = lookahead_steps;
    cfg.max_iterations = max_iterations;
    hmb::AmvmReport rep;
    const auto res = hmb::amvm_multiply(*op->op, x, cfg, rep);
    std::memcpy(b, res.data(), res.size() * sizeof(double));
    if (n_iters) *n_iters = static_cast<int>(rep.iterations.size());
    if (converged) *converged = rep.converged ? 1 : 0;
    if (iters8)
      for (std::size_t i = 0; i < rep.iterations.size(); ++i) {
        const auto& it = rep.iterations[i];
        double* r = iters8 + 8 * i;
        r[0] = it.k;
        r[1] = it.gamma;
        r[2] = it.gamma_pk;
        r[3] = it.marked;
        r[4] = static_cast<double>(it.cumulative_pivots);
        r[5] = it.storage_mb;
        r[6] = it.e_hat;
        r[7] = it.ms;
      }
  });
}

}  // extern "C"
