// oracle/_ref driver -- TEST INFRASTRUCTURE ONLY.
//
// A C ABI over the reference's OWN hot-path code (/root/reference/proj/src/
// {quadrature,mesh,cluster,kernels,aca,hmatrix,expr,amvm,operators}.cpp compiled
// unmodified against oracle/ref_shim/, see oracle/Makefile).  It builds the
// north-star matrix the way the reference would: load_mesh (mesh.cpp:180-
// 219) for the geometry caches, one cluster tree over the triangle support
// boxes (operators.cpp:188-192 / test_hmatrix.cpp:33-37), build_block_
// partition, one CollocSingleOracle per component (kernels.hpp:107-126) at
// the triangle centroids, assemble() six times and the 3x3 BlockGrid with
// the Kelvin symmetry aliasing (baca.cpp:669-687); matvec / amvm_multiply /
// gamma_contributions are the reference's functions on that expression.
//
// The only code here that is not the reference's is (a) this glue and (b)
// the builder-defined self term on the diagonal (the reference has none,
// SURVEY.md 0.4): the same closed form as oracle/hmbem_oracle.cpp
// self_term(), restated.  A second problem kind is the reference test suite's
// CentroidKernelOracle fixture (test_hmatrix.cpp:12-28: 1/|c_i - c_j|, 2 on
// the diagonal).
//
// Never linked into or called by the product (paper_2205_04752_b200/).
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <unistd.h>
#include <vector>

#include "hmbem/amvm.hpp"
#include "hmbem/cluster.hpp"
#include "hmbem/expr.hpp"
#include "hmbem/hmatrix.hpp"
#include "hmbem/kernels.hpp"
#include "hmbem/mesh.hpp"
#include "hmbem/operators.hpp"
#include "hmbem/parallel.hpp"

using namespace hmbem;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

const int kCompR[6] = {0, 0, 0, 1, 1, 2};
const int kCompC[6] = {0, 1, 2, 1, 2, 2};

// builder-defined self term: exact integral of the Kelvin tensor over the
// flat triangle t at its centroid (see oracle/hmbem_oracle.cpp self_term)
Mat3 self_term(const SurfaceMesh& mesh, int t, const MaterialConfig& m) {
  const auto v = mesh.corners(t);
  const Vec3 p = mesh.centroids[t];
  Vec3 nrm = (v[1] - v[0]).cross(v[2] - v[0]);
  nrm = nrm / nrm.norm();
  Real i1 = 0.0;
  Real irc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int e = 0; e < 3; ++e) {
    const Vec3 a = v[e], b = v[(e + 1) % 3];
    Vec3 tt = b - a;
    tt = tt / tt.norm();
    const Vec3 mm = tt.cross(nrm);
    const Vec3 pa = a - p, pb = b - p;
    const Real h = pa.dot(mm);
    const Real s1 = pa.dot(tt), s2 = pb.dot(tt);
    const Real r1 = pa.norm(), r2 = pb.norm();
    const Real lg = std::log((r2 + s2) / (r1 + s1));
    const Real dsin = s2 / r2 - s1 / r1;
    const Real dcos = h / r1 - h / r2;
    i1 += h * lg;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c)
        irc[r][c] += h * (mm[r] * mm[c] * dsin + (mm[r] * tt[c] + tt[r] * mm[c]) * dcos +
                          tt[r] * tt[c] * (lg - dsin));
  }
  const Real cst = (1.0 + m.nu) / (8.0 * M_PI * m.E * (1.0 - m.nu));
  const Real c34 = 3.0 - 4.0 * m.nu;
  Mat3 s;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) s(r, c) = cst * ((r == c ? c34 * i1 : 0.0) + irc[r][c]);
  return s;
}

// The north-star entry oracle: CollocSingleOracle at the centroids, the
// self term on the diagonal.
class KelvinCentroidOracle : public EntryOracle {
 public:
  KelvinCentroidOracle(std::shared_ptr<const GalerkinKernels> k,
                       std::shared_ptr<const Mat> pts, int r, int c, MaterialConfig m,
                       std::shared_ptr<const std::vector<Mat3>> self)
      : inner_(std::move(k), std::move(pts), r, c, m), self_(std::move(self)), r_(r), c_(c) {}
  Index rows() const override { return inner_.rows(); }
  Index cols() const override { return inner_.cols(); }
  Real entry(Index i, Index j) const override {
    if (i == j) return (*self_)[i](r_, c_);
    return inner_.entry(i, j);
  }

 private:
  CollocSingleOracle inner_;
  std::shared_ptr<const std::vector<Mat3>> self_;
  int r_, c_;
};

// test_hmatrix.cpp:12-28
class NewtonCentroidOracle : public EntryOracle {
 public:
  explicit NewtonCentroidOracle(const SurfaceMesh& mesh) : pts_(mesh.centroids) {}
  Index rows() const override { return static_cast<Index>(pts_.size()); }
  Index cols() const override { return static_cast<Index>(pts_.size()); }
  Real entry(Index i, Index j) const override {
    if (i == j) return 2.0;
    return 1.0 / (pts_[i] - pts_[j]).norm();
  }

 private:
  std::vector<Vec3> pts_;
};

}  // namespace

struct hmr_problem {
  std::shared_ptr<SurfaceMesh> mesh;
  MaterialConfig mat;
  std::shared_ptr<GalerkinKernels> kernels;
  std::shared_ptr<ClusterTree> tree;
  std::shared_ptr<const BlockPartition> part;
  int ncomp = 1;
  std::vector<std::shared_ptr<EntryOracle>> oracles;
  std::vector<std::shared_ptr<HMatrix>> h;
  ExprPtr op;  // BlockGrid (Kelvin) or the single leaf (Newton)
  GammaContributions gamma;
};

// The Galerkin operator set of the mixed problem (assemble_operators,
// operators.cpp:187-245) and the right-hand-side operator of assemble_rhs.
struct hmr_ops {
  std::shared_ptr<SurfaceMesh> mesh;
  OperatorSet ops;
  ExprPtr rhs;
};

namespace {
// rhs_operator (baca.cpp:42-55), restated: baca.cpp (preconditioner, BPCG,
// BACA) is not part of _ref, its composition of the right-hand side is
// these lines
ExprPtr rhs_operator_ref(const OperatorSet& ops) {
  const DofLayout& layout = ops.layout;
  const ExprPtr mass = leaf(ops.sparse.mass_d3);
  const ExprPtr top = sum({scale(0.5, mass), ops.kh});
  const ExprPtr bottom = sum({scale(0.5, transpose(mass)), scale(-1.0, transpose(ops.kh))});
  const ExprPtr full = block2x2(scale(-1.0, ops.vh), top, bottom, scale(-1.0, ops.dh));
  const Index m3 = 3 * static_cast<Index>(layout.num_triangles);
  std::vector<Index> rows = dirichlet_triangle_dofs(layout);
  for (Index u : neumann_node_dofs(layout)) rows.push_back(m3 + u);
  return compose({leaf(selection_matrix(rows, full->rows())), full});
}

std::shared_ptr<SurfaceMesh> load_off_mesh(int nv, const double* xyz, int nt, const int* tri,
                                           const std::string& predicate) {
  char path[] = "/tmp/hmr_meshXXXXXX";
  const int fd = mkstemp(path);
  if (fd < 0) throw Error("mkstemp failed");
  close(fd);
  {
    std::ofstream f(path);
    f << "OFF\n" << nv << " " << nt << " 0\n";
    char buf[96];
    for (int v = 0; v < nv; ++v) {
      std::snprintf(buf, sizeof buf, "%.17g %.17g %.17g\n", xyz[3 * v], xyz[3 * v + 1],
                    xyz[3 * v + 2]);
      f << buf;
    }
    for (int t = 0; t < nt; ++t)
      f << "3 " << tri[3 * t] << " " << tri[3 * t + 1] << " " << tri[3 * t + 2] << "\n";
  }
  BoundaryLabeling lab;
  lab.dirichlet_predicate = predicate;
  std::shared_ptr<SurfaceMesh> mesh;
  try {
    mesh = std::make_shared<SurfaceMesh>(load_mesh(path, lab));
  } catch (...) {
    std::remove(path);
    throw;
  }
  std::remove(path);
  return mesh;
}
}  // namespace

#define HMR_API __attribute__((visibility("default")))

extern "C" {

HMR_API const char* hmr_last_error() { return g_err.c_str(); }

// kind 0: Kelvin centroid collocation (6 components, 3x3 grid); kind 1: the
// reference's Newton CentroidKernelOracle fixture (1 component).
HMR_API int hmr_create(int kind, int nv, const double* xyz, int nt, const int* tri, double E,
               double nu, int b_min, double eta, hmr_problem** out) {
  return guard([&] {
    if (!out || !xyz || !tri) throw Error("null argument");
    auto p = std::make_unique<hmr_problem>();
    // the reference's loader computes the caches (areas, normals,
    // centroids, incident triangles) and validates the mesh
    char path[] = "/tmp/hmr_meshXXXXXX";
    const int fd = mkstemp(path);
    if (fd < 0) throw Error("mkstemp failed");
    close(fd);
    {
      std::ofstream f(path);
      f << "OFF\n" << nv << " " << nt << " 0\n";
      char buf[96];
      for (int v = 0; v < nv; ++v) {
        std::snprintf(buf, sizeof buf, "%.17g %.17g %.17g\n", xyz[3 * v], xyz[3 * v + 1],
                      xyz[3 * v + 2]);
        f << buf;
      }
      for (int t = 0; t < nt; ++t)
        f << "3 " << tri[3 * t] << " " << tri[3 * t + 1] << " " << tri[3 * t + 2] << "\n";
    }
    BoundaryLabeling lab;
    lab.dirichlet_predicate = "x1<1e300";  // labels are not used on this path
    try {
      p->mesh = std::make_shared<SurfaceMesh>(load_mesh(path, lab));
    } catch (...) {
      std::remove(path);
      throw;
    }
    std::remove(path);
    p->mat = make_material(E, nu);
    std::vector<Box> boxes(p->mesh->num_triangles());
    for (int t = 0; t < p->mesh->num_triangles(); ++t)
      for (const Vec3& c : p->mesh->corners(t)) boxes[t].absorb(c);
    p->tree = std::make_shared<ClusterTree>(build_cluster_tree(boxes, b_min));
    p->part = std::make_shared<const BlockPartition>(build_block_partition(p->tree, p->tree, eta));
    if (kind == 0) {
      p->ncomp = 6;
      QuadratureConfig qc;
      p->kernels = std::make_shared<GalerkinKernels>(p->mesh, qc);
      auto pts = std::make_shared<Mat>(p->mesh->num_triangles(), 3);
      for (int t = 0; t < p->mesh->num_triangles(); ++t)
        for (int d = 0; d < 3; ++d) (*pts)(t, d) = p->mesh->centroids[t][d];
      auto self = std::make_shared<std::vector<Mat3>>(p->mesh->num_triangles());
      for (int t = 0; t < p->mesh->num_triangles(); ++t)
        (*self)[t] = self_term(*p->mesh, t, p->mat);
      for (int q = 0; q < 6; ++q)
        p->oracles.push_back(std::make_shared<KelvinCentroidOracle>(
            p->kernels, pts, kCompR[q], kCompC[q], p->mat, self));
    } else if (kind == 1) {
      p->ncomp = 1;
      p->oracles.push_back(std::make_shared<NewtonCentroidOracle>(*p->mesh));
    } else {
      throw Error("hmr_create: unknown kind");
    }
    *out = p.release();
  });
}

HMR_API void hmr_destroy(hmr_problem* p) { delete p; }

HMR_API int hmr_set_threads(int n) {
  thread_cap() = n;
  return 0;
}

HMR_API int hmr_partition_json(const hmr_problem* p, char* buf, long long* len) {
  return guard([&] {
    const std::string s = partition_to_json(*p->part);
    if (!buf) {
      *len = static_cast<long long>(s.size()) + 1;
      return;
    }
    if (*len < static_cast<long long>(s.size()) + 1) throw Error("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

HMR_API int hmr_info(const hmr_problem* p, int* n, int* n_blocks, int* ncomp, int* c_sp, int* n_nodes) {
  return guard([&] {
    if (n) *n = p->tree->size();
    if (n_blocks) *n_blocks = static_cast<int>(p->part->blocks.size());
    if (ncomp) *ncomp = p->ncomp;
    if (c_sp) *c_sp = sparsity_constant(*p->part);
    if (n_nodes) *n_nodes = static_cast<int>(p->tree->nodes.size());
  });
}

// perm[n]; nodes[n_nodes][4] = begin, end, child0, child1; blocks[nb][4] =
// row_node, col_node, admissible, level
HMR_API int hmr_tree(const hmr_problem* p, int* perm, int* nodes4, int* blocks4) {
  return guard([&] {
    if (perm) std::copy(p->tree->perm.begin(), p->tree->perm.end(), perm);
    if (nodes4)
      for (std::size_t i = 0; i < p->tree->nodes.size(); ++i) {
        const auto& nd = p->tree->nodes[i];
        nodes4[4 * i] = nd.begin;
        nodes4[4 * i + 1] = nd.end;
        nodes4[4 * i + 2] = nd.child[0];
        nodes4[4 * i + 3] = nd.child[1];
      }
    if (blocks4)
      for (std::size_t b = 0; b < p->part->blocks.size(); ++b) {
        const Block& bl = p->part->blocks[b];
        blocks4[4 * b] = bl.row_node;
        blocks4[4 * b + 1] = bl.col_node;
        blocks4[4 * b + 2] = bl.admissible ? 1 : 0;
        blocks4[4 * b + 3] = bl.level;
      }
  });
}

// bounded CPU samples: keep only the blocks whose row cluster lies inside
// the internal row range [row_begin, row_end) (one subtree of the row tree);
// the reference's assemble / matvec then run on that block-row sample
// (call before hmr_assemble)
HMR_API int hmr_restrict_rows(hmr_problem* p, int row_begin, int row_end) {
  return guard([&] {
    BlockPartition q = *p->part;
    q.blocks.clear();
    for (const Block& b : p->part->blocks) {
      const ClusterNode& rn = p->tree->nodes[b.row_node];
      if (rn.begin >= row_begin && rn.end <= row_end) q.blocks.push_back(b);
    }
    p->part = std::make_shared<const BlockPartition>(std::move(q));
    p->h.clear();
    p->op.reset();
  });
}

HMR_API int hmr_entry(const hmr_problem* p, int comp, long long i, long long j, double* out) {
  return guard([&] { *out = p->oracles.at(comp)->entry(i, j); });
}

// assemble(part, oracle, cfg) per component (hmatrix.cpp:147-186); the grid
// expression as evaluate_interior builds it (baca.cpp:669-687)
HMR_API int hmr_assemble(hmr_problem* p, double eps, double beta, int initial_rank, int lookahead,
                 long long max_rank) {
  return guard([&] {
    AssemblyConfig cfg;
    cfg.eps = eps;
    cfg.beta = beta;
    cfg.initial_rank = initial_rank;
    cfg.lookahead = lookahead;
    cfg.max_rank = static_cast<int>(std::min<long long>(max_rank, 1 << 30));
    p->h.clear();
    for (int q = 0; q < p->ncomp; ++q) p->h.push_back(assemble(p->part, p->oracles[q], cfg));
    if (p->ncomp == 1) {
      p->op = leaf(p->h[0]);
    } else {
      std::vector<ExprPtr> grid(9);
      for (int q = 0; q < 6; ++q) {
        const int r = kCompR[q], c = kCompC[q];
        grid[r * 3 + c] = leaf(p->h[q]);
        if (c != r) grid[c * 3 + r] = grid[r * 3 + c];
      }
      p->op = block_grid(3, 3, std::move(grid));
    }
  });
}

// kcur / klook [ncomp][n_blocks]; -1 on dense blocks
HMR_API int hmr_ranks(const hmr_problem* p, int* kcur, int* klook) {
  return guard([&] {
    if (p->h.empty()) throw Error("assemble first");
    const int nb = static_cast<int>(p->part->blocks.size());
    for (int q = 0; q < p->ncomp; ++q)
      for (int b = 0; b < nb; ++b) {
        const HBlock& hb = p->h[q]->block(b);
        kcur[q * nb + b] = hb.is_lowrank() ? hb.current_rank : -1;
        klook[q * nb + b] = hb.is_lowrank() ? hb.lookahead_rank() : -1;
      }
  });
}

// storage_mb_current summed over the components, total pivots
HMR_API int hmr_storage(const hmr_problem* p, double* mb_current, long long* pivots) {
  return guard([&] {
    double mb = 0.0;
    long long piv = 0;
    for (const auto& h : p->h) {
      mb += h->storage_mb_current();
      piv += h->total_pivots();
    }
    if (mb_current) *mb_current = mb;
    if (pivots) *pivots = piv;
  });
}

// U (m x K, column-major), V (n x K), pivots [K][2]; two-call protocol
HMR_API int hmr_factor(const hmr_problem* p, int comp, int block, int* m, int* n, int* K, int* kcur,
               double* U, double* V, int* piv) {
  return guard([&] {
    const HBlock& hb = p->h.at(comp)->block(block);
    if (!hb.is_lowrank()) throw Error("dense block");
    *m = static_cast<int>(hb.factor.U.rows());
    *n = static_cast<int>(hb.factor.V.rows());
    *K = hb.factor.rank();
    *kcur = hb.current_rank;
    if (U) std::memcpy(U, hb.factor.U.data(), sizeof(double) * hb.factor.U.size());
    if (V) std::memcpy(V, hb.factor.V.data(), sizeof(double) * hb.factor.V.size());
    if (piv)
      for (int l = 0; l < hb.factor.rank(); ++l) {
        piv[2 * l] = hb.factor.pivots[l].first;
        piv[2 * l + 1] = hb.factor.pivots[l].second;
      }
  });
}

// y = A x through the reference's expression matvec (expr.cpp:197-215,
// hmatrix.cpp:22-45); mode 0 current, 1 look-ahead
HMR_API int hmr_matvec(const hmr_problem* p, const double* x, double* y, int mode) {
  return guard([&] {
    if (!p->op) throw Error("assemble first");
    const Index n = p->op->cols();
    Vec xv(n);
    std::copy(x, x + n, xv.data());
    const Vec yv = matvec(*p->op, xv, mode ? Mode::Lookahead : Mode::Current);
    std::copy(yv.data(), yv.data() + yv.size(), y);
  });
}

// gamma_contributions over the expression (amvm.cpp:46-129)
HMR_API int hmr_gamma(hmr_problem* p, const double* x, double* gamma, double* difference,
              int* n_terms) {
  return guard([&] {
    const Index n = p->op->cols();
    Vec xv(n);
    std::copy(x, x + n, xv.data());
    p->gamma = gamma_contributions(p->op, xv);
    if (gamma) *gamma = p->gamma.gamma;
    if (difference)
      std::copy(p->gamma.difference.data(),
                p->gamma.difference.data() + p->gamma.difference.size(), difference);
    if (n_terms) *n_terms = static_cast<int>(p->gamma.terms.size());
  });
}

// mark_blocks on the last gamma (amvm.cpp:131-184): marked term indices and
// the (component, block) of every term
HMR_API int hmr_mark(hmr_problem* p, double theta, int* marked, int* n_marked, double* gamma_pk,
             int* term_comp_block) {
  return guard([&] {
    const int c_sp = operator_sparsity_constant(p->op);
    Real gpk = 0.0;
    const auto m = mark_blocks(p->gamma, theta, c_sp, p->op->rows(), p->op->cols(), &gpk);
    if (marked) std::copy(m.begin(), m.end(), marked);
    if (n_marked) *n_marked = static_cast<int>(m.size());
    if (gamma_pk) *gamma_pk = gpk;
    if (term_comp_block)
      for (std::size_t t = 0; t < p->gamma.terms.size(); ++t) {
        int comp = 0;
        for (int q = 0; q < p->ncomp; ++q)
          if (p->h[q].get() == p->gamma.terms[t].h) comp = q;
        term_comp_block[2 * t] = comp;
        term_comp_block[2 * t + 1] = p->gamma.terms[t].block;
      }
  });
}

// assemble_operators on the labelled mesh (full-mode ACA at eps, beta_stop
// for the stopping rule, eta for admissibility); sizes of the RHS operator
HMR_API int hmr_ops_create(int nv, const double* xyz, int nt, const int* tri,
                           const char* predicate, double E, double nu, int b_min, double eta,
                           double eps, double beta_stop, int lookahead, hmr_ops** out,
                           long long* rows, long long* cols) {
  return guard([&] {
    if (!out || !xyz || !tri || !predicate) throw Error("null argument");
    auto p = std::make_unique<hmr_ops>();
    p->mesh = load_off_mesh(nv, xyz, nt, tri, predicate);
    OperatorConfig cfg;
    cfg.clustering.b_min = b_min;
    cfg.clustering.beta = eta;
    cfg.eps_aca = eps;
    cfg.beta_stop = beta_stop;
    cfg.lookahead = lookahead;
    p->ops = assemble_operators(p->mesh, make_material(E, nu), cfg);
    p->rhs = rhs_operator_ref(p->ops);
    if (rows) *rows = p->rhs->rows();
    if (cols) *cols = p->rhs->cols();
    *out = p.release();
  });
}

HMR_API void hmr_ops_destroy(hmr_ops* p) { delete p; }

// f = rhs_operator x at the current ranks (assemble_rhs without AMVM)
HMR_API int hmr_ops_rhs(const hmr_ops* p, const double* x, double* f) {
  return guard([&] {
    Vec xv(p->rhs->cols());
    std::copy(x, x + xv.size(), xv.data());
    const Vec y = matvec(*p->rhs, xv, Mode::Current);
    std::copy(y.data(), y.data() + y.size(), f);
  });
}

// assemble_rhs with opt.amvm (baca.cpp:57-76): amvm_multiply over the RHS
// operator; iters8 as hmr_amvm
HMR_API int hmr_ops_rhs_amvm(hmr_ops* p, const double* x, double theta, double eps_amvm,
                             int lookahead_steps, int max_iterations, double* f,
                             double* iters8, int* n_iters, int* converged) {
  return guard([&] {
    Vec xv(p->rhs->cols());
    std::copy(x, x + xv.size(), xv.data());
    AmvmConfig cfg;
    cfg.theta = theta;
    cfg.eps_amvm = eps_amvm;
    cfg.lookahead_steps = lookahead_steps;
    cfg.max_iterations = max_iterations;
    auto [res, rep] = amvm_multiply(p->rhs, xv, cfg);
    std::copy(res.data(), res.data() + res.size(), f);
    *n_iters = static_cast<int>(rep.iterations.size());
    *converged = rep.converged ? 1 : 0;
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
      r[7] = 0.0;
    }
  });
}

// amvm_multiply (amvm.cpp:199-268) on the expression; iters8 rows:
// k, gamma, gamma_pk, marked, cumulative_pivots, storage_mb, e_hat, 0
HMR_API int hmr_amvm(hmr_problem* p, const double* x, double theta, double eps_amvm,
             int lookahead_steps, int max_iterations, double* b, double* iters8, int* n_iters,
             int* converged) {
  return guard([&] {
    const Index n = p->op->cols();
    Vec xv(n);
    std::copy(x, x + n, xv.data());
    AmvmConfig cfg;
    cfg.theta = theta;
    cfg.eps_amvm = eps_amvm;
    cfg.lookahead_steps = lookahead_steps;
    cfg.max_iterations = max_iterations;
    auto [res, rep] = amvm_multiply(p->op, xv, cfg);
    std::copy(res.data(), res.data() + res.size(), b);
    *n_iters = static_cast<int>(rep.iterations.size());
    *converged = rep.converged ? 1 : 0;
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
      r[7] = 0.0;
    }
  });
}

}  // extern "C"
