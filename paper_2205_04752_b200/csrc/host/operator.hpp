// Host facade of the B200 H-matrix: keeps the reference's operator API
// (cluster tree, block partition, assemble(), matvec(Mode), promote /
// extend_lookahead, storage accounting, AMVM estimator hooks) and drives the
// device through the C ABI of include/hmgpu.h.
//
// Reference interfaces mirrored (proj/include/hmbem/):
//   AssemblyConfig, HMatrix::{matvec, promote, extend_lookahead,
//     storage_mb_current, storage_mb_tail, total_pivots}   hmatrix.hpp:20-90
//   evaluate_interior's 3x3 Kelvin grid of six aliased component
//     H-matrices                                            baca.cpp:669-687
//   GammaContributions / BlockTerm / mark_blocks /
//     amvm_multiply / AmvmReport                           amvm.hpp:10-71
#pragma once

#include <memory>
#include <string>
#include <functional>
#include <vector>

#include "cluster.hpp"
#include "geometry.hpp"
#include "quadrature.hpp"

struct hmgpu_ctx;

namespace hmb {

struct AssemblyConfig {  // hmatrix.hpp:20-27
  Real eps = 1e-6;
  Real beta = 0.8;        // ACA stopping-rule beta (beta_stop), in (0,1)
  int initial_rank = -1;  // >= 0: coarse mode with this many pivots
  int lookahead = 2;
  long long max_rank = 1LL << 30;
};

enum class Mode { Current = 0, Lookahead = 1 };

struct AssemblyStats {
  long long aca_entries = 0, dense_entries = 0, aca_steps = 0, pivots = 0;
  double ms_total = 0, ms_nearfield = 0, ms_aca = 0;
  int relaunches = 0;
  double counted_flops = 0;  // 30 n_q + 1 per Kelvin component entry
};

// Which rows of the operator this process owns (block-row sharding over
// GPUs).  A rank owns the blocks whose row cluster lies in
// [row_begin, row_end) of the permuted row order.
struct Shard {
  int rank = 0, count = 1;
};

class HOperator {
 public:
  enum Kind { Kelvin = 0, Newton = 1, Dense = 2, Galerkin = 3, KDelta = 4 };

  // Kelvin single-layer collocation at triangle centroids: one cluster tree
  // over the triangle support boxes for rows and columns
  static std::unique_ptr<HOperator> kelvin(const Mesh& mesh, Real E, Real nu,
                                           int b_min, Real eta, int device,
                                           Shard shard = {},
                                           QuadratureConfig qc = {});
  // The single-layer part of evaluate_interior (baca.cpp:625-687): Kelvin
  // collocation at arbitrary points (rows: a tree over the point boxes;
  // columns: the triangle tree), points closer to the surface than
  // min_distance_factor x the largest triangle diameter rejected
  // (baca.cpp:632-643)
  static std::unique_ptr<HOperator> kelvin_points(const Mesh& mesh,
                                                  const std::vector<V3>& points, Real E,
                                                  Real nu, int b_min, Real eta, int device,
                                                  Shard shard = {},
                                                  Real min_distance_factor = 0.5,
                                                  QuadratureConfig qc = {});
  // one cell (r, c) of evaluate_interior's double-layer grid W~ (baca.cpp:
  // 650-651, 674-677): CollocDoubleOracle at the points (rows, point tree)
  // against the vertices (columns, node tree: union of incident triangle boxes)
  static std::unique_ptr<HOperator> kelvin_double_points(
      const Mesh& mesh, const std::vector<V3>& points, int r, int c, Real E, Real nu,
      int b_min, Real eta, int device, Shard shard = {}, Real min_distance_factor = 0.5,
      QuadratureConfig qc = {});
  // Galerkin scalar kernels on the triangle partition of assemble_operators
  // (operators.cpp:186-200, 218-235): which = 0 the six V_kl as the 3x3
  // grid, 1 V_Delta (GalerkinKernels::vkl / vdelta, kernels.cpp:130-149)
  static std::unique_ptr<HOperator> galerkin(const Mesh& mesh, int which, int b_min,
                                             Real eta, int device, Shard shard = {},
                                             QuadratureConfig qc = {},
                                             GalerkinQuadrature gq = {});
  // K_Delta on the triangle x node partition (operators.cpp:186-200):
  // rows triangles, columns vertices (kernels.cpp:151-167)
  static std::unique_ptr<HOperator> kdelta(const Mesh& mesh, int b_min, Real eta,
                                           int device, Shard shard = {},
                                           QuadratureConfig qc = {},
                                           GalerkinQuadrature gq = {});
  // scalar Newton kernel over points; boxes == nullptr => point boxes
  static std::unique_ptr<HOperator> newton(const std::vector<V3>& pts,
                                           const std::vector<Box>* boxes,
                                           Real diag, int b_min, Real eta,
                                           int device, Shard shard = {});
  // explicit column-major matrix with point boxes for rows and columns
  static std::unique_ptr<HOperator> dense(int m, int n, const double* a,
                                          const std::vector<V3>& row_pts,
                                          const std::vector<V3>& col_pts,
                                          int b_min, Real eta, int device,
                                          Shard shard = {});
  ~HOperator();

  Kind kind() const { return kind_; }
  int ncomp() const { return ncomp_; }
  // operator dimensions in DOFs (3 per triangle for Kelvin)
  long long rows() const;
  long long cols() const;
  const ClusterTree& row_tree() const { return *rows_; }
  const ClusterTree& col_tree() const { return cols_ ? *cols_ : *rows_; }
  const BlockPartition& partition() const { return part_; }
  int row_begin() const { return row_begin_; }
  int row_end() const { return row_end_; }
  hmgpu_ctx* gpu() const { return ctx_; }

  AssemblyStats assemble(const AssemblyConfig& cfg);
  const AssemblyConfig& config() const { return cfg_; }
  bool assembled() const { return assembled_; }

  // y = A x (x, y: dofs x nrhs column-major, external component-major order)
  void matvec(const double* x, double* y, int nrhs, Mode mode,
              bool device_ptrs = false) const;
  std::vector<double> matvec(const std::vector<double>& x, Mode mode) const;
  // y = A^T x (HMatrix::matvec_transposed, hmatrix.cpp:47-72): x over rows
  void matvec_transposed(const double* x, double* y, int nrhs, Mode mode,
                         bool device_ptrs = false) const;

  void promote(const std::vector<std::pair<int, int>>& comp_block);
  void extend_lookahead(const std::vector<std::pair<int, int>>& comp_block,
                        int steps);

  // per (comp, block), component-major: -1 for dense / not owned blocks
  void ranks(std::vector<int>& k_cur, std::vector<int>& k_look,
             std::vector<int>* consumed = nullptr,
             std::vector<int>* last_stop = nullptr) const;
  long long total_pivots() const;
  double storage_mb_current() const;
  double storage_mb_tail() const;
  long long matvec_bytes() const;

 private:
  HOperator() = default;
  void init_partition(Real eta, Shard shard);
  void check(int status, const char* what) const;

  Kind kind_ = Kelvin;
  int ncomp_ = 1;
  int n_rows_ = 0, n_cols_ = 0;
  std::unique_ptr<ClusterTree> rows_, cols_;
  BlockPartition part_;
  int row_begin_ = 0, row_end_ = 0;
  AssemblyConfig cfg_;
  bool assembled_ = false;
  hmgpu_ctx* ctx_ = nullptr;
};

// ---- adaptive matvec (Algorithm 2) -----------------------------------------
struct AmvmConfig {  // amvm.hpp:10-15
  Real theta = 0.7;
  Real eps_amvm = 1e-6;
  int lookahead_steps = 2;
  int max_iterations = 100;
};

struct BlockTerm {  // amvm.hpp:19-25; (comp, block) identifies the H-leaf
  int comp = 0, block = 0;
  std::vector<long long> idx;
  std::vector<Real> val;
  Real norm_sq = 0.0;
};

struct GammaContributions {  // amvm.hpp:27-31
  Real gamma = 0.0;
  std::vector<Real> difference;
  std::vector<BlockTerm> terms;
};

GammaContributions gamma_contributions(const HOperator& op, const double* x);
// the same for the transposed occurrence (x over the rows, terms over the columns)
GammaContributions gamma_contributions_transposed(const HOperator& op, const double* x);
std::vector<int> mark_blocks(const GammaContributions& g, Real theta, int c_sp,
                             long long m_rows, long long n_cols,
                             Real* gamma_pk_out = nullptr);

// recv[r * bytes ...] = send of rank r, for every rank (collective)
using AllGather = std::function<void(const void* send, void* recv, long long bytes)>;
// mark_blocks over block-row shards: g holds this rank's terms and the whole
// difference vector, own flags this rank's rows; returns its marked terms
std::vector<int> mark_blocks_sharded(const GammaContributions& g, const std::vector<char>& own,
                                     Real theta, int c_sp, long long m_rows, long long n_cols,
                                     const AllGather& allgather, int nranks, int rank,
                                     Real* gamma_pk_out, int* n_marked_out);

struct AmvmIteration {  // amvm.hpp:50-58
  int k = 0;
  Real gamma = 0.0, gamma_pk = 0.0;
  int marked = 0;
  long long cumulative_pivots = 0;
  Real storage_mb = 0.0;
  Real e_hat = -1.0;
  double ms = 0.0;  // wall time of the iteration (estimator + refinement + matvec)
};

struct AmvmReport {
  std::vector<AmvmIteration> iterations;
  std::string termination;
  bool converged = false;
  int c_sp = 0;
};

std::vector<double> amvm_multiply(HOperator& op, const double* x,
                                  const AmvmConfig& cfg, AmvmReport& report);

}  // namespace hmb
