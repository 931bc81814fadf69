// Minimal Eigen SparseMatrix shim -- TEST INFRASTRUCTURE ONLY (see
// shim_core.hpp).  Compressed column storage with sorted inner indices, as
// Eigen keeps it after setFromTriplets / products.  Arithmetic orders model
// Eigen 3.4 (SparseCore): setFromTriplets sums duplicates in triplet order;
// A*B accumulates, per result column j, over the nonzeros B(k,j) in order
// and A(i,k) in order (conservative_sparse_sparse_product); A*x adds the
// columns in order; A^T*x is a sequential dot per column.
#pragma once

#include "shim_core.hpp"

namespace Eigen {

template <typename S>
class Triplet {
 public:
  Triplet() = default;
  Triplet(Index r, Index c, S v) : r_(r), c_(c), v_(v) {}
  Index row() const { return r_; }
  Index col() const { return c_; }
  S value() const { return v_; }

 private:
  Index r_ = 0, c_ = 0;
  S v_ = 0;
};

template <typename S, int O, typename SI>
class SparseMatrix {
  static_assert(std::is_same_v<S, double> && O == 0, "shim: column-major double only");

 public:
  struct Transposed {
    const SparseMatrix& m;
  };

  SparseMatrix() = default;
  SparseMatrix(Index r, Index c) : rows_(r), cols_(c), outer_(static_cast<std::size_t>(c) + 1, 0) {}
  SparseMatrix(const Transposed& t) { *this = t.m.transposed_copy(); }  // NOLINT

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index outerSize() const { return cols_; }
  Index nonZeros() const { return static_cast<Index>(val_.size()); }
  void makeCompressed() {}
  Transposed transpose() const { return {*this}; }

  template <typename It>
  void setFromTriplets(It begin, It end) {
    // bucket by column in triplet order, then per column sort rows stably
    // and sum duplicates in triplet order
    std::vector<std::vector<std::pair<Index, double>>> col(static_cast<std::size_t>(cols_));
    for (It it = begin; it != end; ++it) {
      if (it->row() < 0 || it->row() >= rows_ || it->col() < 0 || it->col() >= cols_)
        throw std::runtime_error("Eigen shim: triplet out of range");
      col[it->col()].emplace_back(it->row(), it->value());
    }
    outer_.assign(static_cast<std::size_t>(cols_) + 1, 0);
    idx_.clear();
    val_.clear();
    for (Index j = 0; j < cols_; ++j) {
      auto& c = col[j];
      std::stable_sort(c.begin(), c.end(),
                       [](const auto& a, const auto& b) { return a.first < b.first; });
      for (std::size_t q = 0; q < c.size(); ++q) {
        if (q > 0 && c[q].first == c[q - 1].first)
          val_.back() = val_.back() + c[q].second;
        else {
          idx_.push_back(c[q].first);
          val_.push_back(c[q].second);
        }
      }
      outer_[j + 1] = static_cast<Index>(val_.size());
    }
  }

  class InnerIterator {
   public:
    InnerIterator(const SparseMatrix& m, Index outer)
        : m_(m), p_(m.outer_[outer]), end_(m.outer_[outer + 1]), outer_(outer) {}
    explicit operator bool() const { return p_ < end_; }
    InnerIterator& operator++() {
      ++p_;
      return *this;
    }
    Index index() const { return m_.idx_[p_]; }
    Index row() const { return m_.idx_[p_]; }
    Index col() const { return outer_; }
    double value() const { return m_.val_[p_]; }

   private:
    const SparseMatrix& m_;
    Index p_, end_, outer_;
  };

  SparseMatrix transposed_copy() const {
    SparseMatrix t(cols_, rows_);
    std::vector<Index> cnt(static_cast<std::size_t>(rows_) + 1, 0);
    for (Index q : idx_) ++cnt[q + 1];
    for (Index i = 0; i < rows_; ++i) cnt[i + 1] += cnt[i];
    t.outer_ = cnt;
    t.idx_.resize(idx_.size());
    t.val_.resize(val_.size());
    std::vector<Index> pos(cnt.begin(), cnt.end() - 1);
    for (Index j = 0; j < cols_; ++j)
      for (Index p = outer_[j]; p < outer_[j + 1]; ++p) {
        const Index d = pos[idx_[p]]++;
        t.idx_[d] = j;
        t.val_[d] = val_[p];
      }
    return t;
  }

  // A * B
  friend SparseMatrix operator*(const SparseMatrix& a, const SparseMatrix& b) {
    if (a.cols_ != b.rows_) throw std::runtime_error("Eigen shim: spgemm size");
    SparseMatrix r(a.rows_, b.cols_);
    std::vector<double> acc(static_cast<std::size_t>(a.rows_), 0.0);
    std::vector<char> mask(static_cast<std::size_t>(a.rows_), 0);
    std::vector<Index> rows;
    for (Index j = 0; j < b.cols_; ++j) {
      rows.clear();
      for (Index pb = b.outer_[j]; pb < b.outer_[j + 1]; ++pb) {
        const Index k = b.idx_[pb];
        const double y = b.val_[pb];
        for (Index pa = a.outer_[k]; pa < a.outer_[k + 1]; ++pa) {
          const Index i = a.idx_[pa];
          const double x = a.val_[pa];
          if (!mask[i]) {
            mask[i] = 1;
            acc[i] = x * y;
            rows.push_back(i);
          } else {
            acc[i] += x * y;
          }
        }
      }
      std::sort(rows.begin(), rows.end());
      for (Index i : rows) {
        r.idx_.push_back(i);
        r.val_.push_back(acc[i]);
        mask[i] = 0;
      }
      r.outer_[j + 1] = static_cast<Index>(r.val_.size());
    }
    return r;
  }
  friend SparseMatrix operator+(const SparseMatrix& a, const SparseMatrix& b) {
    if (a.rows_ != b.rows_ || a.cols_ != b.cols_)
      throw std::runtime_error("Eigen shim: sparse sum size");
    SparseMatrix r(a.rows_, a.cols_);
    for (Index j = 0; j < a.cols_; ++j) {
      Index p = a.outer_[j], q = b.outer_[j];
      const Index pe = a.outer_[j + 1], qe = b.outer_[j + 1];
      while (p < pe || q < qe) {
        if (q >= qe || (p < pe && a.idx_[p] < b.idx_[q])) {
          r.idx_.push_back(a.idx_[p]);
          r.val_.push_back(a.val_[p++]);
        } else if (p >= pe || b.idx_[q] < a.idx_[p]) {
          r.idx_.push_back(b.idx_[q]);
          r.val_.push_back(b.val_[q++]);
        } else {
          r.idx_.push_back(a.idx_[p]);
          r.val_.push_back(a.val_[p++] + b.val_[q++]);
        }
      }
      r.outer_[j + 1] = static_cast<Index>(r.val_.size());
    }
    return r;
  }
  // -A (SpMat(-t23) in build_sparse_ops, operators.cpp:77)
  friend SparseMatrix operator-(const SparseMatrix& a) {
    SparseMatrix r = a;
    for (double& v : r.val_) v = -v;
    return r;
  }
  friend SparseMatrix operator*(double s, const SparseMatrix& a) {
    SparseMatrix r = a;
    for (double& v : r.val_) v = s * v;
    return r;
  }
  // y = A x
  friend VectorXd operator*(const SparseMatrix& a, const VectorXd& x) {
    if (a.cols_ != x.size()) throw std::runtime_error("Eigen shim: spmv size");
    VectorXd y = VectorXd::Zero(a.rows_);
    for (Index j = 0; j < a.cols_; ++j) {
      const double xj = 1.0 * x[j];
      for (Index p = a.outer_[j]; p < a.outer_[j + 1]; ++p) y[a.idx_[p]] += a.val_[p] * xj;
    }
    return y;
  }
  // y = A^T x
  friend VectorXd operator*(const Transposed& t, const VectorXd& x) {
    const SparseMatrix& a = t.m;
    if (a.rows_ != x.size()) throw std::runtime_error("Eigen shim: spmv^T size");
    VectorXd y = VectorXd::Zero(a.cols_);
    for (Index j = 0; j < a.cols_; ++j) {
      double s = 0.0;
      for (Index p = a.outer_[j]; p < a.outer_[j + 1]; ++p) s += a.val_[p] * x[a.idx_[p]];
      y[j] += 1.0 * s;
    }
    return y;
  }

  // dense copy (Mat(sparse))
  void to_dense(double* out) const {
    std::fill(out, out + rows_ * cols_, 0.0);
    for (Index j = 0; j < cols_; ++j)
      for (Index p = outer_[j]; p < outer_[j + 1]; ++p) out[idx_[p] + j * rows_] = val_[p];
  }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<Index> outer_{0};
  std::vector<Index> idx_;
  std::vector<double> val_;
};

template <typename S, int R, int C, int O, int MR, int MC>
Matrix<S, R, C, O, MR, MC>::Matrix(const SparseMatrix<double>& s) {
  resize(s.rows(), s.cols());
  s.to_dense(data());
}

}  // namespace Eigen
