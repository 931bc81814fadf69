// Minimal Eigen-3 API shim -- TEST INFRASTRUCTURE ONLY.
//
// Purpose: compile the reference's own hot-path sources
// (/root/reference/proj/src/{quadrature,mesh,cluster,kernels,aca,hmatrix,
// expr,amvm}.cpp) UNMODIFIED into oracle/_ref/libhmbem_ref.so, so that the
// CPU restatement (oracle/hmbem_oracle.cpp) and the GPU path can be pinned
// against the reference's code itself.  Eigen3 is not installed in this
// image; this header supplies exactly the subset of its API
// those eight files use (types.hpp:11-18 aliases; the call sites are listed
// in oracle/README_ref.md), nothing more.
//
// Arithmetic model.  Eigen's results depend on its SIMD packet width and
// kernel blocking, which are not recoverable without Eigen; this shim models
// Eigen 3.4 on x86-64 with SSE2 (the reference's Release flags,
// proj/CMakeLists.txt:7-9, set no -march):
//   * dynamic reductions (sum/dot/squaredNorm/norm): two 2-lane packet
//     accumulators, lane sums added, scalar tail (Redux.h,
//     LinearVectorizedTraversal); size-3 reductions sequential;
//   * y = A x, A column-major: per row a sequential sum over the columns,
//     in column blocks of 16/4 once cols >= 128 (GeneralMatrixVector.h);
//   * y = A^T x: per output a 2-lane even/odd sum, lanes added, odd tail;
//   * s * (a b^T): the scalar folded into the left factor
//     (ProductEvaluators.h "scalar * (A * B)" rule);
//   * maxCoeff(&i): first maximum (strict >); v /= s divides.
// These orders are a model, not a pin: the comparisons built on this
// library use the north-star tolerances (ranks +-2, matvec <= 10 eps_ACA),
// never bit equality with a real Eigen build.
#pragma once

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <initializer_list>
#include <limits>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum NoChange_t { NoChange };
enum { ColMajor = 0, RowMajor = 1, AutoAlign = 0, DontAlign = 2 };

template <typename S, int R, int C, int O = 0, int MR = R, int MC = C>
class Matrix;
template <typename S, int O = 0, typename SI = int>
class SparseMatrix;

using VectorXd = Matrix<double, Dynamic, 1>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using Vector3d = Matrix<double, 3, 1>;
using Matrix3d = Matrix<double, 3, 3>;

namespace shim {

// Eigen 3.4 LinearVectorizedTraversal with 2-wide packets (see header).
template <class F>
inline double redux_sum(Index n, F&& t) {
  if (n <= 0) return 0.0;
  if (n < 2) return t(0);
  const Index a1 = n / 2 * 2, a2 = n / 4 * 4;
  double p0a = t(0), p0b = t(1);
  if (a1 > 2) {
    double p1a = t(2), p1b = t(3);
    for (Index i = 4; i < a2; i += 4) {
      p0a += t(i);
      p0b += t(i + 1);
      p1a += t(i + 2);
      p1b += t(i + 3);
    }
    p0a += p1a;
    p0b += p1b;
    if (a1 > a2) {
      p0a += t(a2);
      p0b += t(a2 + 1);
    }
  }
  double r = p0a + p0b;
  for (Index i = a1; i < n; ++i) r += t(i);
  return r;
}

// y = A x, A column-major rows x cols with leading dimension ld.
inline void gemv_cm(const double* A, Index rows, Index cols, Index ld,
                    const double* x, double* y) {
  std::fill(y, y + rows, 0.0);
  if (cols == 0 || rows == 0) return;
  const Index bc = cols < 128 ? cols : (ld * 8 < 32000 ? 16 : 4);
  std::vector<double> c(static_cast<std::size_t>(rows));
  for (Index j2 = 0; j2 < cols; j2 += bc) {
    const Index je = std::min(j2 + bc, cols);
    std::fill(c.begin(), c.end(), 0.0);
    for (Index j = j2; j < je; ++j) {
      const double xj = x[j];
      const double* a = A + j * ld;
      for (Index i = 0; i < rows; ++i) c[i] += a[i] * xj;
    }
    for (Index i = 0; i < rows; ++i) y[i] = c[i] * 1.0 + y[i];
  }
}

// y = A^T x, A column-major n x k with leading dimension ld.
inline void gemv_rm(const double* A, Index n, Index k, Index ld,
                    const double* x, double* y) {
  const Index full = n / 2 * 2;
  for (Index l = 0; l < k; ++l) {
    const double* a = A + l * ld;
    double c0 = 0.0, c1 = 0.0;
    for (Index j = 0; j < full; j += 2) {
      c0 += a[j] * x[j];
      c1 += a[j + 1] * x[j + 1];
    }
    double cc = c0 + c1;
    for (Index j = full; j < n; ++j) cc += a[j] * x[j];
    y[l] = 0.0 + 1.0 * cc;
  }
}

// C = A B (plain, sequential inner sums); A: m x k (lda), B: k x n (ldb).
inline void gemm(const double* A, Index m, Index k, Index lda, const double* B,
                 Index n, Index ldb, bool bt, double* Cm) {
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) {
      double s = 0.0;
      for (Index p = 0; p < k; ++p)
        s += A[i + p * lda] * (bt ? B[j + p * ldb] : B[p + j * ldb]);
      Cm[i + j * m] = s;
    }
}

template <int R, int C>
struct Store {
  static constexpr bool fixed = R > 0 && C > 0;
  using type = std::conditional_t<fixed, std::array<double, fixed ? R * C : 1>,
                                  std::vector<double>>;
};

}  // namespace shim

// ---- views --------------------------------------------------------------
// contiguous vector view: segment(), col()
template <bool Const>
struct VecRef {
  using P = std::conditional_t<Const, const double*, double*>;
  P p;
  Index n;
  Index size() const { return n; }
  Index rows() const { return n; }
  Index cols() const { return 1; }
  const double* data() const { return p; }
  double operator[](Index i) const { return p[i]; }
  double operator()(Index i) const { return p[i]; }
  operator VectorXd() const;
  template <bool C2 = Const, std::enable_if_t<!C2, int> = 0>
  VecRef& operator=(const VectorXd& v);
  template <bool C2 = Const, std::enable_if_t<!C2, int> = 0>
  VecRef& operator+=(const VectorXd& v);
  template <bool C2 = Const, std::enable_if_t<!C2, int> = 0>
  VecRef& operator-=(const VectorXd& v);
  double dot(const VectorXd& v) const;
  double squaredNorm() const {
    return shim::redux_sum(n, [&](Index i) { return p[i] * p[i]; });
  }
  double norm() const { return std::sqrt(squaredNorm()); }
};

// a row vector expression x^T (x a column vector), by reference
template <int N>
struct RowExpr {
  const double* p;
  Index n;
};

// row i of a column-major matrix
template <int C, bool Const>
struct RowRef {
  using P = std::conditional_t<Const, const double*, double*>;
  P p;        // &m(i, 0)
  Index n;    // number of columns
  Index ld;   // column stride
  Matrix<double, C, 1> transpose() const;
  template <bool C2 = Const, int N, std::enable_if_t<!C2, int> = 0>
  RowRef& operator=(const RowExpr<N>& r) {
    if (r.n != n) throw std::runtime_error("Eigen shim: row size mismatch");
    for (Index j = 0; j < n; ++j) p[j * ld] = r.p[j];
    return *this;
  }
  double operator()(Index j) const { return p[j * ld]; }
  Index size() const { return n; }
};

// a range of whole columns of a column-major matrix (middleCols/leftCols)
struct ColsRef;
struct ColsRefT {  // its transpose
  const double* p;
  Index rows, cols, ld;  // of the untransposed block
  VectorXd operator*(const VectorXd& x) const;
};
struct ColsRef {
  const double* p;
  Index rows, cols, ld;
  ColsRefT transpose() const { return {p, rows, cols, ld}; }
  VectorXd operator*(const VectorXd& x) const;
  MatrixXd operator*(const ColsRefT& b) const;
  operator MatrixXd() const;
};

// A^T of a dynamic matrix, by reference
struct MatT {
  const MatrixXd& m;
  VectorXd operator*(const VectorXd& x) const;
  operator MatrixXd() const;
};

// a rectangular block as an assignment target
struct BlockRef {
  double* p;
  Index rows, cols, ld;
  BlockRef& operator=(const MatrixXd& m);
};

// a b^T for 3-vectors (kept unevaluated so that s * (a b^T) folds s into a)
struct Outer3 {
  std::array<double, 3> a, b;
};

// ---- the dense matrix ---------------------------------------------------
template <typename S, int R, int C, int O, int MR, int MC>
class Matrix {
  static_assert(std::is_same_v<S, double>, "shim: double only");

 public:
  using Scalar = double;
  static constexpr bool kFixed = R > 0 && C > 0;
  static constexpr bool kVector = C == 1;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;

  Matrix() {
    if constexpr (kFixed) d_.fill(0.0);
    r_ = R > 0 ? R : 0;
    c_ = C > 0 ? C : 0;
  }
  // size constructors
  template <typename I, std::enable_if_t<std::is_integral_v<I> && (R < 0 && C == 1), int> = 0>
  explicit Matrix(I n) {
    resize(static_cast<Index>(n));
  }
  template <typename I, typename J,
            std::enable_if_t<std::is_integral_v<I> && std::is_integral_v<J> && !kFixed, int> = 0>
  Matrix(I r, J c) {
    resize(static_cast<Index>(r), static_cast<Index>(c));
  }
  // coefficient constructor of a 3-vector
  template <int R2 = R, int C2 = C, std::enable_if_t<R2 == 3 && C2 == 1, int> = 0>
  Matrix(double x, double y, double z) {
    r_ = 3;
    c_ = 1;
    d_ = {x, y, z};
  }
  // size-converting copies (dynamic <-> fixed), as Eigen allows
  template <int R2, int C2, std::enable_if_t<(R2 != R || C2 != C), int> = 0>
  Matrix(const Matrix<double, R2, C2>& o) {
    resize(o.rows(), o.cols());
    std::copy(o.data(), o.data() + o.size(), data());
  }
  explicit Matrix(const SparseMatrix<double>& s);

  // -- shape --
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }

  void resize(Index n) {
    if constexpr (C == 1) resize(n, 1);
    else throw std::runtime_error("Eigen shim: resize(n) on a matrix");
  }
  void resize(Index r, Index c) {
    if constexpr (kFixed) {
      if (r != R || c != C) throw std::runtime_error("Eigen shim: fixed-size resize");
    } else {
      if ((R > 0 && r != R) || (C > 0 && c != C))
        throw std::runtime_error("Eigen shim: resize against a fixed dimension");
      d_.assign(static_cast<std::size_t>(r * c), 0.0);
    }
    r_ = r;
    c_ = c;
  }
  void conservativeResize(NoChange_t, Index c) {
    static_assert(!kFixed, "shim: conservativeResize on a fixed matrix");
    d_.resize(static_cast<std::size_t>(r_ * c), 0.0);  // column-major: cols append
    c_ = c;
  }
  void setZero() { std::fill(d_.begin(), d_.end(), 0.0); }

  // -- factories --
  static Matrix Zero() { return Matrix(); }
  static Matrix Zero(Index n) {
    Matrix m(n);
    return m;
  }
  static Matrix Zero(Index r, Index c) {
    Matrix m(r, c);
    return m;
  }
  static Matrix Constant(double v) {
    Matrix m;
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }
  static Matrix Constant(Index n, double v) {
    Matrix m(n);
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }
  static Matrix Constant(Index r, Index c, double v) {
    Matrix m(r, c);
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, 1.0); }
  static Matrix Identity() {
    Matrix m;
    for (Index i = 0; i < std::min<Index>(R, C); ++i) m(i, i) = 1.0;
    return m;
  }

  // -- access --
  double& operator()(Index i, Index j) { return d_[i + j * r_]; }
  double operator()(Index i, Index j) const { return d_[i + j * r_]; }
  double& operator()(Index i) { return d_[i]; }
  double operator()(Index i) const { return d_[i]; }
  double& operator[](Index i) { return d_[i]; }
  double operator[](Index i) const { return d_[i]; }

  VecRef<false> col(Index j) { return {d_.data() + j * r_, r_}; }
  VecRef<true> col(Index j) const { return {d_.data() + j * r_, r_}; }
  RowRef<C, false> row(Index i) { return {d_.data() + i, c_, r_}; }
  RowRef<C, true> row(Index i) const { return {d_.data() + i, c_, r_}; }
  VecRef<false> segment(Index s, Index n) { return {d_.data() + s, n}; }
  VecRef<true> segment(Index s, Index n) const { return {d_.data() + s, n}; }
  ColsRef middleCols(Index s, Index n) const { return {d_.data() + s * r_, r_, n, r_}; }
  ColsRef leftCols(Index n) const { return middleCols(0, n); }
  BlockRef block(Index i, Index j, Index h, Index w) {
    return {d_.data() + i + j * r_, h, w, r_};
  }

  // x^T of a vector; A^T of a dynamic matrix
  template <int C2 = C, std::enable_if_t<C2 == 1, int> = 0>
  RowExpr<R> transpose() const {
    return {d_.data(), r_};
  }
  template <int C2 = C, std::enable_if_t<C2 != 1, int> = 0>
  MatT transpose() const {
    static_assert(R < 0 && C < 0, "shim: transpose of a fixed matrix");
    return {*this};
  }

  // -- reductions --
  double sum() const {
    return shim::redux_sum(size(), [&](Index i) { return d_[i]; });
  }
  double squaredNorm() const {
    return shim::redux_sum(size(), [&](Index i) { return d_[i] * d_[i]; });
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  template <int R2, int C2>
  double dot(const Matrix<double, R2, C2>& o) const {
    if (o.size() != size()) throw std::runtime_error("Eigen shim: dot size");
    const double* q = o.data();
    return shim::redux_sum(size(), [&](Index i) { return d_[i] * q[i]; });
  }
  double dot(const VecRef<true>& o) const {
    if (o.n != size()) throw std::runtime_error("Eigen shim: dot size");
    return shim::redux_sum(size(), [&](Index i) { return d_[i] * o.p[i]; });
  }
  double dot(const VecRef<false>& o) const { return dot(VecRef<true>{o.p, o.n}); }
  double maxCoeff() const {
    double m = d_[0];
    for (Index i = 1; i < size(); ++i) m = std::max(m, d_[i]);
    return m;
  }
  template <typename I>
  double maxCoeff(I* idx) const {
    Index best = 0;
    for (Index i = 1; i < size(); ++i)
      if (d_[i] > d_[best]) best = i;
    *idx = static_cast<I>(best);
    return d_[best];
  }
  double minCoeff() const {
    double m = d_[0];
    for (Index i = 1; i < size(); ++i) m = std::min(m, d_[i]);
    return m;
  }
  Matrix cwiseAbs() const {
    Matrix m = *this;
    for (auto& v : m.d_) v = std::abs(v);
    return m;
  }
  Matrix cwiseMin(const Matrix& o) const {
    Matrix m = *this;
    for (Index i = 0; i < size(); ++i) m.d_[i] = std::min(d_[i], o.d_[i]);
    return m;
  }
  Matrix cwiseMax(const Matrix& o) const {
    Matrix m = *this;
    for (Index i = 0; i < size(); ++i) m.d_[i] = std::max(d_[i], o.d_[i]);
    return m;
  }
  template <int R2 = R, int C2 = C, std::enable_if_t<R2 == 3 && C2 == 1, int> = 0>
  Matrix cross(const Matrix& o) const {
    const auto& a = d_;
    const auto& b = o.d_;
    return Matrix(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2],
                  a[0] * b[1] - a[1] * b[0]);
  }

  // -- in-place arithmetic (elementwise) --
  Matrix& operator+=(const Matrix& o) {
    check(o);
    for (Index i = 0; i < size(); ++i) d_[i] += o.d_[i];
    return *this;
  }
  Matrix& operator-=(const Matrix& o) {
    check(o);
    for (Index i = 0; i < size(); ++i) d_[i] -= o.d_[i];
    return *this;
  }
  Matrix& operator*=(double s) {
    for (auto& v : d_) v *= s;
    return *this;
  }
  Matrix& operator/=(double s) {
    for (auto& v : d_) v /= s;
    return *this;
  }
  template <int R2 = R, int C2 = C, std::enable_if_t<R2 == 3 && C2 == 3, int> = 0>
  Matrix& operator+=(const Outer3& o) {
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) (*this)(i, j) += o.a[i] * o.b[j];
    return *this;
  }

  void check(const Matrix& o) const {
    if (o.r_ != r_ || o.c_ != c_) throw std::runtime_error("Eigen shim: size mismatch");
  }

 private:
  typename shim::Store<R, C>::type d_{};
  Index r_ = 0, c_ = 0;
};

// ---- elementwise binary operators ---------------------------------------
template <int R, int C>
Matrix<double, R, C> operator+(const Matrix<double, R, C>& a, const Matrix<double, R, C>& b) {
  Matrix<double, R, C> m = a;
  m += b;
  return m;
}
template <int R, int C>
Matrix<double, R, C> operator-(const Matrix<double, R, C>& a, const Matrix<double, R, C>& b) {
  Matrix<double, R, C> m = a;
  m -= b;
  return m;
}
template <int R, int C>
Matrix<double, R, C> operator-(const Matrix<double, R, C>& a) {
  Matrix<double, R, C> m = a;
  for (Index i = 0; i < m.size(); ++i) m.data()[i] = -m.data()[i];
  return m;
}
template <int R, int C>
Matrix<double, R, C> operator*(double s, const Matrix<double, R, C>& a) {
  Matrix<double, R, C> m = a;
  for (Index i = 0; i < m.size(); ++i) m.data()[i] = s * m.data()[i];
  return m;
}
template <int R, int C>
Matrix<double, R, C> operator*(const Matrix<double, R, C>& a, double s) {
  Matrix<double, R, C> m = a;
  for (Index i = 0; i < m.size(); ++i) m.data()[i] = m.data()[i] * s;
  return m;
}
template <int R, int C>
Matrix<double, R, C> operator/(const Matrix<double, R, C>& a, double s) {
  Matrix<double, R, C> m = a;
  for (Index i = 0; i < m.size(); ++i) m.data()[i] = m.data()[i] / s;
  return m;
}
// s * col(l)
inline VectorXd operator*(double s, const VecRef<true>& v) {
  VectorXd m(v.n);
  for (Index i = 0; i < v.n; ++i) m[i] = s * v.p[i];
  return m;
}
inline VectorXd operator*(double s, const VecRef<false>& v) {
  return s * VecRef<true>{v.p, v.n};
}

// ---- products -------------------------------------------------------------
// fixed-size products: coefficient-based, sequential inner sums
template <int R, int K, int C, std::enable_if_t<(R > 0 && K > 0 && C > 0), int> = 0>
Matrix<double, R, C> operator*(const Matrix<double, R, K>& a, const Matrix<double, K, C>& b) {
  Matrix<double, R, C> m;
  for (int j = 0; j < C; ++j)
    for (int i = 0; i < R; ++i) {
      double s = a(i, 0) * b(0, j);
      for (int p = 1; p < K; ++p) s += a(i, p) * b(p, j);
      m(i, j) = s;
    }
  return m;
}
inline VectorXd operator*(const MatrixXd& a, const VectorXd& x) {
  if (a.cols() != x.size()) throw std::runtime_error("Eigen shim: gemv size");
  VectorXd y(a.rows());
  shim::gemv_cm(a.data(), a.rows(), a.cols(), a.rows(), x.data(), y.data());
  return y;
}
inline VectorXd operator*(const MatrixXd& a, const VecRef<true>& x) {
  if (a.cols() != x.n) throw std::runtime_error("Eigen shim: gemv size");
  VectorXd y(a.rows());
  shim::gemv_cm(a.data(), a.rows(), a.cols(), a.rows(), x.p, y.data());
  return y;
}
inline MatrixXd operator*(const MatrixXd& a, const MatrixXd& b) {
  if (a.cols() != b.rows()) throw std::runtime_error("Eigen shim: gemm size");
  MatrixXd m(a.rows(), b.cols());
  shim::gemm(a.data(), a.rows(), a.cols(), a.rows(), b.data(), b.cols(), b.rows(), false,
             m.data());
  return m;
}
// a * b^T of 3-vectors, and s * (a b^T) with s folded into a
inline Outer3 operator*(const Vector3d& a, const RowExpr<3>& bt) {
  return {{a[0], a[1], a[2]}, {bt.p[0], bt.p[1], bt.p[2]}};
}
inline Outer3 operator*(double s, const Outer3& o) {
  return {{o.a[0] * s, o.a[1] * s, o.a[2] * s}, o.b};
}

// ---- view members needing the complete Matrix -------------------------------
template <bool Const>
VecRef<Const>::operator VectorXd() const {
  VectorXd v(n);
  std::copy(p, p + n, v.data());
  return v;
}
template <bool Const>
template <bool C2, std::enable_if_t<!C2, int>>
VecRef<Const>& VecRef<Const>::operator=(const VectorXd& v) {
  if (v.size() != n) throw std::runtime_error("Eigen shim: assign size");
  std::copy(v.data(), v.data() + n, p);
  return *this;
}
template <bool Const>
template <bool C2, std::enable_if_t<!C2, int>>
VecRef<Const>& VecRef<Const>::operator+=(const VectorXd& v) {
  if (v.size() != n) throw std::runtime_error("Eigen shim: += size");
  for (Index i = 0; i < n; ++i) p[i] += v[i];
  return *this;
}
template <bool Const>
template <bool C2, std::enable_if_t<!C2, int>>
VecRef<Const>& VecRef<Const>::operator-=(const VectorXd& v) {
  if (v.size() != n) throw std::runtime_error("Eigen shim: -= size");
  for (Index i = 0; i < n; ++i) p[i] -= v[i];
  return *this;
}
template <bool Const>
double VecRef<Const>::dot(const VectorXd& v) const {
  return shim::redux_sum(n, [&](Index i) { return p[i] * v[i]; });
}
template <int C, bool Const>
Matrix<double, C, 1> RowRef<C, Const>::transpose() const {
  Matrix<double, C, 1> v;
  if constexpr (C < 0) v.resize(n);
  for (Index j = 0; j < n; ++j) v[j] = p[j * ld];
  return v;
}
inline VectorXd ColsRef::operator*(const VectorXd& x) const {
  if (x.size() != cols) throw std::runtime_error("Eigen shim: gemv size");
  VectorXd y(rows);
  shim::gemv_cm(p, rows, cols, ld, x.data(), y.data());
  return y;
}
inline VectorXd ColsRefT::operator*(const VectorXd& x) const {
  if (x.size() != rows) throw std::runtime_error("Eigen shim: gemv^T size");
  VectorXd y(cols);
  shim::gemv_rm(p, rows, cols, ld, x.data(), y.data());
  return y;
}
inline MatrixXd ColsRef::operator*(const ColsRefT& b) const {
  if (cols != b.cols) throw std::runtime_error("Eigen shim: gemm size");
  MatrixXd m(rows, b.rows);
  shim::gemm(p, rows, cols, ld, b.p, b.rows, b.ld, true, m.data());
  return m;
}
inline ColsRef::operator MatrixXd() const {
  MatrixXd m(rows, cols);
  for (Index j = 0; j < cols; ++j) std::copy(p + j * ld, p + j * ld + rows, &m(0, j));
  return m;
}
inline VectorXd MatT::operator*(const VectorXd& x) const {
  if (x.size() != m.rows()) throw std::runtime_error("Eigen shim: gemv^T size");
  VectorXd y(m.cols());
  shim::gemv_rm(m.data(), m.rows(), m.cols(), m.rows(), x.data(), y.data());
  return y;
}
inline MatT::operator MatrixXd() const {
  MatrixXd t(m.cols(), m.rows());
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = 0; i < m.rows(); ++i) t(j, i) = m(i, j);
  return t;
}
inline BlockRef& BlockRef::operator=(const MatrixXd& m) {
  if (m.rows() != rows || m.cols() != cols) throw std::runtime_error("Eigen shim: block size");
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) p[i + j * ld] = m(i, j);
  return *this;
}

}  // namespace Eigen
