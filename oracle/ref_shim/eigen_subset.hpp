// eigen_subset.hpp -- TEST INFRASTRUCTURE (oracle/_ref build only).
//
// A minimal, eager (no expression templates) stand-in for the part of the
// Eigen 3 API the reference sources under /root/reference/proj use, so that
// the unmodified reference compiles here (oracle/Makefile, target `ref`;
// SURVEY.md 7.1 step 1). Eigen itself is not in this image. Only the API
// surface the reference touches is provided:
//   Matrix<double, R, C> (fixed and Dynamic), comma initializer, Zero /
//   Identity / Unit*, block<r,c> / col / head / tail / segment views,
//   transpose, products, norm / squaredNorm / normalized / dot / cross,
//   cwiseAbs / maxCoeff / minCoeff / allFinite / lpNorm<Infinity> / trace /
//   determinant / inverse / asDiagonal / diagonal().array() +=, ldlt().solve(),
//   Quaterniond (from a rotation matrix, toRotationMatrix), AngleAxisd,
//   SelfAdjointEigenSolver (eigenvalues), JacobiSVD (singular values).
// Storage is column-major as in Eigen. Arithmetic is plain sequential double
// loops: results agree with Eigen to rounding (Eigen's vectorised kernels sum
// in other orders); the decompositions restate Eigen's published algorithms
// (LDLT: diagonal pivoting on the largest remaining |diagonal|, as
// Eigen/src/Cholesky/LDLT.h; quaternion from matrix: Shoemake's branch order,
// as Eigen/src/Geometry/Quaternion.h), the same restatements the oracle uses
// (oracle/dynsurf_oracle.cpp:135-182, 441-555).
#pragma once

#include <algorithm>
#include <array>
#include <cfloat>
#include <cmath>
#include <cstddef>
#include <limits>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
inline constexpr int Dynamic = -1;
inline constexpr int Infinity = 10000;

template <typename S, int R, int C>
class Matrix;
template <typename M, int R, int C>
class Block;

namespace detail {
template <typename T>
struct is_matrix : std::false_type {};
template <typename S, int R, int C>
struct is_matrix<Matrix<S, R, C>> : std::true_type {};
template <typename T>
struct is_block : std::false_type {};
template <typename M, int R, int C>
struct is_block<Block<M, R, C>> : std::true_type {};
template <typename T>
inline constexpr bool is_expr_v =
    is_matrix<std::remove_cvref_t<T>>::value || is_block<std::remove_cvref_t<T>>::value;
constexpr int prod_dim(int a, int b) { return a == Dynamic ? Dynamic : b; }
}  // namespace detail

template <typename T>
concept MatExpr = detail::is_expr_v<T>;

// -------------------------------------------------------------- comma init
template <typename M>
class CommaInit {
 public:
  CommaInit(M& m, double v) : m_(m) { put(v); }
  CommaInit& operator,(double v) {
    put(v);
    return *this;
  }
  template <typename V>
    requires requires(const V& x) { x.eval(); }
  CommaInit& operator,(const V& v) {  // vector blocks stacked (column vectors)
    const auto& e = v.eval();
    for (Index k = 0; k < e.size(); ++k) put(e[k]);
    return *this;
  }

 private:
  void put(double v) {  // row by row, as Eigen's comma initializer
    const Index r = k_ / m_.cols(), c = k_ % m_.cols();
    m_(r, c) = v;
    ++k_;
  }
  M& m_;
  Index k_ = 0;
};

// --------------------------------------------------------- diagonal proxy
template <typename M>
class DiagonalArray {
 public:
  explicit DiagonalArray(M& m) : m_(m) {}
  DiagonalArray& operator+=(double v) {
    const Index n = std::min(m_.rows(), m_.cols());
    for (Index i = 0; i < n; ++i) m_(i, i) += v;
    return *this;
  }
  DiagonalArray& operator-=(double v) { return *this += -v; }
  DiagonalArray& array() { return *this; }

 private:
  M& m_;
};

// ------------------------------------------------------------------ matrix
template <typename S, int R, int C>
class Matrix {
 public:
  static constexpr bool kDyn = (R == Dynamic || C == Dynamic);
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  using Scalar = S;

  Matrix() {
    if constexpr (!kDyn) d_.fill(S(0));
    else {
      rows_ = R == Dynamic ? 0 : R;
      cols_ = C == Dynamic ? 0 : C;
    }
  }
  Matrix(Index r, Index c)
    requires kDyn
  {
    resize(r, c);
  }
  explicit Matrix(Index n)
    requires(kDyn && (C == 1 || R == 1))
  {
    if constexpr (C == 1) resize(n, 1);
    else resize(1, n);
  }
  Matrix(S a, S b)
    requires(!kDyn && R * C == 2)
  {
    d_ = {a, b};
  }
  Matrix(S a, S b, S c)
    requires(!kDyn && R * C == 3)
  {
    d_ = {a, b, c};
  }
  Matrix(S a, S b, S c, S e)
    requires(!kDyn && R * C == 4 && (R == 1 || C == 1))
  {
    d_ = {a, b, c, e};
  }
  template <int R2, int C2>
    requires(R2 == R || R2 == Dynamic || R == Dynamic) && (C2 == C || C2 == Dynamic || C == Dynamic)
  Matrix(const Matrix<S, R2, C2>& o) {
    resize(o.rows(), o.cols());
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) (*this)(i, j) = o(i, j);
  }
  template <typename M, int BR, int BC>
  Matrix(const Block<M, BR, BC>& b) : Matrix(b.eval()) {}

  // shape
  Index rows() const {
    if constexpr (kDyn) return rows_;
    else return R;
  }
  Index cols() const {
    if constexpr (kDyn) return cols_;
    else return C;
  }
  Index size() const { return rows() * cols(); }
  void resize(Index r, Index c) {
    if constexpr (kDyn) {
      rows_ = r;
      cols_ = c;
      d_.assign(size_t(r * c), S(0));
    }
  }
  void resize(Index n) {
    if constexpr (C == 1) resize(n, 1);
    else resize(1, n);
  }
  S* data() { return d_.data(); }
  const S* data() const { return d_.data(); }

  // access (column-major)
  S& operator()(Index i, Index j) { return d_[size_t(j * rows() + i)]; }
  const S& operator()(Index i, Index j) const { return d_[size_t(j * rows() + i)]; }
  S& operator()(Index k) { return d_[size_t(k)]; }
  const S& operator()(Index k) const { return d_[size_t(k)]; }
  S& operator[](Index k) { return d_[size_t(k)]; }
  const S& operator[](Index k) const { return d_[size_t(k)]; }
  S& x() { return d_[0]; }
  S& y() { return d_[1]; }
  S& z() { return d_[2]; }
  S& w() { return d_[3]; }
  const S& x() const { return d_[0]; }
  const S& y() const { return d_[1]; }
  const S& z() const { return d_[2]; }
  const S& w() const { return d_[3]; }

  // factories
  static Matrix Zero() { return Matrix(); }
  static Matrix Zero(Index r, Index c)
    requires kDyn
  {
    return Matrix(r, c);
  }
  static Matrix Zero(Index n)
    requires kDyn
  {
    return Matrix(n);
  }
  static Matrix Identity() {
    Matrix m;
    for (Index i = 0; i < std::min<Index>(R, C); ++i) m(i, i) = S(1);
    return m;
  }
  static Matrix Identity(Index r, Index c)
    requires kDyn
  {
    Matrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = S(1);
    return m;
  }
  static Matrix Constant(S v) {
    Matrix m;
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }
  static Matrix Unit(Index k) {
    Matrix m;
    m[k] = S(1);
    return m;
  }
  static Matrix UnitX() { return Unit(0); }
  static Matrix UnitY() { return Unit(1); }
  static Matrix UnitZ() { return Unit(2); }
  static Matrix UnitW() { return Unit(3); }
  Matrix& setZero() {
    std::fill(d_.begin(), d_.end(), S(0));
    return *this;
  }
  Matrix& setIdentity() {
    setZero();
    for (Index i = 0; i < std::min(rows(), cols()); ++i) (*this)(i, i) = S(1);
    return *this;
  }
  CommaInit<Matrix> operator<<(S v) { return CommaInit<Matrix>(*this, v); }
  template <typename V>
    requires requires(const V& x) { x.eval(); }
  CommaInit<Matrix> operator<<(const V& v) {  // column vectors stacked
    const auto& e = v.eval();
    CommaInit<Matrix> ci(*this, e[0]);
    for (Index k = 1; k < e.size(); ++k) ci, e[k];
    return ci;
  }

  const Matrix& eval() const { return *this; }

  // views
  template <int BR, int BC>
  Block<Matrix, BR, BC> block(Index i, Index j) {
    return Block<Matrix, BR, BC>(*this, i, j);
  }
  template <int BR, int BC>
  Block<const Matrix, BR, BC> block(Index i, Index j) const {
    return Block<const Matrix, BR, BC>(*this, i, j);
  }
  Block<Matrix, R, 1> col(Index j) { return Block<Matrix, R, 1>(*this, 0, j); }
  Block<const Matrix, R, 1> col(Index j) const { return Block<const Matrix, R, 1>(*this, 0, j); }
  Block<Matrix, 1, C> row(Index i) { return Block<Matrix, 1, C>(*this, i, 0); }
  Block<const Matrix, 1, C> row(Index i) const { return Block<const Matrix, 1, C>(*this, i, 0); }
  template <int N>
  auto segment(Index k) {
    if constexpr (C == 1) return Block<Matrix, N, 1>(*this, k, 0);
    else return Block<Matrix, 1, N>(*this, 0, k);
  }
  template <int N>
  auto segment(Index k) const {
    if constexpr (C == 1) return Block<const Matrix, N, 1>(*this, k, 0);
    else return Block<const Matrix, 1, N>(*this, 0, k);
  }
  template <int N>
  auto head() {
    return segment<N>(0);
  }
  template <int N>
  auto head() const {
    return segment<N>(0);
  }
  template <int N>
  auto tail() {
    return segment<N>(size() - N);
  }
  template <int N>
  auto tail() const {
    return segment<N>(size() - N);
  }
  DiagonalArray<Matrix> diagonal() { return DiagonalArray<Matrix>(*this); }

  // elementwise / reductions
  Matrix<S, C, R> transpose() const {
    Matrix<S, C, R> t;
    if constexpr (kDyn) t.resize(cols(), rows());
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  S squaredNorm() const {
    S s = 0;
    for (const S& v : d_) s += v * v;
    return s;
  }
  S norm() const { return std::sqrt(squaredNorm()); }
  Matrix normalized() const {
    const S n = norm();
    Matrix m = *this;
    if (n > S(0)) m /= n;
    return m;
  }
  void normalize() { *this = normalized(); }
  template <typename O>
  S dot(const O& other) const {
    const auto& o = other.eval();
    S s = 0;
    for (Index k = 0; k < size(); ++k) s += d_[size_t(k)] * o[k];
    return s;
  }
  template <typename O>
  Matrix cross(const O& other) const {
    const auto& o = other.eval();
    const Matrix& a = *this;
    return Matrix(a[1] * o[2] - a[2] * o[1], a[2] * o[0] - a[0] * o[2], a[0] * o[1] - a[1] * o[0]);
  }
  Matrix cwiseAbs() const {
    Matrix m = *this;
    for (S& v : m.d_) v = std::abs(v);
    return m;
  }
  S maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
  S minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
  S sum() const {
    S s = 0;
    for (const S& v : d_) s += v;
    return s;
  }
  bool allFinite() const {
    for (const S& v : d_)
      if (!std::isfinite(v)) return false;
    return true;
  }
  bool hasNaN() const {
    for (const S& v : d_)
      if (std::isnan(v)) return true;
    return false;
  }
  template <int P>
  S lpNorm() const {
    static_assert(P == Infinity, "only lpNorm<Infinity>");
    S m = 0;
    for (const S& v : d_) m = std::max(m, std::abs(v));
    return m;
  }
  S trace() const {
    S s = 0;
    for (Index i = 0; i < std::min(rows(), cols()); ++i) s += (*this)(i, i);
    return s;
  }
  S determinant() const {
    const Matrix& m = *this;
    if (rows() == 1) return m(0, 0);
    if (rows() == 2) return m(0, 0) * m(1, 1) - m(0, 1) * m(1, 0);
    if (rows() == 3)
      return m(0, 0) * (m(1, 1) * m(2, 2) - m(2, 1) * m(1, 2)) -
             m(1, 0) * (m(0, 1) * m(2, 2) - m(2, 1) * m(0, 2)) +
             m(2, 0) * (m(0, 1) * m(1, 2) - m(1, 1) * m(0, 2));
    // LU with partial pivoting for larger sizes
    Matrix a = m;
    S det = 1;
    const Index n = rows();
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
      if (a(p, k) == S(0)) return S(0);
      if (p != k) {
        for (Index j = 0; j < n; ++j) std::swap(a(k, j), a(p, j));
        det = -det;
      }
      det *= a(k, k);
      for (Index i = k + 1; i < n; ++i) {
        const S f = a(i, k) / a(k, k);
        for (Index j = k; j < n; ++j) a(i, j) -= f * a(k, j);
      }
    }
    return det;
  }
  Matrix inverse() const {  // Gauss-Jordan with partial pivoting
    const Index n = rows();
    Matrix a = *this, inv = *this;
    inv.setIdentity();
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
      for (Index j = 0; j < n; ++j) {
        std::swap(a(k, j), a(p, j));
        std::swap(inv(k, j), inv(p, j));
      }
      const S d = a(k, k);
      for (Index j = 0; j < n; ++j) {
        a(k, j) /= d;
        inv(k, j) /= d;
      }
      for (Index i = 0; i < n; ++i) {
        if (i == k) continue;
        const S f = a(i, k);
        for (Index j = 0; j < n; ++j) {
          a(i, j) -= f * a(k, j);
          inv(i, j) -= f * inv(k, j);
        }
      }
    }
    return inv;
  }
  Matrix<S, (R == 1 ? C : R), (R == 1 ? C : R)> asDiagonal() const {
    Matrix<S, (R == 1 ? C : R), (R == 1 ? C : R)> m;
    for (Index k = 0; k < size(); ++k) m(k, k) = d_[size_t(k)];
    return m;
  }
  class LDLTSolver;
  LDLTSolver ldlt() const { return LDLTSolver(*this); }

  // compound assignment
  template <MatExpr O>
  Matrix& operator+=(const O& other) {
    const auto& o = other.eval();
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) (*this)(i, j) += o(i, j);
    return *this;
  }
  template <MatExpr O>
  Matrix& operator-=(const O& other) {
    const auto& o = other.eval();
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) (*this)(i, j) -= o(i, j);
    return *this;
  }
  Matrix& operator*=(S s) {
    for (S& v : d_) v *= s;
    return *this;
  }
  Matrix& operator/=(S s) {
    for (S& v : d_) v /= s;
    return *this;
  }
  Matrix operator-() const {
    Matrix m = *this;
    for (S& v : m.d_) v = -v;
    return m;
  }

 private:
  template <typename, int, int>
  friend class Matrix;
  std::conditional_t<kDyn, std::vector<S>, std::array<S, size_t(kDyn ? 1 : R * C)>> d_{};
  Index rows_ = 0, cols_ = 0;
};

// ------------------------------------------------------------------- views
template <typename M, int R, int C>
class Block {
 public:
  using S = typename std::remove_const_t<M>::Scalar;
  using Plain = Matrix<S, R, C>;
  Block(M& m, Index i, Index j) : m_(&m), i_(i), j_(j) {}
  Index rows() const { return R; }
  Index cols() const { return C; }
  Index size() const { return R * C; }
  auto& operator()(Index i, Index j) const { return (*m_)(i_ + i, j_ + j); }
  auto& operator[](Index k) const {
    if constexpr (C == 1) return (*m_)(i_ + k, j_);
    else return (*m_)(i_, j_ + k);
  }
  auto& operator()(Index k) const { return (*this)[k]; }
  Plain eval() const {
    Plain p;
    for (Index j = 0; j < C; ++j)
      for (Index i = 0; i < R; ++i) p(i, j) = (*this)(i, j);
    return p;
  }
  operator Plain() const { return eval(); }
  template <MatExpr O>
  Block& operator=(const O& other) {
    const Plain o = Plain(other.eval());
    for (Index j = 0; j < C; ++j)
      for (Index i = 0; i < R; ++i) (*this)(i, j) = o(i, j);
    return *this;
  }
  Block& operator=(const Block& other) { return *this = other.eval(); }
  template <MatExpr O>
  Block& operator+=(const O& other) {
    const Plain o = Plain(other.eval());
    for (Index j = 0; j < C; ++j)
      for (Index i = 0; i < R; ++i) (*this)(i, j) += o(i, j);
    return *this;
  }
  template <MatExpr O>
  Block& operator-=(const O& other) {
    const Plain o = Plain(other.eval());
    for (Index j = 0; j < C; ++j)
      for (Index i = 0; i < R; ++i) (*this)(i, j) -= o(i, j);
    return *this;
  }
  Block& setZero() {
    for (Index j = 0; j < C; ++j)
      for (Index i = 0; i < R; ++i) (*this)(i, j) = S(0);
    return *this;
  }
  auto transpose() const { return eval().transpose(); }
  S norm() const { return eval().norm(); }
  S squaredNorm() const { return eval().squaredNorm(); }
  Plain normalized() const { return eval().normalized(); }
  template <typename O>
  S dot(const O& o) const {
    return eval().dot(o);
  }
  template <typename O>
  Plain cross(const O& o) const {
    return eval().cross(o);
  }
  bool allFinite() const { return eval().allFinite(); }

 private:
  M* m_;
  Index i_, j_;
};

// -------------------------------------------------------------- arithmetic
template <MatExpr A, MatExpr B>
auto operator*(const A& a_, const B& b_) {
  const auto& a = a_.eval();
  const auto& b = b_.eval();
  using MA = std::remove_cvref_t<decltype(a)>;
  using MB = std::remove_cvref_t<decltype(b)>;
  using S = typename MA::Scalar;
  constexpr int R = MA::RowsAtCompileTime, C = MB::ColsAtCompileTime;
  Matrix<S, R, C> out;
  if constexpr (R == Dynamic || C == Dynamic) out.resize(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      S s = 0;
      for (Index k = 0; k < a.cols(); ++k) s += a(i, k) * b(k, j);
      out(i, j) = s;
    }
  return out;
}
template <MatExpr A, MatExpr B>
auto operator+(const A& a_, const B& b_) {
  auto out = std::remove_cvref_t<decltype(a_.eval())>(a_.eval());
  out += b_;
  return out;
}
template <MatExpr A, MatExpr B>
auto operator-(const A& a_, const B& b_) {
  auto out = std::remove_cvref_t<decltype(a_.eval())>(a_.eval());
  out -= b_;
  return out;
}
template <MatExpr A>
auto operator*(const A& a_, double s) {
  auto out = std::remove_cvref_t<decltype(a_.eval())>(a_.eval());
  out *= s;
  return out;
}
template <MatExpr A>
auto operator*(double s, const A& a_) {
  auto out = std::remove_cvref_t<decltype(a_.eval())>(a_.eval());
  out *= s;
  return out;
}
template <MatExpr A>
auto operator/(const A& a_, double s) {
  auto out = std::remove_cvref_t<decltype(a_.eval())>(a_.eval());
  out /= s;
  return out;
}
template <typename M, int R, int C>
auto operator-(const Block<M, R, C>& b) {
  return -b.eval();
}
template <MatExpr A, MatExpr B>
bool operator==(const A& a_, const B& b_) {  // Eigen: cwiseEqual(...).all()
  const auto& a = a_.eval();
  const auto& b = b_.eval();
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i)
      if (!(a(i, j) == b(i, j))) return false;
  return true;
}
template <MatExpr A, MatExpr B>
bool operator!=(const A& a, const B& b) {
  return !(a == b);
}

// -------------------------------------------------------------------- LDLT
namespace shim {
// Optional replacement of the dense (Dynamic-size) LDLT solve -- the
// reference's 6N x 6N LM step (solver.cpp:386) -- by an external solver of the
// same system (the bench's CPU reference arm installs a LAPACK Cholesky via
// dsref_set_dense_solver; parity tests leave it unset). Arguments: n, the
// symmetric matrix (n x n), b, x out; returns 0 on success.
using DenseSolver = int (*)(int n, const double* a, const double* b, double* x);
inline DenseSolver& dense_solver() {
  static DenseSolver f = nullptr;
  return f;
}
inline long long& dense_solves() {
  static long long n = 0;
  return n;
}
}  // namespace shim

// Eigen::LDLT: P^T L D L^T P with diagonal pivoting on the largest remaining
// |diagonal| (LDLT.h, unblocked), zero pivots kept; solve() inverts D with a
// pseudo-inverse below the smallest positive normal number.
template <typename S, int R, int C>
class Matrix<S, R, C>::LDLTSolver {
 public:
  explicit LDLTSolver(const Matrix& a) : n_(a.rows()), a_(size_t(n_ * n_)), perm_(size_t(n_)) {
    for (Index r = 0; r < n_; ++r)
      for (Index c = 0; c < n_; ++c) A(r, c) = a(r, c);
    if (kDyn && shim::dense_solver()) {  // solved externally in solve()
      external_ = true;
      return;
    }
    std::vector<S> temp(static_cast<size_t>(n_));
    for (Index k = 0; k < n_; ++k) {
      Index big = k;
      S bv = std::abs(A(k, k));
      for (Index i = k + 1; i < n_; ++i)
        if (std::abs(A(i, i)) > bv) {
          bv = std::abs(A(i, i));
          big = i;
        }
      perm_[size_t(k)] = big;
      if (big != k) {
        for (Index c = 0; c < k; ++c) std::swap(A(k, c), A(big, c));
        for (Index r = big + 1; r < n_; ++r) std::swap(A(r, k), A(r, big));
        std::swap(A(k, k), A(big, big));
        for (Index i = k + 1; i < big; ++i) {
          const S t = A(i, k);
          A(i, k) = A(big, i);
          A(big, i) = t;
        }
      }
      if (k > 0) {
        for (Index c = 0; c < k; ++c) temp[size_t(c)] = A(c, c) * A(k, c);
        S s = 0;
        for (Index c = 0; c < k; ++c) s += A(k, c) * temp[size_t(c)];
        A(k, k) -= s;
        for (Index r = k + 1; r < n_; ++r) {
          S acc = 0;
          for (Index c = 0; c < k; ++c) acc += A(r, c) * temp[size_t(c)];
          A(r, k) -= acc;
        }
      }
      const S akk = A(k, k);
      const bool valid = std::abs(akk) > S(0);
      if (k == 0 && !valid) {
        zero_all_ = true;
        break;
      }
      if (valid)
        for (Index r = k + 1; r < n_; ++r) A(r, k) /= akk;
    }
  }
  template <MatExpr B>
  Matrix<S, R, 1> solve(const B& b_) const {
    const auto& b = b_.eval();
    Matrix<S, R, 1> x;
    if constexpr (R == Dynamic) x.resize(n_, 1);
    for (Index i = 0; i < n_; ++i) x[i] = b[i];
    if (external_) {
      ++shim::dense_solves();
      Matrix<S, R, 1> out = x;
      if (shim::dense_solver()(int(n_), a_.data(), x.data(), out.data()) == 0) return out;
    }
    if (zero_all_) return x.setZero();
    for (Index k = 0; k < n_; ++k) std::swap(x[k], x[perm_[size_t(k)]]);
    for (Index r = 0; r < n_; ++r) {
      S s = x[r];
      for (Index c = 0; c < r; ++c) s -= A(r, c) * x[c];
      x[r] = s;
    }
    for (Index i = 0; i < n_; ++i) x[i] = std::abs(A(i, i)) > DBL_MIN ? x[i] / A(i, i) : S(0);
    for (Index r = n_ - 1; r >= 0; --r) {
      S s = x[r];
      for (Index c = r + 1; c < n_; ++c) s -= A(c, r) * x[c];
      x[r] = s;
    }
    for (Index k = n_ - 1; k >= 0; --k) std::swap(x[k], x[perm_[size_t(k)]]);
    return x;
  }

 private:
  S& A(Index r, Index c) { return a_[size_t(r * n_ + c)]; }
  const S& A(Index r, Index c) const { return a_[size_t(r * n_ + c)]; }
  Index n_;
  std::vector<S> a_;
  std::vector<Index> perm_;
  bool zero_all_ = false;
  bool external_ = false;
};

// ----------------------------------------------------- symmetric eigen / SVD
namespace detail {
// cyclic Jacobi eigenvalues of a symmetric n x n (row-major) matrix
inline std::vector<double> sym_eigenvalues(int n, std::vector<double> a) {
  auto A = [&](int r, int c) -> double& { return a[size_t(r) * n + c]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += A(p, q) * A(p, q);
    if (off < 1e-300) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (A(p, q) == 0.0) continue;
        const double theta = (A(q, q) - A(p, p)) / (2.0 * A(p, q));
        const double t =
            (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * akq;
          A(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
      }
  }
  std::vector<double> ev(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) ev[size_t(i)] = A(i, i);
  return ev;
}
}  // namespace detail

template <typename M>
class SelfAdjointEigenSolver {
 public:
  static constexpr int N = M::RowsAtCompileTime;
  explicit SelfAdjointEigenSolver(const M& m) {
    const int n = int(m.rows());
    std::vector<double> a(size_t(n) * n);
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < n; ++c) a[size_t(r) * n + c] = m(r, c);
    auto ev = detail::sym_eigenvalues(n, a);
    std::sort(ev.begin(), ev.end());  // increasing, as Eigen
    if constexpr (N == Dynamic) ev_.resize(n);
    for (int i = 0; i < n; ++i) ev_[i] = ev[size_t(i)];
  }
  const Matrix<double, N, 1>& eigenvalues() const { return ev_; }

 private:
  Matrix<double, N, 1> ev_;
};

inline constexpr int ComputeThinU = 0x100, ComputeThinV = 0x200, ComputeFullU = 0x4,
                     ComputeFullV = 0x10;

template <typename M>
class JacobiSVD {
 public:
  static constexpr int N = M::ColsAtCompileTime;
  explicit JacobiSVD(const M& m, int = 0) {
    const int n = int(m.cols());
    std::vector<double> ata(size_t(n) * n, 0.0);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double acc = 0;
        for (int k = 0; k < int(m.rows()); ++k) acc += m(k, i) * m(k, j);
        ata[size_t(i) * n + j] = acc;
      }
    auto ev = detail::sym_eigenvalues(n, ata);
    std::sort(ev.begin(), ev.end(), std::greater<double>());  // decreasing, as Eigen
    for (int i = 0; i < n; ++i) sv_[i] = std::sqrt(std::max(ev[size_t(i)], 0.0));
  }
  const Matrix<double, N, 1>& singularValues() const { return sv_; }

 private:
  Matrix<double, N, 1> sv_;
};

// ---------------------------------------------------------------- geometry
template <typename S>
class Quaternion {
 public:
  Quaternion() = default;
  Quaternion(S w, S x, S y, S z) : w_(w), x_(x), y_(y), z_(z) {}
  // Eigen/src/Geometry/Quaternion.h quaternionbase_assign_impl (Shoemake)
  explicit Quaternion(const Matrix<S, 3, 3>& m) {
    S t = (m(0, 0) + m(1, 1)) + m(2, 2);
    S q[4];  // (w, x, y, z)
    if (t > S(0)) {
      t = std::sqrt(t + S(1));
      q[0] = S(0.5) * t;
      t = S(0.5) / t;
      q[1] = (m(2, 1) - m(1, 2)) * t;
      q[2] = (m(0, 2) - m(2, 0)) * t;
      q[3] = (m(1, 0) - m(0, 1)) * t;
    } else {
      int i = 0;
      if (m(1, 1) > m(0, 0)) i = 1;
      if (m(2, 2) > m(i, i)) i = 2;
      const int j = (i + 1) % 3, k = (j + 1) % 3;
      t = std::sqrt(m(i, i) - m(j, j) - m(k, k) + S(1));
      q[1 + i] = S(0.5) * t;
      t = S(0.5) / t;
      q[0] = (m(k, j) - m(j, k)) * t;
      q[1 + j] = (m(j, i) + m(i, j)) * t;
      q[1 + k] = (m(k, i) + m(i, k)) * t;
    }
    w_ = q[0];
    x_ = q[1];
    y_ = q[2];
    z_ = q[3];
  }
  S w() const { return w_; }
  S x() const { return x_; }
  S y() const { return y_; }
  S z() const { return z_; }
  S norm() const { return std::sqrt(w_ * w_ + x_ * x_ + y_ * y_ + z_ * z_); }
  void normalize() {
    const S n = norm();
    if (n > S(0)) {
      w_ /= n;
      x_ /= n;
      y_ /= n;
      z_ /= n;
    }
  }
  Quaternion normalized() const {
    Quaternion q = *this;
    q.normalize();
    return q;
  }
  Matrix<S, 3, 3> toRotationMatrix() const {  // Quaternion.h toRotationMatrix
    const S tx = S(2) * x_, ty = S(2) * y_, tz = S(2) * z_;
    const S twx = tx * w_, twy = ty * w_, twz = tz * w_;
    const S txx = tx * x_, txy = ty * x_, txz = tz * x_;
    const S tyy = ty * y_, tyz = tz * y_, tzz = tz * z_;
    Matrix<S, 3, 3> r;
    r(0, 0) = S(1) - (tyy + tzz);
    r(0, 1) = txy - twz;
    r(0, 2) = txz + twy;
    r(1, 0) = txy + twz;
    r(1, 1) = S(1) - (txx + tzz);
    r(1, 2) = tyz - twx;
    r(2, 0) = txz - twy;
    r(2, 1) = tyz + twx;
    r(2, 2) = S(1) - (txx + tyy);
    return r;
  }

 private:
  S w_ = 1, x_ = 0, y_ = 0, z_ = 0;
};

template <typename S>
class AngleAxis {
 public:
  AngleAxis(S angle, const Matrix<S, 3, 1>& axis) : angle_(angle), axis_(axis) {}
  Matrix<S, 3, 3> toRotationMatrix() const {  // AngleAxis.h toRotationMatrix
    Matrix<S, 3, 3> r;
    const Matrix<S, 3, 1> sin_axis = std::sin(angle_) * axis_;
    const S c = std::cos(angle_);
    const Matrix<S, 3, 1> cos1_axis = (S(1) - c) * axis_;
    S tmp = cos1_axis.x() * axis_.y();
    r(0, 1) = tmp - sin_axis.z();
    r(1, 0) = tmp + sin_axis.z();
    tmp = cos1_axis.x() * axis_.z();
    r(0, 2) = tmp + sin_axis.y();
    r(2, 0) = tmp - sin_axis.y();
    tmp = cos1_axis.y() * axis_.z();
    r(1, 2) = tmp - sin_axis.x();
    r(2, 1) = tmp + sin_axis.x();
    r(0, 0) = cos1_axis.x() * axis_.x() + c;
    r(1, 1) = cos1_axis.y() * axis_.y() + c;
    r(2, 2) = cos1_axis.z() * axis_.z() + c;
    return r;
  }

 private:
  S angle_;
  Matrix<S, 3, 1> axis_;
};

using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using Quaterniond = Quaternion<double>;
using AngleAxisd = AngleAxis<double>;

}  // namespace Eigen
