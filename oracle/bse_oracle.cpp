// bse_oracle.cpp — CPU ORACLE (test infrastructure only).
//
// A call-by-call restatement of the reference's hot path on LAPACK/BLAS, used ONLY by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg as
// the checker and the timed CPU baseline. Nothing in the product path links or calls it.
//
// The reference itself (/root/reference/proj) cannot be compiled here: Eigen3, lapacke.h /
// cblas.h, doctest and CLI11 are absent. Its arithmetic lives in a third-party
// LAPACK (OpenBLAS + LAPACKE, version unpinned, proj/CMakeLists.txt:13-14). This file
// restates the reference's driver calls, flags and order with the same LAPACK routines,
// linking the OpenBLAS 0.3.31 that ships with scipy in this image (prefixed symbols
// scipy_LAPACKE_* / scipy_cblas_*; LP64). Results agree with the reference build to
// rounding, not bitwise (different OpenBLAS build).
//
// Each function cites the reference file:line it follows.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/bse_gpu.h"

using cd = std::complex<double>;
typedef int lapack_int;

extern "C" {
// LAPACKE / CBLAS prototypes (column-major = 102, lower = 'L'), prefixed in scipy's build.
lapack_int scipy_LAPACKE_zpotrf(int layout, char uplo, lapack_int n, cd* a, lapack_int lda);
lapack_int scipy_LAPACKE_zheevd(int layout, char jobz, char uplo, lapack_int n, cd* a,
                                lapack_int lda, double* w);
lapack_int scipy_LAPACKE_zgesvd(int layout, char jobu, char jobvt, lapack_int m, lapack_int n,
                                cd* a, lapack_int lda, double* s, cd* u, lapack_int ldu, cd* vt,
                                lapack_int ldvt, double* superb);
void scipy_cblas_ztrmm(int layout, int side, int uplo, int transa, int diag, lapack_int m,
                       lapack_int n, const void* alpha, const void* a, lapack_int lda, void* b,
                       lapack_int ldb);
void scipy_cblas_ztrsm(int layout, int side, int uplo, int transa, int diag, lapack_int m,
                       lapack_int n, const void* alpha, const void* a, lapack_int lda, void* b,
                       lapack_int ldb);
void scipy_cblas_zgemm(int layout, int transa, int transb, lapack_int m, lapack_int n,
                       lapack_int k, const void* alpha, const void* a, lapack_int lda,
                       const void* b, lapack_int ldb, const void* beta, void* c,
                       lapack_int ldc);
void scipy_openblas_set_num_threads(int);
int scipy_openblas_get_num_threads(void);
char* scipy_openblas_get_config(void);
}

namespace {

constexpr int kColMajor = 102;
constexpr int kNoTrans = 111, kConjTrans = 113;
constexpr int kUpper = 121, kLower = 122;
constexpr int kNonUnit = 131;
constexpr int kLeft = 141, kRight = 142;

// Column-major complex matrix (the role Eigen::MatrixXcd plays in types.hpp:17-18).
struct Mat {
  int64_t r = 0, c = 0;
  std::vector<cd> d;
  Mat() = default;
  Mat(int64_t rr, int64_t cc) : r(rr), c(cc), d(static_cast<size_t>(rr * cc)) {}
  cd& operator()(int64_t i, int64_t j) { return d[static_cast<size_t>(i + j * r)]; }
  const cd& operator()(int64_t i, int64_t j) const { return d[static_cast<size_t>(i + j * r)]; }
  cd* data() { return d.data(); }
  const cd* data() const { return d.data(); }
  Mat adjoint() const {
    Mat o(c, r);
    for (int64_t j = 0; j < c; ++j)
      for (int64_t i = 0; i < r; ++i) o(j, i) = std::conj((*this)(i, j));
    return o;
  }
};

struct Err {
  int code;
  int block = 0;
  int64_t pivot = -1;
  double dev = 0.0;
  std::string msg;
};

Mat load(int64_t r, int64_t c, const double* p, int64_t ld) {
  Mat m(r, c);
  for (int64_t j = 0; j < c; ++j)
    std::memcpy(static_cast<void*>(&m(0, j)), p + 2 * j * ld, sizeof(cd) * static_cast<size_t>(r));
  return m;
}
void store(const Mat& m, double* p, int64_t ld) {
  for (int64_t j = 0; j < m.c; ++j)
    std::memcpy(p + 2 * j * ld, &m(0, j), sizeof(cd) * static_cast<size_t>(m.r));
}

// backend.cpp:28-45
void hermitian_eig(const Mat& m, std::vector<double>& values, Mat& vectors) {
  const lapack_int n = static_cast<lapack_int>(m.r);
  vectors = m;
  values.assign(static_cast<size_t>(n), 0.0);
  const lapack_int info =
      scipy_LAPACKE_zheevd(kColMajor, 'V', 'L', n, vectors.data(), n, values.data());
  if (info > 0)
    throw Err{BSE_ERR_CONVERGENCE_FAILURE, 0, -1, 0,
              "zheevd failed to converge (info=" + std::to_string(info) + ")"};
  if (info < 0) throw Err{BSE_ERR_GENERIC, 0, -1, 0, "zheevd: invalid argument"};
}

// backend.cpp:47-62
Mat cholesky_lower(const Mat& m) {
  const lapack_int n = static_cast<lapack_int>(m.r);
  Mat l = m;
  const lapack_int info = scipy_LAPACKE_zpotrf(kColMajor, 'L', n, l.data(), n);
  if (info > 0)
    throw Err{BSE_ERR_NOT_POSITIVE_DEFINITE, 0, static_cast<int64_t>(info) - 1, 0,
              "leading minor of order " + std::to_string(info) + " is not positive definite"};
  if (info < 0) throw Err{BSE_ERR_GENERIC, 0, -1, 0, "zpotrf: invalid argument"};
  for (int64_t j = 1; j < n; ++j)
    for (int64_t i = 0; i < j; ++i) l(i, j) = 0.0;
  return l;
}

// backend.cpp:64-86
void svd(const Mat& m, Mat& u, std::vector<double>& s, Mat& v) {
  const lapack_int n = static_cast<lapack_int>(m.r);
  Mat work = m;
  u = Mat(n, n);
  s.assign(static_cast<size_t>(n), 0.0);
  Mat vt(n, n);
  std::vector<double> superb(static_cast<size_t>(std::max<lapack_int>(1, n - 1)));
  const lapack_int info = scipy_LAPACKE_zgesvd(kColMajor, 'A', 'A', n, n, work.data(), n,
                                               s.data(), u.data(), n, vt.data(), n,
                                               superb.data());
  if (info > 0)
    throw Err{BSE_ERR_CONVERGENCE_FAILURE, 0, -1, 0, "zgesvd failed to converge"};
  if (info < 0) throw Err{BSE_ERR_GENERIC, 0, -1, 0, "zgesvd: invalid argument"};
  v = vt.adjoint();
}

// backend.cpp:109-129
Mat tri_solve(const Mat& l, const Mat& rhs, int side, int op) {
  const int64_t n = l.r;
  if ((side == BSE_SIDE_LEFT && rhs.r != n) || (side == BSE_SIDE_RIGHT && rhs.c != n))
    throw Err{BSE_ERR_DIMENSION_MISMATCH, 0, -1, 0,
              "tri_solve: right-hand side does not conform"};
  const double underflow = std::numeric_limits<double>::min();
  for (int64_t i = 0; i < n; ++i)
    if (std::abs(l(i, i)) < underflow)
      throw Err{BSE_ERR_SINGULAR_FACTOR, 0, -1, 0,
                "triangular factor has a vanishing diagonal entry at index " +
                    std::to_string(i)};
  Mat x = rhs;
  const cd one(1.0, 0.0);
  scipy_cblas_ztrsm(kColMajor, side == BSE_SIDE_LEFT ? kLeft : kRight, kLower,
                    op == BSE_OP_NONE ? kNoTrans : kConjTrans, kNonUnit,
                    static_cast<lapack_int>(x.r), static_cast<lapack_int>(x.c), &one, l.data(),
                    static_cast<lapack_int>(n), x.data(), static_cast<lapack_int>(x.r));
  return x;
}

// backend.cpp:131-175
Mat matmul(const Mat& a, const Mat& b, int op_a, int shape_a, int op_b, int shape_b) {
  const int64_t am = op_a == BSE_OP_NONE ? a.r : a.c;
  const int64_t ak = op_a == BSE_OP_NONE ? a.c : a.r;
  const int64_t bk = op_b == BSE_OP_NONE ? b.r : b.c;
  const int64_t bn = op_b == BSE_OP_NONE ? b.c : b.r;
  if (ak != bk)
    throw Err{BSE_ERR_DIMENSION_MISMATCH, 0, -1, 0, "matmul: inner dimensions differ"};
  const cd one(1.0, 0.0), zero(0.0, 0.0);
  const bool tri_a = shape_a != BSE_SHAPE_GENERAL;
  const bool tri_b = shape_b != BSE_SHAPE_GENERAL;
  if (tri_a && !tri_b) {
    if (a.r != a.c)
      throw Err{BSE_ERR_DIMENSION_MISMATCH, 0, -1, 0, "matmul: triangular operand not square"};
    Mat c = op_b == BSE_OP_NONE ? b : b.adjoint();
    scipy_cblas_ztrmm(kColMajor, kLeft, shape_a == BSE_SHAPE_LOWER ? kLower : kUpper,
                      op_a == BSE_OP_NONE ? kNoTrans : kConjTrans, kNonUnit,
                      static_cast<lapack_int>(c.r), static_cast<lapack_int>(c.c), &one, a.data(),
                      static_cast<lapack_int>(a.r), c.data(), static_cast<lapack_int>(c.r));
    return c;
  }
  if (tri_b && !tri_a) {
    if (b.r != b.c)
      throw Err{BSE_ERR_DIMENSION_MISMATCH, 0, -1, 0, "matmul: triangular operand not square"};
    Mat c = op_a == BSE_OP_NONE ? a : a.adjoint();
    scipy_cblas_ztrmm(kColMajor, kRight, shape_b == BSE_SHAPE_LOWER ? kLower : kUpper,
                      op_b == BSE_OP_NONE ? kNoTrans : kConjTrans, kNonUnit,
                      static_cast<lapack_int>(c.r), static_cast<lapack_int>(c.c), &one, b.data(),
                      static_cast<lapack_int>(b.r), c.data(), static_cast<lapack_int>(c.r));
    return c;
  }
  Mat c(am, bn);
  scipy_cblas_zgemm(kColMajor, op_a == BSE_OP_NONE ? kNoTrans : kConjTrans,
                    op_b == BSE_OP_NONE ? kNoTrans : kConjTrans, static_cast<lapack_int>(am),
                    static_cast<lapack_int>(bn), static_cast<lapack_int>(ak), &one, a.data(),
                    static_cast<lapack_int>(a.r), b.data(), static_cast<lapack_int>(b.r), &zero,
                    c.data(), static_cast<lapack_int>(am));
  return c;
}

// backend.cpp:88-107
Mat hpd_sqrt(const Mat& m) {
  std::vector<double> w;
  Mat vec;
  hermitian_eig(m, w, vec);
  const int64_t n = m.r;
  const double lambda_max = w[static_cast<size_t>(n - 1)];
  const double floor = std::numeric_limits<double>::epsilon() * lambda_max;
  for (int64_t i = 0; i < n; ++i)
    if (!(w[static_cast<size_t>(i)] > floor))
      throw Err{BSE_ERR_NOT_POSITIVE_DEFINITE, 0, i, 0,
                "eigenvalue at index " + std::to_string(i) + " is at or below eps*lambda_max"};
  Mat scaled = vec;
  for (int64_t j = 0; j < n; ++j) {
    const double s = std::sqrt(w[static_cast<size_t>(j)]);
    for (int64_t i = 0; i < n; ++i) scaled(i, j) *= s;
  }
  Mat s = matmul(scaled, vec, BSE_OP_NONE, BSE_SHAPE_GENERAL, BSE_OP_ADJOINT, BSE_SHAPE_GENERAL);
  Mat sh = s.adjoint();
  for (size_t i = 0; i < s.d.size(); ++i) s.d[i] = 0.5 * (s.d[i] + sh.d[i]);
  return s;
}

// core.cpp:87-100
void product_pair(const Mat& a, const Mat& b, Mat& m1, Mat& m2) {
  m1 = a;
  m2 = a;
  for (size_t i = 0; i < a.d.size(); ++i) {
    m1.d[i] = a.d[i] + b.d[i];
    m2.d[i] = a.d[i] - b.d[i];
  }
  try {
    cholesky_lower(m1);
  } catch (const Err& e) {
    if (e.code != BSE_ERR_NOT_POSITIVE_DEFINITE) throw;
    throw Err{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M1, e.pivot, 0,
              "A+B is not positive definite: " + e.msg};
  }
  try {
    cholesky_lower(m2);
  } catch (const Err& e) {
    if (e.code != BSE_ERR_NOT_POSITIVE_DEFINITE) throw;
    throw Err{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M2, e.pivot, 0,
              "A-B is not positive definite: " + e.msg};
  }
}

// core.cpp:102-127
Mat assemble_eigenvectors(const Mat& v1, const Mat& v2, const std::vector<double>& l1,
                          const std::vector<double>& l2) {
  const int64_t n = v1.r, k = v1.c;
  if (v2.r != n || v2.c != k || static_cast<int64_t>(l1.size()) != k ||
      static_cast<int64_t>(l2.size()) != k)
    throw Err{BSE_ERR_DIMENSION_MISMATCH, 0, -1, 0, "factor shapes do not conform"};
  for (int64_t j = 0; j < k; ++j) {
    const double x = l1[static_cast<size_t>(j)], y = l2[static_cast<size_t>(j)];
    if (!(x > 0.0) || !(y > 0.0) || !std::isfinite(x) || !std::isfinite(y))
      throw Err{BSE_ERR_NON_POSITIVE_SCALE, 0, -1, 0,
                "scaling factor for column " + std::to_string(j) +
                    " is not a positive finite real"};
  }
  Mat v(2 * n, k);
  for (int64_t j = 0; j < k; ++j) {
    const double s1 = std::pow(l1[static_cast<size_t>(j)] / l2[static_cast<size_t>(j)], 0.25);
    const double s2 = std::pow(l2[static_cast<size_t>(j)] / l1[static_cast<size_t>(j)], 0.25);
    for (int64_t i = 0; i < n; ++i) {
      const cd x = v1(i, j) * s1;
      const cd y = v2(i, j) * s2;
      v(i, j) = 0.5 * (x + y);
      v(n + i, j) = 0.5 * (y - x);
    }
  }
  return v;
}

struct Clamped {
  std::vector<double> lambda;
  std::vector<int64_t> flagged, nonpositive;
  double floor = 0.0;
};

// solvers.cpp:25-45
Clamped lambda_from_squares(const std::vector<double>& d) {
  const int64_t n = static_cast<int64_t>(d.size());
  const double d_max = d[static_cast<size_t>(n - 1)];
  if (!(d_max > 0.0))
    throw Err{BSE_ERR_CONVERGENCE_FAILURE, 0, -1, 0,
              "squared-problem spectrum has no positive eigenvalue"};
  Clamped out;
  out.floor = std::numeric_limits<double>::epsilon() * std::sqrt(d_max);
  out.lambda.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    const double di = d[static_cast<size_t>(i)];
    const double lam = di > 0.0 ? std::sqrt(di) : 0.0;
    if (lam < out.floor) {
      out.lambda[static_cast<size_t>(i)] = out.floor;
      out.flagged.push_back(i);
      if (!(di > 0.0)) out.nonpositive.push_back(i);
    } else {
      out.lambda[static_cast<size_t>(i)] = lam;
    }
  }
  return out;
}

// solvers.cpp:53-65
void rebuild_nonpositive_columns(Mat& v, const Mat& v1, const Mat& v2,
                                 const std::vector<double>& d, const Clamped& cs) {
  const int64_t n = v1.r;
  for (const int64_t j : cs.nonpositive) {
    const double mag = std::max(std::sqrt(std::abs(d[static_cast<size_t>(j)])), cs.floor);
    const cd quarter = std::sqrt(mag) * cd(std::sqrt(2.0) / 2.0, std::sqrt(2.0) / 2.0);
    for (int64_t i = 0; i < n; ++i) {
      const cd x = v1(i, j) * quarter;
      const cd y = v2(i, j) / quarter;
      v(i, j) = 0.5 * (x + y);
      v(n + i, j) = 0.5 * (y - x);
    }
  }
}

// solvers.cpp:69-88
Clamped clamp_singular_ascending(const std::vector<double>& s_desc) {
  const int64_t n = static_cast<int64_t>(s_desc.size());
  const double s_max = s_desc[0];
  if (!(s_max > 0.0))
    throw Err{BSE_ERR_CONVERGENCE_FAILURE, 0, -1, 0, "singular spectrum is identically zero"};
  const double floor = std::numeric_limits<double>::epsilon() * s_max;
  Clamped out;
  out.floor = floor;
  out.lambda.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    const double s = s_desc[static_cast<size_t>(n - 1 - i)];
    if (s < floor) {
      out.lambda[static_cast<size_t>(i)] = floor;
      out.flagged.push_back(i);
    } else {
      out.lambda[static_cast<size_t>(i)] = s;
    }
  }
  return out;
}

struct Result {
  std::vector<double> lambda;
  Mat v;
  std::vector<int64_t> near_singular;
};

// solvers.cpp:94-117
Result solve_sqrt(const Mat& a, const Mat& b) {
  Mat m1, m2;
  product_pair(a, b, m1, m2);
  Mat s;
  try {
    s = hpd_sqrt(m2);
  } catch (const Err& e) {
    if (e.code != BSE_ERR_NOT_POSITIVE_DEFINITE) throw;
    throw Err{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M2, e.pivot, 0,
              "square root of A-B failed: " + e.msg};
  }
  const Mat inner = matmul(m1, s, 0, 0, 0, 0);
  const Mat m = matmul(s, inner, 0, 0, 0, 0);
  std::vector<double> w;
  Mat vm;
  hermitian_eig(m, w, vm);
  const Clamped cs = lambda_from_squares(w);
  const Mat ls = cholesky_lower(s);
  Mat v1 = tri_solve(ls, vm, BSE_SIDE_LEFT, BSE_OP_NONE);
  v1 = tri_solve(ls, v1, BSE_SIDE_LEFT, BSE_OP_ADJOINT);
  const Mat v2 = matmul(s, vm, 0, 0, 0, 0);
  std::vector<double> l1(cs.lambda.size()), ones(cs.lambda.size(), 1.0);
  for (size_t i = 0; i < l1.size(); ++i) l1[i] = cs.lambda[i] * cs.lambda[i];
  Mat v = assemble_eigenvectors(v1, v2, l1, ones);
  rebuild_nonpositive_columns(v, v1, v2, w, cs);
  return Result{cs.lambda, std::move(v), cs.flagged};
}

// solvers.cpp:119-135
Result solve_chol(const Mat& a, const Mat& b) {
  Mat m1, m2;
  product_pair(a, b, m1, m2);
  const Mat l = cholesky_lower(m2);
  Mat m = matmul(l, m1, BSE_OP_ADJOINT, BSE_SHAPE_LOWER, BSE_OP_NONE, BSE_SHAPE_GENERAL);
  m = matmul(m, l, BSE_OP_NONE, BSE_SHAPE_GENERAL, BSE_OP_NONE, BSE_SHAPE_LOWER);
  std::vector<double> w;
  Mat vm;
  hermitian_eig(m, w, vm);
  const Clamped cs = lambda_from_squares(w);
  const Mat v1 = tri_solve(l, vm, BSE_SIDE_LEFT, BSE_OP_ADJOINT);
  const Mat v2 = matmul(l, vm, BSE_OP_NONE, BSE_SHAPE_LOWER, BSE_OP_NONE, BSE_SHAPE_GENERAL);
  std::vector<double> l1(cs.lambda.size()), ones(cs.lambda.size(), 1.0);
  for (size_t i = 0; i < l1.size(); ++i) l1[i] = cs.lambda[i] * cs.lambda[i];
  Mat v = assemble_eigenvectors(v1, v2, l1, ones);
  rebuild_nonpositive_columns(v, v1, v2, w, cs);
  return Result{cs.lambda, std::move(v), cs.flagged};
}

// solvers.cpp:137-161
Result solve_chol_svd(const Mat& a, const Mat& b) {
  Mat m1, m2;
  product_pair(a, b, m1, m2);
  const Mat l1 = cholesky_lower(m1);
  const Mat l2 = cholesky_lower(m2);
  const Mat c = matmul(l1, l2, BSE_OP_ADJOINT, BSE_SHAPE_LOWER, BSE_OP_NONE, BSE_SHAPE_GENERAL);
  Mat u, v;
  std::vector<double> s;
  svd(c, u, s, v);
  const int64_t n = a.r;
  const Clamped cs = clamp_singular_ascending(s);
  Mat u_asc(n, n), v_asc(n, n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      u_asc(i, j) = u(i, n - 1 - j);
      v_asc(i, j) = v(i, n - 1 - j);
    }
  Mat v1 = matmul(l1, u_asc, BSE_OP_NONE, BSE_SHAPE_LOWER, BSE_OP_NONE, BSE_SHAPE_GENERAL);
  Mat v2 = matmul(l2, v_asc, BSE_OP_NONE, BSE_SHAPE_LOWER, BSE_OP_NONE, BSE_SHAPE_GENERAL);
  for (int64_t j = 0; j < n; ++j) {
    const double r = 1.0 / std::sqrt(cs.lambda[static_cast<size_t>(j)]);
    for (int64_t i = 0; i < n; ++i) {
      v1(i, j) *= r;
      v2(i, j) *= r;
    }
  }
  Mat vv = assemble_eigenvectors(v1, v2, cs.lambda, cs.lambda);
  return Result{cs.lambda, std::move(vv), cs.flagged};
}

// solvers.cpp:163-211
Result solve_reference(const Mat& a, const Mat& b) {
  {
    Mat m1, m2;
    product_pair(a, b, m1, m2);
  }
  const int64_t n = a.r;
  Mat ham(2 * n, 2 * n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      ham(i, j) = a(i, j);
      ham(i, n + j) = b(i, j);
      ham(n + i, j) = b(i, j);
      ham(n + i, n + j) = a(i, j);
    }
  Mat l;
  try {
    l = cholesky_lower(ham);
  } catch (const Err& e) {
    if (e.code != BSE_ERR_NOT_POSITIVE_DEFINITE) throw;
    throw Err{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_FULL, e.pivot, 0,
              "BSE Hamiltonian is not positive definite: " + e.msg};
  }
  Mat sigma(2 * n, 2 * n);
  for (int64_t i = 0; i < 2 * n; ++i) sigma(i, i) = i < n ? 1.0 : -1.0;
  Mat k = tri_solve(l, sigma, BSE_SIDE_LEFT, BSE_OP_NONE);
  k = tri_solve(l, k, BSE_SIDE_RIGHT, BSE_OP_ADJOINT);
  std::vector<double> w;
  Mat vec;
  hermitian_eig(k, w, vec);
  int64_t n_pos = 0;
  for (double x : w)
    if (x > 0.0) ++n_pos;
  if (n_pos != n)
    throw Err{BSE_ERR_CONVERGENCE_FAILURE, 0, -1, 0, "pencil inertia is off"};
  Mat wr(2 * n, n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < 2 * n; ++i) wr(i, j) = vec(i, n + j);
  const Mat vw = tri_solve(l, wr, BSE_SIDE_LEFT, BSE_OP_ADJOINT);
  Result out;
  out.lambda.resize(static_cast<size_t>(n));
  out.v = Mat(2 * n, n);
  for (int64_t j = 0; j < n; ++j) {
    const double m_j = w[static_cast<size_t>(n + j)];
    out.lambda[static_cast<size_t>(n - 1 - j)] = 1.0 / m_j;
    const double r = std::sqrt(m_j);
    for (int64_t i = 0; i < 2 * n; ++i) out.v(i, n - 1 - j) = vw(i, j) / r;
  }
  return out;
}

int fail(const Err& e, bse_status* st) {
  if (st) {
    st->code = e.code;
    st->block = e.block;
    st->pivot_index = e.pivot;
    st->relative_deviation = e.dev;
    std::snprintf(st->message, sizeof(st->message), "%s", e.msg.c_str());
  }
  return e.code;
}
int ok(bse_status* st) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->pivot_index = -1;
  }
  return BSE_OK;
}

}  // namespace

extern "C" {

void oracle_set_threads(int t) { scipy_openblas_set_num_threads(t); }
int oracle_get_threads(void) { return scipy_openblas_get_num_threads(); }
const char* oracle_blas_config(void) { return scipy_openblas_get_config(); }

// solvers.cpp:213-221 (dispatcher) — all four methods, for cross-checks.
int oracle_solve(int method, int64_t n, const double* a, const double* b, double* lambda,
                 double* v, int64_t* near_singular, int64_t* n_near, bse_status* st) {
  try {
    const Mat ma = load(n, n, a, n), mb = load(n, n, b, n);
    Result r;
    switch (method) {
      case BSE_METHOD_SQRT: r = solve_sqrt(ma, mb); break;
      case BSE_METHOD_CHOL: r = solve_chol(ma, mb); break;
      case BSE_METHOD_CHOL_SVD: r = solve_chol_svd(ma, mb); break;
      case BSE_METHOD_REFERENCE: r = solve_reference(ma, mb); break;
      default: throw Err{BSE_ERR_INVALID_SPEC, 0, -1, 0, "unknown method"};
    }
    std::memcpy(lambda, r.lambda.data(), sizeof(double) * r.lambda.size());
    store(r.v, v, 2 * n);
    *n_near = static_cast<int64_t>(r.near_singular.size());
    for (size_t i = 0; i < r.near_singular.size(); ++i) near_singular[i] = r.near_singular[i];
    return ok(st);
  } catch (const Err& e) {
    return fail(e, st);
  }
}

int oracle_cholesky_lower(int64_t n, const double* m, double* l, bse_status* st) {
  try {
    store(cholesky_lower(load(n, n, m, n)), l, n);
    return ok(st);
  } catch (const Err& e) {
    return fail(e, st);
  }
}

int oracle_hermitian_eig(int64_t n, const double* m, double* values, double* vectors,
                         bse_status* st) {
  try {
    std::vector<double> w;
    Mat vec;
    hermitian_eig(load(n, n, m, n), w, vec);
    std::memcpy(values, w.data(), sizeof(double) * w.size());
    store(vec, vectors, n);
    return ok(st);
  } catch (const Err& e) {
    return fail(e, st);
  }
}

int oracle_svd(int64_t n, const double* m, double* u, double* s, double* v, bse_status* st) {
  try {
    Mat mu, mv;
    std::vector<double> sv;
    svd(load(n, n, m, n), mu, sv, mv);
    store(mu, u, n);
    std::memcpy(s, sv.data(), sizeof(double) * sv.size());
    store(mv, v, n);
    return ok(st);
  } catch (const Err& e) {
    return fail(e, st);
  }
}

int oracle_tri_solve(int64_t n, const double* l, int64_t rows, int64_t cols, const double* rhs,
                     int side, int op, double* x, bse_status* st) {
  try {
    store(tri_solve(load(n, n, l, n), load(rows, cols, rhs, rows), side, op), x, rows);
    return ok(st);
  } catch (const Err& e) {
    return fail(e, st);
  }
}

int oracle_matmul(int64_t ar, int64_t ac, const double* a, int op_a, int shape_a, int64_t br,
                  int64_t bc, const double* b, int op_b, int shape_b, double* c, bse_status* st) {
  try {
    const Mat r = matmul(load(ar, ac, a, ar), load(br, bc, b, br), op_a, shape_a, op_b, shape_b);
    store(r, c, r.r);
    return ok(st);
  } catch (const Err& e) {
    return fail(e, st);
  }
}

int oracle_product_pair(int64_t n, const double* a, const double* b, double* m1, double* m2,
                        bse_status* st) {
  try {
    Mat x, y;
    product_pair(load(n, n, a, n), load(n, n, b, n), x, y);
    store(x, m1, n);
    store(y, m2, n);
    return ok(st);
  } catch (const Err& e) {
    return fail(e, st);
  }
}

int oracle_assemble_eigenvectors(int64_t n, int64_t k, const double* v1, const double* v2,
                                 const double* l1, const double* l2, double* v, bse_status* st) {
  try {
    std::vector<double> x(l1, l1 + k), y(l2, l2 + k);
    store(assemble_eigenvectors(load(n, k, v1, n), load(n, k, v2, n), x, y), v, 2 * n);
    return ok(st);
  } catch (const Err& e) {
    return fail(e, st);
  }
}

// solvers.cpp:125, 130-133 (the recovery tail of solve_chol / solve_sqrt): lambda_from_squares,
// assemble_eigenvectors with (lambda^2, 1), rebuild_nonpositive_columns.
int oracle_assemble_from_squares(int64_t n, int64_t k, const double* v1, const double* v2,
                                 const double* d, double* lambda, double* v,
                                 int64_t* near_singular, int64_t* n_near_singular,
                                 bse_status* st) {
  try {
    const std::vector<double> w(d, d + k);
    const Clamped cs = lambda_from_squares(w);
    std::vector<double> l1(static_cast<size_t>(k)), ones(static_cast<size_t>(k), 1.0);
    for (int64_t j = 0; j < k; ++j)
      l1[static_cast<size_t>(j)] = cs.lambda[static_cast<size_t>(j)] * cs.lambda[static_cast<size_t>(j)];
    const Mat m1 = load(n, k, v1, n), m2 = load(n, k, v2, n);
    Mat vv = assemble_eigenvectors(m1, m2, l1, ones);
    rebuild_nonpositive_columns(vv, m1, m2, w, cs);
    std::memcpy(lambda, cs.lambda.data(), sizeof(double) * cs.lambda.size());
    for (size_t i = 0; i < cs.flagged.size(); ++i) near_singular[i] = cs.flagged[i];
    *n_near_singular = static_cast<int64_t>(cs.flagged.size());
    store(vv, v, 2 * n);
    return ok(st);
  } catch (const Err& e) {
    return fail(e, st);
  }
}

}  // extern "C"
