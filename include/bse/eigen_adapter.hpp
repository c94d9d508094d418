#pragma once
// Eigen interop for code written against the reference's Eigen-typed API
// (/root/reference/proj/include/bse/types.hpp:17-19: Matrix = Eigen::MatrixXcd,
// RealVector = Eigen::VectorXd). bse::Matrix has Eigen::MatrixXcd's byte layout (column-major
// interleaved complex128), so the conversions are single copies and the views are zero-copy
// Eigen::Map's. Compiled only when Eigen is on the include path; without it this header is
// empty, so it can be included unconditionally (tests/cpp/test_dropin.cpp does).

#if defined(__has_include)
#if __has_include(<Eigen/Dense>)
#define BSE_HAVE_EIGEN 1
#endif
#endif

#ifdef BSE_HAVE_EIGEN
#include <Eigen/Dense>

#include <algorithm>

#include "bse/types.hpp"

namespace bse::eigen {

inline Matrix from_eigen(const Eigen::MatrixXcd& m) {
  Matrix out(m.rows(), m.cols());
  std::copy(m.data(), m.data() + m.size(), out.data());
  return out;
}

inline Eigen::MatrixXcd to_eigen(const Matrix& m) {
  return Eigen::Map<const Eigen::MatrixXcd>(m.data(), m.rows(), m.cols());
}

// zero-copy views of a bse::Matrix (valid while the matrix lives)
inline Eigen::Map<Eigen::MatrixXcd> view(Matrix& m) {
  return Eigen::Map<Eigen::MatrixXcd>(m.data(), m.rows(), m.cols());
}
inline Eigen::Map<const Eigen::MatrixXcd> view(const Matrix& m) {
  return Eigen::Map<const Eigen::MatrixXcd>(m.data(), m.rows(), m.cols());
}

inline Eigen::VectorXd to_eigen(const RealVector& v) {
  return Eigen::Map<const Eigen::VectorXd>(v.data(), static_cast<Eigen::Index>(v.size()));
}

// bse::from_blocks on Eigen blocks (core.cpp:61-75 semantics: Hermitian check within tol,
// then symmetrisation)
inline BseMatrixI from_blocks(const Eigen::MatrixXcd& a, const Eigen::MatrixXcd& b,
                              double tol = kDefaultHermTol) {
  return bse::from_blocks(from_eigen(a), from_eigen(b), tol);
}

}  // namespace bse::eigen
#endif  // BSE_HAVE_EIGEN
