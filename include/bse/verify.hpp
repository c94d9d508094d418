#pragma once
// Drop-in replacement for /root/reference/proj/include/bse/verify.hpp:1-67: structure
// predicates and diagnostics. residual, sigma_orthogonality_error and check_form1/2 run on the
// GPU (DMMA GEMMs + deterministic reductions); check_pairing and
// predicted_error are host-side scalar/sorting formulas like the reference's.

#include "bse/types.hpp"

namespace bse {

/// J = [0 I; -I 0] and Sigma = diag(I, -I) as operators on block-partitioned matrices
/// (verify.cpp:19-43; host data movement, never materialized).
struct SignatureOperators {
  Index n;  // half dimension

  Matrix j_times(const Matrix& x) const;      // J * x
  Matrix times_j(const Matrix& x) const;      // x * J
  Matrix sigma_times(const Matrix& x) const;  // Sigma * x
  Matrix times_sigma(const Matrix& x) const;  // x * Sigma
};

bool check_form1(const Matrix& m, double tol);               // verify.cpp:46-55
bool check_form2(const Matrix& m, double tol);               // verify.cpp:57-68
double sigma_orthogonality_error(const Matrix& v);           // verify.cpp:70-74
RealVector residual(const BseMatrixI& h, const SpectralResult& r);  // verify.cpp:76-93
bool check_pairing(const RealVector& pos, const RealVector& neg, double tol);  // :95-106

struct ErrorModelInput {
  double norm_h;
  double lambda;
  double s_lambda = 1.0;
  double eps = machine_eps();
};
double predicted_error(const ErrorModelInput& in, bool squared_method);  // verify.cpp:108-114

}  // namespace bse
