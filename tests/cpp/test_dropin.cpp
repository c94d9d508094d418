// C++ drop-in check: the reference's test_solvers.cpp cases written against include/bse/*.hpp
// (same names and exception classes), linked to libbse_b200.so. Exit code = failures.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "bse/backend.hpp"
#include "bse/eigen_adapter.hpp"  // empty without Eigen (the reference's Eigen interop when present)
#include "bse/solvers.hpp"
#include "bse/verify.hpp"

static int failures = 0;
#define CHECK(c)                                                  \
  do {                                                            \
    if (!(c)) {                                                   \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);     \
      ++failures;                                                 \
    }                                                             \
  } while (0)

static bse::Matrix scalar(double v) {
  bse::Matrix m(1, 1);
  m(0, 0) = v;
  return m;
}

int main() {
  using namespace bse;
  const double s3 = std::sqrt(3.0);
  for (Method m : {Method::Chol, Method::CholSvd}) {  // test_solvers.cpp:33-42
    const SpectralResult r = solve(m, from_blocks(scalar(2.0), scalar(1.0)));
    CHECK(std::abs(r.lambda[0] - s3) < 1e-13 * s3);
    const Complex ph = r.v(0, 0) / std::abs(r.v(0, 0));
    CHECK(std::abs(r.v(0, 0) / ph - 0.5 * (std::pow(3.0, 0.25) + std::pow(3.0, -0.25))) < 1e-12);
    CHECK(std::abs(r.v(1, 0) / ph - 0.5 * (std::pow(3.0, -0.25) - std::pow(3.0, 0.25))) < 1e-12);
  }
  {  // decoupled B=0 (test_solvers.cpp:44-53)
    Matrix a = Matrix::Zero(3, 3);
    a(0, 0) = 3.0; a(1, 1) = 1.0; a(2, 2) = 2.0;
    const SpectralResult r = solve_chol(from_blocks(a, Matrix::Zero(3, 3)));
    CHECK(std::abs(r.lambda[0] - 1.0) < 1e-13 && std::abs(r.lambda[2] - 3.0) < 1e-13);
  }
  {  // batch driver: items equal the single solves; the failing item's class is thrown
    std::vector<BseMatrixI> hs{from_blocks(scalar(2.0), scalar(1.0)),
                               from_blocks(scalar(5.0), scalar(3.0))};
    const auto rs = solve_batched(Method::Chol, hs);
    CHECK(rs.size() == 2);
    CHECK(std::abs(rs[0].lambda[0] - s3) < 1e-13 * s3);
    CHECK(std::abs(rs[1].lambda[0] - 4.0) < 1e-13 * 4.0);  // sqrt(5^2 - 3^2)
    hs.push_back(from_blocks(scalar(1.0), scalar(2.0)));
    try {
      solve_batched(Method::Chol, hs);
      CHECK(false);
    } catch (const NotDefinite& e) {
      CHECK(e.which() == Block::M2);
      CHECK(std::string(e.what()).find("batch item 2") != std::string::npos);
    }
  }
  try {  // test_solvers.cpp:73-79
    solve_chol_svd(from_blocks(scalar(1.0), scalar(2.0)));
    CHECK(false);
  } catch (const NotDefinite& e) {
    CHECK(e.which() == Block::M2);
    CHECK(std::string(error_kind(e)) == "NotDefinite");
  }
  try {  // test_backend.cpp:78-85
    Matrix m(2, 2);
    m(0, 0) = 1.0; m(0, 1) = 2.0; m(1, 0) = 2.0; m(1, 1) = 1.0;
    cholesky_lower(m);
    CHECK(false);
  } catch (const NotPositiveDefinite& e) {
    CHECK(e.pivot_index() == 1);
  }
  {  // clamp / flag (test_solvers.cpp:168-186)
    Matrix a = Matrix::Zero(2, 2);
    a(0, 0) = 1e-40; a(1, 1) = 1.0;
    const SpectralResult r = solve_chol(from_blocks(a, Matrix::Zero(2, 2)));
    CHECK(r.near_singular.size() == 1 && r.near_singular[0] == 0);
    CHECK(std::abs(r.lambda[0] - machine_eps()) < 1e-6 * machine_eps());
  }
  {  // backend: [[2,1],[1,2]] -> (1, 3)
    Matrix m(2, 2);
    m(0, 0) = 2.0; m(0, 1) = 1.0; m(1, 0) = 1.0; m(1, 1) = 2.0;
    const HermitianEig e = hermitian_eig(m);
    CHECK(std::abs(e.values[0] - 1.0) < 1e-14 && std::abs(e.values[1] - 3.0) < 1e-14);
    const Matrix p = matmul(m, m, {.op_a = Op::Adjoint});
    CHECK(std::abs(p(0, 0) - Complex(5.0)) < 1e-14);
  }
  {  // SQRT / REFERENCE (solvers.cpp:94-117, 163-211): lambda = sqrt(3) for (A, B) = (2, 1)
    const SpectralResult s = solve_sqrt(from_blocks(scalar(2.0), scalar(1.0)));
    const SpectralResult p = solve_reference(from_blocks(scalar(2.0), scalar(1.0)));
    CHECK(std::abs(s.lambda[0] - std::sqrt(3.0)) < 1e-14 && s.method == Method::Sqrt);
    CHECK(std::abs(p.lambda[0] - std::sqrt(3.0)) < 1e-14 && p.method == Method::Reference);
  }
  {  // hpd_sqrt (backend.cpp:88-107) and its NotPositiveDefinite payload
    Matrix m(2, 2);
    m(0, 0) = 4.0; m(1, 1) = 9.0;
    const Matrix s = hpd_sqrt(m);
    CHECK(std::abs(s(0, 0) - Complex(2.0)) < 1e-14 && std::abs(s(1, 1) - Complex(3.0)) < 1e-14);
    m(1, 1) = -1.0;
    try {
      hpd_sqrt(m);
      CHECK(false);
    } catch (const NotPositiveDefinite& e) {
      CHECK(e.pivot_index() == 0);
    }
  }
  {  // verify.hpp on the GPU: residual, Sigma-orthogonality, forms, pairing
    Matrix a(3, 3), b(3, 3);
    for (int i = 0; i < 3; ++i) a(i, i) = 2.0 + i;
    b(0, 1) = b(1, 0) = 0.5;
    const BseMatrixI h = from_blocks(a, b);
    const SpectralResult r = solve_chol(h);
    const RealVector res = residual(h, r);
    CHECK(res.size() == 3 && *std::max_element(res.begin(), res.end()) < 1e-14);
    CHECK(sigma_orthogonality_error(r.v) < 1e-13);
    const SpectralResult neg = negative_spectrum(h, r);
    CHECK(check_pairing(r.lambda, neg.lambda, 1e-14));
    Matrix hm(6, 6);
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) {
        hm(i, j) = a(i, j);
        hm(i, j + 3) = b(i, j);
        hm(i + 3, j) = -b(i, j);
        hm(i + 3, j + 3) = -a(i, j);
      }
    CHECK(check_form1(hm, 1e-14) && check_form2(hm, 1e-14));
    try {
      sigma_orthogonality_error(Matrix(3, 1));
      CHECK(false);
    } catch (const OddDimension&) {
    }
    try {
      check_pairing(RealVector{1.0}, RealVector{}, 0.0);
      CHECK(false);
    } catch (const LengthMismatch&) {
    }
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures;
}
