// include/bse/eigen_adapter.hpp against the mock Eigen (tests/cpp/mock_eigen): conversions are
// exact copies and the views alias the bse::Matrix storage. Host-only (no device call).
#include <cstdio>

#include "bse/eigen_adapter.hpp"

int main() {
#ifndef BSE_HAVE_EIGEN
  std::puts("no Eigen on the include path");
  return 1;
#else
  Eigen::MatrixXcd e(3, 2);
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 3; ++i) e(i, j) = {double(i + 10 * j), double(-j)};
  bse::Matrix m = bse::eigen::from_eigen(e);
  int bad = 0;
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 3; ++i) bad += m(i, j) != e(i, j);
  Eigen::MatrixXcd back = bse::eigen::to_eigen(m);
  for (int k = 0; k < 6; ++k) bad += back.data()[k] != e.data()[k];
  bse::eigen::view(m)(2, 1) = {7.0, 7.0};
  bad += m(2, 1) != bse::Complex(7.0, 7.0);
  std::printf(bad ? "FAILED %d\n" : "OK\n", bad);
  return bad;
#endif
}
