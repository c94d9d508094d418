#pragma once
// Drop-in replacement for /root/reference/proj/include/bse/backend.hpp:1-69 (same contract,
// executed by the B200 kernels through bse_gpu.h).

#include "bse/types.hpp"

namespace bse {

struct HermitianEig {
  RealVector values;
  Matrix vectors;
};
struct CholeskyLower {
  Matrix l;
};
struct SvdTriple {
  Matrix u;
  RealVector s;
  Matrix v;
};

enum class Side { Left, Right };
enum class Op { None, Adjoint };
enum class Shape { General, Lower, Upper };

struct MatmulOpts {
  Op op_a = Op::None;
  Op op_b = Op::None;
  Shape shape_a = Shape::General;
  Shape shape_b = Shape::General;
};

HermitianEig hermitian_eig(const Matrix& m);   // backend.cpp:28-45 (reads the lower triangle)
CholeskyLower cholesky_lower(const Matrix& m);  // backend.cpp:47-62
SvdTriple svd(const Matrix& m);                 // backend.cpp:64-86
Matrix tri_solve(const CholeskyLower& l, const Matrix& rhs, Side side = Side::Left,
                 Op op = Op::None);             // backend.cpp:109-129
Matrix matmul(const Matrix& a, const Matrix& b, const MatmulOpts& opts = {});  // :131-175
Matrix hpd_sqrt(const Matrix& m);               // backend.cpp:88-107 (eigendecomposition)

}  // namespace bse
