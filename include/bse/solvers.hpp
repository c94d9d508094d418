#pragma once
// Drop-in replacement for /root/reference/proj/include/bse/solvers.hpp:1-36.
// solve_chol / solve_chol_svd run on the GPU; solve_sqrt / solve_reference are outside the
// accelerated hot path and throw InvalidSpec("... not accelerated").

#include "bse/types.hpp"

namespace bse {

SpectralResult solve_sqrt(const BseMatrixI& h);
SpectralResult solve_chol(const BseMatrixI& h);      // solvers.cpp:119-135
SpectralResult solve_chol_svd(const BseMatrixI& h);  // solvers.cpp:137-161
SpectralResult solve_reference(const BseMatrixI& h);
SpectralResult solve(Method method, const BseMatrixI& h);  // solvers.cpp:213-221
SpectralResult negative_spectrum(const BseMatrixI& h, const SpectralResult& r);

// B200 extension: device index used by this thread's default context (default 0).
void set_device(int device);

}  // namespace bse
