#pragma once
// Drop-in replacement for /root/reference/proj/include/bse/solvers.hpp:1-36.
// All four solvers run on the GPU: solve_chol / solve_chol_svd are the hot path,
// solve_sqrt / solve_reference are composed from the same device primitives (§8f f2, f3).

#include <vector>

#include "bse/types.hpp"

namespace bse {

SpectralResult solve_sqrt(const BseMatrixI& h);       // solvers.cpp:94-117
SpectralResult solve_chol(const BseMatrixI& h);      // solvers.cpp:119-135
SpectralResult solve_chol_svd(const BseMatrixI& h);  // solvers.cpp:137-161
SpectralResult solve_reference(const BseMatrixI& h);  // solvers.cpp:163-211
SpectralResult solve(Method method, const BseMatrixI& h);  // solvers.cpp:213-221
SpectralResult negative_spectrum(const BseMatrixI& h, const SpectralResult& r);  // :223-236

// B200 extension (SURVEY §8b batch driver): independent matrices of one size, solved in order
// with each upload/download overlapped with the neighbouring solves (bse_solve_batched).
// The first failing item's typed exception is thrown; the message names the item.
std::vector<SpectralResult> solve_batched(Method method, const std::vector<BseMatrixI>& hs);

// B200 extension: device index used by this thread's default context (default 0).
void set_device(int device);

}  // namespace bse
