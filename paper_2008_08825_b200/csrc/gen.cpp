// gen.cpp — seeded synthetic inputs (host, OpenMP).
//
// Input synthesis is not on the hot path; it feeds identical bytes to the GPU solver and
// the CPU oracle. Two families:
//  * bse_gen_gaussian_stream: the reference's GaussianStream (proj/src/gen.cpp:8-38,
//    splitmix64 -> mt19937_64 -> Box-Muller with a spare), for the reference's own test
//    families (random_hermitian, generate_random_definite, random_unitary).
//  * counter-based draws (splitmix64 of (seed, stream, index)) for BASELINE.json's configs:
//    parallel and reproducible bit-for-bit on any host, so a 16384^2 block is generated in
//    a fraction of a second instead of minutes with a sequential engine.
#include <cmath>
#include <cstdint>
#include <random>

#include "../../include/bse_gpu.h"

namespace {

// proj/src/gen.cpp:8-13
inline uint64_t splitmix64_at(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return splitmix64_at(seed, 0x5bd1e995ULL * (stream + 1));
}

inline double uniform_at(uint64_t key, uint64_t idx) {
  return double(splitmix64_at(key, idx) >> 11) * 0x1.0p-53;  // [0,1)
}

inline double normal_at(uint64_t key, uint64_t idx) {
  const double u1 = double((splitmix64_at(key, 2 * idx) >> 11) + 1) * 0x1.0p-53;  // (0,1]
  const double u2 = double(splitmix64_at(key, 2 * idx + 1) >> 11) * 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

}  // namespace

extern "C" {

int bse_gen_normal(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  const uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) out[i] = normal_at(key, uint64_t(i));
  return BSE_OK;
}

int bse_gen_uniform(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  const uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) out[i] = uniform_at(key, uint64_t(i));
  return BSE_OK;
}

// proj/src/gen.cpp:19-38 (GaussianStream::next / next_complex)
int bse_gen_gaussian_stream(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  std::mt19937_64 eng(splitmix64_at(seed, stream));
  bool have_spare = false;
  double spare = 0.0;
  auto next = [&]() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    const double u1 = static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(eng() >> 11) * 0x1.0p-53;
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * M_PI * u2;
    spare = radius * std::sin(angle);
    have_spare = true;
    return radius * std::cos(angle);
  };
  const double h = std::sqrt(2.0) / 2.0;
  for (int64_t i = 0; i < count; ++i) {
    const double re = next();
    const double im = next();
    out[2 * i] = re * h;
    out[2 * i + 1] = im * h;
  }
  return BSE_OK;
}

// BASELINE.json configs 1/2/4/5: A = diag(d) + scale (Z + Z^H)/2, B = scale (W + W^H)/2,
// streams: 0 -> Z, 1 -> W, 2 -> d. Complex: Re/Im ~ N(0,1)/sqrt(2n); real: N(0,1)/sqrt(n).
int bse_gen_dominant(int64_t n, uint64_t seed, int is_complex, double scale, double dlo,
                     double dhi, double* a, double* b) {
  if (n < 1) return BSE_ERR_INVALID_SPEC;
  const uint64_t kz = stream_key(seed, 0), kw = stream_key(seed, 1), kd = stream_key(seed, 2);
  const double sd = is_complex ? 1.0 / std::sqrt(2.0 * double(n)) : 1.0 / std::sqrt(double(n));
  const uint64_t nn = uint64_t(n);
  auto z = [&](uint64_t key, int64_t i, int64_t j, double& re, double& im) {
    const uint64_t idx = uint64_t(i) + uint64_t(j) * nn;
    if (is_complex) {
      re = normal_at(key, 2 * idx) * sd;
      im = normal_at(key, 2 * idx + 1) * sd;
    } else {
      re = normal_at(key, idx) * sd;
      im = 0.0;
    }
  };
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < n; ++i) {
      double zr, zi, tr, ti;
      z(kz, i, j, zr, zi);
      z(kz, j, i, tr, ti);  // (Z^H)_{ij} = conj(Z_{ji})
      double ar = 0.5 * scale * (zr + tr), ai = 0.5 * scale * (zi - ti);
      if (i == j) {
        ar += dlo + (dhi - dlo) * uniform_at(kd, uint64_t(i));
        ai = 0.0;
      }
      z(kw, i, j, zr, zi);
      z(kw, j, i, tr, ti);
      const double br = 0.5 * scale * (zr + tr), bi = (i == j) ? 0.0 : 0.5 * scale * (zi - ti);
      const uint64_t o = 2 * (uint64_t(i) + uint64_t(j) * nn);
      a[o] = ar;
      a[o + 1] = ai;
      b[o] = br;
      b[o + 1] = bi;
    }
  }
  return BSE_OK;
}

}  // extern "C"
