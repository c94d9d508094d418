// gen_api.cpp — the reference's synthetic families in C++ (SURVEY §8f row f4 front ends;
// recipes of proj/src/gen.cpp:8-96): splitmix64 -> mt19937_64 -> Box-Muller Gaussian stream,
// Haar unitary by Householder QR with column phasing, the conditioned family and the random
// definite family. Host arithmetic, OpenMP over columns; not on the solver's hot path.
#include "bse/gen.hpp"

#include <cmath>
#include <vector>

namespace bse {

std::uint64_t splitmix64_at(std::uint64_t seed, std::uint64_t k) {
  std::uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

std::mt19937_64 entry_stream(std::uint64_t seed, std::uint64_t stream) {
  return std::mt19937_64(splitmix64_at(seed, stream));
}

double GaussianStream::next() {
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  // explicit 53-bit uniforms: u1 in (0, 1] keeps the logarithm finite
  const double u1 = static_cast<double>((engine_() >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(engine_() >> 11) * 0x1.0p-53;
  const double rad = std::sqrt(-2.0 * std::log(u1)), ang = 2.0 * M_PI * u2;
  spare_ = rad * std::sin(ang);
  have_spare_ = true;
  return rad * std::cos(ang);
}

Complex GaussianStream::next_complex() {
  const double re = next(), im = next();
  const double h = std::sqrt(2.0) / 2.0;
  return {re * h, im * h};
}

Matrix random_unitary(Index n, std::uint64_t seed) {
  if (n < 1) throw InvalidSpec("random_unitary: n must be >= 1");
  GaussianStream g(seed, 0);
  Matrix r(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) r(i, j) = g.next_complex();
  // Householder QR, reflectors H_k = I - tau_k v_k v_k^H with v_k(k) = 1 and a real beta_k
  // (the zlarfg convention); the reflector tails are kept below the diagonal of r
  std::vector<Complex> tau(static_cast<size_t>(n));
  std::vector<double> beta(static_cast<size_t>(n));
  for (Index k = 0; k < n; ++k) {
    const Complex alpha = r(k, k);
    double xn2 = 0.0;
    for (Index i = k + 1; i < n; ++i) xn2 += std::norm(r(i, k));
    if (xn2 == 0.0 && alpha.imag() == 0.0) {
      tau[k] = 0.0;
      beta[k] = alpha.real();
      continue;
    }
    const double nrm = std::sqrt(std::norm(alpha) + xn2);
    const double b = alpha.real() >= 0.0 ? -nrm : nrm;
    tau[k] = Complex((b - alpha.real()) / b, -alpha.imag() / b);
    const Complex scale = 1.0 / (alpha - b);
    for (Index i = k + 1; i < n; ++i) r(i, k) *= scale;
    beta[k] = b;
    r(k, k) = b;
    // apply H_k^H to the trailing columns: c -= conj(tau) v (v^H c)
#pragma omp parallel for schedule(static)
    for (Index j = k + 1; j < n; ++j) {
      Complex w = r(k, j);
      for (Index i = k + 1; i < n; ++i) w += std::conj(r(i, k)) * r(i, j);
      w *= std::conj(tau[k]);
      r(k, j) -= w;
      for (Index i = k + 1; i < n; ++i) r(i, j) -= r(i, k) * w;
    }
  }
  // Q = H_0 H_1 ... H_{n-1}, accumulated backwards on the identity
  Matrix q = Matrix::Identity(n, n);
  for (Index k = n - 1; k >= 0; --k) {
    if (tau[k] == Complex(0.0)) continue;
#pragma omp parallel for schedule(static)
    for (Index j = k; j < n; ++j) {
      Complex w = q(k, j);
      for (Index i = k + 1; i < n; ++i) w += std::conj(r(i, k)) * q(i, j);
      w *= tau[k];
      q(k, j) -= w;
      for (Index i = k + 1; i < n; ++i) q(i, j) -= r(i, k) * w;
    }
  }
  // phase column j by R(j,j)/|R(j,j)| (here the sign of the real beta_j): Haar distribution
  for (Index j = 0; j < n; ++j) {
    const double ph = beta[j] < 0.0 ? -1.0 : 1.0;
    if (ph < 0.0)
      for (Index i = 0; i < n; ++i) q(i, j) = -q(i, j);
  }
  return q;
}

BseMatrixI generate_conditioned(const GeneratorSpec& spec) {
  if (spec.n < 1) throw InvalidSpec("generate_conditioned: n must be >= 1");
  if (!(spec.kappa >= 3.0))
    throw InvalidSpec("generate_conditioned: kappa must be >= 3 so the spectrum vector is "
                      "nondecreasing from 1");
  const Index n = spec.n;
  std::vector<double> d(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i)
    d[i] = n == 1 ? 1.0 : 1.0 + (spec.kappa / 3.0 - 1.0) * double(i) / double(n - 1);
  const Matrix q = random_unitary(n, spec.seed);
  // A = Q^H D Q, then exactly Hermitian; B = A / 2 keeps A+B and A-B exact multiples of A
  Matrix a(n, n);
#pragma omp parallel for schedule(static)
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) {
      Complex s = 0.0;
      for (Index k = 0; k < n; ++k) s += std::conj(q(k, i)) * d[k] * q(k, j);
      a(i, j) = s;
    }
  Matrix h(n, n), b(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) {
      h(i, j) = 0.5 * (a(i, j) + std::conj(a(j, i)));
      b(i, j) = 0.5 * h(i, j);
    }
  return from_blocks(h, b);
}

BseMatrixI generate_random_definite(Index n, std::uint64_t seed, double shift_margin) {
  if (n < 1) throw InvalidSpec("generate_random_definite: n must be >= 1");
  if (!(shift_margin > 0.0))
    throw InvalidSpec("generate_random_definite: shift_margin must be positive");
  GaussianStream ga(seed, 0), gb(seed, 1);
  Matrix a0(n, n), b0(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) {
      a0(i, j) = ga.next_complex();
      b0(i, j) = gb.next_complex();
    }
  Matrix a(n, n), b(n, n);
  double na = 0.0, nb = 0.0;  // ||.||_1 (max column sum) bounds the 2-norm of a Hermitian
  for (Index j = 0; j < n; ++j) {
    double ca = 0.0, cb = 0.0;
    for (Index i = 0; i < n; ++i) {
      a(i, j) = 0.5 * (a0(i, j) + std::conj(a0(j, i)));
      b(i, j) = 0.5 * (b0(i, j) + std::conj(b0(j, i)));
      ca += std::abs(a(i, j));
      cb += std::abs(b(i, j));
    }
    na = std::max(na, ca);
    nb = std::max(nb, cb);
  }
  for (Index i = 0; i < n; ++i) a(i, i) += na + nb + shift_margin;
  return from_blocks(a, b);
}

}  // namespace bse
