// bse_api.cpp — the C++ drop-in API (include/bse/*.hpp) implemented over the C-ABI
// (include/bse_gpu.h). Host-side validation (from_blocks, shape checks) mirrors
// proj/src/core.cpp and backend.cpp; all numerics run in the CUDA library.
#include <algorithm>
#include <cmath>
#include <limits>
#include <memory>
#include <sstream>

#include "bse/backend.hpp"
#include "bse/solvers.hpp"
#include "bse/verify.hpp"
#include "bse_gpu.h"

namespace bse {

namespace {

thread_local int t_device = 0;

struct CtxHolder {
  bse_ctx* ctx = nullptr;
  int device = -1;
  ~CtxHolder() {
    if (ctx) bse_ctx_destroy(ctx);
  }
};
thread_local CtxHolder t_ctx;

[[noreturn]] void rethrow(const bse_status& st) {
  const std::string msg(st.message);
  switch (st.code) {
    case BSE_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case BSE_ERR_NOT_HERMITIAN: throw NotHermitian(msg, st.relative_deviation);
    case BSE_ERR_NOT_DEFINITE: throw NotDefinite(static_cast<Block>(st.block), msg);
    case BSE_ERR_NOT_POSITIVE_DEFINITE: throw NotPositiveDefinite(msg, st.pivot_index);
    case BSE_ERR_CONVERGENCE_FAILURE: throw ConvergenceFailure(msg);
    case BSE_ERR_SINGULAR_FACTOR: throw SingularFactor(msg);
    case BSE_ERR_NON_POSITIVE_SCALE: throw NonPositiveScale(msg);
    case BSE_ERR_INVALID_SPEC: throw InvalidSpec(msg);
    case BSE_ERR_ODD_DIMENSION: throw OddDimension(msg);
    case BSE_ERR_LENGTH_MISMATCH: throw LengthMismatch(msg);
    case BSE_ERR_CUDA:
    case BSE_ERR_OUT_OF_MEMORY:
    case BSE_ERR_NO_DEVICE: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

void check(int rc, const bse_status& st) {
  if (rc != BSE_OK) rethrow(st);
}

bse_ctx* ctx() {
  if (!t_ctx.ctx || t_ctx.device != t_device) {
    if (t_ctx.ctx) bse_ctx_destroy(t_ctx.ctx);
    t_ctx.ctx = nullptr;
    bse_status st{};
    check(bse_ctx_create(&t_ctx.ctx, t_device, &st), st);
    t_ctx.device = t_device;
  }
  return t_ctx.ctx;
}

const double* dp(const Matrix& m) { return reinterpret_cast<const double*>(m.data()); }
double* dp(Matrix& m) { return reinterpret_cast<double*>(m.data()); }

// core.cpp:45-57
Matrix validated_hermitian(const Matrix& m, double tol, const char* label) {
  const double norm = m.norm();
  double dev2 = 0.0;
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = 0; i < m.rows(); ++i) dev2 += std::norm(m(i, j) - std::conj(m(j, i)));
  const double dev = std::sqrt(dev2);
  if (dev > tol * norm) {
    std::ostringstream os;
    os << "block " << label << " is not Hermitian: relative deviation "
       << (norm > 0 ? dev / norm : dev) << " exceeds tolerance " << tol;
    throw NotHermitian(os.str(), norm > 0 ? dev / norm : dev);
  }
  Matrix out(m.rows(), m.cols());
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = 0; i < m.rows(); ++i) out(i, j) = 0.5 * (m(i, j) + std::conj(m(j, i)));
  return out;
}

SpectralResult run(Method method, const BseMatrixI& h) {
  const Index n = h.n();
  SpectralResult r;
  r.method = method;
  r.lambda.assign(static_cast<size_t>(n), 0.0);
  r.v = Matrix(2 * n, n);
  std::vector<int64_t> ns(static_cast<size_t>(n));
  int64_t nn = 0;
  bse_status st{};
  check(bse_solve(ctx(), static_cast<int>(method), n, dp(h.a()), n, dp(h.b()), n,
                  r.lambda.data(), dp(r.v), 2 * n, ns.data(), &nn, &st),
        st);
  r.near_singular.assign(ns.begin(), ns.begin() + nn);
  return r;
}

}  // namespace

double machine_eps() { return std::numeric_limits<double>::epsilon(); }
double Matrix::norm() const { return std::sqrt(squaredNorm()); }
void set_device(int device) { t_device = device; }

const char* method_name(Method m) {
  switch (m) {
    case Method::Sqrt: return "sqrt";
    case Method::Chol: return "chol";
    case Method::CholSvd: return "chol-svd";
    case Method::Reference: return "reference";
  }
  return "unknown";
}

Method method_from_name(const std::string& name) {
  if (name == "sqrt") return Method::Sqrt;
  if (name == "chol") return Method::Chol;
  if (name == "chol-svd" || name == "cholsvd") return Method::CholSvd;
  if (name == "reference") return Method::Reference;
  throw InvalidSpec("unknown method name: " + name);
}

const char* error_kind(const Error& e) {
  if (dynamic_cast<const DimensionMismatch*>(&e)) return "DimensionMismatch";
  if (dynamic_cast<const NotHermitian*>(&e)) return "NotHermitian";
  if (dynamic_cast<const NotDefinite*>(&e)) return "NotDefinite";
  if (dynamic_cast<const NotPositiveDefinite*>(&e)) return "NotPositiveDefinite";
  if (dynamic_cast<const ConvergenceFailure*>(&e)) return "ConvergenceFailure";
  if (dynamic_cast<const SingularFactor*>(&e)) return "SingularFactor";
  if (dynamic_cast<const NonPositiveScale*>(&e)) return "NonPositiveScale";
  if (dynamic_cast<const OddDimension*>(&e)) return "OddDimension";
  if (dynamic_cast<const LengthMismatch*>(&e)) return "LengthMismatch";
  if (dynamic_cast<const InvalidSpec*>(&e)) return "InvalidSpec";
  if (dynamic_cast<const ParseError*>(&e)) return "ParseError";
  if (dynamic_cast<const IoError*>(&e)) return "IoError";
  if (dynamic_cast<const DeviceError*>(&e)) return "DeviceError";
  return "Error";
}

BseMatrixI from_blocks(const Matrix& a, const Matrix& b, double tol) {
  if (a.rows() != a.cols() || b.rows() != b.cols()) throw DimensionMismatch("blocks must be square");
  if (a.rows() != b.rows()) {
    std::ostringstream os;
    os << "block dimensions differ: A is " << a.rows() << "x" << a.cols() << ", B is "
       << b.rows() << "x" << b.cols();
    throw DimensionMismatch(os.str());
  }
  if (a.rows() < 1) throw DimensionMismatch("blocks must be at least 1x1");
  return BseMatrixI(validated_hermitian(a, tol, "A"), validated_hermitian(b, tol, "B"));
}

Matrix realize_full(const BseMatrixI& h) {  // core.cpp:77-85 (host data movement)
  const Index n = h.n();
  Matrix f(2 * n, 2 * n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) {
      f(i, j) = h.a()(i, j);
      f(i, n + j) = h.b()(i, j);
      f(n + i, j) = -h.b()(i, j);
      f(n + i, n + j) = -h.a()(i, j);
    }
  return f;
}

ProductPair product_pair(const BseMatrixI& h) {
  const Index n = h.n();
  ProductPair p{Matrix(n, n), Matrix(n, n)};
  bse_status st{};
  check(bse_product_pair(ctx(), n, dp(h.a()), n, dp(h.b()), n, dp(p.m1), dp(p.m2), &st), st);
  return p;
}

Matrix assemble_eigenvectors(const HalfSpectralFactors& f) {
  const Index n = f.v1.rows(), k = f.v1.cols();
  if (f.v2.rows() != n || f.v2.cols() != k || Index(f.lambda1.size()) != k ||
      Index(f.lambda2.size()) != k)
    throw DimensionMismatch("factor shapes do not conform");
  Matrix v(2 * n, k);
  bse_status st{};
  check(bse_assemble_eigenvectors(ctx(), n, k, dp(f.v1), n, dp(f.v2), n, f.lambda1.data(),
                                  f.lambda2.data(), dp(v), 2 * n, &st),
        st);
  return v;
}

HermitianEig hermitian_eig(const Matrix& m) {
  if (m.rows() != m.cols()) throw DimensionMismatch("hermitian_eig: expected square");
  const Index n = m.rows();
  HermitianEig e{RealVector(static_cast<size_t>(n)), Matrix(n, n)};
  bse_status st{};
  check(bse_hermitian_eig(ctx(), n, dp(m), n, e.values.data(), dp(e.vectors), n, &st), st);
  return e;
}

CholeskyLower cholesky_lower(const Matrix& m) {
  if (m.rows() != m.cols()) throw DimensionMismatch("cholesky_lower: expected square");
  const Index n = m.rows();
  CholeskyLower l{Matrix(n, n)};
  bse_status st{};
  check(bse_cholesky_lower(ctx(), n, dp(m), n, dp(l.l), n, &st), st);
  return l;
}

SvdTriple svd(const Matrix& m) {
  if (m.rows() != m.cols()) throw DimensionMismatch("svd: expected square");
  const Index n = m.rows();
  SvdTriple t{Matrix(n, n), RealVector(static_cast<size_t>(n)), Matrix(n, n)};
  bse_status st{};
  check(bse_svd(ctx(), n, dp(m), n, dp(t.u), n, t.s.data(), dp(t.v), n, &st), st);
  return t;
}

Matrix tri_solve(const CholeskyLower& l, const Matrix& rhs, Side side, Op op) {
  if (l.l.rows() != l.l.cols()) throw DimensionMismatch("tri_solve: expected square");
  Matrix x(rhs.rows(), rhs.cols());
  bse_status st{};
  const Index ld = rhs.rows() > 0 ? rhs.rows() : 1;
  check(bse_tri_solve(ctx(), l.l.rows(), dp(l.l), l.l.rows(), rhs.rows(), rhs.cols(), dp(rhs),
                      ld, side == Side::Left ? BSE_SIDE_LEFT : BSE_SIDE_RIGHT,
                      op == Op::None ? BSE_OP_NONE : BSE_OP_ADJOINT, dp(x), ld, &st),
        st);
  return x;
}

Matrix matmul(const Matrix& a, const Matrix& b, const MatmulOpts& o) {
  const Index am = o.op_a == Op::None ? a.rows() : a.cols();
  const Index bn = o.op_b == Op::None ? b.cols() : b.rows();
  Matrix c(am, bn);
  bse_status st{};
  auto shp = [](Shape s) {
    return s == Shape::General ? BSE_SHAPE_GENERAL : (s == Shape::Lower ? BSE_SHAPE_LOWER : BSE_SHAPE_UPPER);
  };
  check(bse_matmul(ctx(), a.rows(), a.cols(), dp(a), a.rows() > 0 ? a.rows() : 1,
                   o.op_a == Op::None ? BSE_OP_NONE : BSE_OP_ADJOINT, shp(o.shape_a), b.rows(),
                   b.cols(), dp(b), b.rows() > 0 ? b.rows() : 1,
                   o.op_b == Op::None ? BSE_OP_NONE : BSE_OP_ADJOINT, shp(o.shape_b), dp(c),
                   am > 0 ? am : 1, &st),
        st);
  return c;
}

SpectralResult solve_chol(const BseMatrixI& h) { return run(Method::Chol, h); }
SpectralResult solve_chol_svd(const BseMatrixI& h) { return run(Method::CholSvd, h); }
SpectralResult solve_sqrt(const BseMatrixI& h) { return run(Method::Sqrt, h); }
SpectralResult solve_reference(const BseMatrixI& h) { return run(Method::Reference, h); }
SpectralResult solve(Method method, const BseMatrixI& h) { return run(method, h); }

std::vector<SpectralResult> solve_batched(Method method, const std::vector<BseMatrixI>& hs) {
  std::vector<SpectralResult> out(hs.size());
  if (hs.empty()) return out;
  const Index n = hs[0].n();
  for (const auto& h : hs)
    if (h.n() != n) throw DimensionMismatch("solve_batched: batch items must share one size");
  const size_t k = hs.size();
  std::vector<const double*> pa(k), pb(k);
  std::vector<double*> pl(k), pv(k);
  for (size_t i = 0; i < k; ++i) {
    out[i].method = method;
    out[i].lambda.assign(static_cast<size_t>(n), 0.0);
    out[i].v = Matrix(2 * n, n);
    pa[i] = dp(hs[i].a());
    pb[i] = dp(hs[i].b());
    pl[i] = out[i].lambda.data();
    pv[i] = dp(out[i].v);
  }
  std::vector<int64_t> ns(k * static_cast<size_t>(n)), nn(k);
  int64_t failed = -1;
  bse_status st{};
  check(bse_solve_batched(ctx(), static_cast<int>(method), n, int64_t(k), pa.data(), n, pb.data(),
                          n, pl.data(), pv.data(), 2 * n, ns.data(), nn.data(), &failed, &st),
        st);
  for (size_t i = 0; i < k; ++i)
    out[i].near_singular.assign(ns.begin() + i * n, ns.begin() + i * n + nn[i]);
  return out;
}

SpectralResult negative_spectrum(const BseMatrixI& h, const SpectralResult& r) {
  const Index n = h.n();
  if (r.v.rows() != 2 * n || r.v.cols() != Index(r.lambda.size()))
    throw DimensionMismatch("spectral result does not match the matrix dimension");
  SpectralResult out;
  const Index k = r.v.cols();
  out.lambda.resize(r.lambda.size());
  out.v = Matrix(2 * n, k);
  if (k > 0) {
    bse_status st{};
    check(bse_negative_spectrum(ctx(), n, k, r.lambda.data(), dp(r.v), 2 * n, out.lambda.data(),
                                dp(out.v), 2 * n, &st),
          st);
  }
  out.method = r.method;
  out.near_singular = r.near_singular;
  return out;
}

Matrix hpd_sqrt(const Matrix& m) {
  if (m.rows() != m.cols()) throw DimensionMismatch("hpd_sqrt: expected square");
  const Index n = m.rows();
  Matrix s(n, n);
  bse_status st{};
  check(bse_hpd_sqrt(ctx(), n, dp(m), n, dp(s), n, &st), st);
  return s;
}

// ------------------------------------------------------------------ verify.hpp
Matrix SignatureOperators::j_times(const Matrix& x) const {
  Matrix y(x.rows(), x.cols());
  for (Index j = 0; j < x.cols(); ++j)
    for (Index i = 0; i < n; ++i) {
      y(i, j) = x(n + i, j);
      y(n + i, j) = -x(i, j);
    }
  return y;
}
Matrix SignatureOperators::times_j(const Matrix& x) const {
  Matrix y(x.rows(), x.cols());
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < x.rows(); ++i) {
      y(i, j) = -x(i, n + j);
      y(i, n + j) = x(i, j);
    }
  return y;
}
Matrix SignatureOperators::sigma_times(const Matrix& x) const {
  Matrix y = x;
  for (Index j = 0; j < x.cols(); ++j)
    for (Index i = n; i < 2 * n; ++i) y(i, j) = -y(i, j);
  return y;
}
Matrix SignatureOperators::times_sigma(const Matrix& x) const {
  Matrix y = x;
  for (Index j = n; j < 2 * n; ++j)
    for (Index i = 0; i < x.rows(); ++i) y(i, j) = -y(i, j);
  return y;
}

namespace {
bool check_form(int form, const Matrix& m, double tol) {
  if (m.rows() != m.cols())
    throw DimensionMismatch(std::string(form == 1 ? "check_form1" : "check_form2") +
                            ": matrix must be square");
  int res = 0;
  bse_status st{};
  check(bse_check_form(ctx(), form, m.rows(), dp(m), m.rows() > 0 ? m.rows() : 1, tol, &res, &st),
        st);
  return res != 0;
}
}  // namespace

bool check_form1(const Matrix& m, double tol) { return check_form(1, m, tol); }
bool check_form2(const Matrix& m, double tol) { return check_form(2, m, tol); }

double sigma_orthogonality_error(const Matrix& v) {
  double out = 0.0;
  bse_status st{};
  check(bse_sigma_orthogonality_error(ctx(), v.rows(), v.cols(), dp(v), v.rows() > 0 ? v.rows() : 1,
                                      &out, &st),
        st);
  return out;
}

RealVector residual(const BseMatrixI& h, const SpectralResult& r) {
  const Index n = h.n(), k = r.v.cols();
  if (r.v.rows() != 2 * n || Index(r.lambda.size()) != k)
    throw DimensionMismatch("residual: result does not conform to the matrix");
  RealVector out(static_cast<size_t>(k));
  if (k == 0) return out;
  bse_status st{};
  check(bse_residual(ctx(), n, dp(h.a()), n, dp(h.b()), n, k, r.lambda.data(), dp(r.v), 2 * n,
                     out.data(), &st),
        st);
  return out;
}

bool check_pairing(const RealVector& pos, const RealVector& neg, double tol) {
  if (pos.size() != neg.size()) throw LengthMismatch("check_pairing: spectra have different lengths");
  RealVector p = pos, m(neg.size());
  for (size_t i = 0; i < neg.size(); ++i) m[i] = -neg[i];
  std::sort(p.begin(), p.end());
  std::sort(m.begin(), m.end());
  double scale = 0.0;
  for (double x : pos) scale = std::max(scale, std::fabs(x));
  for (size_t i = 0; i < p.size(); ++i)
    if (!(std::fabs(p[i] - m[i]) <= tol * scale)) return false;
  return true;
}

double predicted_error(const ErrorModelInput& in, bool squared_method) {
  if (squared_method)
    return in.eps * (in.norm_h / in.s_lambda) * std::min(in.norm_h / in.lambda, 1.0 / std::sqrt(in.eps));
  return in.eps * in.norm_h / in.s_lambda;
}

}  // namespace bse
