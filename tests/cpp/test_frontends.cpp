// Host-only checks of the SURVEY §8f row f4 front ends (no GPU calls): Matrix-Market I/O as in
// the reference's proj/tests/test_mm_io.cpp, the generators of test_gen.cpp that do not solve,
// and the flop model / presets of test_bench.cpp. Exit code = failures; argv[1] = scratch dir.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>

#include "bse/bench.hpp"
#include "bse/gen.hpp"
#include "bse/mm_io.hpp"

static int failures = 0;
#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                             \
    }                                                         \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static double diff(const bse::Matrix& a, const bse::Matrix& b) {
  double s = 0.0;
  for (bse::Index j = 0; j < a.cols(); ++j)
    for (bse::Index i = 0; i < a.rows(); ++i) s += std::norm(a(i, j) - b(i, j));
  return std::sqrt(s);
}

static void text(const std::string& path, const char* body) {
  std::ofstream f(path);
  f << body;
}

int main(int argc, char** argv) {
  using namespace bse;
  const std::string dir = argc > 1 ? argv[1] : ".";
  auto file = [&](const char* n) { return dir + "/" + n; };

  {  // complex general array round trip is bit exact
    GaussianStream g(1, 0);
    Matrix m(4, 3);
    for (Index j = 0; j < 3; ++j)
      for (Index i = 0; i < 4; ++i) m(i, j) = g.next_complex();
    mm::write_complex(file("m.mtx"), m);
    const Matrix back = mm::read_complex(file("m.mtx"));
    CHECK(back.rows() == 4 && back.cols() == 3 && diff(back, m) == 0.0);
    mm::write_binary(file("m.bin"), m);  // binary container, same guarantee
    CHECK(diff(mm::read_complex(file("m.bin")), m) == 0.0);
  }
  {  // hermitian array storage restores the upper triangle
    const BseMatrixI h = generate_random_definite(6, 2);
    mm::write_complex(file("a.mtx"), h.a(), mm::Symmetry::Hermitian);
    CHECK(diff(mm::read_complex(file("a.mtx")), h.a()) == 0.0);
    bench::save_matrix_pair(h, file("pa.mtx"), file("pb.bin"));
    const BseMatrixI back = bench::load_matrix_pair(file("pa.mtx"), file("pb.bin"));
    CHECK(diff(back.a(), h.a()) == 0.0 && diff(back.b(), h.b()) == 0.0);
  }
  {  // real array files round trip, incl. subnormal-adjacent magnitudes
    RealMatrix v(3, 1);
    v(0, 0) = 1.0;
    v(1, 0) = std::sqrt(2.0);
    v(2, 0) = 1e-300;
    mm::write_real(file("v.mtx"), v);
    const RealMatrix back = mm::read_real(file("v.mtx"));
    CHECK(back.rows() == 3 && back(0, 0) == v(0, 0) && back(1, 0) == v(1, 0) && back(2, 0) == v(2, 0));
    mm::write_binary(file("v.bin"), v);
    CHECK(mm::read_real(file("v.bin"))(1, 0) == v(1, 0));
    CHECK(throws<ParseError>([&] { mm::read_real(file("m.bin")); }));  // complex field
  }
  {  // coordinate format with hermitian symmetry and a comment line
    text(file("c.mtx"),
         "%%MatrixMarket matrix coordinate complex hermitian\n% a comment line\n2 2 2\n"
         "1 1 2.0 0.0\n2 1 0.5 -0.25\n");
    const Matrix m = mm::read_complex(file("c.mtx"));
    CHECK(m(0, 0) == Complex(2.0, 0.0) && m(1, 0) == Complex(0.5, -0.25));
    CHECK(m(0, 1) == Complex(0.5, 0.25) && m(1, 1) == Complex(0.0, 0.0));
  }
  {  // real and integer fields promote; symmetric coordinate mirrors without conjugation
    text(file("i.mtx"), "%%MatrixMarket matrix coordinate integer symmetric\n3 3 2\n1 1 4\n3 1 -2\n");
    const Matrix m = mm::read_complex(file("i.mtx"));
    CHECK(m(0, 0) == Complex(4.0, 0.0) && m(2, 0) == Complex(-2.0, 0.0) && m(0, 2) == Complex(-2.0, 0.0));
    const RealMatrix r = mm::read_real(file("i.mtx"));
    CHECK(r(0, 2) == -2.0);
  }
  {  // malformed inputs: ParseError with the line number; IoError for missing files
    struct Case {
      const char* body;
      long line;
    };
    const Case cases[] = {
        {"%%MatrixMarket matrix array real general\n2 2\n1.0\n", 3},             // too few
        {"%%MatrixMarket matrix array real general\n1 1\n1.0\n2.0\n", 4},        // extra
        {"%%MatrixMarket matrix array real general\n1 1\nabc\n", 3},             // numeric
        {"%%MatrixMarket matrix array real general\n1 1\n1.0 2.0\n", 3},         // trailing
        {"%%MatrixMarket vector array real general\n1 1\n1.0\n", 1},             // object
        {"MatrixMarket matrix array real general\n1 1\n1.0\n", 1},               // banner
        {"%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n", 3},  // upper
        {"%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", 3},  // range
        {"%%MatrixMarket matrix array real symmetric\n2 3\n1.0\n", 2},           // square
        {"", 0},                                                                  // empty
    };
    int k = 0;
    for (const Case& c : cases) {
      const std::string p = file(("bad" + std::to_string(k++) + ".mtx").c_str());
      text(p, c.body);
      long line = -1;
      try {
        mm::read_complex(p);
      } catch (const ParseError& e) {
        line = e.line();
      } catch (...) {
      }
      CHECK(line == c.line);
    }
    CHECK(throws<IoError>([&] { mm::read_complex(file("does_not_exist.mtx")); }));
    CHECK(throws<IoError>([&] { mm::write_complex(dir + "/no/such/dir/x.mtx", Matrix(1, 1)); }));
    CHECK(throws<DimensionMismatch>(
        [&] { mm::write_complex(file("r.mtx"), Matrix(2, 3), mm::Symmetry::Hermitian); }));
  }
  {  // generators (test_gen.cpp cases that do not solve)
    const Matrix q = random_unitary(1, 5);
    CHECK(std::abs(std::abs(q(0, 0)) - 1.0) < 1e-15);
    const Matrix q16 = random_unitary(16, 7);
    double dev = 0.0;
    for (Index j = 0; j < 16; ++j)
      for (Index i = 0; i < 16; ++i) {
        Complex s = 0.0;
        for (Index k = 0; k < 16; ++k) s += std::conj(q16(k, i)) * q16(k, j);
        dev += std::norm(s - (i == j ? 1.0 : 0.0));
      }
    CHECK(std::sqrt(dev) <= 1e-13);
    CHECK(diff(random_unitary(8, 3), random_unitary(8, 3)) == 0.0);
    CHECK(diff(random_unitary(8, 3), random_unitary(8, 4)) > 1e-3);
    CHECK(throws<InvalidSpec>([] { generate_conditioned({8, 2.9999, 0}); }));
    CHECK(throws<InvalidSpec>([] { generate_conditioned({8, 1.0, 0}); }));
    CHECK(!throws<InvalidSpec>([] { generate_conditioned({8, 3.0, 0}); }));
    const BseMatrixI h1 = generate_conditioned({12, 50.0, 9}), h2 = generate_conditioned({12, 50.0, 9});
    CHECK(diff(h1.a(), h2.a()) == 0.0 && diff(h1.b(), h2.b()) == 0.0);
    CHECK(diff(generate_random_definite(5, 1).a(), generate_random_definite(5, 1).a()) == 0.0);
    CHECK(diff(generate_random_definite(5, 1).a(), generate_random_definite(5, 2).a()) > 0.0);
    CHECK(throws<InvalidSpec>([] { generate_random_definite(4, 1, 0.0); }));
    CHECK(splitmix64_at(0, 0) != splitmix64_at(0, 1) && splitmix64_at(0, 0) != splitmix64_at(1, 0));
    GaussianStream g(11, 0);
    double s = 0.0, s2 = 0.0;
    const int n = 20000;
    for (int i = 0; i < n; ++i) {
      const double x = g.next();
      s += x;
      s2 += x * x;
    }
    CHECK(std::abs(s / n) < 0.05 && std::abs(s2 / n - 1.0) < 0.05);
  }
  {  // flop model and presets (test_bench.cpp)
    CHECK(bench::flop_estimate(Method::Chol, 3) == 40.0 * 27.0 / 3.0);
    CHECK(bench::flop_estimate(Method::CholSvd, 300) == 74.0 * 27e6 / 3.0);
    CHECK(bench::flop_model(Method::Sqrt).coeff_num == 86 && bench::flop_model(Method::Reference).coeff_num == 112);
    CHECK(throws<InvalidSpec>([] { bench::flop_estimate(Method::Chol, 0); }));
    const bench::BenchConfig t2 = bench::preset("table2");
    CHECK(t2.sizes == std::vector<Index>{200} && t2.kappas == (std::vector<double>{10.0, 1e3, 1e6, 1e9}));
    CHECK(t2.methods.size() == 4 && t2.seed == 1);
    const bench::BenchConfig f3 = bench::preset("fig3");
    CHECK(f3.kappas.size() == 11 && f3.kappas.front() == 1.0 && f3.kappas.back() == 1e10);
    const bench::BenchConfig f2 = bench::preset("fig2");
    CHECK(f2.repeats == 3 && f2.methods == (std::vector<Method>{Method::Sqrt, Method::Chol, Method::CholSvd}));
    CHECK(throws<InvalidSpec>([] { bench::preset("nope"); }));
    bench::BenchConfig bad;
    CHECK(throws<InvalidSpec>([&] { bench::run_accuracy_experiment(bad); }));
    bad.sizes = {8};
    bad.kappas = {10.0};
    bad.methods = {Method::Chol};
    bad.repeats = 0;
    CHECK(throws<InvalidSpec>([&] { bench::run_runtime_experiment(bad); }));
  }
  std::printf(failures ? "FAILED %d\n" : "OK\n", failures);
  return failures;
}
