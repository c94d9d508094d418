// cli.cpp — the `bse` command-line tool (surface of proj/src/cli.cpp:1-335:
// subcommands generate / solve / verify / bench, their options, the BSE_SEED fallback, the
// exit-code table and the `error: <Kind>: <detail>` line). Own small argument parser and a
// minimal JSON reader for `bench --config` (the reference links CLI11 and nlohmann::json).
#include "bse/cli.hpp"

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <vector>

#include "bse/bench.hpp"
#include "bse/gen.hpp"
#include "bse/mm_io.hpp"
#include "bse/solvers.hpp"
#include "bse/types.hpp"
#include "bse/verify.hpp"

namespace bse::cli {

namespace {

struct Usage : std::runtime_error {  // exit code 2
  using std::runtime_error::runtime_error;
};

int exit_code(const Error& e) {
  if (dynamic_cast<const DimensionMismatch*>(&e)) return 3;
  if (dynamic_cast<const NotHermitian*>(&e)) return 4;
  if (dynamic_cast<const NotDefinite*>(&e)) return 5;
  if (dynamic_cast<const NotPositiveDefinite*>(&e)) return 6;
  if (dynamic_cast<const ConvergenceFailure*>(&e)) return 7;
  if (dynamic_cast<const SingularFactor*>(&e)) return 8;
  if (dynamic_cast<const NonPositiveScale*>(&e)) return 9;
  if (dynamic_cast<const OddDimension*>(&e)) return 10;
  if (dynamic_cast<const LengthMismatch*>(&e)) return 11;
  if (dynamic_cast<const InvalidSpec*>(&e)) return 12;
  if (dynamic_cast<const ParseError*>(&e)) return 13;
  if (dynamic_cast<const IoError*>(&e)) return 14;
  return 1;
}

std::string g17(double x) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", x);
  return buf;
}

const char* kHelp = R"(bse — dense structured eigensolvers and benchmarks for BSE matrices of form I
(B200 GPU implementation)

Usage:
  bse generate --n N (--kappa K | --random-definite) [--seed S] [--shift-margin M] --a A --b B
  bse solve --method {sqrt,chol,chol-svd,reference} --a A --b B [--negative]
            [--out-values FILE] [--out-vectors FILE]
  bse verify --a A --b B [--values FILE --vectors FILE] [--tol T]
  bse bench (--preset {table2,fig3,fig2} | --experiment {accuracy,sigma,runtime} | --config JSON)
            [--sizes N...] [--kappas K...] [--methods M...] [--repeats R] [--seed S] [--out CSV]
  --seed falls back to the BSE_SEED environment variable.

File formats:
  Matrices are Matrix Market files (dense `array` or sparse `coordinate`, real or complex,
  general/symmetric/hermitian), written with 17 significant digits so save -> load round
  trips are bit-exact. Paths ending in ".bin" use the raw BSEMAT01 container instead
  (for large n).

Exit codes:
  0 success                  7 ConvergenceFailure
  2 usage error              8 SingularFactor
  3 DimensionMismatch        9 NonPositiveScale
  4 NotHermitian            10 OddDimension
  5 NotDefinite             11 LengthMismatch
  6 NotPositiveDefinite     12 InvalidSpec
                            13 ParseError
                            14 IoError
On failure a machine-readable line `error: <Kind>: <detail>` is printed to standard error.
)";

// ---------------------------------------------------------------- argument parsing
// Options are `--name value`, `--name v1 v2 ...` (multi) or bare flags.
struct Spec {
  std::set<std::string> single, multi, flags;
};

struct Parsed {
  std::map<std::string, std::vector<std::string>> opt;
  bool has(const std::string& k) const { return opt.count(k) > 0; }
  const std::string& one(const std::string& k) const { return opt.at(k).front(); }
};

Parsed parse(int argc, char** argv, int first, const Spec& spec) {
  Parsed p;
  for (int i = first; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("--", 0) != 0) throw Usage("unexpected argument '" + a + "'");
    const std::string k = a.substr(2);
    if (spec.flags.count(k)) {
      p.opt[k] = {};
      continue;
    }
    const bool multi = spec.multi.count(k) > 0;
    if (!multi && !spec.single.count(k)) throw Usage("unknown option '" + a + "'");
    if (p.has(k)) throw Usage("option '" + a + "' given twice");
    std::vector<std::string> vals;
    while (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) {
      vals.push_back(argv[++i]);
      if (!multi) break;
    }
    if (vals.empty()) throw Usage("option '" + a + "' needs a value");
    p.opt[k] = vals;
  }
  return p;
}

void require(const Parsed& p, const std::string& k) {
  if (!p.has(k)) throw Usage("--" + k + " is required");
}

template <typename T>
T to_num(const std::string& s, const std::string& what) {
  std::istringstream ss(s);
  T v{};
  if (!(ss >> v) || !ss.eof()) throw Usage("invalid value '" + s + "' for --" + what);
  return v;
}

void check_member(const std::string& v, const std::set<std::string>& ok, const std::string& opt) {
  if (!ok.count(v)) throw Usage("--" + opt + ": '" + v + "' is not one of the allowed values");
}

bool seed_from(const Parsed& p, std::uint64_t& seed) {
  if (p.has("seed")) {
    seed = to_num<std::uint64_t>(p.one("seed"), "seed");
    return true;
  }
  if (const char* env = std::getenv("BSE_SEED")) {
    seed = to_num<std::uint64_t>(env, "seed (BSE_SEED)");
    return true;
  }
  return false;
}

// ---------------------------------------------------------------- minimal JSON (bench --config)
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
};

class JsonReader {
 public:
  JsonReader(const std::string& text, const std::string& path) : t_(text), path_(path) {}
  Json document() {
    Json v = value();
    ws();
    if (p_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& m) const {
    throw ParseError(path_ + ": " + m + " at offset " + std::to_string(p_), 0);
  }
  void ws() {
    while (p_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[p_]))) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < t_.size() && t_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  std::string string_lit() {
    if (!eat('"')) fail("expected a string");
    std::string s;
    while (p_ < t_.size() && t_[p_] != '"') {
      if (t_[p_] == '\\') {
        if (++p_ >= t_.size()) break;
        const char e = t_[p_];
        s += e == 'n' ? '\n' : e == 't' ? '\t' : e;
      } else {
        s += t_[p_];
      }
      ++p_;
    }
    if (p_ >= t_.size()) fail("unterminated string");
    ++p_;
    return s;
  }
  Json value() {
    ws();
    if (p_ >= t_.size()) fail("unexpected end of input");
    Json v;
    const char c = t_[p_];
    if (c == '{') {
      ++p_;
      v.kind = Json::Obj;
      if (eat('}')) return v;
      do {
        const std::string k = string_lit();
        if (!eat(':')) fail("expected ':'");
        v.obj[k] = value();
      } while (eat(','));
      if (!eat('}')) fail("expected '}'");
    } else if (c == '[') {
      ++p_;
      v.kind = Json::Arr;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      if (!eat(']')) fail("expected ']'");
    } else if (c == '"') {
      v.kind = Json::Str;
      v.str = string_lit();
    } else if (t_.compare(p_, 4, "true") == 0 || t_.compare(p_, 5, "false") == 0) {
      v.kind = Json::Bool;
      v.b = t_[p_] == 't';
      p_ += v.b ? 4 : 5;
    } else if (t_.compare(p_, 4, "null") == 0) {
      p_ += 4;
    } else {
      const char* s = t_.c_str() + p_;
      char* end = nullptr;
      v.num = std::strtod(s, &end);
      if (end == s) fail("unexpected character");
      v.kind = Json::Num;
      p_ += size_t(end - s);
    }
    return v;
  }
  const std::string& t_;
  std::string path_;
  size_t p_ = 0;
};

const Json& expect(const Json& j, Json::Kind k, const std::string& key, const std::string& path) {
  if (j.kind != k) throw ParseError(path + ": key '" + key + "' has the wrong type", 0);
  return j;
}

// ---------------------------------------------------------------- subcommands
int do_generate(const Parsed& p) {
  require(p, "n");
  require(p, "a");
  require(p, "b");
  const bool rnd = p.has("random-definite");
  if (!rnd && !p.has("kappa")) throw Usage("--kappa is required (unless --random-definite)");
  std::uint64_t seed = 0;
  seed_from(p, seed);
  const Index n = to_num<Index>(p.one("n"), "n");
  const BseMatrixI h =
      rnd ? generate_random_definite(
                n, seed, p.has("shift-margin") ? to_num<double>(p.one("shift-margin"), "shift-margin") : 1.0)
          : generate_conditioned({n, to_num<double>(p.one("kappa"), "kappa"), seed});
  bench::save_matrix_pair(h, p.one("a"), p.one("b"));
  std::cout << "wrote " << p.one("a") << " and " << p.one("b") << " (n = " << h.n() << ")\n";
  return 0;
}

int do_solve(const Parsed& p) {
  require(p, "method");
  require(p, "a");
  require(p, "b");
  check_member(p.one("method"), {"sqrt", "chol", "chol-svd", "reference"}, "method");
  const std::string out_values = p.has("out-values") ? p.one("out-values") : "eigenvalues.mtx";
  const std::string out_vectors = p.has("out-vectors") ? p.one("out-vectors") : "eigenvectors.mtx";
  const BseMatrixI h = bench::load_matrix_pair(p.one("a"), p.one("b"));
  const Method method = method_from_name(p.one("method"));
  const SpectralResult r = solve(method, h);
  SpectralResult full = r;  // positive half, then (--negative) the mirrored half
  if (p.has("negative")) {
    const SpectralResult neg = negative_spectrum(h, r);
    const Index n2 = r.v.rows(), k = r.v.cols();
    full.lambda.insert(full.lambda.end(), neg.lambda.begin(), neg.lambda.end());
    full.v = Matrix(n2, 2 * k);
    for (Index j = 0; j < k; ++j)
      for (Index i = 0; i < n2; ++i) {
        full.v(i, j) = r.v(i, j);
        full.v(i, k + j) = neg.v(i, j);
      }
  }
  if (mm::is_binary_path(out_values)) mm::write_binary(out_values, RealMatrix(full.lambda));
  else mm::write_real(out_values, RealMatrix(full.lambda));
  if (mm::is_binary_path(out_vectors)) mm::write_binary(out_vectors, full.v);
  else mm::write_complex(out_vectors, full.v);

  std::cout << "method: " << method_name(method) << "\nn: " << h.n() << "\neigenvalues (ascending):";
  const size_t shown = std::min<size_t>(r.lambda.size(), 8);
  for (size_t i = 0; i < shown; ++i) std::cout << " " << g17(r.lambda[i]);
  if (shown < r.lambda.size()) std::cout << " ...";
  std::cout << "\n";
  const RealVector res = residual(h, full);
  double rmax = 0.0;
  for (double x : res) rmax = std::max(rmax, x);
  std::cout << "max residual: " << g17(rmax) << "\n";
  std::cout << "sigma_dev: " << g17(sigma_orthogonality_error(r.v)) << "\n";
  if (!r.near_singular.empty())
    std::cout << "near-singular eigenvalues clamped: " << r.near_singular.size() << "\n";
  std::cout << "wrote " << out_values << " and " << out_vectors << "\n";
  return 0;
}

int do_verify(const Parsed& p) {
  require(p, "a");
  require(p, "b");
  const double tol = p.has("tol") ? to_num<double>(p.one("tol"), "tol") : 1e-12;
  const BseMatrixI h = bench::load_matrix_pair(p.one("a"), p.one("b"));
  const Matrix full = realize_full(h);
  const bool f1 = check_form1(full, tol), f2 = check_form2(full, tol);
  std::cout << "check_form1: " << (f1 ? "pass" : "fail") << "\n";
  std::cout << "check_form2: " << (f2 ? "pass" : "fail") << "\n";
  if (p.has("values") && p.has("vectors")) {
    const RealMatrix vals = mm::read_real(p.one("values"));
    SpectralResult r;
    r.lambda = vals.col(0);
    r.v = mm::read_complex(p.one("vectors"));
    const RealVector res = residual(h, r);
    double rmax = 0.0;
    for (double x : res) rmax = std::max(rmax, x);
    std::cout << "columns: " << r.v.cols() << "\n";
    std::cout << "max residual: " << g17(rmax) << "\n";
    std::cout << "sigma_dev: " << g17(sigma_orthogonality_error(r.v)) << "\n";
  }
  return 0;
}

int do_bench(const Parsed& p) {
  const std::set<std::string> methods{"sqrt", "chol", "chol-svd", "reference"};
  if (!p.has("preset") && !p.has("experiment") && !p.has("config"))
    throw Usage("one of --preset, --experiment or --config is required");
  bench::BenchConfig cfg;
  std::string experiment;
  if (p.has("preset")) {
    const std::string name = p.one("preset");
    check_member(name, {"table2", "fig3", "fig2"}, "preset");
    cfg = bench::preset(name);
    experiment = name == "table2" ? "accuracy" : name == "fig3" ? "sigma" : "runtime";
  }
  if (p.has("experiment")) {
    check_member(p.one("experiment"), {"accuracy", "sigma", "runtime"}, "experiment");
    experiment = p.one("experiment");
  }
  if (p.has("config")) {
    const std::string path = p.one("config");
    std::ifstream f(path);
    if (!f) throw IoError("cannot open config file " + path);
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string text = ss.str();
    const Json j = JsonReader(text, path).document();
    if (j.kind != Json::Obj) throw ParseError(path + ": the config must be a JSON object", 0);
    for (const auto& [k, v] : j.obj) {
      if (k == "experiment") {
        experiment = expect(v, Json::Str, k, path).str;
      } else if (k == "sizes" || k == "kappas") {
        expect(v, Json::Arr, k, path);
        if (k == "sizes") cfg.sizes.clear();
        else cfg.kappas.clear();
        for (const Json& e : v.arr) {
          expect(e, Json::Num, k, path);
          if (k == "sizes") cfg.sizes.push_back(static_cast<Index>(e.num));
          else cfg.kappas.push_back(e.num);
        }
      } else if (k == "methods") {
        expect(v, Json::Arr, k, path);
        cfg.methods.clear();
        for (const Json& e : v.arr) cfg.methods.push_back(method_from_name(expect(e, Json::Str, k, path).str));
      } else if (k == "repeats") {
        cfg.repeats = static_cast<int>(expect(v, Json::Num, k, path).num);
      } else if (k == "seed") {
        cfg.seed = static_cast<std::uint64_t>(expect(v, Json::Num, k, path).num);
      } else if (k == "out") {
        cfg.output_path = expect(v, Json::Str, k, path).str;
      }
    }
  }
  if (p.has("sizes")) {
    cfg.sizes.clear();
    for (const auto& s : p.opt.at("sizes")) cfg.sizes.push_back(to_num<Index>(s, "sizes"));
  }
  if (p.has("kappas")) {
    cfg.kappas.clear();
    for (const auto& s : p.opt.at("kappas")) cfg.kappas.push_back(to_num<double>(s, "kappas"));
  }
  if (p.has("methods")) {
    cfg.methods.clear();
    for (const auto& s : p.opt.at("methods")) {
      check_member(s, methods, "methods");
      cfg.methods.push_back(method_from_name(s));
    }
  }
  if (p.has("repeats")) {
    const int r = to_num<int>(p.one("repeats"), "repeats");
    if (r > 0) cfg.repeats = r;
  }
  std::uint64_t seed = 0;
  if (seed_from(p, seed)) cfg.seed = seed;
  if (p.has("out")) cfg.output_path = p.one("out");

  std::string csv;
  if (experiment == "accuracy") csv = bench::run_accuracy_experiment(cfg);
  else if (experiment == "sigma") csv = bench::run_sigma_experiment(cfg);
  else if (experiment == "runtime") csv = bench::run_runtime_experiment(cfg);
  else if (experiment.empty()) throw InvalidSpec("bench: the config file names no experiment");
  else throw InvalidSpec("unknown experiment '" + experiment + "'");
  if (cfg.output_path.empty()) {
    std::cout << csv;
  } else {
    std::ofstream out(cfg.output_path);
    if (!out) throw IoError("cannot open " + cfg.output_path + " for writing");
    out << csv;
    std::cout << "wrote " << cfg.output_path << "\n";
  }
  return 0;
}

}  // namespace

int run(int argc, char** argv) {
  try {
    if (argc < 2) throw Usage("a subcommand is required (generate, solve, verify, bench)");
    const std::string cmd = argv[1];
    for (int i = 1; i < argc; ++i) {
      const std::string a = argv[i];
      if (a == "--help" || a == "-h") {
        std::cout << kHelp;
        return 0;
      }
    }
    if (cmd == "generate")
      return do_generate(parse(argc, argv, 2, {{"n", "kappa", "seed", "shift-margin", "a", "b"}, {}, {"random-definite"}}));
    if (cmd == "solve")
      return do_solve(parse(argc, argv, 2, {{"method", "a", "b", "out-values", "out-vectors"}, {}, {"negative"}}));
    if (cmd == "verify")
      return do_verify(parse(argc, argv, 2, {{"a", "b", "values", "vectors", "tol"}, {}, {}}));
    if (cmd == "bench")
      return do_bench(parse(argc, argv, 2,
                            {{"preset", "experiment", "repeats", "seed", "out", "config"},
                             {"sizes", "kappas", "methods"}, {}}));
    throw Usage("unknown subcommand '" + cmd + "'");
  } catch (const Usage& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return 2;
  } catch (const Error& e) {
    std::cerr << "error: " << error_kind(e) << ": " << e.what() << "\n";
    return exit_code(e);
  } catch (const std::exception& e) {
    std::cerr << "error: Internal: " << e.what() << "\n";
    return 1;
  }
}

}  // namespace bse::cli
