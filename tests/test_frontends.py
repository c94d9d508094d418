"""Matrix-Market I/O, generators, bench harness and the `bse` CLI
(include/bse/{mm_io,gen,bench,cli}.hpp; csrc/host/*.cpp), mirroring the reference's
proj/tests/test_mm_io.cpp, test_gen.cpp, test_bench.cpp and cli_tests.cmake.

CPU tests: the host-only C++ checks (tests/cpp/test_frontends.cpp) and every CLI path that
fails before the first device call (usage errors, parse / I/O errors, NotHermitian).
GPU tests: solve / verify / bench through the CLI, and the CSV experiments.
"""
import os
import re
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
PKG = os.path.join(ROOT, "paper_2008_08825_b200")
BSE = os.path.join(PKG, "bin", "bse")


def run(args, cwd, env=None):
    e = dict(os.environ)
    e.pop("BSE_SEED", None)
    e.update(env or {})
    return subprocess.run([BSE] + args, cwd=cwd, capture_output=True, text=True, timeout=600,
                          env=e)


def write(path, body):
    with open(path, "w") as f:
        f.write(body)


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(BSE):
        subprocess.check_call(["make", "-s", "bin/bse"], cwd=PKG)
    return BSE


# ------------------------------------------------------------------ CPU
def test_frontends_host_cpp(tmp_path):
    exe = tmp_path / "test_frontends"
    subprocess.check_call(["g++", "-std=c++17", f"-I{ROOT}/include",
                           os.path.join(HERE, "cpp", "test_frontends.cpp"), f"-L{PKG}",
                           "-lbse_b200", f"-Wl,-rpath,{PKG}", "-o", str(exe)])
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


def test_cli_usage_errors(cli, tmp_path):
    assert run([], tmp_path).returncode == 2
    assert run(["solve", "--definitely-not-a-flag"], tmp_path).returncode == 2
    assert run(["nope"], tmp_path).returncode == 2
    assert run(["solve", "--method", "qr", "--a", "a", "--b", "b"], tmp_path).returncode == 2
    assert run(["generate", "--n", "4", "--seed", "1", "--a", "x.mtx", "--b", "y.mtx"],
               tmp_path).returncode == 2  # no --kappa and no --random-definite
    assert run(["bench", "--sizes", "8"], tmp_path).returncode == 2  # no experiment selection
    h = run(["--help"], tmp_path)
    assert h.returncode == 0 and "Exit codes" in h.stdout and "13 ParseError" in h.stdout


def test_cli_host_side_errors(cli, tmp_path):
    write(tmp_path / "broken.mtx", "%%MatrixMarket matrix array real general\n2 2\n1.0\n")
    r = run(["solve", "--method", "chol", "--a", "broken.mtx", "--b", "broken.mtx"], tmp_path)
    assert r.returncode == 13 and "error: ParseError: broken.mtx:3:" in r.stderr
    r = run(["solve", "--method", "chol", "--a", "missing.mtx", "--b", "missing.mtx"], tmp_path)
    assert r.returncode == 14 and "error: IoError" in r.stderr
    write(tmp_path / "nh.mtx", "%%MatrixMarket matrix array real general\n2 2\n0.0\n1.0\n0.0\n0.0\n")
    write(tmp_path / "z2.mtx", "%%MatrixMarket matrix array real general\n2 2\n0.0\n0.0\n0.0\n0.0\n")
    r = run(["solve", "--method", "chol", "--a", "nh.mtx", "--b", "z2.mtx"], tmp_path)
    assert r.returncode == 4 and "error: NotHermitian" in r.stderr
    write(tmp_path / "one.mtx", "%%MatrixMarket matrix array real general\n1 1\n1.0\n")
    r = run(["solve", "--method", "chol", "--a", "one.mtx", "--b", "z2.mtx"], tmp_path)
    assert r.returncode == 3 and "error: DimensionMismatch" in r.stderr
    write(tmp_path / "cfg.json", '{"experiment": "accuracy", "sizes": [8,')
    r = run(["bench", "--config", "cfg.json"], tmp_path)
    assert r.returncode == 13 and "error: ParseError" in r.stderr


def test_cli_generate_files(cli, tmp_path):
    r = run(["generate", "--n", "12", "--kappa", "50", "--seed", "3", "--a", "g_a.mtx", "--b",
             "g_b.mtx"], tmp_path)
    assert r.returncode == 0 and "(n = 12)" in r.stdout
    with open(tmp_path / "g_a.mtx") as f:
        assert f.readline().strip() == "%%MatrixMarket matrix array complex hermitian"
    # BSE_SEED is the --seed fallback; the same seed gives the same bytes
    r2 = run(["generate", "--n", "12", "--kappa", "50", "--a", "e_a.mtx", "--b", "e_b.mtx"],
             tmp_path, env={"BSE_SEED": "3"})
    assert r2.returncode == 0
    assert open(tmp_path / "g_a.mtx").read() == open(tmp_path / "e_a.mtx").read()
    r3 = run(["generate", "--n", "5", "--random-definite", "--seed", "1", "--a", "x.bin", "--b",
              "y.bin"], tmp_path)
    assert r3.returncode == 0 and os.path.getsize(tmp_path / "x.bin") == 32 + 25 * 16
    r4 = run(["generate", "--n", "8", "--kappa", "2", "--a", "k_a.mtx", "--b", "k_b.mtx"], tmp_path)
    assert r4.returncode == 12 and "error: InvalidSpec" in r4.stderr


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_cli_solve_canonical_and_errors(cli, tmp_path):
    write(tmp_path / "a.mtx", "%%MatrixMarket matrix array real general\n1 1\n2.0\n")
    write(tmp_path / "b.mtx", "%%MatrixMarket matrix array real general\n1 1\n1.0\n")
    r = run(["solve", "--method", "chol-svd", "--a", "a.mtx", "--b", "b.mtx"], tmp_path)
    assert r.returncode == 0, r.stderr
    assert re.search(r"1\.7320508", r.stdout)
    assert (tmp_path / "eigenvalues.mtx").exists() and (tmp_path / "eigenvectors.mtx").exists()
    write(tmp_path / "bad_b.mtx", "%%MatrixMarket matrix array real general\n1 1\n3.0\n")
    r = run(["solve", "--method", "chol", "--a", "a.mtx", "--b", "bad_b.mtx"], tmp_path)
    assert r.returncode == 5 and "error: NotDefinite" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["sqrt", "chol", "chol-svd", "reference"])
def test_cli_generate_solve_verify_round_trip(cli, tmp_path, method):
    assert run(["generate", "--n", "12", "--kappa", "50", "--seed", "3", "--a", "g_a.mtx", "--b",
                "g_b.mtx"], tmp_path).returncode == 0
    r = run(["solve", "--method", method, "--a", "g_a.mtx", "--b", "g_b.mtx", "--negative",
             "--out-values", "vals.mtx", "--out-vectors", "vecs.mtx"], tmp_path)
    assert r.returncode == 0, r.stderr
    res = float(re.search(r"max residual: (\S+)", r.stdout).group(1))
    assert res <= 100 * 24 * 2.2e-16
    v = run(["verify", "--a", "g_a.mtx", "--b", "g_b.mtx"], tmp_path)
    assert v.returncode == 0 and "check_form1: pass" in v.stdout
    v = run(["verify", "--a", "g_a.mtx", "--b", "g_b.mtx", "--values", "vals.mtx", "--vectors",
             "vecs.mtx"], tmp_path)
    assert v.returncode == 0 and "columns: 24" in v.stdout
    assert float(re.search(r"max residual: (\S+)", v.stdout).group(1)) <= 100 * 24 * 2.2e-16
    # the binary container carries the same solve bit-for-bit
    assert run(["generate", "--n", "12", "--kappa", "50", "--seed", "3", "--a", "g_a.bin", "--b",
                "g_b.bin"], tmp_path).returncode == 0
    rb = run(["solve", "--method", method, "--a", "g_a.bin", "--b", "g_b.bin", "--out-values",
              "vals.bin", "--out-vectors", "vecs.bin"], tmp_path)
    assert rb.returncode == 0
    first = lambda out: re.search(r"eigenvalues \(ascending\):(.*)", out).group(1)  # noqa: E731
    assert first(rb.stdout) == first(r.stdout)


def _rows(csv_text):
    return [line.split(",") for line in csv_text.strip().splitlines()]


@pytest.mark.gpu
def test_cli_bench_accuracy_deterministic(cli, tmp_path):
    args = ["bench", "--preset", "table2", "--seed", "9", "--sizes", "24", "--kappas", "10",
            "1000", "--methods", "chol", "chol-svd"]
    assert run(args + ["--out", "run1.csv"], tmp_path).returncode == 0
    assert run(args + ["--out", "run2.csv"], tmp_path).returncode == 0
    r1 = _rows(open(tmp_path / "run1.csv").read())
    r2 = _rows(open(tmp_path / "run2.csv").read())
    assert r1[0] == ["method", "n", "kappa", "rel_err_min_eig", "runtime_s", "seed", "status"]
    assert len(r1) == 5
    for a, b in zip(r1[1:], r2[1:]):
        assert a[:4] + a[5:] == b[:4] + b[5:]  # every column but the timing
        assert a[6] == "ok" and float(a[3]) < 1e-9


@pytest.mark.gpu
def test_cli_bench_sigma_runtime_and_config(cli, tmp_path):
    r = run(["bench", "--experiment", "sigma", "--sizes", "16", "--kappas", "1", "10",
             "--methods", "chol-svd", "--seed", "2"], tmp_path)
    rows = _rows(r.stdout)
    assert rows[0] == ["method", "n", "kappa", "sigma_dev", "seed", "status"]
    assert rows[1][5] == "InvalidSpec" and rows[1][3] == "nan"  # kappa = 1 is not in the family
    assert rows[2][5] == "ok" and float(rows[2][3]) < 1e-11
    write(tmp_path / "cfg.json", '{"experiment": "runtime", "sizes": [8, 16], '
                                 '"methods": ["sqrt", "chol"], "repeats": 3, "seed": 6}')
    r = run(["bench", "--config", "cfg.json", "--out", "rt.csv"], tmp_path)
    assert r.returncode == 0, r.stderr
    rows = _rows(open(tmp_path / "rt.csv").read())
    assert rows[0] == ["method", "n", "median_runtime_s", "repeats", "status"]
    assert len(rows) == 5
    assert all(row[3] == "3" and row[4] == "ok" and float(row[2]) >= 0.0 for row in rows[1:])
