"""The hsolve_bench command line and the bench harness (reference
cli.cpp:220-291, bench.cpp:51-195), after proj/tests/test_cli.cpp: usage
errors exit 2 (CPU), gen / solve / sweep / --config on the GPU."""
import os
import subprocess

import pytest

import paper_2605_13209_b200 as hs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2605_13209_b200", "bin", "hsolve_bench")

REFERENCE_COLUMNS = (
    "algo,n,block_size,fraction,workers_a,workers_b,slowdown_a,slowdown_b,reps,"
    "runtime_ms_median,runtime_ms_mean,compute_ms_median,iters,recomputes,true_residual,"
    "bytes_total,bytes_scalar,bytes_subvector,bytes_block,bytes_block_row,border_shifts,"
    "status,seed").split(",")


def run(*args, timeout=600):
    if not os.path.exists(BIN):
        pytest.skip("hsolve_bench not built")
    p = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout, p.stderr


def csv_rows(path):
    lines = open(path).read().splitlines()
    head = lines[0].split(",")
    rows = [dict(zip(head, ln.split(","))) for ln in lines[1:] if not ln.startswith("#")]
    return lines, head, rows


@pytest.mark.parametrize("args", [
    ["solve", "cg", "--size", "64", "--fraction", "1.5"],
    ["solve", "banana", "--size", "64"],
    ["solve", "cg"],                       # neither --matrix nor --size
    ["nonsense"],
    [],
    ["sweep", "--sizes", "64", "--fractions", ""],
    ["sweep", "--sizes", "64", "--fractions", "zero"],
    ["sweep", "--sizes", "x,y", "--fractions", "0.5"],
    ["gen", "--size", "32"],               # missing --output
    ["solve", "cg", "--size", "sixty"],
    ["solve", "cg", "--size", "64", "--bogus", "1"],
    ["solve", "cg", "--size", "64", "--workers-a", "0"],
    ["solve", "cg", "--size", "64", "--eps", "-1"],
    ["solve", "cg", "--size", "64", "--config", "/tmp/hsolve_no_such.ini"],
])
def test_usage_errors_exit_2(args):
    # test_cli.cpp:54-63 (+ parse errors the reference gets from CLI11)
    code, _, err = run(*args)
    assert code == 2, (args, err)
    assert "error" in err


def test_help_exits_0():
    code, out, _ = run("--help")
    assert code == 0 and "gen" in out and "sweep" in out


def test_csv_header_keeps_reference_columns_first():
    # the reference schema (bench.cpp csv_header) unchanged, GPU columns after
    code, out, _ = run("solve", "cg", "--size", "64", "--fraction", "1.5")
    src = open(os.path.join(ROOT, "paper_2605_13209_b200", "host", "bench.cpp")).read()
    for c in REFERENCE_COLUMNS:
        assert f'"{c}"' in src


@pytest.mark.gpu
def test_gen_writes_loadable_bspd1(tmp_path):
    # test_cli.cpp:65-73
    p = str(tmp_path / "g.bspd")
    code, _, err = run("gen", "--size", "48", "--block-size", "8", "--seed", "7",
                       "--output", p)
    assert code == 0, err
    m = hs.load_matrix(p)
    assert (m.n, m.b) == (48, 8)
    ref = hs.generate_spd(48, 8, seed=7)
    assert m.values.tobytes() == ref.values.tobytes()


@pytest.mark.gpu
def test_solve_emits_one_row(tmp_path):
    # test_cli.cpp:75-87
    out = str(tmp_path / "o.csv")
    code, _, err = run("solve", "cg", "--size", "96", "--block-size", "16", "--fraction",
                       "0.85", "--eps", "1e-6", "--reps", "2", "--output", out)
    assert code == 0, err
    lines, head, rows = csv_rows(out)
    assert len(lines) == 2
    assert head[:len(REFERENCE_COLUMNS)] == REFERENCE_COLUMNS
    r = rows[0]
    assert (r["status"], r["algo"], r["n"], r["fraction"]) == ("converged", "cg", "96", "0.85")
    assert float(r["iters_per_s"]) > 0 and r["gpus"] == "1"


@pytest.mark.gpu
def test_solve_on_saved_matrix(tmp_path):
    # test_cli.cpp:89-101
    p, out = str(tmp_path / "m.bspd"), str(tmp_path / "o.csv")
    assert run("gen", "--size", "64", "--block-size", "16", "--output", p)[0] == 0
    code, _, err = run("solve", "cholesky", "--matrix", p, "--fraction", "0.5", "--reps",
                       "1", "--output", out)
    assert code == 0, err
    _, _, rows = csv_rows(out)
    assert rows[0]["status"] == "ok" and rows[0]["block_size"] == "16"
    assert float(rows[0]["true_residual"]) < 1e-9
    assert float(rows[0]["gflops"]) > 0


@pytest.mark.gpu
def test_non_timing_columns_bit_identical(tmp_path):
    # test_cli.cpp:103-124
    out = str(tmp_path / "o.csv")
    args = ["solve", "cg", "--size", "96", "--block-size", "16", "--fraction", "0.75",
            "--reps", "2", "--seed", "9", "--output", out]
    assert run(*args)[0] == 0
    _, head, first = csv_rows(out)
    assert run(*args)[0] == 0
    _, _, second = csv_rows(out)
    timing = {"runtime_ms_median", "runtime_ms_mean", "compute_ms_median",
              "factor_ms_median", "solve_ms_median", "iters_per_s", "gflops"}
    for c in head:
        if c not in timing:
            assert first[0][c] == second[0][c], c


@pytest.mark.gpu
def test_homogeneous_endpoints_zero_traffic(tmp_path):
    # test_cli.cpp:126-138 (a single-GPU run issues no collectives)
    out = str(tmp_path / "o.csv")
    for f in ("0.0", "1.0"):
        assert run("solve", "cholesky", "--size", "64", "--block-size", "16", "--fraction",
                   f, "--reps", "1", "--output", out)[0] == 0
        _, _, rows = csv_rows(out)
        for c in ("bytes_total", "bytes_scalar", "bytes_subvector", "border_shifts"):
            assert rows[0][c] == "0", c


@pytest.mark.gpu
def test_reps1_median_equals_mean(tmp_path):
    out = str(tmp_path / "o.csv")
    assert run("solve", "cg", "--size", "64", "--block-size", "16", "--fraction", "0.5",
               "--reps", "1", "--output", out)[0] == 0
    _, _, rows = csv_rows(out)
    assert rows[0]["runtime_ms_median"] == rows[0]["runtime_ms_mean"]


@pytest.mark.gpu
def test_sweep_grid_and_summary(tmp_path):
    # test_cli.cpp:149-171
    out = str(tmp_path / "o.csv")
    code, _, err = run("sweep", "--sizes", "64", "--block-sizes", "16", "--fractions",
                       "0.0:1.0:0.5", "--reps", "1", "--summary", "--output", out)
    assert code == 0, err
    lines = open(out).read().splitlines()
    assert len(lines) == 1 + 6 + 2
    body = [ln for ln in lines[1:] if not ln.startswith("# argmin")]
    assert sum(ln.startswith("cg,") for ln in body) == 3
    assert sum(ln.startswith("cholesky,") for ln in body) == 3
    assert sum(ln.startswith("# argmin") for ln in lines) == 2


@pytest.mark.gpu
def test_sweep_records_failing_row(tmp_path):
    # test_cli.cpp:173-185
    out = str(tmp_path / "o.csv")
    code, _, _ = run("sweep", "--sizes", "32", "--block-sizes", "8", "--fractions", "0.5",
                     "--reps", "1", "--max-iters", "1", "--eps", "1e-15", "--output", out)
    assert code == 1
    _, _, rows = csv_rows(out)
    assert [r["status"] for r in rows] == ["not_converged", "ok"]


@pytest.mark.gpu
def test_config_file_defaults_and_override(tmp_path):
    # test_cli.cpp:187-206
    cfg, out = str(tmp_path / "c.ini"), str(tmp_path / "o.csv")
    open(cfg, "w").write("[solve]\nsize=96\nblock-size=16\nfraction=0.5\nreps=1\n")
    code, _, err = run("solve", "cg", "--config", cfg, "--fraction", "0.25", "--output", out)
    assert code == 0, err
    _, _, rows = csv_rows(out)
    assert rows[0]["n"] == "96" and rows[0]["fraction"] == "0.25"


@pytest.mark.gpu
def test_solve_cholesky_with_int8_emulation(tmp_path):
    out = str(tmp_path / "o.csv")
    code, _, err = run("solve", "cholesky", "--size", "1024", "--block-size", "128",
                       "--reps", "1", "--fp64-emulation-slices", "8", "--output", out)
    assert code == 0, err
    _, _, rows = csv_rows(out)
    assert rows[0]["status"] == "ok" and float(rows[0]["true_residual"]) < 1e-9
    assert run("solve", "cholesky", "--size", "64", "--fp64-emulation-slices", "9")[0] == 2
