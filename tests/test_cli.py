"""The sssvd-gpu command line, re-expressing proj/tests/test_cli.cpp:
subcommands, report schema v1, triplet/filter CSV layouts and exit codes. Host-only
subcommands and configuration errors run on CPU; solve / verify / bench need the B200."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import sssvd_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2109_13655_b200", "sssvd-gpu")


def run_cli(args, cwd=None, timeout=600):
    p = subprocess.run([CLI] + args.split(), capture_output=True, text=True, cwd=cwd, timeout=timeout)
    return p.returncode, p.stdout, p.stderr


def test_cli_built():
    assert os.access(CLI, os.X_OK)
    rc, out, _ = run_cli("--help")
    assert rc == 0 and "filter-plot" in out


def test_configuration_errors_exit_2():                                  # test_cli.cpp:84-91
    assert run_cli("solve --model 1 --interval 1.2 0.8 --mode ss-svd")[0] == 2      # a > b
    assert run_cli("solve --model 1 --interval 0.8 1.2 --N 31")[0] == 2             # odd N
    assert run_cli("solve --model 2 --interval 0 0.1 --mode ss-svd-nt")[0] == 2     # a = 0 with exp
    assert run_cli("solve --model 1 --interval 0.8 1.2 --L 80")[0] == 2             # L*M > n
    assert run_cli("solve --input /does/not/exist.mtx --interval 0.8 1.2")[0] != 0


def test_parse_errors_use_cli11_codes():
    assert run_cli("")[0] == 106
    assert run_cli("solve --bogus 1")[0] == 109
    assert run_cli("solve --model 1 --L x")[0] == 104
    assert run_cli("solve --model 3")[0] == 105


def test_bad_input_file_exits_2(tmp_path):
    p = tmp_path / "bad.mtx"
    p.write_text("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n")
    rc, _, err = run_cli(f"solve --input {p} --interval 0.8 1.2")
    assert rc == 2 and "unsupported field" in err


def test_model_writes_mtx_and_truth(tmp_path):                           # test_cli.cpp:93-105 (first half)
    prefix = str(tmp_path / "m1")
    assert run_cli(f"model --which 1 --rows 120 --cols 40 --out {prefix}")[0] == 0
    from paper_2109_13655_b200 import sssvd
    a = sssvd.read_matrix_market(prefix + ".mtx")
    assert not a.is_sparse() and (a.rows(), a.cols()) == (120, 40)
    truth = np.loadtxt(prefix + ".truth.csv", delimiter=",", skiprows=1)[:, 1]
    assert np.array_equal(truth, orc.model_spectrum(1, 40))
    ref, *_ = orc.build_model(1, 120, 40, 7)                     # same normal stream, Householder Q
    assert np.max(np.abs(a.dense() - ref.dense)) <= 1e-14
    assert np.max(np.abs(np.linalg.svd(a.dense(), compute_uv=False)[::-1] - truth)) <= 1e-14
    assert open(prefix + ".mtx").read().splitlines()[1] == "% model 1 seed 7"


def test_filter_plot_csv(tmp_path):                                      # test_cli.cpp:107-127
    prefix = str(tmp_path / "f")
    rc, _, _ = run_cli(f"filter-plot --interval 1e-3 1e-1 --transform exp --log --points 40 "
                       f"--sigma-min 1e-6 --sigma-max 1 --out {prefix}")
    assert rc == 0
    lines = open(prefix + ".filter.csv").read().splitlines()
    assert lines[0].startswith("# interval=") and "transform=exp" in lines[0]
    assert lines[1] == "sigma,abs_f"
    rows = [l for l in lines[2:] if l]
    assert len(rows) == 40
    rule = orc.ContourRule(1e-3, 1e-1, 32, 0.1, orc.SpectralTransform("exp"))
    for r in rows:
        s, f = map(float, r.split(","))
        assert f == abs(orc.eval_filter(rule, s)) or abs(f - abs(orc.eval_filter(rule, s))) <= 1e-15 * max(f, 1e-300)
    assert run_cli(f"filter-plot --interval 1e-3 1e-1 --points 0 --out {prefix}0")[0] == 2


@pytest.mark.gpu
def test_solve_model_writes_report_and_triplets(tmp_path):               # test_cli.cpp:47-66
    prefix = str(tmp_path / "run")
    rc, out, err = run_cli(f"solve --model 1 --interval 0.8 1.2 --mode ss-svd --out {prefix}")
    assert rc == 0, err
    j = json.load(open(prefix + ".report.json"))
    assert j["schema_version"] == 1
    assert j["counts"]["nonspurious_in_interval"] == 40
    assert j["accuracy"]["max_rel_error_nonspurious"] <= 1e-10
    assert j["config"]["mode"] == "ss-svd" and j["config"]["transform"] == "identity"
    assert j["matrix"] == {"rows": 1000, "cols": 200, "source": "model1"}
    assert len(j["triplets"]) == j["counts"]["candidates"]
    header = open(prefix + ".triplets.csv").readline().strip()
    assert header == "index,sigma,in_interval,spurious,tau,residual_exact,residual_estimated,galerkin"
    assert "non-spurious in-interval 40" in out


@pytest.mark.gpu
def test_empty_interval_report(tmp_path):                                # test_cli.cpp:68-78
    prefix = str(tmp_path / "empty")
    rc, _, _ = run_cli(f"solve --model 1 --interval 5.0 6.0 --mode ss-svd --out {prefix}")
    assert rc == 0
    j = json.load(open(prefix + ".report.json"))
    assert j["empty"] is True and j["counts"]["in_interval"] == 0 and "note" in j


@pytest.mark.gpu
def test_model_round_trips_through_solve_input(tmp_path):                # test_cli.cpp:93-105
    m1 = str(tmp_path / "m1")
    assert run_cli(f"model --which 1 --rows 120 --cols 40 --out {m1}")[0] == 0
    r = str(tmp_path / "r")
    rc, _, err = run_cli(f"solve --input {m1}.mtx --interval 0.2 0.33 --L 6 --M 3 --N 16 --out {r}")
    assert rc == 0, err
    j = json.load(open(r + ".report.json"))
    assert j["counts"]["nonspurious_in_interval"] > 0 and j["matrix"]["source"].endswith("m1.mtx")


@pytest.mark.gpu
def test_solve_sparse_input_with_normalize(tmp_path):
    """coordinate .mtx through the sparse upload path, --normalize rescales sigma_max to ~1."""
    import scipy.sparse as sp
    from paper_2109_13655_b200 import sssvd
    rng = np.random.default_rng(3)
    a = sp.random(400, 150, density=0.05, random_state=rng, data_rvs=rng.standard_normal) + sp.eye(400, 150)
    path = str(tmp_path / "s.mtx")
    sssvd.write_matrix_market(path, sssvd.ProblemMatrix.from_sparse(a), "")
    smax = np.linalg.svd(a.toarray(), compute_uv=False)[0]
    r = str(tmp_path / "s")
    rc, _, err = run_cli(f"solve --input {path} --interval 0.5 0.7 --L 8 --M 4 --normalize --out {r}")
    assert rc == 0, err
    j = json.load(open(r + ".report.json"))
    assert abs(j["matrix"]["normalized_scale"] - smax) <= 1e-5 * smax
    assert j["counts"]["nonspurious_in_interval"] > 0


@pytest.mark.gpu
def test_verify_clean_and_injected_noise():                              # test_cli.cpp:129-133
    rc, out, err = run_cli("verify --model 1 --interval 0.8 1.2 --L 10 --M 4")
    assert rc == 0, out + err
    assert "PASS  Galerkin identity" in out and "PASS  moment identity" in out
    assert run_cli("verify --model 1 --interval 0.8 1.2 --L 10 --M 4 --inject-noise 1e-2")[0] == 1


@pytest.mark.gpu
def test_bench_table(tmp_path):
    """bench.hpp:60-100: both models x four modes (the L-scaling sweep skipped)."""
    prefix = str(tmp_path / "b")
    rc, out, err = run_cli(f"bench --no-scaling --out {prefix}")
    assert rc == 0, err
    j = json.load(open(prefix + ".bench.json"))
    assert j["schema_version"] == 1 and len(j["rows"]) == 8
    assert all(r["error"] == "" for r in j["rows"])
    m1 = {r["mode"]: r for r in j["rows"] if r["model"] == 1}
    assert m1["ss-svd"]["t_hat"] == 40 and m1["ss-svd"]["max_rel_error"] <= 1e-10
