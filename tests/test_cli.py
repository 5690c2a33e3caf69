"""The bnmc_b200 CLI (paper_1210_5128_b200/csrc/cli.cpp): the reference CLI's
`learn`, `eval --sweep` and `bench` (tools/bnmc.cpp) on the B200 backend.
Outputs are compared byte for byte with the reference's own driver steps run
through oracle/_ref (summary minus '#' timing lines, trace CSV, best edges,
sweep metrics, BNSC cache) — the CLI reproducibility contract of
proj/tests/cli_test.sh."""
import os
import subprocess

import numpy as np
import pytest

from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1210_5128_b200", "bnmc_b200")
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module", autouse=True)
def built():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_1210_5128_b200", "csrc")])


def run(*args, check=True):
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check:
        assert p.returncode == 0, p.stderr
    return p


def no_comments(path):
    return "".join(l for l in open(path) if not l.startswith("#"))


def test_usage_and_data_errors_exit_codes(tmp_path):
    """bnmc.cpp:454-465: usage 2, data 3 (checked before any device call)."""
    assert run(check=False).returncode == 2
    assert run("frobnicate", check=False).returncode == 2
    assert run("learn", "--bogus", "1", check=False).returncode == 2
    assert run("learn", "--out-prefix", tmp_path / "x", check=False).returncode == 2  # no --data
    assert run("learn", "--data", tmp_path / "missing.csv", "--out-prefix", tmp_path / "x",
               check=False).returncode == 3
    (tmp_path / "d.csv").write_text("a,b\n0,1\n1,0\n")
    assert run("learn", "--data", tmp_path / "d.csv", "--out-prefix", tmp_path / "x",
               "--max-parents", "9", check=False).returncode == 2
    assert run("learn", "--data", tmp_path / "d.csv", "--out-prefix", tmp_path / "x", "--pst",
               "--unrank", check=False).returncode == 2
    (tmp_path / "bad.csv").write_text("a,b\n0,1,1\n")
    assert run("learn", "--data", tmp_path / "bad.csv", "--out-prefix", tmp_path / "x",
               check=False).returncode == 3
    assert run("eval", "--truth", tmp_path / "none.edges", check=False).returncode == 3


def _instance(tmp_path, n=10, m=600, seed=3, priors=True):
    cells, truth = ref.generate(n, 3, m, [3] * n, seed=seed)
    ref.write_dataset_csv(cells, [3] * n, tmp_path / "d.csv")
    ref.write_edge_list(truth, tmp_path / "truth.edges")
    if priors:
        ref.write_prior_csv(ref.synth_priors(n, truth, seed=seed), tmp_path / "p.csv")
    return cells, truth


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("k2,strict,priors", [(False, False, True), (True, True, False)])
def test_learn_outputs_identical_to_reference(tmp_path, k2, strict, priors):
    _instance(tmp_path, priors=priors)
    kw = dict(s=3, iterations=400, seed=11, workers=4, track_top=5, k2=k2, strict=strict,
              priors_path=(tmp_path / "p.csv") if priors else None)
    ref.learn(tmp_path / "d.csv", tmp_path / "ref", **kw)
    args = ["learn", "--data", tmp_path / "d.csv", "--out-prefix", tmp_path / "ours",
            "--max-parents", 3, "--iterations", 400, "--seed", 11, "--workers", 4,
            "--track-top", 5]
    if priors:
        args += ["--priors", tmp_path / "p.csv"]
    if k2:
        args += ["--k2"]
    if strict:
        args += ["--strict-paper-tracker"]
    out = run(*args).stdout
    assert "best_score:" in out
    assert no_comments(tmp_path / "ours.summary.txt") == no_comments(tmp_path / "ref.summary.txt")
    for ext in (".trace.csv", ".best.edges"):
        assert open(tmp_path / f"ours{ext}").read() == open(tmp_path / f"ref{ext}").read(), ext


@needs_ref
@pytest.mark.gpu
def test_save_and_load_cache_round_trip(tmp_path):
    cells, _ = _instance(tmp_path, priors=False)
    common = ["--data", tmp_path / "d.csv", "--max-parents", 3, "--iterations", 200, "--seed", 2]
    run("learn", *common, "--out-prefix", tmp_path / "a", "--save-cache", tmp_path / "c.bnsc")
    run("learn", *common, "--out-prefix", tmp_path / "b", "--load-cache", tmp_path / "c.bnsc")
    for ext in (".trace.csv", ".best.edges"):
        assert open(tmp_path / f"a{ext}").read() == open(tmp_path / f"b{ext}").read()
    assert no_comments(tmp_path / "a.summary.txt") == no_comments(tmp_path / "b.summary.txt")
    # the BNSC file is the reference's ScoreCache::save, byte for byte
    ref.Cache.build(cells, [3] * cells.shape[1], 3).save(str(tmp_path / "r.bnsc"))
    assert open(tmp_path / "c.bnsc", "rb").read() == open(tmp_path / "r.bnsc", "rb").read()
    # a cache built with other scoring parameters is rejected (DataError -> 3)
    p = run("learn", *common, "--ess", 2.0, "--out-prefix", tmp_path / "e", "--load-cache",
            tmp_path / "c.bnsc", check=False)
    assert p.returncode == 3


@needs_ref
@pytest.mark.gpu
def test_eval_sweep_identical_to_reference(tmp_path):
    _instance(tmp_path, n=9, m=500, seed=8, priors=False)
    ref.eval_sweep(tmp_path / "truth.edges", tmp_path / "d.csv", tmp_path / "ref.csv", s=3,
                   iterations=150, seed=4, workers=2)
    run("eval", "--truth", tmp_path / "truth.edges", "--sweep", "--data", tmp_path / "d.csv",
        "--out", tmp_path / "ours.csv", "--max-parents", 3, "--iterations", 150, "--seed", 4,
        "--workers", 2)
    assert open(tmp_path / "ours.csv").read() == open(tmp_path / "ref.csv").read()
    # plain eval of a learned graph against the truth
    out = run("eval", "--truth", tmp_path / "truth.edges", "--learned", tmp_path / "truth.edges").stdout
    assert out.splitlines()[1].startswith("eval,0.5,0.5,0,")


@pytest.mark.gpu
def test_bench_csv_schema(tmp_path):
    run("bench", "--scaling-nodes", "8,13", "--reps", 5, "--chains", 64, "--chain-iters", 20,
        "--out", tmp_path / "b.csv")
    rows = [l.split(",") for l in open(tmp_path / "b.csv").read().splitlines()]
    assert rows[0] == ["phase", "nodes", "workers", "candidates", "reps", "seconds", "speedup"]
    phases = [r[0] for r in rows[1:]]
    assert phases == ["preprocess", "iteration", "iteration_batched", "chain_iteration"] * 2
    assert all(float(r[5]) > 0 for r in rows[1:])
