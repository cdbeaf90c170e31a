"""The device-routed CLI (paper_2001_04179_b200.cli): the
reference's flags, exit codes and seed derivation; on the GPU the full
generate -> solve -> bench -> rates flow through the B200 solver and the
native MatrixMarket reader.  (tools/ref_cli_plugin.py additionally runs the
reference's own test_cli.py against this CLI on the GPU box.)"""

import csv

import numpy as np
import pytest

from paper_2001_04179_b200 import cli


def test_usage_errors_exit_1():
    assert cli.main(["solve"]) == cli.EXIT_USAGE
    assert cli.main(["frobnicate"]) == cli.EXIT_USAGE
    assert cli.main(["generate", "--type", "2", "--m", "3000", "--n", "2000", "--out", "/tmp/x"]) == cli.EXIT_USAGE


def test_derive_seed_is_seedsequence():
    want = int(np.random.SeedSequence(7, spawn_key=(1, 0)).generate_state(1, np.uint64)[0])
    assert cli.derive_seed(7, 1, 0) == want
    assert cli.derive_seed(7, 1, 0) != cli.derive_seed(7, 1, 1)


def test_config_file_tokens(tmp_path):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("# comment\ntype = 2\nm = 10\ninconsistent = true\nverbose = off\n")
    assert cli._with_config(["solve", "--config", str(cfg), "--seed", "4"]) == [
        "solve", "--type", "2", "--m", "10", "--inconsistent", "--seed", "4"]


def test_host_only_algorithms_are_usage_errors(tmp_path):
    with pytest.raises(cli.UsageError, match="not on the B200 path"):
        cli._check_algo("rdbk")
    with pytest.raises(cli.UsageError, match="unknown algorithm"):
        cli._check_algo("cg")


@pytest.mark.gpu
def test_generate_solve_bench_rates_on_device(tmp_path, capsys):
    out = tmp_path / "prob"
    assert cli.main(["generate", "--type", "1", "--m", "30", "--n", "18", "--rank", "10", "--kappa", "2",
                     "--inconsistent", "--seed", "5", "--out", str(out)]) == cli.EXIT_OK
    assert "declared_rank = 10" in (out / "meta.txt").read_text()
    curve = tmp_path / "curve.csv"
    assert cli.main(["solve", "--problem", str(out), "--algo", "rebk", "--tau", "5", "--alpha", "1x", "--seed", "2",
                     "--curve", str(curve)]) == cli.EXIT_OK
    text = capsys.readouterr().out
    assert "converged      true" in text and "rho_hat" in text and "device         cuda:0" in text
    rows = list(csv.DictReader(open(curve)))
    assert rows[0]["iteration"] == "0" and float(rows[-1]["error"]) <= 1e-5
    assert cli.main(["solve", "--problem", str(out), "--algo", "dsbgs", "--tau", "5", "--alpha", "1",
                     "--seed", "2", "--max-iters", "200"]) in (cli.EXIT_OK, cli.EXIT_NO_CONVERGENCE)
    bench = tmp_path / "b.csv"
    assert cli.main(["bench", "--problem", str(out), "--algo", "rek,rebk", "--tau", "5", "--alpha", "1x",
                     "--trials", "2", "--seed", "9", "--out", str(bench)]) == cli.EXIT_OK
    rows = list(csv.DictReader(open(bench)))
    assert sum(r["kind"] == "aggregate" for r in rows) == 2
    assert cli.main(["rates", "--problem", str(out), "--tau", "5", "--alpha", "0.75x,1x,2.25x"]) == cli.EXIT_OK
    assert cli.main(["solve", "--problem", str(out), "--algo", "rek", "--max-iters", "5",
                     "--seed", "2"]) == cli.EXIT_NO_CONVERGENCE
