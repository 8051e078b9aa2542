"""The chainscan front end (cli.py): the reference's test_cli.py cases that the
B200 run / bench / diff wiring covers (test_cli.py:20-239).  Usage errors are
checked on the CPU; running chains needs the device."""

import json
import os

import pytest

from paper_2508_18413_b200 import cli


def test_usage_errors_exit_1(tmp_path):
    assert cli.main([]) == cli.USAGE
    assert cli.main(["run", "--sampler", "nuts"]) == cli.USAGE
    assert cli.main(["run", "--sampler", "gibbs", "--method", "block-quasi-deer"]) == cli.USAGE
    assert cli.main(["run", "--config", str(tmp_path / "missing.cfg")]) == cli.USAGE
    bad = tmp_path / "bad.cfg"
    bad.write_text("T = 10\nnot_a_key = 3\n")
    assert cli.main(["run", "--config", str(bad)]) == cli.USAGE


def test_config_precedence_flag_over_file_over_default(tmp_path):
    f = tmp_path / "run.cfg"
    f.write_text("# comment\nT = 300\neps = 0.2\nfull-trace = yes\n")
    ns = cli.parser().parse_args(["run", "--config", str(f), "--T", "50"])
    cfg = cli.merge(ns, cli.read_config(str(f)))
    assert cfg.T == 50 and cfg.eps == 0.2 and cfg.full_trace is True and cfg.sampler == "mala"
    assert cli.echo(cfg)["clip"] == "inf"


@pytest.mark.gpu
def test_run_sequential_and_parallel_then_diff(cuda_device, tmp_path):
    # test_cli.py:83-95: a quasi-DEER run matches the sequential chain
    a, b = str(tmp_path / "seq.bin"), str(tmp_path / "par.bin")
    common = ["--sampler", "hmc", "--target", "std-normal:2", "--eps", "0.3", "--T", "2000", "--B", "2",
              "--seed", "3"]
    assert cli.main(["run", *common, "--method", "sequential", "--out", a]) == cli.OK
    assert cli.main(["run", *common, "--method", "quasi-deer", "--clip", "1", "--atol", "1e-7", "--rtol", "1e-6",
                     "--max-iters", "400", "--out", b]) == cli.OK
    rep = json.load(open(b + ".report.json"))
    assert [c["seed"] for c in rep["chains"]] == [3, 2]  # seed ^ b
    assert all(c["converged"] and c["engine"] in ("fused", "streamed") for c in rep["chains"])
    assert cli.main(["diff", a, b, "--out", str(tmp_path / "d.csv")]) == cli.OK
    rows = open(tmp_path / "d.csv").read().splitlines()
    assert rows[0] == "step,max_abs_error,within_tolerance" and len(rows) == 2001


@pytest.mark.gpu
def test_config_echo_reproduces_the_trace(cuda_device, tmp_path):
    # test_cli.py:139-161: feeding the echoed config back reproduces the bytes
    out = str(tmp_path / "a.bin")
    assert cli.main(["run", "--sampler", "mala", "--target", "std-normal:2", "--method", "deer-dense",
                     "--T", "512", "--eps", "0.3", "--out", out]) == cli.OK
    echo = json.load(open(out + ".report.json"))["config"]
    cfgf = tmp_path / "echo.cfg"
    echo["out"] = str(tmp_path / "b.bin")
    cfgf.write_text("".join(f"{k} = {v}\n" for k, v in echo.items() if v is not None))
    assert cli.main(["run", "--config", str(cfgf)]) == cli.OK
    with open(out, "rb") as fa, open(str(tmp_path / "b.bin"), "rb") as fb:
        assert fa.read() == fb.read()


@pytest.mark.gpu
def test_divergence_exits_2(cuda_device, tmp_path):
    # test_cli.py:185-192: plain quasi-DEER on the headline HMC chain diverges
    assert cli.main(["run", "--sampler", "hmc", "--target", "rosenbrock", "--eps", "0.5", "--T", "3000",
                     "--method", "quasi-deer", "--out", str(tmp_path / "x.bin")]) == cli.DIVERGED


@pytest.mark.gpu
def test_bench_csv_schema(cuda_device, tmp_path):
    # test_cli.py:196-211
    out = tmp_path / "b.csv"
    assert cli.main(["bench", "--sampler", "mala", "--target", "std-normal:2", "--method",
                     "sequential,deer-dense,quasi-deer", "--T", "256,512", "--B", "1", "--reps", "2",
                     "--warmups", "1", "--out", str(out)]) == cli.OK
    rows = open(out).read().splitlines()
    assert rows[0] == "sampler,method,B,T,median_seconds,iterations,converged_fraction,status"
    assert len(rows) == 7 and all(r.endswith(",ok") for r in rows[1:])


@pytest.mark.gpu
def test_orthogonal_run_matches_plain(cuda_device, tmp_path):
    a, b = str(tmp_path / "p.bin"), str(tmp_path / "o.bin")
    common = ["--sampler", "mala", "--target", "std-normal:4", "--T", "800", "--eps", "0.3", "--method",
              "quasi-deer", "--atol", "1e-7", "--rtol", "1e-6"]
    assert cli.main(["run", *common, "--out", a]) == cli.OK
    assert cli.main(["run", *common, "--orthogonal", "--out", b]) == cli.OK
    assert cli.main(["diff", a, b, "--atol", "1e-5", "--rtol", "1e-4"]) == cli.OK
    assert os.path.exists(b + ".json")
