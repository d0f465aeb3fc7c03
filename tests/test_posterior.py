"""Posterior wire format and CLI plumbing."""

import json

import pytest

from paper_2010_08454_b200.cli import main
from paper_2010_08454_b200.posterior import parse_posterior, serialize_posterior


class _D:
    def __init__(self, support, log_z=-1.25):
        self.support = support
        self.log_z = log_z


def test_tsv_ordering_probability_descending_ties_by_text():
    d = _D([(False, 0.25), (True, 0.75)])
    assert serialize_posterior(d, "tsv") == "true\t0.75\nfalse\t0.25\n"
    d = _D([(3, 0.25), (10, 0.25), (2, 0.5)])
    assert serialize_posterior(d, "tsv").splitlines() == ["2\t0.5", "10\t0.25", "3\t0.25"]


def test_json_uniform_example_and_roundtrip():
    d = _D([(2, 0.5), (1, 0.5)], log_z=-0.6931471805599453)
    text = serialize_posterior(d, "json")
    obj = json.loads(text)
    assert obj["support"] == [{"value": 1, "prob": 0.5}, {"value": 2, "prob": 0.5}]
    assert obj["log_z"] == -0.6931471805599453
    back = parse_posterior(text, "json")
    assert back["support"] == [(1, 0.5), (2, 0.5)]


@pytest.mark.parametrize("fmt", ["tsv", "json"])
def test_roundtrip_exact_and_byte_identical(fmt):
    d = _D([(4, 0.1234567890123456789), (2, 1 / 3), (3, 1 - 1 / 3 - 0.1234567890123456789), (None, 0.0)])
    t1, t2 = serialize_posterior(d, fmt), serialize_posterior(d, fmt)
    assert t1 == t2
    back = parse_posterior(t1, fmt)
    want = sorted(d.support, key=lambda vp: (-vp[1], str(vp[0])))
    assert [p for _, p in back["support"]] == [p for _, p in want]
    assert [v for v, _ in back["support"]] == [v for v, _ in want]


def test_empty_support_refused_in_tsv():
    with pytest.raises(ValueError):
        serialize_posterior(_D([]), "tsv")
    assert json.loads(serialize_posterior(_D([]), "json"))["support"] == []


def test_cli_usage_errors_exit_1(tmp_path):
    assert main(["run", "--model", "nope"]) == 1
    assert main(["run", "--model", "poly", "--thin", "0"]) == 1
    assert main([]) == 1
    assert main(["run", str(tmp_path / "missing.cup")]) == 1
    bad = tmp_path / "bad.cup"
    bad.write_text("model <- function() { shift(k, 1) }; importance(model, 10)")
    assert main(["run", str(bad)]) == 1  # compile error


@pytest.mark.gpu
def test_cli_run_is_deterministic_and_serialised(cuda, capsys):
    assert main(["run", "--model", "poly", "--samples", "200000", "--seed", "3", "--format", "tsv"]) == 0
    a = capsys.readouterr().out
    assert main(["run", "--model", "poly", "--samples", "200000", "--seed", "3", "--format", "tsv"]) == 0
    b = capsys.readouterr().out
    assert a == b  # same config => byte-identical posterior (SPEC.md cli invariants)
    rows = parse_posterior(a, "tsv")["support"]
    assert {v for v, _ in rows} <= {2, 3, 4} and abs(sum(p for _, p in rows) - 1) < 1e-12
    assert main(["run", "--model", "hmm", "--samples", "50000", "--points", "50", "--format", "json"]) == 0
    obj = json.loads(capsys.readouterr().out)
    assert obj["support"] and obj["log_z"] < 0


@pytest.mark.gpu
def test_cli_bench_checks_then_times(cuda, capsys):
    assert main(["bench", "--filter", "poly", "--repeats", "2"]) == 0
    out = capsys.readouterr().out
    assert "poly" in out and " ok" in out


@pytest.mark.gpu
def test_cli_run_program_file(cuda, capsys, tmp_path):
    prog = tmp_path / "coin.cup"
    prog.write_text("""
      flips <- [1, 1, 1, 1, 1, 1, 1, 1, 0, 0];
      model <- function() {
        p <- sample(beta(1, 1));
        factor(reduce(function(acc, f) { acc + dist-score(bernoulli(p), f > 0.5) }, 0.0, flips));
        p > 0.5
      };
      importance(model, 400000)
    """)
    assert main(["run", str(prog), "--seed", "2", "--format", "json"]) == 0
    obj = json.loads(capsys.readouterr().out)
    probs = {e["value"]: e["prob"] for e in obj["support"]}
    # posterior Beta(9, 3): P(p > 0.5) = 1 - I_0.5(9, 3) = 0.96728515625
    assert abs(probs[True] - 0.96728515625) < 0.01


def test_cli_flags_and_multi_gpu_relaunch():
    """--particles (alias of --samples), --smc-steps, --chains and
    --gpus N, which re-runs the same command one process per GPU under torch.distributed.run."""
    from paper_2010_08454_b200 import cli

    cmd = cli.relaunch_command(["run", "--model", "hmm", "--gpus", "8", "--particles", "1000000",
                                "--smc-steps", "50"], 8)
    i = cmd.index("-m")
    assert cmd[i:i + 2] == ["-m", "torch.distributed.run"] and "--nproc-per-node=8" in cmd
    assert "--master-addr=127.0.0.1" in cmd
    tail = cmd[cmd.index("paper_2010_08454_b200"):]
    assert tail == ["paper_2010_08454_b200", "run", "--model", "hmm", "--particles", "1000000", "--smc-steps", "50"]
    assert "--gpus" not in " ".join(tail)
    assert cli.relaunch_command(["run", "x.cup", "--gpus=2"], 2)[-2:] == ["run", "x.cup"]
