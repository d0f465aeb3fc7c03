"""The paper's benchmark corpus (§5.1 table "Benchmark programs"), re-derived in CuPPL
under examples/ (the corpus is reconstructed from the descriptions), compiled for
the GPU and checked against known answers — the "sidecar expectations" of SPEC.md:509."""

import math
from pathlib import Path

import numpy as np
import pytest

from paper_2010_08454_b200 import frontend

EX = Path(__file__).resolve().parent.parent / "examples"
NAMES = ["biasedcoin", "customdist", "linear_regression", "logistic_regression", "binomial",
         "sevenscientists", "linefitting", "enumerate_geometric"]


def _src(name):
    return (EX / f"{name}.cup").read_text()


def _vec(src, name):
    """A top-level numeric vector of a program (for the closed-form expectations)."""
    from paper_2010_08454_b200 import lang

    for b, e in lang.parse(src).bindings:
        if b == name:
            return np.array([float(x.value) if isinstance(x, lang.Num) else -float(x.arg.value) for x in e.elems])
    raise KeyError(name)


@pytest.mark.parametrize("name", NAMES)
def test_example_compiles(name):
    m = frontend.compile_program(_src(name))
    frontend._nvrtc_cubin(m.cuda, 1)
    assert m.engine == {"linear_regression": "mcmc", "logistic_regression": "mcmc",
                        "enumerate_geometric": "enumerate"}.get(name, "importance")


@pytest.mark.gpu
def test_biasedcoin(cuda):
    from paper_2010_08454_b200 import Rng, infer

    post = infer.run_importance(frontend.compile_program(_src("biasedcoin")), 2_000_000, Rng(1))
    assert abs(post.mean["value"] - 0.75) < 0.005  # Beta(9, 3)


@pytest.mark.gpu
def test_customdist(cuda):
    from paper_2010_08454_b200 import Rng, infer

    post = infer.run_importance(frontend.compile_program(_src("customdist")), 2_000_000, Rng(2))
    assert abs(post.mean["value"] - 3.0) < 0.01 and abs(post.stats["var_value"] - 5.0) < 0.05


@pytest.mark.gpu
def test_binomial(cuda):
    from paper_2010_08454_b200 import Rng, infer

    post = infer.run_importance(frontend.compile_program(_src("binomial")), 2_000_000, Rng(3))
    pmf = [math.comb(10, k) * 0.3 ** k * 0.7 ** (10 - k) for k in range(11)]
    got = dict(post.support)
    for k in range(11):  # beyond the record's 8 bins: the K3 second pass (full support)
        assert abs(got.get(k, 0.0) - pmf[k]) < 2e-3, (k, got.get(k), pmf[k])
    assert 8 in got and abs(sum(got.values()) - 1.0) < 1e-9
    assert abs(post.mean["value"] - 3.0) < 0.01


@pytest.mark.gpu
def test_linear_regression_mcmc(cuda):
    from paper_2010_08454_b200 import Rng, infer

    src = _src("linear_regression")
    xs, ys = _vec(src, "xs"), _vec(src, "ys")
    X = np.stack([xs, np.ones_like(xs)], axis=1)
    prec = X.T @ X + np.eye(2) / 100.0
    mean = np.linalg.solve(prec, X.T @ ys)
    post = infer.run_lmh(frontend.compile_program(src), 3000, Rng(4), chains=1024, burn_in=500)
    got = np.array([post.mean["v0"], post.mean["v1"]])
    assert np.all(np.abs(got - mean) < 0.05), (got, mean)
    assert 0.0 < post.stats["acceptance"] < 1.0


@pytest.mark.gpu
def test_logistic_regression_mcmc(cuda):
    from paper_2010_08454_b200 import Rng, infer

    src = _src("logistic_regression")
    xs, ys = _vec(src, "xs"), _vec(src, "ys")
    w, b = np.meshgrid(np.linspace(-5, 25, 601), np.linspace(-15, 15, 601), indexing="ij")
    z = w[..., None] * xs + b[..., None]
    ll = (ys * -np.logaddexp(0, -z) + (1 - ys) * -np.logaddexp(0, z)).sum(-1) - (w ** 2 + b ** 2) / 200.0
    p = np.exp(ll - ll.max())
    p /= p.sum()
    mean = np.array([(p * w).sum(), (p * b).sum()])
    post = infer.run_lmh(frontend.compile_program(src), 4000, Rng(5), chains=1024, burn_in=1000)
    got = np.array([post.mean["v0"], post.mean["v1"]])
    assert np.all(np.abs(got - mean) < 0.15 * np.maximum(1.0, np.abs(mean))), (got, mean)


@pytest.mark.gpu
def test_sevenscientists(cuda):
    from paper_2010_08454_b200 import Rng, infer

    src = _src("sevenscientists")
    xs = _vec(src, "xs")
    mu = np.linspace(-20, 30, 5001)
    s = np.linspace(0.1, 25.0, 4001)
    # p(x | mu) = mean over s ~ U(0.1, 25) of N(x; mu, s), per measurement
    logp = -mu ** 2 / (2 * 50.0 ** 2)
    for x in xs:
        dens = np.exp(-0.5 * ((x - mu[:, None]) / s) ** 2) / (s * math.sqrt(2 * math.pi))
        logp = logp + np.log(dens.mean(axis=1))
    p = np.exp(logp - logp.max())
    p /= p.sum()
    mean = float((p * mu).sum())
    post = infer.run_importance(frontend.compile_program(src), 2_000_000, Rng(6))
    assert abs(post.mean["value"] - mean) < 0.3, (post.mean["value"], mean, post.ess)


@pytest.mark.gpu
def test_linefitting(cuda):
    from oracle import exact
    from paper_2010_08454_b200 import Rng, infer

    src = _src("linefitting")
    xs, ys = _vec(src, "xs"), _vec(src, "ys")
    p_exact, _, _, logz = exact.poly_posterior(np.float32(xs).astype(float), np.float32(ys).astype(float))
    post = infer.run_importance(frontend.compile_program(src), 2_000_000, Rng(7))
    got = dict(post.support)
    for d, p in p_exact.items():
        se = math.sqrt(max(p * (1 - p), 1e-8) / post.ess)
        assert abs(got.get(d, 0.0) - p) < 5 * se + 1e-3, (d, got.get(d), p)
    assert abs(post.log_z - logz) < 5 / math.sqrt(post.ess) + 0.02


@pytest.mark.gpu
def test_enumerate_geometric_and_cli(cuda, capsys):
    from paper_2010_08454_b200 import cli, infer

    post = infer.run_enumeration(frontend.compile_program(_src("enumerate_geometric")))
    got = dict(post.support)
    z = 1.0 - 0.5 ** 20  # paths recursing past max_depth = 20 are cut and the rest renormalised
    assert set(got) == set(range(20))  # the whole support, beyond the record's 8 bins
    for k in range(20):
        assert abs(got[k] - 0.5 ** (k + 1) / z) < 1e-6
    assert cli.main(["run", str(EX / "enumerate_geometric.cup"), "--format", "tsv"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0].split("\t")[0] == "0" and abs(float(lines[0].split("\t")[1]) - 0.5) < 1e-6
    assert lines[1].split("\t")[0] == "1" and abs(float(lines[1].split("\t")[1]) - 0.25) < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_example_through_the_cli(cuda, capsys, name):
    """`run FILE.cup --format json` for every corpus program: exit code 0 and a posterior that
    parses back."""
    from paper_2010_08454_b200 import cli
    from paper_2010_08454_b200.posterior import parse_posterior

    args = ["run", str(EX / f"{name}.cup"), "--format", "json", "--seed", "3"]
    if name in ("linear_regression", "logistic_regression"):
        args += ["--samples", "200", "--chains", "256"]
    elif name != "enumerate_geometric":
        args += ["--particles", "200000"]
    assert cli.main(args) == 0
    out = parse_posterior(capsys.readouterr().out, "json")
    assert "support" in out
    if name in ("binomial", "enumerate_geometric", "linefitting"):
        assert abs(sum(p for _, p in out["support"]) - 1.0) < 1e-6
