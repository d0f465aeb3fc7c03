"""Programs that compute with engine results (builtins.py:116-123): engine
calls bound at top level run on the GPU and return empirical DistValues; dist-var / dist-score
and arithmetic over them run on the host (paper_2010_08454_b200/program.py)."""

import math

import pytest

from paper_2010_08454_b200 import program
from paper_2010_08454_b200.frontend import CompileError

COIN = """
flips <- [1.0, 1.0, 0.0, 1.0, 1.0, 1.0, 0.0, 1.0, 1.0, 1.0];
coin <- function() {
  p <- sample(beta(1, 1));
  map(function(f) { observe(bernoulli(p), f > 0.5) }, flips);
  p
};
post <- importance(coin, 1000000);
v <- dist-var(post);
[v, dist-var(beta(9, 3)), dist-var(normal(0, 10))]
"""

DISCRETE = """
model <- function() {
  k <- sample(uniform-discrete(0, 4));
  factor(-0.5 * to-real(k));
  k
};
post <- enumerate(model, 100);
[dist-var(post), dist-score(post, 2), dist-score(post, 7)]
"""


def test_program_structure_compiles_on_cpu():
    cp = program.CompiledProgram(COIN)
    kinds = [s[0] for s in cp.steps]
    assert kinds.count("engine") == 1 and cp.result_engine is None
    assert cp.engines[0].engine == "importance" and cp.engines[0].default_n == 1_000_000
    cp2 = program.CompiledProgram(DISCRETE)
    assert cp2.engines[0].engine == "enumerate"


def test_host_code_over_parametric_distributions():
    ev = program._HostEval({})
    from paper_2010_08454_b200 import lang

    res = ev.ev(lang.parse("x <- 1; [dist-var(normal(0, 10)), dist-var(bernoulli(0.5)), "
                           "dist-var(uniform-discrete(2, 5)), 2 * 3 + 1]").result)
    assert res[0] == 100.0 and res[1] == 0.25 and abs(res[2] - 2 / 3) < 1e-12 and res[3] == 7


def test_engine_call_inside_an_expression_is_rejected():
    with pytest.raises(CompileError):
        program.run_program("m <- function() { sample(bernoulli(0.5)) }; dist-var(importance(m, 10))", None)


@pytest.mark.gpu
def test_gpu_dist_var_of_importance_posterior(cuda):
    """importance(coin-model, ...) inside a program, then dist-var of the result:
    the Beta(9, 3) posterior variance within Monte Carlo error."""
    from paper_2010_08454_b200 import Rng

    v, exact, prior = program.run_program(COIN, Rng(7))
    assert exact == pytest.approx(27 / 1872) and prior == 100.0
    assert abs(v - exact) < 0.02 * exact


@pytest.mark.gpu
def test_gpu_dist_score_of_enumerated_posterior(cuda):
    """Exact enumeration: P(k) ∝ exp(-k/2) on {0..3}; dist-score is its log-mass, -inf off the
    support; dist-var the weighted variance."""
    from paper_2010_08454_b200 import Rng

    var, s2, s7 = program.run_program(DISCRETE, Rng(1))
    w = [math.exp(-0.5 * k) for k in range(4)]
    z = sum(w)
    p = [x / z for x in w]
    m = sum(k * q for k, q in enumerate(p))
    assert s2 == pytest.approx(math.log(p[2]), abs=1e-5)
    assert s7 == -math.inf
    assert var == pytest.approx(sum(q * (k - m) ** 2 for k, q in enumerate(p)), abs=1e-5)


@pytest.mark.gpu
def test_gpu_program_with_two_engines(cuda):
    """Two engine bindings in one program run on rng.split(0) and rng.split(1); the result
    combines them on the host."""
    from paper_2010_08454_b200 import Rng

    src = """
    a <- function() { sample(normal(0, 1)) };
    b <- function() { sample(normal(0, 2)) };
    pa <- importance(a, 400000);
    pb <- importance(b, 400000);
    dist-var(pb) / dist-var(pa)
    """
    r = program.run_program(src, Rng(3))
    assert abs(r - 4.0) < 0.1
