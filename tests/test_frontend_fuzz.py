"""Differential testing of the model compiler: seeded random CuPPL programs (tests/fuzz_programs.py
— every draw kind, arithmetic, pure and effectful ifs, factors, observe loops over data, scalar
and tuple returns) compiled for the GPU, their log-weights compared with the fp64 interpreter on
the GPU's recorded draws. Tolerance: SURVEY.md D11 (1e-5 relative + 1e-6) plus the program's
own fp32 conditioning — ten times the distance between the fp64 interpreter and the same
interpreter rounding every operation to fp32 (oracle/dsl_eval.Fp32Interpreter). Random
expression trees cancel (x - y with x ~ y, pow of large arguments), where no fixed relative
tolerance holds for any fp32 evaluation; for well-conditioned programs the extra term is ~0."""

import math

import numpy as np


def tol_ok(got: float, ref: float, ref32: float) -> bool:
    """D11 plus the program's fp32 conditioning (module docstring)."""
    cond = abs(ref32 - ref) if math.isfinite(ref32) else 0.0
    return abs(got - ref) <= 1e-5 * abs(ref) + 1e-6 + 10.0 * cond
import pytest

from fuzz_programs import program
from paper_2010_08454_b200 import frontend

SEEDS = list(range(40))


def test_fuzz_programs_compile():
    for seed in SEEDS:
        m = frontend.compile_program(program(seed))
        if seed % 8 == 0:
            frontend._nvrtc_cubin(m.cuda, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_gpu_fuzz_program_matches_interpreter(cuda, seed):
    from oracle.dsl_eval import Fp32Interpreter, Interpreter
    from paper_2010_08454_b200 import Rng, infer

    src = program(seed)
    m = frontend.compile_program(src)
    n = 2048
    post = infer.run_importance(m, n, Rng(seed), return_traces=True)
    lw = post.traces["log_weight"].cpu().numpy().astype(float)
    draws = post.traces["draws"].cpu().numpy().astype(float)
    it, it32 = Interpreter(src), Fp32Interpreter(src)
    for i in range(0, n, 67):
        ref, _ = it.run(draws[i])
        if math.isinf(ref) or math.isnan(ref):
            assert not np.isfinite(lw[i]) or math.isinf(ref), (seed, i, lw[i], ref)
            continue
        assert tol_ok(lw[i], ref, it32.run(draws[i])[0]), (seed, i, lw[i], ref, draws[i], src)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS[:12])
def test_gpu_fuzz_program_masked_lanes(cuda, seed, monkeypatch):
    """The same programs built with 8 particles per thread even where control flow depends on
    particle values (masked lane form, dsl_lanes.cuh)."""
    monkeypatch.setenv("CUPPL_DSL_LANES", "8")
    test_gpu_fuzz_program_matches_interpreter(cuda, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", list(range(16)))
def test_gpu_fuzz_enumeration_matches_forced_choice_oracle(cuda, seed):
    from fuzz_programs import discrete_program
    from oracle.dsl_eval import Enumerator
    from paper_2010_08454_b200 import infer

    src = discrete_program(seed)
    post = infer.run_enumeration(frontend.compile_program(src))
    ref, log_z = Enumerator(src).posterior()
    got = dict(post.support)
    assert set(got) == {k for k, p in ref.items() if p > 0}, (seed, src)
    for k, p in ref.items():
        assert abs(got.get(k, 0.0) - p) < 1e-12, (seed, k, got.get(k), p, src)
    assert abs(post.log_z - log_z) < 1e-10 * max(1.0, abs(log_z)), (seed, post.log_z, log_z)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", list(range(12)))
def test_gpu_fuzz_lmh_matches_enumeration(cuda, seed):
    """LMH on random finite-support programs (mcmc) against their exact enumeration: total
    variation of the return value's distribution (negative values included)."""
    from fuzz_programs import discrete_program
    from paper_2010_08454_b200 import Rng, infer

    src = discrete_program(seed)
    ex = dict(infer.run_enumeration(frontend.compile_program(src)).support)
    mc = infer.run_lmh(frontend.compile_program(src.replace("enumerate(model, 100000)", "mcmc(model, 10)")),
                       3000, Rng(seed), chains=512, burn_in=300)
    got = dict(mc.support)
    assert not mc.support_truncated
    tv = 0.5 * sum(abs(got.get(k, 0.0) - ex.get(k, 0.0)) for k in set(ex) | set(got))
    assert tv < 0.04, (seed, tv, got, ex, src)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", list(range(8)))
def test_gpu_fuzz_importance_matches_enumeration(cuda, seed):
    """Importance sampling of the same random finite-support programs against their exact
    enumeration (negative and > 7 returns go through the full-support second pass)."""
    from fuzz_programs import discrete_program
    from paper_2010_08454_b200 import Rng, infer

    src = discrete_program(seed)
    ex = infer.run_enumeration(frontend.compile_program(src))
    post = infer.run_importance(frontend.compile_program(src.replace("enumerate(model, 100000)",
                                                                     "importance(model, 1000)")),
                                1_000_000, Rng(seed))
    got, exd = dict(post.support), dict(ex.support)
    tv = 0.5 * sum(abs(got.get(k, 0.0) - exd.get(k, 0.0)) for k in set(exd) | set(got))
    assert tv < 0.01 and not post.support_truncated, (seed, tv, got, exd)
    assert abs(post.log_z - ex.log_z) < 0.01


@pytest.mark.gpu
@pytest.mark.parametrize("seed", list(range(12)))
def test_gpu_fuzz_vector_program_matches_interpreter(cuda, seed):
    """Random programs over drawn vectors (repeat of draws with literal or drawn length, reduces,
    Horner over data, indexing by a drawn integer, per-datum draws in map, vector returns)."""
    from fuzz_programs import vector_program
    from oracle.dsl_eval import Fp32Interpreter, Interpreter
    from paper_2010_08454_b200 import Rng, infer

    src = vector_program(seed)
    post = infer.run_importance(frontend.compile_program(src), 2048, Rng(seed), return_traces=True)
    lw = post.traces["log_weight"].cpu().numpy().astype(float)
    draws = post.traces["draws"].cpu().numpy().astype(float)
    it, it32 = Interpreter(src), Fp32Interpreter(src)
    for i in range(0, 2048, 61):
        ref, _ = it.run(draws[i])
        assert tol_ok(lw[i], ref, it32.run(draws[i])[0]), (seed, i, lw[i], ref, src)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1, 3, 4, 9, 13])
def test_gpu_fuzz_lmh_matches_importance_on_vector_programs(cuda, seed):
    """LMH on programs whose trace dimension changes (a drawn vector length: the trace database
    reuses sites by position and kind) against importance sampling of the same
    program: posterior means within a tenth of a posterior sd."""
    from fuzz_programs import vector_program
    from paper_2010_08454_b200 import Rng, infer

    src = vector_program(seed)
    isd = infer.run_importance(frontend.compile_program(src), 4_000_000, Rng(seed))
    mc = infer.run_lmh(frontend.compile_program(src.replace("importance(model, 1000)", "mcmc(model, 10)")),
                       4000, Rng(seed), chains=1024, burn_in=1000)
    sd = max(isd.stats["var_value"], 1e-12) ** 0.5
    assert abs(isd.mean["value"] - mc.mean["value"]) < 0.1 * sd, (seed, isd.mean, mc.mean, sd)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", list(range(8)))
def test_gpu_fuzz_misc_operators(cuda, seed):
    """Integer % and /, floor, to-int, pow, && || !, int-valued ifs, closures over draws."""
    from fuzz_programs import misc_program
    from oracle.dsl_eval import Fp32Interpreter, Interpreter
    from paper_2010_08454_b200 import Rng, infer

    src = misc_program(seed)
    post = infer.run_importance(frontend.compile_program(src), 2048, Rng(seed), return_traces=True)
    lw = post.traces["log_weight"].cpu().numpy().astype(float)
    draws = post.traces["draws"].cpu().numpy().astype(float)
    it, it32 = Interpreter(src), Fp32Interpreter(src)
    for i in range(0, 2048, 61):
        ref, _ = it.run(draws[i])
        assert tol_ok(lw[i], ref, it32.run(draws[i])[0]), (seed, i, lw[i], ref, src)
