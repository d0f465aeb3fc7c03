"""Whole CuPPL programs whose engine results are values (builtins.py:116-123).

In the reference, `importance(model, n)`, `mcmc(model, n)` and `enumerate(model, n)` are
builtins of type ((unit -> t), int) -> ~t: the program gets an empirical DistValue back and may
compute with it, e.g. "importance(coin-model, 100000) inside a program, then dist-var of the
result". Here a program may bind engine results at top level,

    model <- function() { ... };
    post  <- importance(model, 100000);
    v     <- dist-var(post);
    [v, dist-score(post, true)]

Each engine binding compiles its model (frontend.compile_parsed, the same NVRTC sm_100a path
as a program whose result is the engine call) and runs it on the GPU in program order; the
result is an EmpiricalDistribution. The remaining top-level code is evaluated on the host over
those values: numbers, booleans, arithmetic and comparisons, vectors, distribution
constructors (dists.py, the reference's parameter order builtins.py:86-94), dist-var
(analytic for parametric kinds, the weighted variance for the empirical kind)
and dist-score (the log-mass of a value in an empirical posterior's support, or the parametric
density through the batch K8 kernel). Engine n and the per-engine Philox streams: engine
binding k runs with rng.split(k) so programs are reproducible from one seed.
"""

from __future__ import annotations

import math

from . import lang
from .errors import CupError, InferRuntimeError, UnsupportedDistError
from .frontend import CompileError, compile_parsed

ENGINES = ("importance", "mcmc", "enumerate")


def _is_engine(e) -> bool:
    return isinstance(e, lang.Call) and isinstance(e.fn, lang.Var) and e.fn.name in ENGINES


def _free_vars(e, out: set) -> set:
    """Names referenced by an expression (over-approximation: ignores shadowing)."""
    if isinstance(e, lang.Var):
        out.add(e.name)
    elif isinstance(e, (list, tuple)):
        for x in e:
            _free_vars(x, out)
    elif hasattr(e, "__dataclass_fields__"):
        for f in e.__dataclass_fields__:
            _free_vars(getattr(e, f), out)
    return out


class Empirical:
    """An engine result as a program value: the empirical DistValue (values.py 'empirical' kind)."""

    def __init__(self, engine: str, post):
        self.engine = engine
        self.post = post  # infer.EmpiricalDistribution

    def var(self) -> float:
        """Weighted variance of the returned value."""
        st = self.post.stats
        if "var_value" in st:
            return float(st["var_value"])
        if self.post.support and all(isinstance(v, (int, bool)) for v, _ in self.post.support):
            m = sum(float(v) * p for v, p in self.post.support)
            return sum(p * (float(v) - m) ** 2 for v, p in self.post.support)
        raise UnsupportedDistError("dist-var needs a scalar-valued posterior (builtins.py:100: ~a -> real)")

    def score(self, v) -> float:
        """Natural log of the posterior mass of v (discrete support; -inf outside it)."""
        if not self.post.support:
            raise UnsupportedDistError("dist-score of an empirical posterior over real values: each value "
                                       "has singleton support (SPEC.md:448); only discrete posteriors are scored")
        for x, p in self.post.support:
            if x == v and isinstance(x, bool) == isinstance(v, bool):
                return math.log(p) if p > 0 else -math.inf
        return -math.inf


class CompiledProgram:
    """A parsed program with its engine bindings compiled for the GPU."""

    def __init__(self, source: str, data: dict | None = None, max_depth: int = 20):
        prog = lang.parse(source)
        self.source = source
        self.prog = prog
        engine_names = set()
        self.steps = []  # ("engine", name, CompiledModel, n) | ("host", name, expr)
        model_bindings = []
        for name, e in prog.bindings:
            deps = _free_vars(e, set())
            if _is_engine(e):
                if len(e.args) != 2:
                    raise CompileError(f"{e.fn.name} takes (model, n)")
                sub = lang.Program(bindings=list(model_bindings), result=e)
                cm = compile_parsed(sub, source, data, max_depth)
                self.steps.append(("engine", name, cm, cm.default_n))
                engine_names.add(name)
            elif deps & engine_names:
                self.steps.append(("host", name, e))
                engine_names.add(name)  # host values derived from posteriors stay on the host
            else:
                model_bindings.append((name, e))
                self.steps.append(("host", name, e))
        self.result = prog.result
        self.result_engine = None
        if _is_engine(prog.result):
            sub = lang.Program(bindings=list(model_bindings), result=prog.result)
            self.result_engine = compile_parsed(sub, source, data, max_depth)
        self.data = data or {}

    @property
    def engines(self) -> list:
        out = [cm for kind, *rest in self.steps if kind == "engine" for cm in [rest[1]]]
        if self.result_engine is not None:
            out.append(self.result_engine)
        return out

    def run(self, rng, *, chains: int = 4096):
        """Run every engine in program order (engine k on rng.split(k)) and evaluate the result."""
        from . import infer

        env: dict = {k: list(v) for k, v in self.data.items()}
        k = 0

        def run_engine(cm):
            nonlocal k
            r = rng.split(k)
            k += 1
            if cm.engine == "enumerate":
                return Empirical("enumerate", infer.run_enumeration(cm, cm.default_n))
            if cm.engine == "mcmc":  # as `cuppl run`: n steps in each of `chains` chains
                return Empirical("mcmc", infer.run_lmh(cm, cm.default_n, r, chains=chains))
            return Empirical("importance", infer.run_importance(cm, cm.default_n, r))

        for step in self.steps:
            if step[0] == "engine":
                env[step[1]] = run_engine(step[2])
            else:
                _, name, e = step
                if isinstance(e, lang.Lambda):
                    env[name] = e  # model functions: used only by engines
                    continue
                env[name] = _HostEval(env).ev(e)
        if self.result_engine is not None:
            return run_engine(self.result_engine).post
        v = _HostEval(env).ev(self.result)
        return v.post if isinstance(v, Empirical) else v


def run_program(source: str, rng, *, data: dict | None = None, chains: int = 4096):
    """Compile and run a whole program; returns its final value (an EmpiricalDistribution when
    the value is an engine result)."""
    return CompiledProgram(source, data).run(rng, chains=chains)


class _HostEval:
    """Top-level code over engine results (module docstring)."""

    CONSTRUCTORS = {"normal": "normal", "bernoulli": "bernoulli", "poisson": "poisson",
                    "uniform-discrete": "uniform_discrete", "uniform-continuous": "uniform_continuous",
                    "beta": "beta", "exponential": "exponential", "categorical": "categorical"}

    def __init__(self, env: dict):
        self.env = env

    def ev(self, e):
        if isinstance(e, lang.Num):
            return e.value
        if isinstance(e, lang.Bool):
            return e.value
        if isinstance(e, lang.Var):
            if e.name not in self.env:
                raise CompileError(f"unbound variable {e.name}")
            return self.env[e.name]
        if isinstance(e, lang.VecLit):
            return [self.ev(x) for x in e.elems]
        if isinstance(e, lang.Unary):
            a = self.ev(e.arg)
            return -a if e.op == "-" else (not a)
        if isinstance(e, lang.BinOp):
            a, b = self.ev(e.lhs), self.ev(e.rhs)
            op = e.op
            if op in ("&&", "||"):
                return (a and b) if op == "&&" else (a or b)
            if op == "/" and isinstance(a, int) and isinstance(b, int) and not isinstance(a, bool):
                return int(a / b)
            return {"+": lambda: a + b, "-": lambda: a - b, "*": lambda: a * b, "/": lambda: a / b,
                    "%": lambda: math.fmod(a, b), "==": lambda: a == b, "!=": lambda: a != b,
                    "<": lambda: a < b, "<=": lambda: a <= b, ">": lambda: a > b, ">=": lambda: a >= b}[op]()
        if isinstance(e, lang.If):
            return self.ev(e.then if self.ev(e.cond) else e.orelse)
        if isinstance(e, lang.Index):
            return self.ev(e.vec)[int(self.ev(e.idx))]
        if isinstance(e, lang.Call) and isinstance(e.fn, lang.Var):
            return self.call(e.fn.name, e.args)
        raise CompileError(f"{type(e).__name__} is not supported in top-level code over engine results")

    def call(self, name, args):
        from . import dists

        vals = [self.ev(a) for a in args]
        if name in self.CONSTRUCTORS:
            return getattr(dists, self.CONSTRUCTORS[name])(*vals)
        if name == "dist-var":
            d = vals[0]
            return d.var() if isinstance(d, Empirical) else dists.variance(d)
        if name == "dist-score":
            d, v = vals
            if isinstance(d, Empirical):
                return d.score(v)
            import torch

            x = torch.tensor([float(v)], device="cuda")
            return float(dists.score(d, x).cpu()[0])
        if name in ("exp", "log", "sqrt", "abs", "floor"):
            x = float(vals[0])
            if name == "log":
                return math.log(x) if x > 0 else (-math.inf if x == 0 else math.nan)
            return {"exp": math.exp, "sqrt": math.sqrt, "abs": abs, "floor": math.floor}[name](x)
        if name == "length":
            return len(vals[0])
        if name == "to-real":
            return float(vals[0])
        if name == "to-int":
            return int(vals[0])
        if name in ENGINES:
            raise CompileError("engine calls in expressions must be bound at top level")
        raise CompileError(f"{name} is not available in top-level code over engine results")


__all__ = ["CompiledProgram", "Empirical", "run_program", "CupError", "InferRuntimeError"]
