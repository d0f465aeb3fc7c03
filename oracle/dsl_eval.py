"""fp64 interpreter of CuPPL GPU-subset programs with INJECTED draws — TEST INFRASTRUCTURE.

Parity oracle of the model compiler (paper_2010_08454_b200/frontend.py): it evaluates the
same AST (paper_2010_08454_b200/lang.py) directly, with the importance engine's semantics
(SPEC.md:399-407): `sample(d)` returns the next injected draw (the GPU records every draw of a
particle in program order), `factor(x)` adds x to the log-weight, `observe(d, v)` adds
dist-score(d, v) (cuppl/desugar.py:37-39); `repeat` evaluates its function eagerly in index
order, `reduce` is a left fold, `map` applies elementwise. Scores use
oracle/semantics.py. Data vectors are rounded to fp32 like the GPU's.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2010_08454_b200 import lang

from . import semantics as sem

_TAGS = {"normal": sem.NORMAL, "bernoulli": sem.BERNOULLI, "poisson": sem.POISSON,
         "uniform-discrete": sem.UNIFORM_DISCRETE, "uniform-continuous": sem.UNIFORM_CONTINUOUS,
         "beta": sem.BETA, "exponential": sem.EXPONENTIAL, "categorical": sem.CATEGORICAL}
_KIND = {"normal": float, "uniform-continuous": float, "beta": float, "exponential": float,
         "uniform-discrete": int, "poisson": int, "bernoulli": bool, "categorical": int}


class _Fn:
    def __init__(self, params, body, env):
        self.params, self.body, self.env = params, body, env


class _Dist:
    def __init__(self, kind, args):
        self.kind, self.args = kind, args


class Interpreter:
    F32_LITERALS = True  # literals and data as the fp32 GPU kernels see them

    def _rl(self, v):
        return float(np.float32(v)) if self.F32_LITERALS else float(v)

    def __init__(self, source: str, data: dict | None = None):
        self.prog = lang.parse(source)
        self.globals = {}
        for name, arr in (data or {}).items():
            self.globals[name] = [self._rl(v) for v in np.asarray(arr).reshape(-1)]
        for name, e in self.prog.bindings:
            if isinstance(e, lang.VecLit):
                self.globals[name] = [self._rl(self._const(x)) for x in e.elems]
            else:
                self.globals[name] = self.ev(e, {})
        res = self.prog.result
        self.model = self.ev(res.args[0], {})

    def _const(self, e):
        if isinstance(e, lang.Num):
            return e.value
        if isinstance(e, lang.Unary) and e.op == "-":
            return -self._const(e.arg)
        raise ValueError("non-constant vector element")

    def run(self, draws):
        """One particle: injected draws (in program order) -> (log-weight, return value)."""
        self._draws = list(draws)
        self._k = 0
        self._lw = 0.0
        ret = self.apply(self.model, [])
        return self._lw, ret

    # ------------------------------------------------------------------------------------
    def apply(self, f, args):
        env = dict(f.env)
        env.update(zip(f.params, args))
        return self.ev(f.body, env)

    def ev(self, e, env):
        if isinstance(e, lang.Num):
            return self._rl(e.value) if isinstance(e.value, float) else e.value
        if isinstance(e, lang.Bool):
            return e.value
        if isinstance(e, lang.Var):
            if e.name in env:
                return env[e.name]
            return self.globals[e.name]
        if isinstance(e, lang.Lambda):
            return _Fn(e.params, e.body, dict(env))
        if isinstance(e, lang.Block):
            env = dict(env)
            for name, rhs in e.stmts:
                v = self.ev(rhs, env)
                if name is not None:
                    env[name] = v
            return self.ev(e.result, env)
        if isinstance(e, lang.Unary):
            a = self.ev(e.arg, env)
            return -a if e.op == "-" else (not a)
        if isinstance(e, lang.BinOp):
            a, b = self.ev(e.lhs, env), self.ev(e.rhs, env)
            op = e.op
            if op == "+":
                return a + b
            if op == "-":
                return a - b
            if op == "*":
                return a * b
            if op == "/":
                return int(a / b) if isinstance(a, int) and isinstance(b, int) else a / b
            if op == "%":
                return math.fmod(a, b)
            return {"==": a == b, "!=": a != b, "<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b,
                    "&&": a and b, "||": a or b}[op]
        if isinstance(e, lang.If):
            return self.ev(e.then if self.ev(e.cond, env) else e.orelse, dict(env))
        if isinstance(e, lang.Index):
            return self.ev(e.vec, env)[int(self.ev(e.idx, env))]
        if isinstance(e, lang.VecLit):
            return [self.ev(x, env) for x in e.elems]
        if isinstance(e, lang.Call):
            return self.call(e, env)
        raise ValueError(type(e).__name__)

    def call(self, e, env):
        if isinstance(e.fn, lang.Var) and e.fn.name not in env and e.fn.name not in self.globals:
            n = e.fn.name
            args = [self.ev(a, env) for a in e.args] if n not in ("repeat", "map", "reduce") else None
            if n in _TAGS:
                return _Dist(n, args)
            if n in ("sample", "sample*"):
                d = args[0]
                v = self._draws[self._k]
                self._k += 1
                return _KIND[d.kind](v)
            if n == "factor":
                self._lw += float(args[0])
                return None
            if n in ("observe", "dist-score"):
                d, v = args
                s = sem.dist_score(_TAGS[d.kind], d.args, v)
                if n == "dist-score":
                    return s
                self._lw += s
                return None
            if n in ("exp", "log", "sqrt", "abs", "floor"):
                x = float(args[0])
                if n == "log":
                    return math.log(x) if x > 0 else (-math.inf if x == 0 else math.nan)
                return {"exp": math.exp, "sqrt": math.sqrt, "abs": abs, "floor": math.floor}[n](x)
            if n == "pow":
                return float(args[0]) ** float(args[1])
            if n == "to-real":
                return float(args[0])
            if n == "to-int":
                return int(args[0])
            if n == "length":
                return len(args[0])
            f = self.ev(e.args[0], env)
            if n == "repeat":
                return [self.apply(f, [i]) for i in range(int(self.ev(e.args[1], env)))]
            if n == "map":
                return [self.apply(f, [x]) for x in self.ev(e.args[1], env)]
            if n == "reduce":
                acc = self.ev(e.args[1], env)
                for x in self.ev(e.args[2], env):
                    acc = self.apply(f, [acc, x])
                return acc
            raise ValueError(n)
        f = self.ev(e.fn, env)
        return self.apply(f, [self.ev(a, env) for a in e.args])


class _NeedChoice(Exception):
    def __init__(self, support):
        super().__init__()
        self.support = support


class Enumerator(Interpreter):
    """Exact enumeration by re-execution (SPEC.md:438's brute-force forced-choice oracle):
    a run with a choice prefix either completes or asks for the next choice point's support;
    every completed path contributes exp(sum of choice log-masses + factors). Literals and data
    stay fp64, as in the GPU's fp64 enumeration kernels (frontend.py)."""

    F32_LITERALS = False

    def run_forced(self, prefix):
        self._prefix = prefix
        self._k = 0
        self._lw = 0.0
        ret = self.apply(self.model, [])
        return self._lw, ret

    def call(self, e, env):
        if isinstance(e.fn, lang.Var) and e.fn.name in ("sample", "sample*") and e.fn.name not in env:
            d = self.ev(e.args[0], env)
            if d.kind == "bernoulli":
                support = [True, False]
            elif d.kind == "uniform-discrete":
                support = list(range(int(d.args[0]), int(d.args[1])))
            elif d.kind == "categorical":
                support = list(range(len(d.args[0])))
            else:
                raise ValueError(f"{d.kind} has no finite support")
            if self._k >= len(self._prefix):
                raise _NeedChoice(support)
            v = self._prefix[self._k]
            self._k += 1
            self._lw += sem.dist_score(_TAGS[d.kind], d.args, v)
            return v
        return super().call(e, env)

    def posterior_bfs(self, max_executions: int):
        """The reference's breadth-first traversal: a FIFO frontier of choice
        prefixes, children in support order; stops after max_executions completed paths and
        normalises over them."""
        from collections import deque

        mass, done, q = {}, 0, deque([[]])
        while q and done < max_executions:
            prefix = q.popleft()
            try:
                lw, ret = self.run_forced(prefix)
            except _NeedChoice as need:
                q.extend(prefix + [v] for v in need.support)
                continue
            key = tuple(ret) if isinstance(ret, list) else ret
            mass[key] = mass.get(key, 0.0) + math.exp(lw)
            done += 1
        z = sum(mass.values())
        return {k: v / z for k, v in mass.items()}, math.log(z)

    def posterior(self):
        """{return value: probability}, log evidence (fp64)."""
        mass, stack = {}, [[]]
        while stack:
            prefix = stack.pop()
            try:
                lw, ret = self.run_forced(prefix)
            except _NeedChoice as need:
                stack.extend(prefix + [v] for v in need.support)
                continue
            key = tuple(ret) if isinstance(ret, list) else ret
            mass[key] = mass.get(key, 0.0) + math.exp(lw)
        z = sum(mass.values())
        return {k: v / z for k, v in mass.items()}, math.log(z)


def _f32(x):
    return float(np.float32(x)) if isinstance(x, float) else x


class Fp32Interpreter(Interpreter):
    """The same interpreter rounding every real-valued operation to fp32 (round to nearest per
    operation; no FMA contraction, correctly rounded functions). Its distance from the fp64
    result measures how much fp32 arithmetic itself moves a given program's log-weight — the
    conditioning term of the compiler's parity tolerance (tests/test_frontend_fuzz.py): random
    expression trees can cancel, where no fixed relative tolerance holds for any fp32 code."""

    def run(self, draws):
        self._draws = [_f32(float(d)) for d in draws]
        self._k = 0
        self._lw = 0.0
        ret = self.apply(self.model, [])
        return self._lw, ret

    def ev(self, e, env):
        v = super().ev(e, env)
        if isinstance(e, (lang.BinOp, lang.Unary)):
            return _f32(v)
        return v

    def call(self, e, env):
        if isinstance(e.fn, lang.Var) and e.fn.name in ("factor", "observe") and e.fn.name not in env \
                and e.fn.name not in self.globals:
            before = self._lw
            out = super().call(e, env)
            self._lw = _f32(self._lw) if self._lw != before else self._lw
            return out
        return _f32(super().call(e, env))
