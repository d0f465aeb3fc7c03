"""GPU model compiler: CuPPL source -> CUDA C++ -> NVRTC (sm_100a) -> importance sampling.

SURVEY.md §8(f) row 1 (the paper's NVVM code-generation story): a model
written in CuPPL reaches the GPU without a hand-registered descriptor.

    src = '''
      xs <- [-1.0, 0.0, 1.0];  ys <- [2.1, 0.9, 0.2];
      model <- function() {
        a <- sample(normal(0, 10));
        b <- sample(normal(0, 10));
        factor(reduce(function(acc, i) { acc + dist-score(normal(a * xs[i] + b, 1), ys[i]) },
                      0, repeat(function(i) { i }, length(xs))));
        [a, b]
      };
      importance(model, 100000)
    '''
    m = frontend.compile_program(src)
    post = infer.run_importance(m, 10**8, Rng(1))

Semantics (the reference's importance engine): each particle runs the model
once; `sample(d)` draws from the prior, `factor(x)` adds x to the log-weight, `observe(d, v)`
is factor(dist-score(d, v)) (cuppl/desugar.py:37-39). Every particle owns one word stream
(Philox blocks (pid, 0..), tag CUPPL_TAG_DSL) consumed in program order by the reference draw
algorithms (rng.py:43-117; csrc/draws.cuh) — the GPU form of rng.split(i).

The compiler is a staged evaluator: the program is evaluated at compile time over symbolic
values (scalars are C++ expressions, data vectors live in one device buffer, user functions
and closures are inlined at their call sites), and side effects (draws, factors) are emitted
as CUDA statements in program order. `repeat` / `map` are fused into the `reduce` that
consumes them unless they draw, in which case they are materialised in program order into a
bounded local array. The supported subset is first-order: scalars (real, int, bool), vectors
of bounded length, no recursion, no unit-returning user functions as values.

The kernel fuses the model with the importance-sampling record (log-sum-exp, ESS, mode,
moments of the returned components, histogram of a discrete return or of a returned vector's
length) exactly like the hand-written kernels (csrc/is_accum.cuh).

Engines: a program's result selects the kernel — `importance(model, n)` (above),
`enumerate(model, n)` (forced choices: thread p runs the path given by the base-R digits of p,
SPEC.md:438) and `mcmc(model, n)` (many single-site LMH chains with a per-thread trace
database).

Lanes (csrc/dsl_lanes.cuh): the body is emitted once in lane-polymorphic C++ (VF / VI / VB,
sel, to_f, lifted math, mask-aware draws). Importance kernels are built with several particles
per thread when that compiles without spills and the program has no particle-dependent
control flow; otherwise with one. Peepholes: Gaussian-likelihood reduces (and map / repeat of
observe) become packed FFMA2 loops over pairs of data points; literal-init reduces are peeled
with exact constant folds.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import lang
from .errors import CupError, InferRuntimeError, InvalidDistParamError

CSRC = Path(__file__).resolve().parent / "csrc"
INCLUDE = Path(__file__).resolve().parent.parent / "include"
TAG_DSL = 8  # CUPPL_TAG_DSL
TAG_DSL_MH = 9  # CUPPL_TAG_DSL_MH: LMH step streams, id = step << 32 | chain
MAX_STATS = 16  # cuppl_is_record.stat_w
MAX_BINS = 8   # cuppl_is_record.bin_w
MCMC_BINS, MCMC_BIN_LO = 128, -32  # chain histograms of integer returns: values [-32, 96)
MAX_TRACE_DRAWS = 256
MAX_CONST_DATA = 16_000  # floats kept in the module's __constant__ bank (64 KB); larger: __ldg
# Bytes of padding before the constant-bank data (multiple of 8): where the data starts
# relative to 32-byte bank boundaries changes the speed of the point loops (is_kernels.cuh
# kXyOffset). Measured on the dsl-linreg bench: 16 bytes past a 32-byte boundary 103.2 ms per
# 1e9 particles, offsets 0 / 8 / 24 bytes 104.4-104.9 ms. CUPPL_DC_PAD_BYTES overrides it
# (tuning only).
_DC_PAD = int(os.environ.get("CUPPL_DC_PAD_BYTES", "16")) // 8
DATA_SYM = "DATA"        # resolved by the kernel prelude to the constant bank or the buffer
DSL_LANES = 8            # particles per thread of an importance kernel (CUPPL_DSL_LANES overrides)


class CompileError(CupError):
    kind = "compile"


# ----------------------------------------------------------------------------- values ----
@dataclass
class S:
    """A scalar: C++ expression `code` of type real | int | bool."""

    code: str
    ty: str
    pure: bool = True  # no side effects (draws / factors) were needed to produce it
    mul: tuple | None = None  # packed product (x, y): a following add fuses into one fma2
    finite: bool = False  # known finite (a literal, an element of finite data): 0 * x == 0


@dataclass
class DataVec:
    off: int
    n: int
    finite: bool = True  # every element is a finite number (checked when the data are bound)

    def length(self):
        return S(str(self.n), "int")

    def bound(self):
        return self.n

    def elem(self, comp, i: S):
        if i.ty == "int2":  # elements i, i + 1 as one 8-byte load (offsets are even, i is even)
            return S(f"{DATA_SYM}2({self.off} + ({i.code}))", "real2")
        return S(f"{DATA_SYM}({self.off} + ({i.code}))", "real", finite=self.finite)


@dataclass
class LocVec:
    var: str
    bound_: int
    length_: S
    ty: str

    def length(self):
        return self.length_

    def bound(self):
        return self.bound_

    def elem(self, comp, i: S):
        if _is_literal(i.code) or self.bound_ > 8:
            return S(f"{self.var}[{i.code}]", self.ty)
        # small vector, computed index: a select chain over static elements keeps the array
        # in registers (a dynamic index would spill it to local memory)
        k = comp.g.let(i, "k")
        code = f"{self.var}[{self.bound_ - 1}]"
        for j in range(self.bound_ - 2, -1, -1):
            code = f"sel({k.code} == {j}, {self.var}[{j}], {code})"
        return S(code, self.ty)


@dataclass
class LazyVec:
    """repeat(f, n) / map(f, v) with a pure element function: elements built on demand."""

    length_: S
    bound_: int | None
    gen: object  # callable(compiler, index S) -> value

    def length(self):
        return self.length_

    def bound(self):
        return self.bound_

    def elem(self, comp, i: S):
        return self.gen(comp, i)


@dataclass
class ConstVec:
    """A vector literal of model values (a returned tuple such as [a, b])."""

    items: list

    def length(self):
        return S(str(len(self.items)), "int")

    def bound(self):
        return len(self.items)


@dataclass
class Fn:
    params: list
    body: object
    env: dict
    name: str = "<lambda>"


@dataclass
class Dist:
    kind: str
    args: list


_DISTS = {  # name: (arity, sample type)
    "normal": (2, "real"), "uniform-continuous": (2, "real"), "uniform-discrete": (2, "int"),
    "bernoulli": (1, "bool"), "beta": (2, "real"), "exponential": (1, "real"), "poisson": (1, "int"),
    "categorical": (1, "int"),  # categorical(weights): a vector of static length
}
MAX_CATEGORIES = 32
_KIND_CODE = {"normal": 0, "uniform-continuous": 1, "uniform-discrete": 2, "bernoulli": 3, "beta": 4,
              "exponential": 5, "poisson": 6, "categorical": 7}
_MATH1 = {"exp": "expf", "log": "logf", "sqrt": "sqrtf", "abs": "fabsf", "floor": "floorf"}
_CMP = {"==", "!=", "<", "<=", ">", ">="}


# ----------------------------------------------------------------------------- codegen ---
class _Gen:
    def __init__(self, data: list):
        self.lines: list[str] = []
        self.ind = 2
        self.n = 0
        self.data = data  # flat float list of all data vectors
        self.draw_bound = 0  # upper bound of sample calls per particle
        self.loop_mult = [1]
        self.depth = 0
        self.bounds: dict = {}  # C variable of a uniform-discrete draw -> largest value
        self.masks: list = []  # (indent, C name) of the open particle masks, innermost last
        self.calls: list = []  # user functions being inlined (recursion depth per function)
        self.masked = False  # some control flow depends on particle values

    def fresh(self, p="t"):
        self.n += 1
        return f"{p}{self.n}"

    def emit(self, line: str):
        self.lines.append(" " * self.ind + line)

    def open(self, head: str):
        self.emit(head + " {")
        self.ind += 2

    def close(self):
        self.ind -= 2
        self.emit("}")
        while self.masks and self.masks[-1][0] > self.ind:
            self.masks.pop()

    def mask(self):
        """The innermost open particle mask (None at the top level of the model)."""
        return self.masks[-1][1] if self.masks else None

    def open_masked(self, cond: str):
        """`if (cond)` on particle values (dsl_lanes.cuh): the block runs when some lane needs
        it, and its effects apply to the lanes of mask (outer masks && cond)."""
        m = self.fresh("m")
        self.masked = True
        outer = self.mask()
        self.emit(f"const auto {m} = {outer + ' && ' if outer else ''}({cond});")
        self.open(f"if (lanes_any({m}))")
        self.masks.append((self.ind, m))

    def assign(self, var: str, expr: str):
        """var = expr in the active lanes."""
        m = self.mask()
        self.emit(f"masked_set({var}, {m}, {expr});" if m else f"{var} = {expr};")

    def add_lw(self, x: str):
        m = self.mask()
        self.emit(f"masked_add(lw, {m}, {x});" if m else f"lw += {x};")

    def valid_m(self) -> str:
        m = self.mask()
        return f"valid && {m}" if m else "valid"

    def draw_m(self) -> str:
        return self.mask() or "true"

    def let(self, v: S, hint="t") -> S:
        if v.code.isidentifier() or _is_literal(v.code):
            return v
        name = self.fresh(hint)
        self.emit(f"const auto {name} = {v.code};")
        return S(name, v.ty, v.pure, finite=v.finite)


def _cty(ty):
    return {"real": "VF", "int": "VI", "bool": "VB", "real2": "VF2", "int2": "int"}[ty]


class _PairUnsupported(Exception):
    """An operation without a packed (two data points per instruction) form: the peephole
    falls back to the scalar loop."""


def _pair(v: S) -> str:
    """f32x2 code of a scalar (broadcast) or packed value."""
    if v.ty == "real2":
        return v.code
    if v.ty in ("int2", "bool"):
        raise _PairUnsupported(v.ty)
    r = _real(v)
    return f"pack2({r}, {r})"


def _is_literal(code: str) -> bool:
    try:
        float(code.rstrip("f"))
        return True
    except ValueError:
        return code in ("true", "false")


# Real arithmetic of the model being compiled: fp32 (importance / mcmc kernels)
# or fp64 (enumerate: path probabilities are exact to ~1e-15, SPEC.md:438 asks 1e-12); set by
# compile_parsed for the duration of one compilation.
_F64 = False
_COMPILE_LOCK = __import__("threading").Lock()


def _fconst(x: float) -> str:
    """A real constant folded at compile time, in the model's real type."""
    return repr(float(x)) if _F64 else repr(float(np.float32(x))) + "f"


def _lit(v) -> S:
    if isinstance(v, bool):
        return S("true" if v else "false", "bool")
    if isinstance(v, int):
        return S(str(v), "int", finite=True)
    if _F64:
        return S(repr(float(v)), "real", finite=math.isfinite(v))
    f = float(np.float32(v))
    return S(repr(f) + "f", "real", finite=math.isfinite(f))


def _real_lit(v: S, value: float) -> bool:
    return v.ty == "real" and _is_literal(v.code) and float(v.code.rstrip("f")) == value


def _real(v: S) -> str:
    if v.ty in ("real2", "int2"):
        raise _PairUnsupported(v.ty)
    return f"to_f({v.code})" if v.ty != "real" else v.code


def _scalar(v, what) -> S:
    if not isinstance(v, S):
        raise CompileError(f"{what}: expected a scalar, got {type(v).__name__}")
    return v


class _Compiler:
    def __init__(self, prog: lang.Program, data: dict | None, max_depth: int = 20):
        self.prog = prog
        self.g = _Gen([])
        self.globals: dict = {}
        self.external = dict(data or {})
        self.model = None
        self.default_n = None
        self.engine = "importance"
        self.radix = 1  # enumeration: largest support size of a choice point
        self.max_depth = max_depth  # enumeration: recursion bound per function

    # -------------------------------------------------------------- top level ----
    def _data_vec(self, values) -> DataVec:
        arr = np.asarray(values, dtype=np.float64).reshape(-1)
        if len(self.g.data) % 2:  # even offsets: pairs of elements load as one f32x2
            self.g.data.append(0.0)
        off = len(self.g.data)
        vals = arr if _F64 else np.float32(arr)
        self.g.data.extend(vals.tolist())
        return DataVec(off, len(arr), bool(np.isfinite(vals).all()))

    def top(self):
        for name, e in self.prog.bindings:
            self.globals[name] = self._global_value(name, e)
        res = self.prog.result
        if not (isinstance(res, lang.Call) and isinstance(res.fn, lang.Var)
                and res.fn.name in ("importance", "enumerate", "mcmc")):
            raise CompileError("the program result must be importance(model, n), mcmc(model, n) or "
                               "enumerate(model, max_executions)")
        self.engine = res.fn.name
        if len(res.args) != 2:
            raise CompileError(f"{self.engine} takes (model, n)")
        m = self._global_value("<model>", res.args[0])
        if not isinstance(m, Fn) or m.params:
            raise CompileError("importance's first argument must be a zero-argument model function")
        n = self._global_value("<n>", res.args[1])
        if not (isinstance(n, S) and n.ty == "int" and _is_literal(n.code)):
            raise CompileError("importance's sample count must be an integer constant")
        self.model, self.default_n = m, int(n.code)

    def _global_value(self, name, e):
        if isinstance(e, lang.VecLit):
            vals = []
            for x in e.elems:
                v = self._global_value(name, x)
                if not (isinstance(v, S) and _is_literal(v.code)):
                    raise CompileError(f"top-level vector {name} must hold numeric constants")
                vals.append(float(v.code.rstrip("f")) if v.code not in ("true", "false") else float(v.code == "true"))
            return self._data_vec(vals)
        if isinstance(e, lang.Num):
            return _lit(e.value)
        if isinstance(e, lang.Bool):
            return _lit(e.value)
        if isinstance(e, lang.Unary) and e.op == "-" and isinstance(e.arg, lang.Num):
            return _lit(-e.arg.value)
        if isinstance(e, lang.Lambda):
            return Fn(e.params, e.body, self.globals, name)
        if isinstance(e, lang.Var):
            return self._lookup(e.name, self.globals)
        raise CompileError(f"top-level binding {name}: only constants, numeric vectors and functions "
                           "are supported outside the model")

    def _lookup(self, name, env):
        if name in env:
            return env[name]
        if name in self.globals:
            return self.globals[name]
        if name in self.external:
            v = self._data_vec(self.external.pop(name))
            self.globals[name] = v
            return v
        raise CompileError(f"unbound variable {name}")

    # -------------------------------------------------------------- expressions --
    def ev(self, e, env):
        g = self.g
        if isinstance(e, lang.Num):
            return _lit(e.value)
        if isinstance(e, lang.Bool):
            return _lit(e.value)
        if isinstance(e, lang.Var):
            if e.name in _DISTS or e.name in _MATH1:
                raise CompileError(f"builtin {e.name} must be applied")
            return self._lookup(e.name, env)
        if isinstance(e, lang.Lambda):
            return Fn(e.params, e.body, dict(env))
        if isinstance(e, lang.Block):
            env = dict(env)
            for name, rhs in e.stmts:
                v = self.ev(rhs, env)
                if isinstance(v, S) and not v.pure:
                    v = g.let(v)
                if name is not None:
                    env[name] = g.let(v, "v") if isinstance(v, S) else v
            return self.ev(e.result, env)
        if isinstance(e, lang.Unary):
            a = _scalar(self.ev(e.arg, env), e.op)
            if a.ty in ("real2", "int2"):
                if e.op != "-" or a.ty == "int2":
                    raise _PairUnsupported(e.op)
                return S(f"mul2({a.code}, pack2(-1.f, -1.f))", "real2", a.pure)
            if e.op == "-" and a.ty in ("int", "real") and _is_literal(a.code):
                return _lit(-int(a.code) if a.ty == "int" else -float(a.code.rstrip("f")))  # a constant
            if e.op == "-":
                return S(f"(-{a.code})", a.ty if a.ty != "bool" else "int", a.pure)
            return S(f"(!{a.code})", "bool", a.pure)
        if isinstance(e, lang.BinOp):
            return self._binop(e, env)
        if isinstance(e, lang.If):
            return self._if(e, env)
        if isinstance(e, lang.Index):
            v = self.ev(e.vec, env)
            i = _scalar(self.ev(e.idx, env), "index")
            if i.ty == "int2" and not isinstance(v, DataVec):
                raise _PairUnsupported("pair index into a non-data vector")
            if i.ty not in ("int", "int2"):
                raise CompileError("vector index must be an int")
            if isinstance(v, ConstVec):
                if not _is_literal(i.code):
                    raise CompileError("a vector literal of model values is indexed by constants only")
                return v.items[int(i.code)]
            if not hasattr(v, "elem"):
                raise CompileError("indexing a non-vector")
            return v.elem(self, i)
        if isinstance(e, lang.VecLit):
            items = [self.ev(x, env) for x in e.elems]
            if all(isinstance(x, S) and _is_literal(x.code) for x in items):
                return self._data_vec([float(x.code.rstrip("f")) if x.ty != "bool" else float(x.code == "true")
                                       for x in items])
            return ConstVec([_scalar(x, "vector element") for x in items])
        if isinstance(e, lang.Call):
            return self._call(e, env)
        raise CompileError(f"unsupported expression {type(e).__name__}")

    def _binop(self, e, env):
        a = _scalar(self.ev(e.lhs, env), e.op)
        b = _scalar(self.ev(e.rhs, env), e.op)
        pure = a.pure and b.pure
        if "real2" in (a.ty, b.ty) or "int2" in (a.ty, b.ty):
            if e.op == "+":
                if a.mul is not None:
                    return S(f"fma2({a.mul[0]}, {a.mul[1]}, {_pair(b)})", "real2", pure)
                if b.mul is not None:
                    return S(f"fma2({b.mul[0]}, {b.mul[1]}, {_pair(a)})", "real2", pure)
                return S(f"add2({_pair(a)}, {_pair(b)})", "real2", pure)
            if e.op == "-":
                return S(f"fma2({_pair(b)}, pack2(-1.f, -1.f), {_pair(a)})", "real2", pure)
            if e.op == "*":
                pa, pb = _pair(a), _pair(b)
                return S(f"mul2({pa}, {pb})", "real2", pure, mul=(pa, pb))
            raise _PairUnsupported(e.op)
        if e.op in ("&&", "||"):
            return S(f"({a.code} {e.op} {b.code})", "bool", pure)
        if e.op in _CMP:
            if "real" in (a.ty, b.ty):
                return S(f"({_real(a)} {e.op} {_real(b)})", "bool", pure)
            return S(f"({a.code} {e.op} {b.code})", "bool", pure)
        if a.ty == "int" and b.ty == "int":
            return S(f"({a.code} {e.op} {b.code})", "int", pure)
        if a.ty == "real" and b.ty == "real":  # exact folds (up to the sign of a zero)
            if e.op == "*" and (_real_lit(a, 0.0) and b.finite or _real_lit(b, 0.0) and a.finite):
                return S("0.0f", "real", pure, finite=True)
            if e.op == "*" and _real_lit(a, 1.0):
                return b
            if e.op == "*" and _real_lit(b, 1.0) or e.op in ("+", "-") and _real_lit(b, 0.0):
                return a
            if e.op == "+" and _real_lit(a, 0.0):
                return b
        if e.op == "%":
            return S(f"fmodf({_real(a)}, {_real(b)})", "real", pure)
        return S(f"({_real(a)} {e.op} {_real(b)})", "real", pure)

    def _if(self, e, env):
        g = self.g
        c = _scalar(self.ev(e.cond, env), "if condition")
        mark, b0 = len(g.lines), g.draw_bound
        if not (self._effects(e.then, env) or self._effects(e.orelse, env)):
            # pure branches: both evaluated, one select (no probe of effectful branches: with
            # recursion that would evaluate every level twice)
            t = self.ev(e.then, dict(env))
            f = self.ev(e.orelse, dict(env))
            g.draw_bound = b0
            if len(g.lines) == mark and isinstance(t, S) and isinstance(f, S) and t.pure and f.pure:
                ty = "real" if "real" in (t.ty, f.ty) else t.ty
                tc, fc = (_real(t), _real(f)) if ty == "real" else (t.code, f.code)
                return S(f"sel({c.code}, {tc}, {fc})", ty, c.pure)
        # side effects in a branch: emit real control flow (draws happen on the taken path only)
        del g.lines[mark:]
        res = g.fresh("r")
        g.emit(f"VF {res} = 0.f;")
        cv = g.let(c, "c")
        g.open_masked(cv.code)
        t = self.ev(e.then, dict(env))
        tt = t.ty if isinstance(t, S) else None
        if isinstance(t, S):
            g.assign(res, _real(t))
        g.close()
        bt, g.draw_bound = g.draw_bound - b0, b0
        g.open_masked(f"!{cv.code}")
        f = self.ev(e.orelse, dict(env))
        if isinstance(f, S):
            g.assign(res, _real(f))
        g.close()
        g.draw_bound = b0 + max(bt, g.draw_bound - b0)  # draws per path: the longer branch
        if tt is None:
            return None
        ty = "real" if "real" in (tt, f.ty) else tt
        return S(res if ty == "real" else f"to_{ty[0]}({res})", ty, False)

    # -------------------------------------------------------------- calls --------
    def _call(self, e, env):
        g = self.g
        if isinstance(e.fn, lang.Var) and e.fn.name not in env and e.fn.name not in self.globals:
            name = e.fn.name
            if name in _DISTS:
                arity, _ = _DISTS[name]
                if len(e.args) != arity:
                    raise CompileError(f"{name} takes {arity} argument(s)")
                if name == "categorical":
                    return Dist(name, [self._cat_weights(self.ev(e.args[0], env))])
                return Dist(name, [_scalar(self.ev(a, env), name) for a in e.args])
            if name in ("sample", "sample*"):
                d = self.ev(e.args[0], env)
                if not isinstance(d, Dist):
                    raise CompileError("sample expects a distribution")
                return self._sample(d)
            if name == "factor":
                x = _scalar(self.ev(e.args[0], env), "factor")
                g.add_lw(_real(x))
                return None
            if name == "observe":
                d = self.ev(e.args[0], env)
                v = _scalar(self.ev(e.args[1], env), "observe")
                g.add_lw(self._score(d, v))
                return None
            if name == "dist-score":
                d = self.ev(e.args[0], env)
                v = _scalar(self.ev(e.args[1], env), "dist-score")
                return S(self._score(d, v), "real")
            if name in _MATH1:
                x = _scalar(self.ev(e.args[0], env), name)
                return S(f"{_MATH1[name]}({_real(x)})", "real", x.pure)
            if name == "pow":
                a, b = (_scalar(self.ev(x, env), "pow") for x in e.args)
                if _is_literal(b.code) and float(b.code.rstrip("f")) == 2.0:
                    a = g.let(a, "p")
                    return S(f"({_real(a)} * {_real(a)})", "real", a.pure)
                return S(f"powf({_real(a)}, {_real(b)})", "real", a.pure and b.pure)
            if name == "to-real":
                x = _scalar(self.ev(e.args[0], env), name)
                return S(_real(x), "real", x.pure)
            if name == "to-int":
                x = _scalar(self.ev(e.args[0], env), name)
                return S(f"to_i({x.code})", "int", x.pure)
            if name == "length":
                v = self.ev(e.args[0], env)
                return v.length()
            if name == "repeat":
                return self._repeat(e, env)
            if name == "map":
                return self._map(e, env)
            if name == "reduce":
                return self._reduce(e, env)
            raise CompileError(f"{name} is not supported in GPU models")
        f = self.ev(e.fn, env)
        if not isinstance(f, Fn):
            raise CompileError("calling a non-function")
        return self._apply(f, [self.ev(a, env) for a in e.args])

    def _apply(self, f: Fn, args):
        if len(args) != len(f.params):
            raise CompileError(f"{f.name} takes {len(f.params)} argument(s)")
        if self.engine == "enumerate" and self.g.calls.count(id(f.body)) >= self.max_depth:
            # bounded recursion (geometric with max_depth 20): a path that would
            # recurse deeper is cut — zero mass; the enumeration posterior renormalises the rest
            self.g.emit(f"dead = true;  // recursion deeper than max_depth = {self.max_depth}")
            return S("0", "int")
        self.g.depth += 1
        if self.g.depth > 64 + (self.max_depth if self.engine == "enumerate" else 0):
            raise CompileError("recursion is not supported in GPU models (enumeration bounds it by max_depth)")
        self.g.calls.append(id(f.body))
        env = dict(f.env)
        for p, a in zip(f.params, args):
            env[p] = self.g.let(a, "a") if isinstance(a, S) else a
        try:
            return self.ev(f.body, env)
        finally:
            self.g.depth -= 1
            self.g.calls.pop()

    def _emit_draw(self, k: str, a, v: str, decl: bool = True):
        """Draw from the particle's / step's word stream into `v` (the reference algorithms,
        csrc/draws.cuh; the same consumption as the batch dist_sample kernel)."""
        g = self.g
        ty = _DISTS[k][1]
        lhs = f"const {_cty(ty)} {v}" if decl else v
        m = g.draw_m()
        if k == "normal":
            g.emit(f"{lhs} = fmaf({_real(a[1])}, draw_normal(ws, {m}), {_real(a[0])});")
        elif k == "uniform-continuous":
            g.emit(f"{lhs} = fmaf({_real(a[1])} - {_real(a[0])}, draw_uniform(ws, {m}), {_real(a[0])});")
        elif k == "uniform-discrete":
            g.emit(f"err |= ud_check({g.valid_m()}, {a[0].code}, {a[1].code}, pid, first_bad);")
            g.emit(f"{lhs} = ud_draw(ws, {a[0].code}, {a[1].code}, {m});")
        elif k == "bernoulli":
            g.emit(f"{lhs} = draw_uniform(ws, {m}) < {_real(a[0])};")
        elif k == "beta":
            gx, gy = g.fresh("gx"), g.fresh("gy")
            g.emit(f"const auto {gx} = draw_gamma(ws, {_real(a[0])}, {m});")
            g.emit(f"const auto {gy} = draw_gamma(ws, {_real(a[1])}, {m});")
            g.emit(f"{lhs} = {gx} / ({gx} + {gy});")
        elif k == "exponential":
            g.emit(f"{lhs} = -logf(draw_uniform_pos(ws, {m})) / {_real(a[0])};")
        elif k == "poisson":
            g.emit(f"err |= pois_check({g.valid_m()}, {_real(a[0])}, pid, first_bad);")
            g.emit(f"{lhs} = draw_poisson(ws, {_real(a[0])}, {m});")
        elif k == "categorical":  # k = #{j < n-1 : w_0 + .. + w_j <= u * sum w}
            w = a[0]
            tot, wmin = self._cat_total(w), g.fresh("cmin")
            g.emit(f"const auto {wmin} = {self._fold('fminf', w)};")
            g.emit(f"err |= cat_check({g.valid_m()}, {tot}, {wmin}, pid, first_bad);")
            u = g.fresh("cu")
            g.emit(f"const auto {u} = draw_uniform(ws, {m}) * {tot};")
            terms, cum = [], None
            for j in range(len(w) - 1):
                c = g.fresh("cc")
                g.emit(f"const auto {c} = {w[j] if cum is None else f'{cum} + {w[j]}'};")
                terms.append(f"to_i({c} <= {u})")
                cum = c
            g.emit(f"{lhs} = {' + '.join(terms) if terms else '0'};")

    def _sample(self, d: Dist) -> S:
        g = self.g
        g.draw_bound += g.loop_mult[-1]
        a = d.args if d.kind == "categorical" else [g.let(x) for x in d.args]
        v = g.fresh("x")
        k = d.kind
        if self.engine == "enumerate":
            return self._choose(d, a, v)
        if k == "uniform-discrete" and _is_literal(a[1].code):
            g.bounds[v] = max(int(a[1].code) - 1, 0)
        if k == "categorical":
            g.bounds[v] = len(a[0]) - 1
        ty = _DISTS[k][1]
        if self.engine == "mcmc":
            return self._lmh_site(d, a, v, ty)
        self._emit_draw(k, a, v)
        g.emit(f"store_draw(draws_out, idx, {g.valid_m()}, nd, {v});")
        g.emit(f"nd += to_i({g.mask()});" if g.mask() else "nd += 1;")
        return S(v, ty, False)

    def _lmh_site(self, d: Dist, a, v: str, ty: str) -> S:
        """LMH: the nd-th sample call of this execution reuses the trace database entry nd when
        its kind matches and it is not the proposed site; otherwise it
        draws fresh from the step's stream. The site's score under the current parameters enters
        the log-joint; fresh sites also enter l_fresh and reused ones are marked for l_stale."""
        g = self.g
        kc = _KIND_CODE[d.kind]
        fv, re, sc = g.fresh("fv"), g.fresh("re"), g.fresh("sc")
        g.emit(f"const bool {re} = nd < oldLen && oldKind[nd] == {kc} && nd != kstar;")
        g.emit(f"float {fv};")
        g.open(f"if ({re})")
        g.emit(f"{fv} = oldVal[nd];")
        g.emit("reused |= 1ull << nd;")
        g.close()
        g.open("else")
        tmp = g.fresh("x")
        self._emit_draw(d.kind, a, tmp)
        g.emit(f"{fv} = static_cast<float>({tmp});")
        g.close()
        val = {"real": fv, "int": f"static_cast<int>({fv})", "bool": f"({fv} != 0.f)"}[ty]
        g.emit(f"const {_cty(ty)} {v} = {val};")
        g.emit(f"const float {sc} = {self._score(d, S(v, ty))};")
        g.emit(f"if (!{re}) lfresh += {sc};")
        g.emit(f"lw += {sc};")
        g.emit(f"newVal[nd] = {fv}; newKind[nd] = {kc}; newScore[nd] = {sc}; ++nd;")
        return S(v, ty, False)

    def _choose(self, d: Dist, a, v) -> S:
        """Enumeration: the next choice is the next base-R digit of the path index (forced
        choices); its log-mass is added to the path weight; a digit outside the
        site's support kills the path."""
        g = self.g
        k = d.kind
        if k == "bernoulli":
            self.radix = max(self.radix, 2)
            g.emit("{ const unsigned dg = static_cast<unsigned>(rem % ENUM_R); rem /= ENUM_R; ++nd;")
            g.emit(f"  if (dg > 1u) dead = true;")
            g.emit(f"  lw += dg == 0u ? logf({_real(a[0])}) : log1pf(-{_real(a[0])});")
            g.emit(f"  chosen = dg == 0u; }}")
            g.emit(f"const bool {v} = chosen;")
            return S(v, "bool", False)
        if k == "uniform-discrete":
            if not (_is_literal(a[0].code) and _is_literal(a[1].code)):
                raise CompileError("enumeration needs uniform-discrete bounds known at compile time")
            lo, hi = int(a[0].code), int(a[1].code)
            if hi <= lo:
                raise CompileError("uniform-discrete(a, b) needs b > a (SPEC.md:347)")
            self.radix = max(self.radix, hi - lo)
            g.bounds[v] = hi - 1
            g.emit("{ const unsigned dg = static_cast<unsigned>(rem % ENUM_R); rem /= ENUM_R; ++nd;")
            g.emit(f"  if (dg >= {hi - lo}u) dead = true;")
            g.emit(f"  lw += {_fconst(-math.log(hi - lo))};")
            g.emit(f"  chosen_i = {lo} + static_cast<int>(dg); }}")
            g.emit(f"const int {v} = chosen_i;")
            return S(v, "int", False)
        if k == "categorical":
            w = a[0]
            n = len(w)
            self.radix = max(self.radix, n)
            g.bounds[v] = n - 1
            tot = self._cat_total(w)
            g.emit("{ const unsigned dg = static_cast<unsigned>(rem % ENUM_R); rem /= ENUM_R; ++nd;")
            g.emit(f"  if (dg >= {n}u) dead = true;")
            g.emit(f"  chosen_i = static_cast<int>(dg);")
            g.emit(f"  lw += dg < {n}u ? score_categorical(chosen_i, {n}, {self._cat_pick(w, 'chosen_i')}, {tot}) : 0.f; }}")
            g.emit(f"const int {v} = chosen_i;")
            return S(v, "int", False)
        from .errors import ContinuousDistError

        raise ContinuousDistError(f"enumeration needs finite-support distributions; {k} is not "
                                  "(SPEC.md:394)")

    def _score(self, d, v: S) -> str:
        if not isinstance(d, Dist):
            raise CompileError("dist-score / observe expect a distribution")
        a = d.args
        k = d.kind
        if k == "normal":
            sd = a[1]
            if _is_literal(sd.code):  # fold 1/sd and -ln sd - ln(2 pi)/2: one FFMA chain per point
                sdv = float(sd.code.rstrip("f"))
                if not sdv > 0:
                    raise CompileError("normal(mean, sd): sd must be > 0")
                inv = _fconst(1.0 / sdv)
                c = _fconst(-math.log(sdv) - 0.5 * math.log(2 * math.pi))
                z = self.g.fresh("z")
                self.g.emit(f"const auto {z} = ({_real(v)} - {_real(a[0])}) * {inv};")
                return f"fmaf(-0.5f * {z}, {z}, {c})"
            return f"score_normal({_real(v)}, {_real(a[0])}, {_real(sd)})"
        if k == "uniform-continuous":
            return f"score_uniform_continuous({_real(v)}, {_real(a[0])}, {_real(a[1])})"
        if k == "uniform-discrete":
            return f"score_uniform_discrete({v.code}, {a[0].code}, {a[1].code})"
        if k == "bernoulli":
            return f"score_bernoulli({v.code}, {_real(a[0])})"
        if k == "beta":
            return f"score_beta({_real(v)}, {_real(a[0])}, {_real(a[1])})"
        if k == "exponential":
            return f"score_exponential({_real(v)}, {_real(a[0])})"
        if k == "categorical":
            kk = self.g.let(S(f"to_i({v.code})", "int"), "k")
            return (f"score_categorical({kk.code}, {len(a[0])}, {self._cat_pick(a[0], kk.code)}, "
                    f"{self._cat_total(a[0])})")
        return f"score_poisson({v.code}, {_real(a[0])})"

    # -------------------------------------------------------------- categorical --
    def _cat_weights(self, vec) -> list:
        """The weight vector of categorical(w) as C expressions (static length <= MAX_CATEGORIES)."""
        if isinstance(vec, ConstVec):
            items = [_real(_scalar(x, "categorical weight")) for x in vec.items]
        elif hasattr(vec, "elem"):
            n = vec.length()
            if not (_is_literal(n.code) and n.ty == "int"):
                raise CompileError("categorical needs a weight vector of static length")
            items = [_real(self.g.let(vec.elem(self, S(str(j), "int")), "w")) for j in range(int(n.code))]
        else:
            raise CompileError("categorical expects a vector of weights")
        if not 1 <= len(items) <= MAX_CATEGORIES:
            raise CompileError(f"categorical supports 1..{MAX_CATEGORIES} categories")
        return items

    def _fold(self, fn: str, w: list) -> str:
        code = w[-1]
        for x in reversed(w[:-1]):
            code = f"{fn}({x}, {code})"
        return code

    def _cat_total(self, w: list) -> str:
        code = w[0]
        for x in w[1:]:
            code = f"({code} + {x})"
        return self.g.let(S(code, "real"), "ctot").code

    def _cat_pick(self, w: list, k: str) -> str:
        code = w[-1]
        for j in range(len(w) - 2, -1, -1):
            code = f"sel({k} == {j}, {w[j]}, {code})"
        return code

    def _repeat(self, e, env):
        g = self.g
        f = self.ev(e.args[0], env)
        n = _scalar(self.ev(e.args[1], env), "repeat length")
        if not isinstance(f, Fn) or len(f.params) != 1:
            raise CompileError("repeat expects a one-argument function")
        n = g.let(n, "n")
        bound = self._bound_of(n)
        # a pure element function is fused into its consumer; one that draws is evaluated now,
        # in order, into a bounded local array (the reference evaluates repeat eagerly)
        if not self._effects(f.body, f.env):
            return LazyVec(n, bound, lambda comp, i: comp._apply(f, [i]))
        if self._observe_loop(f, LazyVec(n, bound, lambda comp, i: i)):
            return None
        probe_v = self._sandbox()._apply(f, [S("i_probe", "int")])
        keep = isinstance(probe_v, S)  # a unit-valued body (observe, factor) runs for its effects
        if bound is None and keep:
            raise CompileError("a repeat that draws needs a bounded length (constant, data length or a "
                               "uniform-discrete draw)")
        arr, i = g.fresh("vec"), g.fresh("i")
        if keep:
            g.emit(f"{_cty(probe_v.ty)} {arr}[{bound}];")
        depth = self._loop(i, n, bound)
        g.loop_mult.append(g.loop_mult[-1] * (bound or 1))
        v = self._apply(f, [S(i, "int")])
        g.loop_mult.pop()
        if keep:
            g.emit(f"{arr}[{i}] = {v.code};")
        for _ in range(depth):
            g.close()
        return LocVec(arr, bound, n, probe_v.ty) if keep else None

    def _observe_loop(self, f: Fn, v) -> bool:
        """map / repeat of `observe(normal(m, sd), y)` with a constant sd: the observes of a
        data loop are one Gaussian-likelihood reduce (the packed peephole below) whose sum is
        added to the log-weight once — the same terms, summed in a different order."""
        body = f.body
        while isinstance(body, lang.Block) and not body.stmts:
            body = body.result
        if not (len(f.params) == 1 and isinstance(body, lang.Call) and isinstance(body.fn, lang.Var)
                and body.fn.name == "observe" and len(body.args) == 2):
            return False
        d = body.args[0]
        if not (isinstance(d, lang.Call) and isinstance(d.fn, lang.Var) and d.fn.name == "normal"
                and len(d.args) == 2):
            return False
        if any(name in f.env or name in self.globals for name in ("observe", "normal", "dist-score")):
            return False
        acc = "__observe_acc"
        red = Fn([acc, f.params[0]], lang.BinOp("+", lang.Var(acc), lang.Call(lang.Var("dist-score"),
                                                                               [d, body.args[1]])),
                 f.env, "<observe loop>")
        r = self._gaussian_reduce(red, S("0.f", "real"), v)
        if r is None:
            return False
        self.g.add_lw(_real(r))
        return True

    def _gaussian_reduce(self, f: Fn, init: S, v):
        """reduce(function(acc, x) { acc + dist-score(normal(m, sd), y) }, init, v) with a
        constant sd: sum (y - m)^2 with one FFMA per element, constants applied once
        (-0.5/sd^2 * sum + n (-ln sd - ln(2 pi)/2)), as the hand-written kernels do."""
        body = f.body
        while isinstance(body, lang.Block) and not body.stmts:
            body = body.result
        if not (isinstance(body, lang.BinOp) and body.op == "+" and isinstance(body.lhs, lang.Var)
                and body.lhs.name == f.params[0] and isinstance(body.rhs, lang.Call)
                and isinstance(body.rhs.fn, lang.Var) and body.rhs.fn.name == "dist-score"
                and len(body.rhs.args) == 2 and isinstance(body.rhs.args[0], lang.Call)
                and isinstance(body.rhs.args[0].fn, lang.Var) and body.rhs.args[0].fn.name == "normal"
                and len(body.rhs.args[0].args) == 2):
            return None
        g = self.g
        env0 = dict(f.env, **{f.params[0]: S("0.f", "real"), f.params[1]: S("0", "int")})
        if self._effects(body.rhs, env0):
            return None
        sd = self._sandbox().ev(body.rhs.args[0].args[1], dict(env0))
        if not (isinstance(sd, S) and _is_literal(sd.code) and float(sd.code.rstrip("f")) > 0):
            return None
        sdv = float(sd.code.rstrip("f"))
        n = v.length()
        if _is_literal(n.code) and int(n.code) >= 2 and isinstance(v, (DataVec, LazyVec)):
            packed = self._gaussian_reduce_packed(f, body, v, int(n.code), init, sdv)
            if packed is not None:
                return packed
        acc, i = g.fresh("ss"), g.fresh("i")
        g.emit(f"VF {acc} = 0.f;")
        n = v.length()
        depth = self._loop(i, n, v.bound())
        env = dict(f.env)
        env[f.params[0]] = S("0.f", "real")
        env[f.params[1]] = g.let(v.elem(self, S(i, "int")), "e")
        m = _scalar(self.ev(body.rhs.args[0].args[0], env), "normal mean")
        y = _scalar(self.ev(body.rhs.args[1], env), "observed value")
        z = g.fresh("z")
        g.emit(f"const auto {z} = {_real(y)} - {_real(m)};")
        g.assign(acc, f"fmaf({z}, {z}, {acc})")
        for _ in range(depth):
            g.close()
        k = _fconst(-0.5 / (sdv * sdv))
        c = _fconst(-math.log(sdv) - 0.5 * math.log(2 * math.pi))
        return S(f"({_real(init)} + fmaf({k}, {acc}, to_f({n.code}) * {c}))", "real", False)

    def _gaussian_reduce_packed(self, f: Fn, body, v, n: int, init: S, sdv: float):
        """The Gaussian-likelihood reduce over pairs of elements: elements (i, i + 1) of the
        data as one f32x2, the particle's scalars broadcast, so each FFMA2 / FADD2 covers two
        data points (the hand-written kernels pack two particles instead). None if some
        operation has no packed form (or the model computes in fp64)."""
        if _F64:
            return None
        sb = self._sandbox()
        try:  # dry run: every operation of m and y must have a packed form
            envp = dict(f.env)
            envp[f.params[0]] = S("0.f", "real")
            envp[f.params[1]] = v.elem(sb, S("ip", "int2"))
            m2 = sb.ev(body.rhs.args[0].args[0], envp)
            y2 = sb.ev(body.rhs.args[1], envp)
            _pair(m2), _pair(y2)
        except (_PairUnsupported, CompileError):
            return None
        g = self.g
        acc, i = g.fresh("ss"), g.fresh("i")
        g.emit(f"VF2 {acc} = pack2(0.f, 0.f);")
        g.emit("#pragma unroll 4")
        g.open(f"for (int {i} = 0; {i} + 1 < {n}; {i} += 2)")
        env = dict(f.env)
        env[f.params[0]] = S("0.f", "real")
        env[f.params[1]] = g.let(v.elem(self, S(i, "int2")), "e")
        m = self.ev(body.rhs.args[0].args[0], env)
        y = self.ev(body.rhs.args[1], env)
        z = g.fresh("z")
        g.emit(f"const auto {z} = fma2({_pair(m)}, pack2(-1.f, -1.f), {_pair(y)});")
        g.emit(f"{acc} = fma2({z}, {z}, {acc});")
        g.close()
        tot = g.fresh("ss")
        g.emit(f"VF {tot} = hsum2({acc});")
        if n % 2:  # odd length: the last element, scalar
            env = dict(f.env)
            env[f.params[0]] = S("0.f", "real")
            env[f.params[1]] = g.let(v.elem(self, S(str(n - 1), "int")), "e")
            m = _scalar(self.ev(body.rhs.args[0].args[0], env), "normal mean")
            y = _scalar(self.ev(body.rhs.args[1], env), "observed value")
            z = g.fresh("z")
            g.emit(f"const auto {z} = {_real(y)} - {_real(m)};")
            g.emit(f"{tot} = fmaf({z}, {z}, {tot});")
        k = _fconst(-0.5 / (sdv * sdv))
        c = _fconst(-math.log(sdv) - 0.5 * math.log(2 * math.pi))
        return S(f"({_real(init)} + fmaf({k}, {tot}, {_fconst(n)} * {c}))", "real", False)

    def _loop(self, i: str, n: S, bound, start: int = 0):
        """Open `for i < n`: small known bounds are unrolled with a guard (static indices keep
        bounded vectors in registers); long data loops are partially unrolled."""
        g = self.g
        if bound is not None and bound <= 16:
            g.emit("#pragma unroll")
            g.open(f"for (int {i} = {start}; {i} < {bound}; ++{i})")
            if not (_is_literal(n.code) and int(n.code) == bound):
                g.open_masked(f"{i} < {n.code}")
                return 2
            return 1
        g.emit("#pragma unroll 4")
        g.open(f"for (int {i} = 0; {i} < {n.code}; ++{i})")
        return 1

    def _bound_of(self, n: S):
        if _is_literal(n.code) and n.ty == "int":
            return int(n.code)
        return self.g.bounds.get(n.code)

    def _map(self, e, env):
        g = self.g
        f = self.ev(e.args[0], env)
        v = self.ev(e.args[1], env)
        if not isinstance(f, Fn) or len(f.params) != 1 or not hasattr(v, "elem"):
            raise CompileError("map expects (function, vector)")
        if not self._effects(f.body, f.env):
            return LazyVec(v.length(), v.bound(), lambda comp, i: comp._apply(f, [v.elem(comp, i)]))
        if self._observe_loop(f, v):
            return None
        # effects: evaluated now, element by element in order (the reference's eager map)
        bound = v.bound()
        probe = self._sandbox()._apply(f, [v.elem(self._sandbox(), S("i_probe", "int"))])
        keep = isinstance(probe, S) and bound is not None
        arr, i = g.fresh("vec"), g.fresh("i")
        if keep:
            g.emit(f"{_cty(probe.ty)} {arr}[{bound}];")
        depth = self._loop(i, v.length(), bound)
        g.loop_mult.append(g.loop_mult[-1] * (bound or 1))
        r = self._apply(f, [v.elem(self, S(i, "int"))])
        g.loop_mult.pop()
        if keep:
            g.emit(f"{arr}[{i}] = {r.code};")
        for _ in range(depth):
            g.close()
        return LocVec(arr, bound, v.length(), probe.ty) if keep else None

    def _reduce(self, e, env):
        g = self.g
        f = self.ev(e.args[0], env)
        init = _scalar(self.ev(e.args[1], env), "reduce init")
        v = self.ev(e.args[2], env)
        if not isinstance(f, Fn) or len(f.params) != 2 or not hasattr(v, "elem"):
            raise CompileError("reduce expects (function(acc, x), init, vector)")
        fused = self._gaussian_reduce(f, init, v)
        if fused is not None:
            return fused
        acc, i = g.fresh("acc"), g.fresh("i")
        # the accumulator type is the body's type given a real (or int) accumulator
        ty = "real" if init.ty == "real" else init.ty
        sb = self._sandbox()
        r = sb._apply(f, [S("acc_probe", ty), v.elem(sb, S("i_probe", "int"))])
        if isinstance(r, S) and r.ty == "real":
            ty = "real"
        g.emit(f"{_cty(ty)} {acc} = {init.code if ty != 'real' else _real(init)};")
        n = v.length()
        bound = v.bound()
        start = 0
        if ty == "real" and init.ty == "real" and _is_literal(init.code) and bound is not None and 1 <= bound <= 16:
            # peel element 0: the body sees the literal init, so e.g. Horner's first step
            # 0 * x + c folds to c (frontend _binop) instead of a multiply-add by zero
            if not _is_literal(n.code):
                g.open_masked(f"0 < {n.code}")
            if not _is_literal(n.code) or int(n.code) >= 1:
                r0 = self._apply(f, [init, v.elem(self, S("0", "int"))])
                g.assign(acc, _real(r0))
            if not _is_literal(n.code):
                g.close()
            start = 1
            if bound == 1:
                return S(acc, ty, False)
        depth = self._loop(i, n, bound, start)
        g.loop_mult.append(g.loop_mult[-1] * (bound - start if bound else 1))
        x = v.elem(self, S(i, "int"))
        r = self._apply(f, [S(acc, ty), x])
        g.loop_mult.pop()
        g.assign(acc, r.code if ty != 'real' else _real(r))
        for _ in range(depth):
            g.close()
        return S(acc, ty, False)

    # -------------------------------------------------------------- helpers ----
    def _sandbox(self):
        """A throwaway copy for type probes: nothing it emits or binds reaches this compiler."""
        c = _Compiler.__new__(_Compiler)
        c.prog, c.model, c.default_n = self.prog, self.model, self.default_n
        c.engine, c.radix, c.max_depth = self.engine, self.radix, self.max_depth
        c.globals, c.external = dict(self.globals), dict(self.external)
        c.g = _Gen(list(self.g.data))
        c.g.n, c.g.bounds, c.g.calls = self.g.n, dict(self.g.bounds), list(self.g.calls)
        return c

    def _effects(self, node, env, seen=None) -> bool:
        """Conservative: does evaluating `node` draw or add to the log-weight?"""
        seen = seen if seen is not None else set()
        if isinstance(node, lang.Call):
            if isinstance(node.fn, lang.Var):
                name = node.fn.name
                if name in ("sample", "sample*", "factor", "observe"):
                    return True
                f = env.get(name, self.globals.get(name))
                if isinstance(f, Fn) and id(f) not in seen:
                    seen.add(id(f))
                    if self._effects(f.body, f.env, seen):
                        return True
            return any(self._effects(x, env, seen) for x in [node.fn] + node.args)
        if isinstance(node, lang.Var):
            f = env.get(node.name, self.globals.get(node.name))
            if isinstance(f, Fn) and id(f) not in seen:
                seen.add(id(f))
                return self._effects(f.body, f.env, seen)
            return False
        if isinstance(node, (list, tuple)):
            return any(self._effects(x, env, seen) for x in node)
        if hasattr(node, "__dataclass_fields__"):
            return any(self._effects(getattr(node, k), env, seen) for k in node.__dataclass_fields__)
        return False

    # -------------------------------------------------------------- the model ----
    def compile(self):
        self.top()
        self.g.bounds = {}
        return self._apply(self.model, [])


@dataclass
class CompiledModel:
    """A CuPPL model compiled for the GPU (importance sampling)."""

    source: str
    cuda: str
    data: np.ndarray
    n_stats: int
    n_bins: int
    stat_names: list
    return_kind: str  # "real" | "int" | "bool" | "vector" | "none"
    return_width: int
    max_draws: int
    default_n: int
    engine: str = "importance"
    radix: int = 1
    masked: bool = False  # particle-dependent control flow (lane builds are opt-in)
    f64: bool = False  # fp64 model arithmetic and record (enumerate)
    bin_lo: int = 0  # histogram bin k holds the integer return value bin_lo + k
    kind: str = "dsl"
    _fn: object = field(default=None, repr=False)


_KERNEL = r'''
#define MAXD {maxd}
{f64_define}
#include "dsl_lanes.cuh"
#include "is_accum.cuh"
using namespace cuppl;
{f64_prelude}
{data_decl}
// LANES particles per thread (dsl_lanes.cuh): particle (base + p * 256 + threadIdx.x) is lane p
extern "C" __global__ void __launch_bounds__(256)
cuppl_dsl_model(const float* __restrict__ D, unsigned long long pid_begin, unsigned long long n,
                unsigned int k0, unsigned int k1, cuppl_is_record* block_recs, unsigned int* counter,
                cuppl_is_record* rec_out, {real_t}* lw_out, float* draws_out, float* ret_out,
                unsigned int* err_out) {{
  {acc_t}<{ns}, {nb}> acc;
  acc.init();
  const PhiloxKey key{{k0, k1}};
  unsigned int err = 0u;
  unsigned long long first_bad = ~0ull;  // smallest particle id with invalid parameters
  // block-uniform chunk loop (lanes past the end run masked): the model body stays in
  // uniform control flow, so warp-uniform data indices use the uniform datapath
  for (unsigned long long base = blockIdx.x * (256ull * LANES); base < n;
       base += static_cast<unsigned long long>(gridDim.x) * (256ull * LANES)) {{
    VU64 idx;
    VB valid;
#pragma unroll
    for (int p_ = 0; p_ < LANES; ++p_) {{
      lane_ref(idx, p_) = base + p_ * 256ull + threadIdx.x;
      lane_ref(valid, p_) = lane_ref(idx, p_) < n;
    }}
    const VU64 pid = idx + pid_begin;
    VStream ws;
    ws.init(key, pid, {tag}u);
    VF lw = 0.f;
    VI nd = 0;
{enum_init}
{body}
{enum_final}
#pragma unroll
    for (int p_ = 0; p_ < LANES; ++p_) {{
      const unsigned long long idx_ = lane_at(idx, p_);
      if (lane_at(valid, p_)) {{
        const {real_t} lw_ = lane_at(lw, p_);
        {real_t} f[{ns_arr}] = {{{stats}}};
        acc.add(lw_, pid_begin + idx_, f, lane_at({bin}, p_));
        if (lw_out) lw_out[idx_] = lw_;
        if (ret_out) {{
{ret_store}
        }}
      }}
    }}
    (void)nd;
  }}
  if (err) {{
    atomicOr(err_out, err);
    atomicMin(reinterpret_cast<unsigned long long*>(err_out + 2), first_bad);
  }}
  is_epilogue(acc, block_recs, counter, rec_out);
}}
'''


_MCMC_KERNEL = r"""
#define MAXD {maxd}
#include "dsl_lanes.cuh"
using namespace cuppl;
{data_decl}
// many independent LMH chains, one thread each (SPEC.md:408-416); the trace database of the
// current state (old*) and of the proposal (new*) live in per-thread arrays
extern "C" __global__ void __launch_bounds__(128)
cuppl_dsl_mcmc(const float* __restrict__ D, unsigned int n_chains, unsigned int chain_begin,
               unsigned int n_steps, unsigned int burn_in, unsigned int thin, unsigned int k0,
               unsigned int k1, double* stats_out, unsigned int* err_out) {{
  const PhiloxKey key{{k0, k1}};
  unsigned int err = 0u;
  unsigned long long first_bad = ~0ull;  // smallest chain id with invalid parameters
  const bool valid = true;
  for (unsigned int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_chains; c += gridDim.x * blockDim.x) {{
    const unsigned int chain = chain_begin + c;
    const unsigned long long pid = chain;
    float oldVal[MAXD], newVal[MAXD], oldScore[MAXD], newScore[MAXD];
    unsigned char oldKind[MAXD], newKind[MAXD];
    int oldLen = 0;
    float ll = 0.f;
    float curf[{ns_arr}];
    int curbin = -1;
    double sums[{ns_arr}], binc[{nb_arr}], nrec = 0.0, nacc = 0.0;
    for (int k = 0; k < {ns_arr}; ++k) {{ curf[k] = 0.f; sums[k] = 0.0; }}
    for (int k = 0; k < {nb_arr}; ++k) binc[k] = 0.0;
    for (unsigned int s = 0; s < n_steps; ++s) {{  // sample s: the initial trace, then s MH steps
      WordStream ws;
      ws.init(key, (static_cast<unsigned long long>(s) << 32) | chain, {tag}u);
      int kstar = -1;  // proposed site: uniform over the current trace database
      if (s > 0 && oldLen > 0) kstar = static_cast<int>(ws.randint(static_cast<unsigned>(oldLen)));
      float lw = 0.f, lfresh = 0.f;
      int nd = 0;
      unsigned long long reused = 0ull;
{body}
      float f[{ns_arr}] = {{{stats}}};
      const int bin = {bin};
      float lstale = 0.f;  // old sites the proposal did not reuse (incl. the proposed one)
      for (int i = 0; i < oldLen; ++i)
        if (!((reused >> i) & 1ull)) lstale += oldScore[i];
      bool accept = true;
      if (s > 0) {{  // SURVEY.md D8: single-site prior-proposal ratio with the |DB| terms
        const float la = (lw - ll) + logf(static_cast<float>(oldLen > 0 ? oldLen : 1)) -
                         logf(static_cast<float>(nd > 0 ? nd : 1)) + lstale - lfresh;
        accept = logf(ws.uniform_pos()) < la;
        nacc += accept ? 1.0 : 0.0;
      }}
      if (accept) {{
        for (int i = 0; i < nd; ++i) {{
          oldVal[i] = newVal[i];
          oldScore[i] = newScore[i];
          oldKind[i] = newKind[i];
        }}
        oldLen = nd;
        ll = lw;
        for (int k = 0; k < {ns_arr}; ++k) curf[k] = f[k];
        curbin = bin;
      }}
      if (s >= burn_in && (s - burn_in) % thin == 0) {{
        for (int k = 0; k < {ns_arr}; ++k) sums[k] += curf[k];
        if (curbin >= 0 && curbin < {nb_arr}) binc[curbin] += 1.0;
        nrec += 1.0;
      }}
      (void)lfresh;
    }}
    double* out = stats_out + static_cast<unsigned long long>(c) * ({ns_arr} + {nb_arr} + 2);
    for (int k = 0; k < {ns_arr}; ++k) out[k] = sums[k];
    for (int k = 0; k < {nb_arr}; ++k) out[{ns_arr} + k] = binc[k];
    out[{ns_arr} + {nb_arr}] = nrec;
    out[{ns_arr} + {nb_arr} + 1] = nacc;
  }}
  if (err) {{
    atomicOr(err_out, err);
    atomicMin(reinterpret_cast<unsigned long long*>(err_out + 2), first_bad);
  }}
}}
"""


def _return_parts(ret, g: _Gen, int_bins: tuple = (0, MAX_BINS)):
    """(stat expressions, stat names, bin expression, n_bins, kind, width, stores); a store is
    (component index, value expression) of ret_out[idx * width + k]. An integer return is
    histogrammed over values [lo, lo + n) of int_bins = (lo, n)."""
    if ret is None:
        return [], [], "0", 0, "none", 0, []
    if isinstance(ret, S):
        v = g.let(ret, "ret")
        st = [_real(v), f"{_real(v)} * {_real(v)}"]
        if ret.ty in ("int", "bool"):
            lo, nb = int_bins if ret.ty == "int" else (0, MAX_BINS)
            b = f"sel(({v.code}) >= {lo} && ({v.code}) < {lo + nb}, to_i({v.code}) - ({lo}), -1)"
            return st, ["value", "value^2"], b, nb, ret.ty, 1, [(0, _real(v))]
        return st, ["value", "value^2"], "0", 0, "real", 1, [(0, _real(v))]
    if isinstance(ret, ConstVec):
        items = [g.let(x, "ret") for x in ret.items]
        if 2 * len(items) > MAX_STATS:
            raise CompileError(f"at most {MAX_STATS // 2} returned components")
        st = [_real(x) for x in items] + [f"{_real(x)} * {_real(x)}" for x in items]
        names = [f"v{k}" for k in range(len(items))] + [f"v{k}^2" for k in range(len(items))]
        return st, names, "0", 0, "vector", len(items), [(k, _real(x)) for k, x in enumerate(items)]
    if isinstance(ret, LocVec):
        if ret.bound_ > MAX_STATS // 2:
            raise CompileError(f"returned vectors are bounded by {MAX_STATS // 2} elements")
        comps = [f"sel({k} < {ret.length_.code}, to_f({ret.var}[{k}]), 0.f)" for k in range(ret.bound_)]
        names = [f"v{k}" for k in range(ret.bound_)]
        b = f"sel(({ret.length_.code}) >= 0 && ({ret.length_.code}) < {MAX_BINS}, to_i({ret.length_.code}), -1)"
        store = list(enumerate(comps)) + [(ret.bound_, f"to_f({ret.length_.code})")]
        return comps, names, b, MAX_BINS, "vector", ret.bound_ + 1, store
    raise CompileError(f"unsupported return value {type(ret).__name__}")


def compile_program(source: str, data: dict | None = None, max_depth: int = 20) -> CompiledModel:
    """Parse and compile a CuPPL program whose result is importance(model, n), enumerate(model,
    n) or mcmc(model, n). max_depth bounds recursion in enumerated programs.
    Programs that bind engine results and compute with them (dist-var of a posterior,
    SPEC.md:432) run through program.run_program."""
    return compile_parsed(lang.parse(source), source, data, max_depth)


def compile_parsed(prog, source: str, data: dict | None = None, max_depth: int = 20) -> CompiledModel:
    """compile_program of an already parsed lang.Program."""
    global _F64
    res = prog.result
    f64 = isinstance(res, lang.Call) and isinstance(res.fn, lang.Var) and res.fn.name == "enumerate"
    with _COMPILE_LOCK:
        _F64 = f64
        try:
            return _compile_parsed(prog, source, data, max_depth)
        finally:
            _F64 = False


def _compile_parsed(prog, source: str, data: dict | None, max_depth: int) -> CompiledModel:
    comp = _Compiler(prog, data, max_depth)
    ret = comp.compile()
    g = comp.g
    int_bins = (MCMC_BIN_LO, MCMC_BINS) if comp.engine == "mcmc" else (0, MAX_BINS)
    stats, names, bin_expr, nb, kind, width, store = _return_parts(ret, g, int_bins)
    bin_lo = int_bins[0] if kind == "int" else 0
    lane_stats = [f"lane_at({x}, p_)" for x in stats]
    maxd = g.draw_bound if 0 < g.draw_bound <= MAX_TRACE_DRAWS else 1
    body = "\n".join("  " + line for line in g.lines)
    data_arr = np.asarray(g.data if g.data else [0.0], dtype=np.float64 if _F64 else np.float32)
    rt = "double" if _F64 else "float"
    if _F64 and len(data_arr) > MAX_CONST_DATA // 2:
        raise CompileError(f"enumerate programs hold up to {MAX_CONST_DATA // 2} data values (fp64 constant bank)")
    if len(data_arr) <= MAX_CONST_DATA:  # warp-uniform indices: constant-cache broadcasts
        pad = _DC_PAD * (1 if _F64 else 2)  # elements before the data (DC_PAD_BYTES)
        data_decl = (f"__constant__ __align__(32) {rt} DCP[{pad + len(data_arr)}];\n"
                     f"#define DC (DCP + {pad})\n"
                     f"__device__ __forceinline__ {rt} dat(int i) {{ return DC[i]; }}\n"
                     "CUPPL_LIFT(dat)  // a per-particle index: one constant-bank read per lane\n"
                     f"#define {DATA_SYM}(i) dat(i)\n"
                     f"#define {DATA_SYM}2(i) (*reinterpret_cast<const f32x2*>(&DC[i]))")
    else:
        data_decl = (f"#define {DATA_SYM}(i) __ldg(D + (i))\n"
                     f"#define {DATA_SYM}2(i) __ldg(reinterpret_cast<const unsigned long long*>(D + (i)))")
    enum_init = enum_final = ""
    if comp.engine == "enumerate":
        radix = max(comp.radix, 2)
        maxd = max(g.draw_bound, 1)
        data_decl += f"\n#define ENUM_R {radix}ull"
        enum_init = ("    unsigned long long rem = pid;  // base-R digits: the forced choices of this path\n"
                     "    bool dead = false, chosen = false;\n    int chosen_i = 0;\n    (void)chosen; (void)chosen_i;")
        # a path that made nd < MAXD choices stands for R^(MAXD - nd) indices: divide them out
        # draws_out carries each index's number of choices (int32) in enumeration launches:
        # the breadth-first truncation of run_enumeration ranks paths by (choices, digits)
        enum_final = (f"    if (dead) lw = neg_inf_f();\n"
                      f"    lw -= static_cast<double>(MAXD - nd) * {repr(math.log(radix))};\n"
                      f"    if (draws_out && valid) reinterpret_cast<int*>(draws_out)[idx] = dead ? -1 : nd;")
    if comp.engine == "mcmc":
        if g.draw_bound > 64:
            raise CompileError("mcmc supports up to 64 sample calls per execution")
        cuda = _MCMC_KERNEL.format(maxd=max(g.draw_bound, 1), data_decl=data_decl, ns_arr=max(len(stats), 1),
                                   nb_arr=max(nb, 1), stats=", ".join(stats) if stats else "0.f",
                                   bin=bin_expr if nb else "-1", tag=TAG_DSL_MH,
                                   body="\n".join("    " + line for line in g.lines))
        return CompiledModel(source=source, cuda=cuda, data=data_arr, n_stats=len(stats), n_bins=nb,
                             stat_names=names, return_kind=kind, return_width=width,
                             max_draws=g.draw_bound, default_n=comp.default_n, engine="mcmc",
                             bin_lo=bin_lo)
    f64_define = "#define CUPPL_F64 1" if _F64 else ""
    # fp64 models: the body's float math names resolve to the double functions (dsl_lanes.cuh
    # CUPPL_F64 keeps VF = double and the score functions' fp64 forms)
    f64_prelude = ("#define expf exp\n#define logf log\n#define log1pf log1p\n#define sqrtf sqrt\n"
                   "#define fabsf fabs\n#define floorf floor\n#define fmodf fmod\n#define powf pow\n"
                   "#define fmaf fma\n#define fminf fmin\n#define fmaxf fmax") if _F64 else ""
    cuda = _KERNEL.format(maxd=maxd, data_decl=data_decl, enum_init=enum_init, enum_final=enum_final,
                          f64_define=f64_define, f64_prelude=f64_prelude,
                          acc_t="ThreadAccF64" if _F64 else "ThreadAcc", real_t=rt,
                          ns=len(stats), nb=nb, ns_arr=max(len(stats), 1),
                          stats=", ".join(lane_stats) if stats else "0.f", bin=bin_expr, tag=TAG_DSL,
                          body=body, ret_store="\n".join(f"          ret_out[idx_ * {width} + {k}] = lane_at({x}, p_);"
                                                         for k, x in store))
    return CompiledModel(source=source, cuda=cuda, data=data_arr, n_stats=len(stats), n_bins=nb,
                         stat_names=names, return_kind=kind, return_width=width,
                         max_draws=g.draw_bound, default_n=comp.default_n, engine=comp.engine,
                         radix=max(comp.radix, 2) if comp.engine == "enumerate" else 1, masked=g.masked,
                         f64=_F64)


# ----------------------------------------------------------------------------- JIT -------
_MODULES: dict = {}


def _nvrtc_cubin(src: str, lanes: int = 1, extra: tuple = ()) -> bytes:
    from cuda.bindings import nvrtc

    def ok(r, what):
        err = r[0]
        if err != nvrtc.nvrtcResult.NVRTC_SUCCESS:
            raise InferRuntimeError(f"NVRTC {what} failed: {err}")
        return r[1:] if len(r) > 2 else (r[1] if len(r) == 2 else None)

    prog = ok(nvrtc.nvrtcCreateProgram(src.encode(), b"cuppl_model.cu", 0, [], []), "create")
    opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo", b"-default-device",
            f"-DLANES={lanes}".encode(), f"-I{CSRC}".encode(), f"-I{INCLUDE}".encode()]
    opts += [o.encode() for o in extra]
    r = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
    if r[0] != nvrtc.nvrtcResult.NVRTC_SUCCESS:
        size = ok(nvrtc.nvrtcGetProgramLogSize(prog), "log size")
        log = b" " * size
        nvrtc.nvrtcGetProgramLog(prog, log)
        raise CompileError("NVRTC compilation failed:\n" + log.decode(errors="replace"))
    size = ok(nvrtc.nvrtcGetCUBINSize(prog), "cubin size")
    cubin = b" " * size
    ok(nvrtc.nvrtcGetCUBIN(prog, cubin), "cubin")
    nvrtc.nvrtcDestroyProgram(prog)
    return cubin


def _lanes_to_try(model: CompiledModel) -> list:
    """Lane counts to build, best first. Programs with particle-dependent control flow build
    at one particle per thread unless CUPPL_DSL_LANES asks otherwise: their masked lane form
    is correct but measured slower (Fig.1: 6.0e10 particles/s at 1 lane, 4.3e10 at 2, 2.9e10
    at 8 — per-lane conditional draws and a select per masked update)."""
    if model.engine != "importance":
        return [1]
    env = os.environ.get("CUPPL_DSL_LANES")
    want = int(env) if env else (1 if model.masked else DSL_LANES)
    return [k for k in (8, 4, 2) if k <= want] + [1]


def _function(model: CompiledModel):
    """Load (once per process and source) the compiled kernel; returns (CUfunction, lanes).
    Importance kernels are first built with DSL_LANES particles per thread; a program whose
    control flow depends on particle values does not compile that way (dsl_lanes.cuh), and a
    build that spills registers is not kept: both fall back to one particle per thread."""
    from cuda.bindings import driver as cu

    h = hashlib.sha256(model.cuda.encode() + model.data.tobytes() + repr(_lanes_to_try(model)).encode()).hexdigest()
    if h not in _MODULES:
        import torch

        torch.cuda.init()  # the primary context torch uses is current for the driver calls
        name = b"cuppl_dsl_mcmc" if model.engine == "mcmc" else b"cuppl_dsl_model"
        lane_divergent = False
        for lanes in _lanes_to_try(model):
            if lanes > 1 and lane_divergent:
                continue
            try:
                cubin = _nvrtc_cubin(model.cuda, lanes)
            except CompileError:
                if lanes == 1:
                    raise
                lane_divergent = True  # a type error in lane form: no lane count will build
                continue
            err, mod = cu.cuModuleLoadData(cubin)
            if err != cu.CUresult.CUDA_SUCCESS:
                raise InferRuntimeError(f"cuModuleLoadData failed: {err}")
            err, fn = cu.cuModuleGetFunction(mod, name)
            if err != cu.CUresult.CUDA_SUCCESS:
                raise InferRuntimeError(f"cuModuleGetFunction failed: {err}")
            err, local = cu.cuFuncGetAttribute(cu.CUfunction_attribute.CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, fn)
            if lanes > 1 and err == cu.CUresult.CUDA_SUCCESS and local > 0:
                cu.cuModuleUnload(mod)
                continue
            break
        if " float DCP[" in model.cuda or " double DCP[" in model.cuda:  # data in the module's constant bank
            err, dptr, size = cu.cuModuleGetGlobal(mod, b"DCP")
            pad_bytes = size - model.data.nbytes
            if err != cu.CUresult.CUDA_SUCCESS or pad_bytes not in (0, _DC_PAD * 8):
                raise InferRuntimeError(f"cuModuleGetGlobal(DCP) failed: {err}")
            err, = cu.cuMemcpyHtoD(int(dptr) + pad_bytes, model.data.ctypes.data, model.data.nbytes)
            if err != cu.CUresult.CUDA_SUCCESS:
                raise InferRuntimeError(f"cuMemcpyHtoD(DC) failed: {err}")
        _MODULES[h] = (mod, fn, lanes)
    return _MODULES[h][1], _MODULES[h][2]


def _raise_param_error(err, what: str):
    """Map a kernel error word [flags, 0, first failing id (u64)] to InvalidDistParamError and
    reset it."""
    w = err.cpu().numpy()
    if not w[0]:
        return
    first = int(w[2:4].view(np.uint64)[0])
    err.copy_(err.new_tensor([0, 0, -1, -1]))
    if w[0] & 1:
        msg = "uniform-discrete(a, b) needs b > a (SPEC.md:347)"
    elif w[0] & 2:
        msg = "categorical(w): weights must be >= 0 and not all 0 (SURVEY.md D5)"
    else:
        msg = "poisson(rate): rate must be finite, >= 0 and < 2^31"
    raise InvalidDistParamError(f"{msg}; first failing {what}: {first}")


class DslLauncher:
    """Launcher of a compiled model with the IsLauncher interface (launch(lo, hi, key, ...),
    .rec): infer.run_importance shards and merges it like the hand-written kernels."""

    def __init__(self, model: CompiledModel, device=None):
        import torch

        from . import _native as N

        self.model = model
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        props = torch.cuda.get_device_properties(self.device)
        self.sms = props.multi_processor_count
        self.max_grid = self.sms * 8
        self.data = torch.from_numpy(model.data).to(self.device)
        self.ws = torch.zeros(256 + self.max_grid * N.REC_BYTES, dtype=torch.uint8, device=self.device)
        self.rec = torch.empty(N.REC_BYTES, dtype=torch.uint8, device=self.device)
        # error word: [flags, 0, first failing particle id (u64, all ones when none)]
        self.err = torch.tensor([0, 0, -1, -1], dtype=torch.int32, device=self.device)
        self.fn, self.lanes = _function(model)

    def launch(self, pid_begin: int, pid_end: int, key: int, lw_out=None, draws_out=None, ret_out=None,
               rec_out=None, stream=None, **_):
        import torch
        from cuda.bindings import driver as cu

        from . import _native as N

        n = pid_end - pid_begin
        if n <= 0:
            raise ValueError("empty particle range")
        grid = int(min(self.max_grid, (n + 256 * self.lanes - 1) // (256 * self.lanes)))
        rec = self.rec if rec_out is None else rec_out
        counter = self.ws[:4]
        blocks = self.ws[256:]
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        vals = [C.c_uint64(self.data.data_ptr()), C.c_uint64(pid_begin), C.c_uint64(n),
                C.c_uint32(key & 0xFFFFFFFF), C.c_uint32(key >> 32), C.c_uint64(blocks.data_ptr()),
                C.c_uint64(counter.data_ptr()), C.c_uint64(rec.data_ptr()), C.c_uint64(N.ptr(lw_out) or 0),
                C.c_uint64(N.ptr(draws_out) or 0), C.c_uint64(N.ptr(ret_out) or 0),
                C.c_uint64(self.err.data_ptr())]
        ptrs = (C.c_void_p * len(vals))(*[C.addressof(v) for v in vals])
        err, = cu.cuLaunchKernel(self.fn, grid, 1, 1, 256, 1, 1, 0, st, C.addressof(ptrs), 0)
        if err != cu.CUresult.CUDA_SUCCESS:
            raise InferRuntimeError(f"cuLaunchKernel failed: {err}")

    def check_errors(self):
        _raise_param_error(self.err, "particle")

    def trace_of(self, pid: int, key: int):
        """Return value of one particle (re-executed: the streams are counter-based)."""
        import torch

        w = max(self.model.return_width, 1)
        out = torch.empty(w, dtype=torch.float32, device=self.device)
        rec = torch.empty_like(self.rec)
        self.launch(pid, pid + 1, key, ret_out=out, rec_out=rec)
        v = out.cpu().numpy().astype(float).tolist()
        k = self.model.return_kind
        if k in ("int", "bool"):
            return int(v[0]) if k == "int" else bool(v[0])
        if k == "real":
            return v[0]
        if k == "vector" and self.model.n_bins:  # bounded vector: components then length
            return v[:int(v[-1])]
        return v


def distribution_from_record(model: CompiledModel, rec, n: int, launcher: DslLauncher, key: int):
    """EmpiricalDistribution of a compiled model from its merged record."""
    from .errors import AllZeroWeightError
    from .infer import EmpiricalDistribution, record_to_dict

    if rec.n_finite == 0:
        raise AllZeroWeightError("every particle has log-weight -inf (SPEC.md:421)")
    S_, S2, M = rec.sum_w, rec.sum_w2, rec.max_lw
    out = EmpiricalDistribution(n=n, record=record_to_dict(rec))
    out.log_z = M + math.log(S_) - math.log(n)
    out.ess = S_ * S_ / S2
    out.mode_log_weight = rec.argmax_lw
    out.mode_index = int(rec.argmax_pid)
    out.mode = launcher.trace_of(out.mode_index, key)
    st = np.array(rec.stat_w[:model.n_stats]) / S_
    out.mean = {name: float(v) for name, v in zip(model.stat_names, st) if not name.endswith("^2")}
    half = model.n_stats // 2
    if model.stat_names and model.stat_names[-1].endswith("^2"):
        out.stats = {f"var_{model.stat_names[k]}": float(st[half + k] - st[k] ** 2) for k in range(half)}
    if model.n_bins:
        bins = np.array(rec.bin_w[:model.n_bins]) / S_
        conv = bool if model.return_kind == "bool" else int
        out.support = [(conv(k), float(p)) for k, p in enumerate(bins) if p > 0]
        out.support_truncated = False
        if model.return_kind == "int" and bins.sum() < 1.0 - 1e-6:
            full = _full_int_support(model, n, launcher, key)
            if full is not None:
                out.support = full
            else:
                out.support_truncated = True
    return out


def _full_int_support(model: CompiledModel, n: int, launcher: DslLauncher, key: int):
    """The record histograms returned values 0..MAX_BINS-1; when weight falls outside, re-run
    the (counter-based, hence identical) particles with their log-weights and returned values
    materialised and histogram the whole support with K3 (exact fixed-point bins). One process
    and n <= 2^30 only; None otherwise."""
    import torch

    from .infer import _world, normalize_tensors

    if n > 1 << 30 or _world(None)[1] > 1:
        return None
    lw = torch.empty(n, dtype=torch.float64 if model.f64 else torch.float32, device=launcher.device)
    ret = torch.empty(n, dtype=torch.float32, device=launcher.device)
    rec = torch.empty_like(launcher.rec)
    launcher.launch(0, n, key, lw_out=lw, ret_out=ret, rec_out=rec)
    v = ret.to(torch.int64)
    lo, hi = int(v.min()), int(v.max())
    if hi - lo >= 1 << 20:
        return None
    res = normalize_tensors(lw, (v - lo).to(torch.int32), hi - lo + 1)
    return [(lo + k, float(p)) for k, p in enumerate(res["probs"]) if p > 0]


def run_mcmc(model: CompiledModel, n_steps: int, rng, *, chains: int = 4096, burn_in: int = 0, thin: int = 1,
             chain_begin: int = 0, device=None) -> dict:
    """Launch the compiled LMH kernel: `chains` chains of `n_steps` steps. Returns per-chain
    statistics [chains, n_stats + n_bins + 2] (sums of the returned components, bin counts,
    records, acceptances) as a numpy array."""
    import torch
    from cuda.bindings import driver as cu

    from .rng import key_of

    dev = device or torch.device("cuda", torch.cuda.current_device())
    data = torch.from_numpy(model.data).to(dev)
    fn, _ = _function(model)
    width = max(model.n_stats, 1) + max(model.n_bins, 1) + 2
    stats = torch.zeros((chains, width), dtype=torch.float64, device=dev)
    err = torch.tensor([0, 0, -1, -1], dtype=torch.int32, device=dev)
    key = key_of(rng)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    grid = int(min((chains + 127) // 128, sms * 16))
    vals = [C.c_uint64(data.data_ptr()), C.c_uint32(chains), C.c_uint32(chain_begin), C.c_uint32(n_steps),
            C.c_uint32(burn_in), C.c_uint32(thin), C.c_uint32(key & 0xFFFFFFFF), C.c_uint32(key >> 32),
            C.c_uint64(stats.data_ptr()), C.c_uint64(err.data_ptr())]
    ptrs = (C.c_void_p * len(vals))(*[C.addressof(v) for v in vals])
    st = torch.cuda.current_stream(dev).cuda_stream
    e, = cu.cuLaunchKernel(fn, grid, 1, 1, 128, 1, 1, 0, st, C.addressof(ptrs), 0)
    if e != cu.CUresult.CUDA_SUCCESS:
        raise InferRuntimeError(f"cuLaunchKernel failed: {e}")
    _raise_param_error(err, "chain")
    return stats.cpu().numpy()
