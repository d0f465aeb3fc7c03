"""Seeded random CuPPL programs for differential testing of the model compiler against the
fp64 interpreter (tests/test_frontend_fuzz.py). Expressions stay numerically tame: bounded
arguments for exp / log / sqrt, literal sds, no division by values near zero."""

import random

DISTS = ["normal", "uniform-continuous", "beta", "exponential", "bernoulli", "uniform-discrete", "poisson"]


class _Gen:
    def __init__(self, seed):
        self.r = random.Random(seed)
        self.reals = []   # names of real-valued model variables
        self.ints = []
        self.bools = []
        self.n = 0

    def name(self):
        self.n += 1
        return f"v{self.n}"

    def real_atom(self):
        r = self.r
        if self.reals and r.random() < 0.7:
            return r.choice(self.reals)
        if self.ints and r.random() < 0.3:
            return f"to-real({r.choice(self.ints)})"
        return f"{r.uniform(-3, 3):.3f}"

    def real_expr(self, depth=0):
        r = self.r
        if depth >= 2 or r.random() < 0.35:
            return self.real_atom()
        k = r.random()
        a, b = self.real_expr(depth + 1), self.real_expr(depth + 1)
        if k < 0.25:
            return f"({a} + {b})"
        if k < 0.45:
            return f"({a} - {b})"
        if k < 0.65:
            return f"({a} * {b})"
        if k < 0.72:
            return f"({a} / (abs({b}) + 1.0))"
        if k < 0.79:
            return f"exp({a} / 20.0)"
        if k < 0.86:
            return f"log(abs({a}) + 1.0)"
        if k < 0.92:
            return f"sqrt(abs({a}))"
        if self.bools:
            return f"if ({r.choice(self.bools)}) {{ {a} }} else {{ {b} }}"
        return f"if ({a} > {b}) {{ {a} }} else {{ {b} }}"

    def draw(self):
        r = self.r
        k = r.choice(DISTS)
        v = self.name()
        if k == "normal":
            s = f"sample(normal({self.real_expr(1)}, {r.uniform(0.5, 5):.2f}))"
            self.reals.append(v)
        elif k == "uniform-continuous":
            lo = r.uniform(-5, 0)
            s = f"sample(uniform-continuous({lo:.2f}, {lo + r.uniform(0.5, 5):.2f}))"
            self.reals.append(v)
        elif k == "beta":
            s = f"sample(beta({r.uniform(0.5, 4):.2f}, {r.uniform(0.5, 4):.2f}))"
            self.reals.append(v)
        elif k == "exponential":
            s = f"sample(exponential({r.uniform(0.2, 3):.2f}))"
            self.reals.append(v)
        elif k == "bernoulli":
            s = f"sample(bernoulli({r.uniform(0.1, 0.9):.2f}))"
            self.bools.append(v)
        elif k == "uniform-discrete":
            lo = r.randint(-3, 2)
            s = f"sample(uniform-discrete({lo}, {lo + r.randint(1, 5)}))"
            self.ints.append(v)
        else:
            s = f"sample(poisson({r.uniform(0.5, 6):.2f}))"
            self.ints.append(v)
        return f"  {v} <- {s};"

    def effect(self):
        r = self.r
        k = r.random()
        if k < 0.3:
            return f"  factor(-abs({self.real_expr()}) / 4.0);"
        if k < 0.55:
            return (f"  observe(normal({self.real_expr(1)}, {r.uniform(0.5, 3):.2f}), {r.uniform(-3, 3):.2f});")
        if k < 0.75:
            return ("  map(function(i) { observe(normal(" + self.real_expr(1) + " * xs[i], "
                    f"{r.uniform(0.5, 3):.2f}), ys[i]) }}, repeat(function(i) {{ i }}, length(xs)));")
        if k < 0.9:
            return ("  factor(reduce(function(acc, i) { acc - abs(" + self.real_expr(1)
                    + " - ys[i]) / 10.0 }, 0.0, repeat(function(i) { i }, length(ys))));")
        c = r.choice(self.bools) if self.bools else f"({self.real_expr(1)} > 0.0)"
        return (f"  if ({c}) {{ factor({self.real_expr(1)} / 10.0) }} else "
                f"{{ observe(normal({self.real_expr(1)}, 2.0), 0.5) }};")


def program(seed: int) -> str:
    g = _Gen(seed)
    r = g.r
    n_pts = r.randint(1, 9)
    xs = ", ".join(f"{r.uniform(-2, 2):.3f}" for _ in range(n_pts))
    ys = ", ".join(f"{r.uniform(-2, 2):.3f}" for _ in range(n_pts))
    lines = [f"xs <- [{xs}];", f"ys <- [{ys}];", "model <- function() {"]
    for _ in range(r.randint(2, 5)):
        lines.append(g.draw())
        if r.random() < 0.6:
            lines.append(g.effect())
    lines.append(g.effect())
    if r.random() < 0.5 or not g.reals:
        ret = g.real_expr()
    else:
        ret = "[" + ", ".join(r.sample(g.reals, min(len(g.reals), 3))) + "]"
    lines.append(f"  {ret}")
    lines.append("};")
    lines.append("importance(model, 1000)")
    return "\n".join(lines) + "\n"


def discrete_program(seed: int) -> str:
    """A random finite-support program for enumerate(model, n): bernoulli / uniform-discrete /
    categorical choice points (at most 5), factors and observes of real expressions of them, an
    integer return."""
    r = random.Random(10_000 + seed)
    ints, bools, lines = [], [], ["model <- function() {"]
    n = 0
    for _ in range(r.randint(2, 5)):
        n += 1
        v = f"d{n}"
        k = r.random()
        if k < 0.35:
            lines.append(f"  {v} <- sample(bernoulli({r.uniform(0.1, 0.9):.2f}));")
            bools.append(v)
        elif k < 0.7:
            lo = r.randint(-2, 2)
            lines.append(f"  {v} <- sample(uniform-discrete({lo}, {lo + r.randint(2, 4)}));")
            ints.append(v)
        else:
            w = ", ".join(f"{r.uniform(0.1, 2):.2f}" for _ in range(r.randint(2, 4)))
            lines.append(f"  {v} <- sample(categorical([{w}]));")
            ints.append(v)
        if (ints or bools) and r.random() < 0.7:
            def term():
                if ints and (not bools or r.random() < 0.6):
                    return f"to-real({r.choice(ints)})"
                b = r.choice(bools)
                return f"if ({b}) {{ {r.uniform(-2, 2):.2f} }} else {{ {r.uniform(-2, 2):.2f} }}"
            e = term() if r.random() < 0.5 else f"({term()} * {r.uniform(-1.5, 1.5):.2f} + {term()})"
            if r.random() < 0.5:
                lines.append(f"  factor(-abs({e}) / 2.0);")
            else:
                lines.append(f"  observe(normal({e}, {r.uniform(0.5, 2):.2f}), {r.uniform(-2, 2):.2f});")
    if ints:
        ret = " + ".join(r.sample(ints, min(len(ints), 2)))
    else:
        ret = f"if ({bools[0]}) {{ 1 }} else {{ 0 }}"
    if bools and r.random() < 0.5:
        ret = f"if ({r.choice(bools)}) {{ {ret} }} else {{ 7 }}"
    lines += [f"  {ret}", "};", "enumerate(model, 100000)"]
    return "\n".join(lines) + "\n"


def vector_program(seed: int) -> str:
    """Random programs over drawn vectors: repeat of draws (literal or uniform-discrete length),
    reduce / map over them and over data, indexing by drawn integers, vector returns."""
    r = random.Random(20_000 + seed)
    n_pts = r.randint(1, 7)
    xs = ", ".join(f"{r.uniform(-2, 2):.3f}" for _ in range(n_pts))
    ys = ", ".join(f"{r.uniform(-2, 2):.3f}" for _ in range(n_pts))
    lines = [f"xs <- [{xs}];", f"ys <- [{ys}];", "model <- function() {"]
    length = str(r.randint(1, 5)) if r.random() < 0.5 else "k"
    if length == "k":
        lines.append(f"  k <- sample(uniform-discrete(1, {r.randint(2, 6)}));")
    lines.append(f"  c <- repeat(function(i) {{ sample(normal({r.uniform(-1, 1):.2f}, {r.uniform(0.5, 3):.2f})) }}, {length});")
    choice = r.random()
    if choice < 0.3:  # sum of squares of the vector as a factor
        lines.append("  factor(-reduce(function(acc, v) { acc + v * v }, 0.0, c) / 4.0);")
    elif choice < 0.6:  # a polynomial over the data (Horner over the drawn coefficients)
        lines.append("  factor(-reduce(function(acc, i) { acc + pow(ys[i] - reduce(function(p, j) { "
                     "p * xs[i] + c[length(c) - 1 - j] }, 0.0, repeat(function(j) { j }, length(c))), 2) }, "
                     "0.0, repeat(function(i) { i }, length(xs))) / 8.0);")
    else:  # an element picked by a drawn index
        lines.append("  j <- sample(uniform-discrete(0, length(c)));")
        lines.append(f"  observe(normal(c[j], {r.uniform(0.5, 2):.2f}), {r.uniform(-1, 1):.2f});")
    if r.random() < 0.5:  # per-datum draws inside map
        lines.append(f"  map(function(y) {{ e <- sample(normal(0.0, {r.uniform(0.5, 2):.2f})); "
                     f"observe(normal(e, 1.0), y) }}, ys);")
    if r.random() < 0.5:
        lines.append("  c")
    else:
        lines.append("  reduce(function(acc, v) { acc + v }, 0.0, c)")
    lines += ["};", "importance(model, 1000)"]
    return "\n".join(lines) + "\n"


def misc_program(seed: int) -> str:
    """Operators the other generators do not reach: integer % and /, floor, to-int, pow with
    non-2 exponents, && || !, int-valued ifs, closures over drawn values, a discrete return."""
    r = random.Random(30_000 + seed)
    lines = ["model <- function() {"]
    lines.append(f"  a <- sample(uniform-discrete({r.randint(-4, 0)}, {r.randint(2, 7)}));")
    lines.append(f"  b <- sample(uniform-discrete(1, {r.randint(3, 6)}));")
    lines.append(f"  x <- sample(normal({r.uniform(-1, 1):.2f}, {r.uniform(0.5, 2):.2f}));")
    lines.append(f"  t <- sample(bernoulli({r.uniform(0.2, 0.8):.2f}));")
    lines.append(f"  scale <- function(v) {{ v * x + {r.uniform(-1, 1):.2f} }};")  # closure over x
    ops = [
        "to-real(a % b)", "to-real(a / b)", "floor(x * 1.7)", "to-real(to-int(x * 2.3))",
        f"pow(abs(x) + 0.5, {r.choice([0.5, 1.5, 3.0])})", "scale(to-real(b))",
        "if (t && a > 0) { 1.5 } else { -0.5 }", "if (t || !(b > 2)) { x } else { -x }",
        "to-real(if (a >= b) { a - b } else { b - a })",
    ]
    for _ in range(r.randint(2, 4)):
        e = r.choice(ops)
        if r.random() < 0.5:
            lines.append(f"  factor(-abs({e}) / 3.0);")
        else:
            lines.append(f"  observe(normal({e}, {r.uniform(0.7, 2):.2f}), {r.uniform(-1, 1):.2f});")
    ret = r.choice(["a % b + 3", "if (t) { a } else { b }", "to-int(floor(x)) + 5", "a * b"])
    lines += [f"  {ret}", "};", "importance(model, 1000)"]
    return "\n".join(lines) + "\n"
