"""Runtime values on the inference boundary (mirrors pkg/src/cuppl/values.py).

`DistValue` keeps the reference's fixed 1-tag + 3-slot layout (values.py:86-98,
PAPER.md:589-594); `value_key` / `value_eq` give the structural identity used to merge
posterior support (values.py:101-129); `render_value` / `json_value` the
posterior serialisation forms (values.py:132-180).
"""

from __future__ import annotations

from .errors import TypeMismatchError

# Tags: constructor order of pkg/src/cuppl/builtins.py:86-94, then categorical.
NORMAL, BERNOULLI, POISSON, UNIFORM_DISCRETE, UNIFORM_CONTINUOUS, BETA, EXPONENTIAL, CATEGORICAL = range(8)
TAG_NAMES = ("normal", "bernoulli", "poisson", "uniform-discrete", "uniform-continuous", "beta",
             "exponential", "categorical")
DISCRETE_TAGS = frozenset({BERNOULLI, POISSON, UNIFORM_DISCRETE, CATEGORICAL})


class DistValue:
    """Fixed-size distribution value: one tag and three payload slots."""

    __slots__ = ("tag", "p0", "p1", "p2")

    def __init__(self, tag, p0=0, p1=0, p2=0):
        self.tag = tag
        self.p0 = p0
        self.p1 = p1
        self.p2 = p2

    def __repr__(self):
        return f"<dist tag={self.tag} {self.p0} {self.p1} {self.p2}>"


def value_key(v):
    """Hashable structural key; distinct scalar types never collide (values.py:101-122)."""
    if v is None:
        return ("u",)
    if v is True or v is False:
        return ("b", v)
    t = type(v)
    if t is int:
        return ("i", v)
    if t is float:
        return ("r", v)
    if t is str:
        return ("s", v)
    if t is tuple:
        return ("t",) + tuple(value_key(x) for x in v)
    if t is list:
        return ("v",) + tuple(value_key(x) for x in v)
    if t is DistValue:
        return ("d", v.tag, value_key(v.p0), value_key(v.p1), value_key(v.p2))
    raise TypeMismatchError(f"value of kind {t.__name__} has no structural identity")


def value_eq(a, b):
    return value_key(a) == value_key(b)


def render_value(v):
    if v is None:
        return "()"
    if v is True:
        return "true"
    if v is False:
        return "false"
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        return repr(v)
    if isinstance(v, str):
        return v
    if isinstance(v, tuple):
        return "(" + ", ".join(render_value(x) for x in v) + ")"
    if isinstance(v, list):
        return "[" + ", ".join(render_value(x) for x in v) + "]"
    if isinstance(v, DistValue):
        return f"<dist:{v.tag}>"
    return repr(v)


def json_value(v):
    if v is None or isinstance(v, (bool, int, float, str)):
        return v
    if isinstance(v, (tuple, list)):
        return [json_value(x) for x in v]
    raise TypeMismatchError(f"cannot serialize {type(v).__name__} to JSON")
