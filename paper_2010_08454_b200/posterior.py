"""Posterior wire format: serialize_posterior / parse_posterior.

tsv  -- one `value TAB probability` row per support point, probability descending, ties by
        the value's text ascending; probabilities are written with repr() so parsing gives the
        identical floats back.
json -- {"support": [{"value": v, "prob": p}, ...], "log_z": z, ...} with the same ordering;
        extra summary keys (n, ess, mode, mean) are carried alongside.

Values render with values.render_value / values.json_value (the reference's forms,
pkg/src/cuppl/values.py:132-180). Same inputs give byte-identical text (SPEC.md, cli
invariants). A posterior whose return value is real-valued has singleton support per
particle; it has no finite support list, so its tsv form is refused and its json
form carries the summaries with an empty support.
"""

from __future__ import annotations

import json
import math

from .values import json_value, render_value


def _ordered(support):
    return sorted(((v, float(p)) for v, p in support), key=lambda vp: (-vp[1], render_value(vp[0])))


def _finite(x):
    if x is None:
        return None
    x = float(x)
    return x if math.isfinite(x) else repr(x)


def serialize_posterior(d, fmt: str = "tsv") -> str:
    """EmpiricalDistribution (or anything with .support / .log_z) -> text."""
    support = list(getattr(d, "support", []) or [])
    if fmt == "tsv":
        if not support:
            raise ValueError("serialize_posterior: empty support (real-valued return); use json")
        return "".join(f"{render_value(v)}\t{p!r}\n" for v, p in _ordered(support))
    if fmt == "json":
        obj = {"support": [{"value": json_value(v), "prob": p} for v, p in _ordered(support)],
               "log_z": _finite(getattr(d, "log_z", None))}
        for k in ("n", "ess", "mode_log_weight", "mode_index"):
            if hasattr(d, k):
                v = getattr(d, k)
                obj[k] = _finite(v) if isinstance(v, float) else v
        mode = getattr(d, "mode", None)
        if mode is not None:
            obj["mode"] = json_value(list(mode) if isinstance(mode, tuple) else mode)
        mean = getattr(d, "mean", None)
        if mean:
            obj["mean"] = {k: (None if v is None else json_value(v) if not hasattr(v, "tolist") else v.tolist())
                           for k, v in mean.items()}
        return json.dumps(obj, sort_keys=False, separators=(",", ":")) + "\n"
    raise ValueError(f"unknown posterior format {fmt!r} (tsv | json)")


def _parse_scalar(text: str):
    if text == "true":
        return True
    if text == "false":
        return False
    if text == "()":
        return None
    try:
        return int(text)
    except ValueError:
        pass
    try:
        return float(text)
    except ValueError:
        return text


def parse_posterior(text: str, fmt: str = "tsv") -> dict:
    """Inverse of serialize_posterior: {"support": [(value, prob)], "log_z": ...}. Scalar values
    (bool, int, float, unit, str) round-trip exactly; json values come back as json types."""
    if fmt == "tsv":
        support = []
        for line in text.splitlines():
            if not line:
                continue
            v, p = line.rsplit("\t", 1)
            support.append((_parse_scalar(v), float(p)))
        return {"support": support, "log_z": None}
    if fmt == "json":
        obj = json.loads(text)
        obj["support"] = [(e["value"], float(e["prob"])) for e in obj["support"]]
        return obj
    raise ValueError(f"unknown posterior format {fmt!r} (tsv | json)")
