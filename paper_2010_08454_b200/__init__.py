"""paper_2010_08454_b200 — B200-native (sm_100a) inference hot path of CuPPL (arXiv 2010.08454).

Public surface mirrors the reference package's inference API and runtime
types (pkg/src/cuppl/rng.py, values.py, errors.py):

    from paper_2010_08454_b200 import infer, models, dists, Rng
    post = infer.run_importance(models.LinearRegression.synthetic(), 10**9, Rng(1))

All engines run in libcuppl_gpu.so (csrc/, C ABI in include/cuppl_gpu.h).
"""

from . import dists, errors, infer, models, values  # noqa: F401
from .rng import Rng  # noqa: F401

__all__ = ["dists", "errors", "infer", "models", "values", "Rng"]
