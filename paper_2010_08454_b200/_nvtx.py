"""NVTX ranges per engine phase (tracing row), for ncu `--nvtx` filters and
timeline tools. Off unless CUPPL_NVTX=1, so the hot loops pay nothing by default."""

from __future__ import annotations

import contextlib
import functools
import os

ENABLED = os.environ.get("CUPPL_NVTX") == "1"


@contextlib.contextmanager
def phase(name: str):
    if not ENABLED:
        yield
        return
    import torch

    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()


def traced(name: str):
    """Decorator: the whole call inside one NVTX range."""
    def wrap(fn):
        @functools.wraps(fn)
        def inner(*a, **kw):
            with phase(name):
                return fn(*a, **kw)
        return inner
    return wrap
