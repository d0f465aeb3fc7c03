"""CPU tests of the C-ABI boundary: the library loads without a GPU, exports every symbol the
header declares, matches the ctypes layouts, and validates arguments before touching CUDA."""

import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADERS = sorted((ROOT / "include").glob("*.h"))


def declared_functions():
    names = []
    for h in HEADERS:
        names += re.findall(r"CUPPL_API\s+[\w\s\*]+?\b(cuppl_\w+)\s*\(", h.read_text())
    return names


def test_header_declares_functions():
    names = declared_functions()
    assert "cuppl_is_linreg" in names and "cuppl_abi_version" in names
    assert len(names) == len(set(names))


def test_library_exports_every_declared_symbol(native_lib):
    for name in declared_functions():
        assert hasattr(native_lib, name), f"{name} not exported"


def test_ctypes_signatures_cover_header(native_lib):
    from paper_2010_08454_b200 import _native

    assert set(declared_functions()) == set(_native.signatures())


def test_abi_version(native_lib):
    assert native_lib.cuppl_abi_version() == 1


def test_record_layout_matches_header():
    from paper_2010_08454_b200 import _native

    text = (ROOT / "include" / "cuppl_gpu.h").read_text()
    body = re.search(r"typedef struct cuppl_is_record \{(.*?)\} cuppl_is_record;", text, re.S).group(1)
    fields = re.findall(r"^\s*(?:double|uint64_t)\s+(\w+)", body, re.M)
    assert fields == [f for f, _ in _native.IsRecord._fields_]
    assert C.sizeof(_native.IsRecord) == 256
    body = re.search(r"typedef struct cuppl_dist \{(.*?)\} cuppl_dist;", text, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";"):  # every declarator: "double p0, p1, p2" -> p0, p1, p2
        decl = decl.strip()
        if not decl:
            continue
        head, *rest = decl.split(",")
        fields.append(re.search(r"(\w+)\s*$", head).group(1))
        fields += [r.strip().lstrip("*").strip() for r in rest]
    assert fields == [f for f, _ in _native.Dist._fields_]
    assert C.sizeof(_native.Dist) == 40


def test_smc_model_layout_matches_header():
    from paper_2010_08454_b200 import _native

    text = (ROOT / "include" / "cuppl_gpu.h").read_text()
    body = re.search(r"typedef struct cuppl_smc_model \{(.*?)\} cuppl_smc_model;", text, re.S).group(1)
    fields = re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(\w+);", body, re.M)
    assert fields == [f for f, _ in _native.SmcModel._fields_]
    assert C.sizeof(_native.SmcModel) == 48


def test_smc_arguments_rejected_before_cuda(native_lib):
    """SMC entry points validate their arguments on the host and name the problem."""
    from paper_2010_08454_b200 import _native

    L = _native.lib()
    m = _native.SmcModel()
    m.n_states, m.inv_sd, m.c = 4, 1.0, -0.9189385
    mu = np.zeros(4, dtype=np.float32)
    alias = np.zeros(4 * 4, dtype=np.uint64)
    m.alias_trans = alias.ctypes.data
    m.alias_init = alias.ctypes.data
    m.mu = mu.ctypes.data
    n = 4096
    wsb = L.cuppl_smc_workspace_bytes(n)
    ws = np.zeros(wsb, dtype=np.uint8)
    x = np.zeros(n, dtype=np.uint8)
    mk = np.zeros(2, dtype=np.int32)
    # NULL population buffer
    rc = L.cuppl_smc_init(C.byref(m), n, 0, 1, 0.0, None, mk.ctypes.data, ws.ctypes.data, wsb, None)
    assert rc == _native.E_ARGUMENT and b"NULL" in L.cuppl_last_error()
    # rank boundaries are multiples of 16
    rc = L.cuppl_smc_init(C.byref(m), n, 8, 1, 0.0, x.ctypes.data, mk.ctypes.data, ws.ctypes.data, wsb, None)
    assert rc == _native.E_ARGUMENT and b"16" in L.cuppl_last_error()
    # workspace too small
    rc = L.cuppl_smc_init(C.byref(m), n, 0, 1, 0.0, x.ctypes.data, mk.ctypes.data, ws.ctypes.data, wsb - 1, None)
    assert rc != _native.OK
    # rank outside the world
    rc = L.cuppl_smc_resample(C.byref(m), n, n, 1, 0, 3, 2, 0.0, 0.0, x.ctypes.data, mk.ctypes.data,
                              ws.ctypes.data, ws.ctypes.data, ws.ctypes.data, None, mk.ctypes.data,
                              ws.ctypes.data, ws.ctypes.data, wsb, None)
    assert rc == _native.E_ARGUMENT and b"world" in L.cuppl_last_error()
    # populations of 2^31 or more: the comb's 64-bit arithmetic would overflow
    rc = L.cuppl_smc_resample(C.byref(m), n, 1 << 31, 1, 0, 0, 1, 0.0, 0.0, x.ctypes.data, mk.ctypes.data,
                              ws.ctypes.data, ws.ctypes.data, ws.ctypes.data, None, mk.ctypes.data,
                              ws.ctypes.data, ws.ctypes.data, wsb, None)
    assert rc == _native.E_CAPACITY and b"2^31" in L.cuppl_last_error()
    # too many states for the one-byte population
    m.n_states = 300
    rc = L.cuppl_smc_init(C.byref(m), n, 0, 1, 0.0, x.ctypes.data, mk.ctypes.data, ws.ctypes.data, wsb, None)
    assert rc != _native.OK


def test_invalid_params_rejected_before_cuda(native_lib):
    """Parameter validation happens on the host, so it works (and maps errors) without a GPU."""
    from paper_2010_08454_b200 import _native, errors

    d = _native.Dist()
    d.tag = 0
    d.p0, d.p1 = 0.0, -1.0  # normal(0, -1)
    rc = native_lib.cuppl_dist_sample(C.byref(d), 1, 7, 0, 10, None, None)
    assert rc == _native.E_INVALID_PARAM
    with pytest.raises(errors.InvalidDistParamError):
        _native.check(rc)
    d.tag = 3
    d.p0, d.p1 = 5.0, 2.0  # uniform-discrete(5, 2)
    assert native_lib.cuppl_dist_sample(C.byref(d), 1, 7, 0, 10, None, None) == _native.E_INVALID_PARAM
    d.tag = 99
    rc = native_lib.cuppl_dist_sample(C.byref(d), 1, 7, 0, 10, None, None)
    assert rc == _native.E_UNSUPPORTED
    with pytest.raises(errors.UnsupportedDistError):
        _native.check(rc)
    xs = np.zeros(4, dtype=np.float32)
    fp = C.POINTER(C.c_float)
    rc = native_lib.cuppl_is_linreg(xs.ctypes.data_as(fp), xs.ctypes.data_as(fp), 4, 0.0, 0, 10, 1,
                                    None, None, None, None, None, 0, None)
    assert rc == _native.E_INVALID_PARAM


def test_host_record_merge_matches_oracle(native_lib, oracle_lib):
    """cuppl_is_record_merge (host code of the library) == oracle ordered merge."""
    from oracle import refstream
    from paper_2010_08454_b200 import infer, models

    m = models.PolyRegression.synthetic()
    n, key = 20_000, refstream.key_of(5)
    full, _ = oracle_lib.is_poly(m.xs, m.ys, 0, n, key, threads=1)
    parts = []
    for r in range(4):
        lo, hi = infer.shard_range(n, r, 4)
        d, _ = oracle_lib.is_poly(m.xs, m.ys, lo, hi, key, threads=1)
        rec = infer.N.IsRecord()
        for k, v in d.items():
            if k in ("stat_w", "bin_w"):
                getattr(rec, k)[:] = list(v)
            else:
                setattr(rec, k, v)
        parts.append(rec)
    got = infer.record_to_dict(infer.merge_records(parts))
    assert got["argmax_pid"] == full["argmax_pid"] and got["n_total"] == n
    assert got["sum_w"] == pytest.approx(full["sum_w"], rel=1e-12)
    assert np.allclose(got["stat_w"], full["stat_w"], rtol=1e-11, atol=1e-300)
    assert math.isfinite(got["max_lw"])


def test_shard_range_partitions():
    from paper_2010_08454_b200.infer import shard_range

    for n in (1, 7, 10**11 + 3):
        for R in (1, 2, 3, 8):
            rs = [shard_range(n, r, R) for r in range(R)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(R - 1))


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No CPU fallback: without the built library every entry point raises NativeLibraryError."""
    from paper_2010_08454_b200 import _native, errors

    monkeypatch.setattr(_native, "LIB_PATH", tmp_path / "libcuppl_gpu.so")
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(errors.NativeLibraryError, match="no CPU fallback"):
        _native.lib()
    with pytest.raises(errors.NativeLibraryError):
        _native.check(_native.E_CUDA)  # status mapping needs the library's message too
