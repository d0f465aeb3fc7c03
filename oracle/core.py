"""ctypes binding of oracle/liboracle.so (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py)."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"


class OrRecord(C.Structure):
    """Layout of or_record == cuppl_is_record (include/cuppl_gpu.h)."""

    _fields_ = [
        ("max_lw", C.c_double),
        ("sum_w", C.c_double),
        ("sum_w2", C.c_double),
        ("argmax_lw", C.c_double),
        ("argmax_pid", C.c_uint64),
        ("n_finite", C.c_uint64),
        ("n_total", C.c_uint64),
        ("reserved", C.c_uint64),
        ("stat_w", C.c_double * 16),
        ("bin_w", C.c_double * 8),
    ]

    def as_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_ if f not in ("stat_w", "bin_w")}
        d["stat_w"] = np.array(self.stat_w[:])
        d["bin_w"] = np.array(self.bin_w[:])
        return d


def _source_hash() -> str:
    import hashlib

    h = hashlib.sha256()
    for p in sorted(HERE.glob("*.c")) + [HERE / "Makefile"]:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def build() -> Path:
    """Compile the C restatement (make, in-tree). Content-hash stamped, so a copied tree whose
    modification times are not preserved still rebuilds exactly when the sources changed."""
    stamp = LIB_PATH.with_suffix(".sha256")
    h = _source_hash()
    if LIB_PATH.exists() and stamp.exists() and stamp.read_text().strip() == h:
        return LIB_PATH
    subprocess.run(["make", "-s", "-B", "-C", str(HERE)], check=True)
    stamp.write_text(h)
    return LIB_PATH


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        P = C.POINTER
        u32p, f32p, f64p, i32p, u64p = (P(C.c_uint32), P(C.c_float), P(C.c_double),
                                        P(C.c_int32), P(C.c_uint64))
        L.or_philox.argtypes = [u32p, u32p, u32p]
        L.or_philox_blocks.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, u32p]
        L.or_u01_open0.argtypes = [C.c_uint32]
        L.or_u01_open0.restype = C.c_double
        L.or_u01_closed0.argtypes = [C.c_uint32]
        L.or_u01_closed0.restype = C.c_double
        L.or_lemire.argtypes = [C.c_uint32, C.c_uint32, u32p]
        L.or_box_muller.argtypes = [C.c_uint32, C.c_uint32, f64p, f64p]
        L.or_poly_draw.argtypes = [C.c_uint64, C.c_uint64, P(C.c_int), f64p]
        L.or_poly_lw.argtypes = [C.c_int, f64p, f32p, f32p, C.c_int]
        L.or_poly_lw.restype = C.c_double
        L.or_is_poly.argtypes = [f32p, f32p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, f32p,
                                 f64p, i32p, f64p, P(OrRecord), C.c_int]
        L.or_is_linreg.argtypes = [f32p, f32p, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                   C.c_uint64, f32p, f64p, f64p, P(OrRecord), C.c_int]
        L.or_dist_sample.argtypes = [C.c_int, C.c_double, C.c_double, u64p, C.c_int, C.c_uint64,
                                     C.c_uint32, C.c_uint64, C.c_uint64, f64p, i32p]
        L.or_rec_merge.argtypes = [P(OrRecord), P(OrRecord)]
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def philox(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox(_ptr(c, C.c_uint32), _ptr(k, C.c_uint32), _ptr(out, C.c_uint32))
    return out


def philox_blocks(key: int, first_id: int, block: int, tag: int, count: int) -> np.ndarray:
    out = np.zeros((count, 4), dtype=np.uint32)
    lib().or_philox_blocks(key, first_id, block, tag, count, _ptr(out, C.c_uint32))
    return out


def is_poly(xs, ys, pid_begin, pid_end, key, injected=None, traces=False, threads=0):
    xs = np.ascontiguousarray(xs, dtype=np.float32)
    ys = np.ascontiguousarray(ys, dtype=np.float32)
    n = pid_end - pid_begin
    inj = None if injected is None else np.ascontiguousarray(injected, dtype=np.float32)
    lw = np.zeros(n) if traces else None
    deg = np.zeros(n, dtype=np.int32) if traces else None
    coef = np.zeros((n, 4)) if traces else None
    rec = OrRecord()
    rc = lib().or_is_poly(_ptr(xs, C.c_float), _ptr(ys, C.c_float), len(xs), pid_begin, pid_end,
                          key, _ptr(inj, C.c_float), _ptr(lw, C.c_double), _ptr(deg, C.c_int32),
                          _ptr(coef, C.c_double), C.byref(rec), threads)
    assert rc == 0
    return rec.as_dict(), (lw, deg, coef)


def is_linreg(xs, ys, sigma, pid_begin, pid_end, key, injected=None, traces=False, threads=0):
    xs = np.ascontiguousarray(xs, dtype=np.float32)
    ys = np.ascontiguousarray(ys, dtype=np.float32)
    n = pid_end - pid_begin
    inj = None if injected is None else np.ascontiguousarray(injected, dtype=np.float32)
    lw = np.zeros(n) if traces else None
    coef = np.zeros((n, 2)) if traces else None
    rec = OrRecord()
    rc = lib().or_is_linreg(_ptr(xs, C.c_float), _ptr(ys, C.c_float), len(xs), float(sigma),
                            pid_begin, pid_end, key, _ptr(inj, C.c_float), _ptr(lw, C.c_double),
                            _ptr(coef, C.c_double), C.byref(rec), threads)
    assert rc == 0
    return rec.as_dict(), (lw, coef)


def dist_sample(tag: int, p0: float, p1: float, key: int, stream_tag: int, first_id: int,
                count: int, table: np.ndarray | None = None):
    """Returns float64 samples for continuous kinds, int32 for discrete ones."""
    discrete = tag in (1, 2, 3, 7)
    outf = None if discrete else np.zeros(count)
    outi = np.zeros(count, dtype=np.int32) if discrete else None
    tbl = None if table is None else np.ascontiguousarray(table, dtype=np.uint64)
    K = 0 if table is None else len(table) + 1
    rc = lib().or_dist_sample(tag, p0, p1, _ptr(tbl, C.c_uint64), K, key, stream_tag, first_id,
                              count, _ptr(outf, C.c_double), _ptr(outi, C.c_int32))
    assert rc == 0
    return outi if discrete else outf


def default_threads() -> int:
    return os.cpu_count() or 1


# ---------------------------------------------------------------------------- SMC -------
class OrSmcStats(C.Structure):
    _fields_ = [("M", C.c_float), ("status", C.c_uint32), ("T", C.c_uint64), ("s1", C.c_double),
                ("s2", C.c_double)]


def _smc_sig(L):
    P = C.POINTER
    if getattr(L, "_smc_sig", False):
        return
    L.or_smc_init.argtypes = [C.c_uint64, C.c_uint64, P(C.c_uint64), C.c_int, P(C.c_float), C.c_float,
                              C.c_float, C.c_float, P(C.c_int32), P(C.c_float)]
    L.or_smc_step.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, P(C.c_uint64), C.c_int, P(C.c_float),
                              C.c_float, C.c_float, C.c_float, P(C.c_int32), P(C.c_float), P(C.c_int32),
                              P(C.c_float), P(C.c_uint64), P(OrSmcStats), P(C.c_uint64)]
    L.or_smc_step.restype = C.c_int
    L.or_comb_target.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64]
    L.or_comb_target.restype = C.c_uint64
    L.or_comb_word.argtypes = [C.c_uint64, C.c_uint32]
    L.or_comb_word.restype = C.c_uint32
    L.or_alias_build.argtypes = [P(C.c_double), C.c_int, P(C.c_uint64)]
    L.or_alias_draw.argtypes = [P(C.c_uint64), C.c_int, C.c_uint32]
    L.or_alias_draw.restype = C.c_int
    L.or_exp_repro.argtypes = [C.c_float]
    L.or_exp_repro.restype = C.c_float
    L._smc_sig = True


def alias_table(weights) -> np.ndarray:
    """or_alias_build: u64 entries thr | alias << 40."""
    L = lib()
    _smc_sig(L)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.zeros(len(w), dtype=np.uint64)
    L.or_alias_build(_ptr(w, C.c_double), len(w), _ptr(out, C.c_uint64))
    return out


def alias_draw(table: np.ndarray, w: int) -> int:
    L = lib()
    _smc_sig(L)
    t = np.ascontiguousarray(table, dtype=np.uint64)
    return L.or_alias_draw(_ptr(t, C.c_uint64), len(t), w)


def smc_run(model, n: int, key: int, steps: int | None = None, record_ancestors: bool = False,
            hist_steps=None):
    """Exact CPU restatement of run_smc (or_smc_*). Returns a dict of per-step statistics,
    final population, integer filtering histograms and optionally ancestors per step."""
    L = lib()
    _smc_sig(L)
    S = model.n_states
    T = steps or model.T
    thrA = np.ascontiguousarray(np.concatenate([alias_table(model.A[s]) for s in range(S)]), dtype=np.uint64)
    thr0 = alias_table(model.pi0)
    mu = np.ascontiguousarray(model.mu, dtype=np.float32)
    ys = np.ascontiguousarray(model.ys, dtype=np.float32)
    inv_sd = np.float32(1.0 / model.sd)
    c = np.float32(-np.log(model.sd) - 0.5 * np.log(2 * np.pi))
    x = np.zeros(n, dtype=np.int32)
    lw = np.zeros(n, dtype=np.float32)
    x2 = np.zeros(n, dtype=np.int32)
    lw2 = np.zeros(n, dtype=np.float32)
    anc = np.zeros(n, dtype=np.uint64) if record_ancestors else None
    hist_steps = set(hist_steps if hist_steps is not None else [T - 1])
    u64p = C.POINTER(C.c_uint64)
    L.or_smc_init(n, key, _ptr(thr0, C.c_uint64), S, _ptr(mu, C.c_float), float(ys[0]),
                  float(inv_sd), float(c), _ptr(x, C.c_int32), _ptr(lw, C.c_float))
    out = {"M": np.zeros(T, np.float32), "T": np.zeros(T, np.uint64), "s1": np.zeros(T), "s2": np.zeros(T),
           "hist": {}, "ancestors": []}
    for t in range(T):
        st = OrSmcStats()
        h = np.zeros(S, dtype=np.uint64) if t in hist_steps else None
        last = t + 1 >= T
        rc = L.or_smc_step(n, key, t, _ptr(thrA, C.c_uint64), S, _ptr(mu, C.c_float),
                           float(ys[t + 1]) if not last else 0.0, float(inv_sd), float(c),
                           _ptr(x, C.c_int32), _ptr(lw, C.c_float),
                           None if last else _ptr(x2, C.c_int32), None if last else _ptr(lw2, C.c_float),
                           None if (last or anc is None) else anc.ctypes.data_as(u64p), C.byref(st),
                           None if h is None else h.ctypes.data_as(u64p))
        out["M"][t], out["T"][t], out["s1"][t], out["s2"][t] = st.M, st.T, st.s1, st.s2
        if h is not None:
            out["hist"][t] = h
        if rc != 0:
            out["status"] = (rc, t)
            break
        if not last:
            if anc is not None:
                out["ancestors"].append(anc.copy())
            x, x2 = x2, x
            lw, lw2 = lw2, lw
    out["x"], out["lw"] = x, lw
    out["log_z_steps"] = out["M"].astype(np.float64) + np.log(out["s1"]) - np.log(n)
    out["log_z"] = float(out["log_z_steps"].sum())
    return out


# ---------------------------------------------------------------------------- MH --------
def _mh_sig(L):
    P = C.POINTER
    if getattr(L, "_mh_sig", False):
        return
    L.or_mh_gmm_chain.argtypes = [P(C.c_float), C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint32,
                                  C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, P(C.c_double),
                                  P(C.c_double), P(C.c_double), C.c_uint32, P(C.c_int32), P(C.c_double)]
    L.or_mh_gmm_chain.restype = C.c_double
    L.or_mh_gmm.argtypes = [P(C.c_float), C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint32, C.c_uint32,
                            C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, P(C.c_double), P(C.c_double),
                            P(C.c_double), C.c_int]
    L._mh_sig = True


def mh_gmm(ys, K, prior_sd, sigma, n_chains, n_steps, key, chain_begin=0, burn_in=0, thin=1, threads=0):
    L = lib()
    _mh_sig(L)
    y = np.ascontiguousarray(ys, dtype=np.float32)
    mu = np.zeros((n_chains, K))
    ll = np.zeros(n_chains)
    st = np.zeros((n_chains, 2 * K + 2))
    L.or_mh_gmm(_ptr(y, C.c_float), len(y), K, prior_sd, sigma, n_chains, chain_begin, n_steps, burn_in, thin,
                key, _ptr(mu, C.c_double), _ptr(ll, C.c_double), _ptr(st, C.c_double), threads)
    return mu, ll, st


def mh_gmm_init(ys, K, prior_sd, sigma, chain, key):
    """Initial trace of one chain: (labels, means, log-likelihood)."""
    L = lib()
    _mh_sig(L)
    y = np.ascontiguousarray(ys, dtype=np.float32)
    z = np.zeros(len(y), dtype=np.int32)
    mu = np.zeros(K)
    st = np.zeros(2 * K + 2)
    ll0 = C.c_double()
    L.or_mh_gmm_chain(_ptr(y, C.c_float), len(y), K, prior_sd, sigma, chain, 0, 0, 1, key, _ptr(mu, C.c_double),
                      _ptr(st, C.c_double), None, 0, _ptr(z, C.c_int32), C.byref(ll0))
    return z, mu, ll0.value


def rec_from_dict(d: dict) -> OrRecord:
    r = OrRecord()
    for k, v in d.items():
        if k in ("stat_w", "bin_w"):
            getattr(r, k)[:] = [float(x) for x in v]
        else:
            setattr(r, k, v)
    return r


def merge_records(recs: list) -> dict:
    """or_rec_merge over window records (dicts) in window order: the record of their union."""
    L = lib()
    out = rec_from_dict(recs[0])
    for d in recs[1:]:
        b = rec_from_dict(d)
        L.or_rec_merge(C.byref(out), C.byref(b))
    return out.as_dict()


# ---------------------------------------------------------------- generic resampling --------
class OrResampleStats(C.Structure):
    _fields_ = [("M", C.c_float), ("status", C.c_uint32), ("T", C.c_uint64), ("s1", C.c_double),
                ("s2", C.c_double)]


def resample(lw, payload, key: int, t: int):
    """or_resample: systematic resampling of fp32 log-weights with a payload
    array whose first axis is the particle; returns (payload_out, ancestors, stats dict)."""
    L = lib()
    if not getattr(L, "_rs_sig", False):
        P = C.POINTER
        L.or_resample.argtypes = [C.c_uint64, P(C.c_float), C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                  C.c_void_p, P(C.c_uint64), P(OrResampleStats)]
        L.or_resample.restype = C.c_int
        L._rs_sig = True
    w = np.ascontiguousarray(lw, dtype=np.float32)
    n = len(w)
    pay = np.ascontiguousarray(payload)
    assert pay.shape[0] == n
    nbytes = pay.nbytes // n if n else 0
    out = np.empty_like(pay)
    anc = np.zeros(n, dtype=np.uint64)
    st = OrResampleStats()
    rc = L.or_resample(n, _ptr(w, C.c_float), pay.ctypes.data, nbytes, key, t, out.ctypes.data,
                       anc.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(st))
    stats = {"M": st.M, "T": st.T, "s1": st.s1, "s2": st.s2, "status": rc}
    return out, anc, stats
