"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the batched pricing / Greeks /
implied-vol path.  Never imported by the product package; only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline / reference arms use
it, always as the checker (or the timed CPU reference), never as the thing
measured on the GPU.

``fvoracle.cpp`` is a statement-for-statement C++ restatement of
/root/reference/pkg/src/fastvol/{batch,pricing,greeks,solver,lbr,
distributions}.py that calls the REAL glibc libm and the REAL scipy erfcx
(``scipy.special.cython_special``); this module builds/loads it, restates the
batch front end (``batch.py:_assemble``/``validate``, numpy) and turns the
per-row exception codes into the exception the reference would raise
(``batch.py:_run_chunked`` surfaces the lowest failing row).

Pinned against the live reference by tests/golden/*.npz (made by
tests/golden/gen_golden.py) -- see tests/test_oracle_golden.py.
"""

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fvoracle.cpp")
BUILD_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(BUILD_DIR, "liborc.so")

MODEL_IDS = {"black": 0, "black76": 0, "b76": 0, "bs": 1, "black_scholes": 1,
             "bsm": 2, "black_scholes_merton": 2}
IV_STATUS = np.array(["converged", "fell_back_to_bisection", "below_intrinsic",
                      "above_upper_bound", "max_iterations"], dtype=object)
GREEK_STATUS = np.array(["ok", "step_function_edge"], dtype=object)
REGIONS = ("far_low", "near_low", "near_high", "far_high")

_lock = threading.Lock()
_lib = None


class OracleDomainError(ValueError):
    """Stands in for fastvol.errors.DomainError (a ValueError subclass)."""


class OracleBatchError(Exception):
    def __init__(self, kind, index, detail):
        self.kind, self.index, self.detail = kind, index, detail
        super().__init__(f"{kind} at row {index}: {detail}")


CXXFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fno-builtin", "-fopenmp",
            "-shared", "-fPIC"]


def build(force=False):
    """Compile fvoracle.cpp with g++: no FMA contraction (CPython rounds every
    op), -fno-builtin so every libm call really reaches glibc (gcc would
    otherwise fold pow(x, 2.0) into x*x, which glibc's pow is not), OpenMP."""
    os.makedirs(BUILD_DIR, exist_ok=True)
    stamp = LIB + ".cmd"
    cmd = ["g++"] + CXXFLAGS + ["-o", LIB, SRC, "-lm"]
    fresh = (os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC)
             and os.path.exists(stamp) and open(stamp).read() == " ".join(cmd))
    if fresh and not force:
        return LIB
    tmp = LIB + ".tmp%d" % os.getpid()
    subprocess.run(["g++"] + CXXFLAGS + ["-o", tmp, SRC, "-lm"], check=True)
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(" ".join(cmd))
    return LIB


def _scipy_erfcx_ptr():
    import scipy.special.cython_special as cs
    cap = cs.__pyx_capi__["__pyx_fuse_1erfcx"]
    get = ctypes.pythonapi.PyCapsule_GetPointer
    get.restype = ctypes.c_void_p
    get.argtypes = [ctypes.py_object, ctypes.c_char_p]
    return get(cap, b"double (double, int __pyx_skip_dispatch)")


def _asym_tables():
    """lbr.py:59-62, restated: _ASYM_FACTS and _ASYM_PASCAL."""
    from scipy.linalg import pascal
    from scipy.special import factorial2
    facts = np.concatenate([[1.0], [float(factorial2(n)) * (-1.0) ** ((n + 1) // 2)
                                    for n in range(1, 34, 2)]])
    pas = 2.0 * pascal(36, kind="lower")[:, 1::2][1::2, :].T
    return (np.ascontiguousarray(facts, dtype=np.float64),
            np.ascontiguousarray(np.asarray(pas, dtype=np.float64)))


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            facts, pas = _asym_tables()
            L.orc_init(ctypes.c_void_p(_scipy_erfcx_ptr()),
                       facts.ctypes.data_as(ctypes.c_void_p),
                       pas.ctypes.data_as(ctypes.c_void_p))
            L.orc_normalized_black.restype = ctypes.c_double
            L.orc_normalized_black.argtypes = [ctypes.c_double, ctypes.c_double,
                                               ctypes.POINTER(ctypes.c_int)]
            L.orc_norm_cdf.restype = ctypes.c_double
            L.orc_norm_cdf.argtypes = [ctypes.c_double]
            L.orc_inv_norm_cdf.restype = ctypes.c_double
            L.orc_inv_norm_cdf.argtypes = [ctypes.c_double]
            _lib = L
    return _lib


def set_threads(n):
    """OpenMP thread count used by the oracle's batch loops."""
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def _col(a, n):
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 0:
        a = a.reshape(1)
    if a.shape[0] == 1 and n != 1:
        a = np.broadcast_to(a, (n,))
    return np.ascontiguousarray(a)


def _model_id(model):
    if isinstance(model, (int, np.integer)):
        return int(model)
    name = getattr(model, "value", model)
    return MODEL_IDS[str(name).lower()]


# --------------------------------------------------------------------------
# batch.py front end (numpy restatement of _assemble / validate)
# --------------------------------------------------------------------------
def parse_flags(flags):
    """batch.py:78-88: case-insensitive 'c'/'p' -> +1/-1, BadFlag at first bad row."""
    if isinstance(flags, str):
        flags = [flags]
    out = np.empty(len(flags), dtype=np.int8)
    for i, f in enumerate(flags):
        if f == "c" or f == "C":
            out[i] = 1
        elif f == "p" or f == "P":
            out[i] = -1
        else:
            raise OracleBatchError("BadFlag", i, f"option flag must be 'c' or 'p', got {f!r}")
    return out


def assemble(model, flag, underlying, strike, t, r, q=0.0, sigma=None, price=None):
    """batch.py:127-148 -> (n, dict of full-length contiguous columns)."""
    theta = parse_flags(flag)
    raw = {"underlying": underlying, "strike": strike, "t": t, "r": r, "q": q}
    if sigma is not None:
        raw["sigma"] = sigma
    if price is not None:
        raw["price"] = price
    lengths = [theta.shape[0]] + [np.atleast_1d(np.asarray(v, dtype=np.float64)).shape[0]
                                  for v in raw.values()]
    n = max(lengths, default=1)
    if 0 in lengths:
        n = 0
    for i, length in enumerate(lengths):
        if length not in (1, n):
            raise OracleBatchError("ShapeMismatch", i,
                                   f"length {length} incompatible with batch size {n}")
    table = {"flag": theta if theta.shape[0] == n else np.broadcast_to(theta, (n,))}
    for name, values in raw.items():
        arr = np.atleast_1d(np.asarray(values, dtype=np.float64))
        if arr.ndim != 1:
            raise OracleBatchError("ShapeMismatch", 0, f"column {name} is not 1-D")
        if arr.shape[0] == 1 and n != 1:
            arr = np.broadcast_to(arr, (n,))
        if arr.shape[0] != n:
            raise OracleBatchError("ShapeMismatch", 0,
                                   f"column {name} has length {arr.shape[0]}, expected {n}")
        table[name] = arr
    for name, col in table.items():
        if col.dtype.kind != "f":
            continue
        bad = np.flatnonzero(~np.isfinite(col))
        if bad.size:
            raise OracleBatchError("NonFiniteInput", int(bad[0]), f"column {name} is not finite")
    for name in ("underlying", "strike"):
        bad = np.flatnonzero(~(table[name] > 0.0))
        if bad.size:
            raise OracleBatchError("DomainError", int(bad[0]), f"column {name} must be positive")
    for name in ("t", "sigma"):
        if name in table:
            bad = np.flatnonzero(table[name] < 0.0)
            if bad.size:
                raise OracleBatchError("DomainError", int(bad[0]), f"column {name} must be >= 0")
    if _model_id(model) != 2 and np.any(table["q"] != 0.0):
        idx = int(np.flatnonzero(table["q"] != 0.0)[0])
        mname = {0: "black", 1: "bs"}[_model_id(model)]
        raise OracleBatchError("DomainError", idx,
                               f"model {mname} does not accept a dividend yield")
    return n, {k: np.ascontiguousarray(v) for k, v in table.items()}


# --------------------------------------------------------------------------
# per-row exception codes -> the exception the reference raises
# --------------------------------------------------------------------------
def _repr_value(v, is_np):
    return repr(np.float64(v)) if is_np else repr(float(v))


def exception_for(code, val=0.0, is_np=False):
    """Map an oracle/kernel exception code to the reference's exception."""
    code = int(code)
    if code == 1:
        return OverflowError("math range error")
    if code == 2:
        return ValueError("math domain error")
    if code == 3:
        return ZeroDivisionError("float division by zero")
    if code == 4:
        return OverflowError(34, "Numerical result out of range")
    if code == 5:
        return OracleDomainError("F and K must be positive")
    if code == 6:
        return OracleDomainError(f"atm_inverse requires beta in (0, 1), got {_repr_value(val, is_np)}")
    if code == 7:
        return OracleDomainError(f"inv_norm_cdf requires p in (0, 1), got {_repr_value(val, is_np)}")
    if code == 8:
        return OracleDomainError(f"normalized_black requires x <= 0, got {_repr_value(val, is_np)}")
    if code == 9:
        return OracleDomainError(f"normalized_black requires s > 0, got {_repr_value(val, is_np)}")
    if code == 10:
        return OracleDomainError(f"objective_branch requires s > 0, got {_repr_value(val, is_np)}")
    raise AssertionError(f"unknown exception code {code}")


def exception_text(exc):
    return f"{type(exc).__name__}: {exc}"


class RowResult(dict):
    """Columns plus per-row exception arrays (exc, exc_val, exc_np)."""

    def raise_first(self):
        bad = np.flatnonzero(self["exc"])
        if bad.size:
            i = int(bad[0])
            raise exception_for(self["exc"][i], self["exc_val"][i], bool(self["exc_np"][i]))


def _exc_arrays(n):
    return np.zeros(n, np.int8), np.zeros(n, np.float64), np.zeros(n, np.int8)


def rows_price(model, flag, un, k, t, r, q, sg):
    """fill() of batch_price on already-assembled columns, per-row exceptions."""
    n = len(flag)
    cols = [np.ascontiguousarray(flag, dtype=np.int8)] + [_col(c, n) for c in (un, k, t, r, q, sg)]
    out = np.empty(n)
    exc, ev, en = _exc_arrays(n)
    lib().orc_batch_price(ctypes.c_int(_model_id(model)), *[_p(c) for c in cols],
                          ctypes.c_int64(n), _p(out), _p(exc), _p(ev), _p(en))
    return RowResult(price=out, exc=exc, exc_val=ev, exc_np=en)


def rows_greeks(model, flag, un, k, t, r, q, sg):
    n = len(flag)
    cols = [np.ascontiguousarray(flag, dtype=np.int8)] + [_col(c, n) for c in (un, k, t, r, q, sg)]
    outs = [np.empty(n) for _ in range(5)]
    st = np.empty(n, np.int8)
    exc, ev, en = _exc_arrays(n)
    lib().orc_batch_greeks(ctypes.c_int(_model_id(model)), *[_p(c) for c in cols],
                           ctypes.c_int64(n), *[_p(o) for o in outs], _p(st),
                           _p(exc), _p(ev), _p(en))
    return RowResult(delta=outs[0], gamma=outs[1], theta=outs[2], rho=outs[3], vega=outs[4],
                     status_code=st, exc=exc, exc_val=ev, exc_np=en)


def rows_iv(model, method, flag, un, k, t, r, q, px):
    n = len(flag)
    cols = [np.ascontiguousarray(flag, dtype=np.int8)] + [_col(c, n) for c in (un, k, t, r, q, px)]
    iv = np.empty(n)
    st = np.empty(n, np.int8)
    iters = np.empty(n, np.int32)
    reg = np.empty(n, np.int8)
    exc, ev, en = _exc_arrays(n)
    m = {"halley": 0, "lbr": 1}[method]
    lib().orc_batch_iv(ctypes.c_int(_model_id(model)), ctypes.c_int(m), *[_p(c) for c in cols],
                       ctypes.c_int64(n), _p(iv), _p(st), _p(iters), _p(reg),
                       _p(exc), _p(ev), _p(en))
    return RowResult(iv=iv, status_code=st, iterations=iters, region=reg,
                     exc=exc, exc_val=ev, exc_np=en)


# --------------------------------------------------------------------------
# batch.py public entry points (oracle flavour): same semantics, dict result
# --------------------------------------------------------------------------
def batch_price(model, flag, underlying, strike, t, r, q=0.0, sigma=None):
    n, tb = assemble(model, flag, underlying, strike, t, r, q, sigma=sigma)
    if "sigma" not in tb:
        raise OracleBatchError("DomainError", 0, "batch_price requires sigma")
    res = rows_price(model, tb["flag"], tb["underlying"], tb["strike"], tb["t"], tb["r"],
                     tb["q"], tb["sigma"])
    res.raise_first()
    cols = dict(tb)
    cols["price"] = res["price"]
    return cols


def batch_iv(model, method, flag, underlying, strike, t, r, price=None, q=0.0):
    if method not in ("halley", "lbr"):
        raise OracleBatchError("DomainError", 0, f"unknown IV method {method!r}")
    n, tb = assemble(model, flag, underlying, strike, t, r, q, price=price)
    if "price" not in tb:
        raise OracleBatchError("DomainError", 0, "batch_iv requires price")
    res = rows_iv(model, method, tb["flag"], tb["underlying"], tb["strike"], tb["t"], tb["r"],
                  tb["q"], tb["price"])
    res.raise_first()
    cols = dict(tb)
    cols["iv"] = res["iv"]
    cols["status"] = IV_STATUS[res["status_code"]]
    return cols


def batch_greeks(model, flag, underlying, strike, t, r, q=0.0, sigma=None):
    n, tb = assemble(model, flag, underlying, strike, t, r, q, sigma=sigma)
    if "sigma" not in tb:
        raise OracleBatchError("DomainError", 0, "batch_greeks requires sigma")
    res = rows_greeks(model, tb["flag"], tb["underlying"], tb["strike"], tb["t"], tb["r"],
                      tb["q"], tb["sigma"])
    res.raise_first()
    cols = dict(tb)
    for g in ("delta", "gamma", "theta", "rho", "vega"):
        cols[g] = res[g]
    cols["status"] = GREEK_STATUS[res["status_code"]]
    return cols


def normalized_black(x, s):
    br = ctypes.c_int(-1)
    v = lib().orc_normalized_black(float(x), float(s), ctypes.byref(br))
    return v, br.value
