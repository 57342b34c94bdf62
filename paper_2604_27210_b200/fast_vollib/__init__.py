"""The paper's public API (fast-vollib, PAPER.md:64-110 and Table 1,
PAPER.md:155-176) on the B200 path.

fast-vollib mirrors py_vollib_vectorized's names and conventions; the
reference implementation of its arithmetic is ``fastvol``'s batch engine
(SURVEY.md section 0 name map), so every function here is a thin front end
over ``paper_2604_27210_b200.batch`` (bit-identical to ``fastvol.batch``):

    fast_black / fast_black_scholes / fast_black_scholes_merton -> batch_price
    fast_implied_volatility (BS / BSM) / fast_implied_volatility_black
                                                   -> batch_iv(..., "halley")
    jackel.jackel_iv_black (LBR)                   -> batch_iv(BLACK76, "lbr")
    vectorized_{delta,gamma,theta,rho,vega}, get_all_greeks -> batch_greeks

Common keywords: ``flag`` ('c'/'p', scalar or array),
``return_as`` ('dataframe' (default), 'series', 'numpy' / 'array', 'dict',
'json'), ``dtype`` (output dtype, float64 default), ``backend`` and
``return_native``.  Inputs broadcast like the reference's batch engine
(length-1 columns extend to N).  Torch CUDA tensors are used in place: the
call runs device-resident (no host copies) and, with ``return_native=True``,
returns CUDA tensors.

Backend resolution: ``backend=`` keyword, then
``set_backend``, then the ``FAST_VOLLIB_BACKEND`` environment variable, then
'auto'.  This build has exactly one execution engine, the B200 CUDA path
('b200', alias 'cuda'); 'auto' resolves to it and fails loudly when no GPU
or built library is present -- there is no CPU fallback.  Asking for the
paper's 'numpy' / 'torch' / 'jax' engines raises ``BackendUnavailable``.
"""

import json
import os
import warnings

import numpy as np

from .. import _native
from ..batch import batch_greeks, batch_iv, batch_price
from ..models import Model
from . import jackel  # noqa: F401  (fast_vollib.jackel)
from ._device import device_call_greeks, device_call_iv, device_call_price, is_cuda_tensor

ENV_BACKEND = "FAST_VOLLIB_BACKEND"
BACKENDS = ("auto", "b200", "cuda")
_PAPER_BACKENDS = ("numpy", "torch", "jax")
_backend = None

GREEKS = ("delta", "gamma", "theta", "rho", "vega")
RETURN_AS = ("dataframe", "series", "numpy", "array", "dict", "json")

_MODELS = {"black": Model.BLACK76, "black76": Model.BLACK76, "black_scholes": Model.BLACK_SCHOLES,
           "bs": Model.BLACK_SCHOLES, "black_scholes_merton": Model.BLACK_SCHOLES_MERTON,
           "bsm": Model.BLACK_SCHOLES_MERTON}


class BackendUnavailable(RuntimeError):
    """The requested execution backend does not exist in this build."""


# ---------------------------------------------------------------------------
# backend resolution
# ---------------------------------------------------------------------------
def set_backend(name):
    """Select the default backend ('auto', 'b200' / 'cuda'); None resets."""
    global _backend
    if name is not None:
        _check_backend(name)
    _backend = name


def get_backend():
    """The backend a call without ``backend=`` resolves to."""
    return resolve_backend(None)


def _check_backend(name):
    key = str(name).lower()
    if key in _PAPER_BACKENDS:
        raise BackendUnavailable(
            f"backend {name!r} is not part of this build: the only execution engine is the B200 CUDA "
            "path ('b200'); there is no CPU/torch/jax fallback")
    if key not in BACKENDS:
        raise ValueError(f"unknown backend {name!r}; expected one of {BACKENDS}")
    return key


def resolve_backend(backend):
    """keyword > set_backend > $FAST_VOLLIB_BACKEND > 'auto'; always 'b200'."""
    for cand in (backend, _backend, os.environ.get(ENV_BACKEND)):
        if cand:
            _check_backend(cand)
            break
    return "b200"


def _engine(backend):
    resolve_backend(backend)
    return _native.lib_for_compute()         # fails loudly without a GPU / built library


# ---------------------------------------------------------------------------
# output containers
# ---------------------------------------------------------------------------
def _format(columns, return_as, dtype, index_len):
    """columns: ordered {name: 1-D array}."""
    kind = str(return_as).lower()
    if kind not in RETURN_AS:
        raise ValueError(f"return_as must be one of {RETURN_AS}, got {return_as!r}")
    cols = {k: np.asarray(v).astype(dtype, copy=False) for k, v in columns.items()}
    if kind in ("numpy", "array"):
        if len(cols) == 1:
            return next(iter(cols.values()))
        return np.column_stack(list(cols.values())) if index_len else np.empty((0, len(cols)), dtype)
    if kind == "dict":
        return cols
    if kind == "json":
        return json.dumps({k: [None if not np.isfinite(x) else float(x) for x in v] for k, v in cols.items()})
    import pandas as pd
    if kind == "series":
        if len(cols) != 1:
            raise ValueError("return_as='series' needs a single output column; use 'dataframe'")
        name, v = next(iter(cols.items()))
        return pd.Series(v, name=name)
    return pd.DataFrame(cols)


def _model(model, q):
    key = str(getattr(model, "value", model)).lower()
    if key not in _MODELS:
        raise ValueError(f"unknown model {model!r}")
    m = _MODELS[key]
    if m is Model.BLACK_SCHOLES and q is not None and _any_nonzero(q):
        m = Model.BLACK_SCHOLES_MERTON         # py_vollib_vectorized: q given -> BSM
    return m


def _any_nonzero(x):
    if hasattr(x, "is_cuda"):                  # torch tensor: reduce where it lives
        return bool((x != 0).any())
    return bool(np.any(np.asarray(x) != 0.0))


def _qcol(q):
    return 0.0 if q is None else q


def _iv_errors(iv, status, on_error):
    if on_error not in ("warn", "ignore", "raise"):
        raise ValueError("on_error must be 'warn', 'ignore' or 'raise'")
    if on_error == "ignore":
        return
    bad = np.isnan(np.asarray(iv))
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        msg = (f"{int(bad.sum())} of {bad.size} implied volatilities could not be found "
               f"(first: row {i}, status {status[i]!r}); they are NaN")
        if on_error == "raise":
            raise ValueError(msg)
        warnings.warn(msg, RuntimeWarning, stacklevel=3)


# ---------------------------------------------------------------------------
# pricing
# ---------------------------------------------------------------------------
def _price(model, flag, und, K, t, r, sigma, q, return_as, dtype, backend, return_native):
    lib = _engine(backend)
    if is_cuda_tensor(und, K, t, r, sigma, q):
        out = device_call_price(lib, model, flag, und, K, t, r, _qcol(q), sigma)
        if return_native:
            return out
        return _format({"Price": out.cpu().numpy()}, return_as, dtype, out.numel())
    tb = batch_price(model, flag, und, K, t, r, _qcol(q), sigma=sigma)
    return _format({"Price": tb["price"]}, return_as, dtype, tb.length)


def fast_black(flag, F, K, t, r, sigma, *, return_as="dataframe", dtype=np.float64, backend=None,
               return_native=False):
    """Black-76 prices on forward F (pricing.py:49-53)."""
    return _price(Model.BLACK76, flag, F, K, t, r, sigma, None, return_as, dtype, backend, return_native)


def fast_black_scholes(flag, S, K, t, r, sigma, *, return_as="dataframe", dtype=np.float64, backend=None,
                       return_native=False):
    """Black-Scholes prices on spot S (pricing.py:64-67)."""
    return _price(Model.BLACK_SCHOLES, flag, S, K, t, r, sigma, None, return_as, dtype, backend,
                  return_native)


def fast_black_scholes_merton(flag, S, K, t, r, sigma, q, *, return_as="dataframe", dtype=np.float64,
                              backend=None, return_native=False):
    """Black-Scholes-Merton prices with continuous dividend yield q
    (pricing.py:56-61)."""
    return _price(Model.BLACK_SCHOLES_MERTON, flag, S, K, t, r, sigma, q, return_as, dtype, backend,
                  return_native)


# ---------------------------------------------------------------------------
# implied volatility (Halley + bisection; solver.py:49-161)
# ---------------------------------------------------------------------------
def _iv(model, method, price, und, K, t, r, flag, q, on_error, return_as, dtype, backend, return_native):
    lib = _engine(backend)
    if is_cuda_tensor(price, und, K, t, r, q):
        iv, status = device_call_iv(lib, model, method, flag, und, K, t, r, _qcol(q), price)
        if return_native:
            return iv
        ivh = iv.cpu().numpy()
        _iv_errors(ivh, status.cpu().numpy(), on_error)
        return _format({"IV": ivh}, return_as, dtype, ivh.size)
    tb = batch_iv(model, method, flag, und, K, t, r, price=price, q=_qcol(q))
    _iv_errors(tb["iv"], tb["status"], on_error)
    return _format({"IV": tb["iv"]}, return_as, dtype, tb.length)


def fast_implied_volatility(price, S, K, t, r, flag, q=None, *, on_error="warn", model="black_scholes",
                            return_as="dataframe", dtype=np.float64, backend=None, return_native=False):
    """Implied volatility of spot-model quotes (BS, or BSM when ``q`` is
    given / model='black_scholes_merton'); Halley with bisection fallback."""
    m = _model(model, q)
    return _iv(m, "halley", price, S, K, t, r, flag, q, on_error, return_as, dtype, backend, return_native)


def fast_implied_volatility_black(price, F, K, r, t, flag, *, on_error="warn", return_as="dataframe",
                                  dtype=np.float64, backend=None, return_native=False):
    """Implied volatility of Black-76 (futures-style) quotes; note the
    py_vollib argument order (price, F, K, r, t, flag)."""
    return _iv(Model.BLACK76, "halley", price, F, K, t, r, flag, None, on_error, return_as, dtype, backend,
               return_native)


# ---------------------------------------------------------------------------
# Greeks (greeks.py:45-104): per-day theta, per-1% vega and rho
# ---------------------------------------------------------------------------
def _greeks(names, flag, S, K, t, r, sigma, q, model, return_as, dtype, backend, return_native):
    m = _model(model, q)
    lib = _engine(backend)
    if is_cuda_tensor(S, K, t, r, sigma, q):
        outs = device_call_greeks(lib, m, flag, S, K, t, r, _qcol(q), sigma)
        if return_native:
            return outs[names[0]] if len(names) == 1 else {k: outs[k] for k in names}
        cols = {k: outs[k].cpu().numpy() for k in names}
        return _format(cols, return_as, dtype, len(next(iter(cols.values()))))
    tb = batch_greeks(m, flag, S, K, t, r, _qcol(q), sigma=sigma)
    return _format({k: tb[k] for k in names}, return_as, dtype, tb.length)


def get_all_greeks(flag, S, K, t, r, sigma, q=None, *, model="black_scholes", return_as="dataframe",
                   dtype=np.float64, backend=None, return_native=False):
    """delta, gamma, theta, rho, vega in one batched call (d1/d2, Phi, phi
    computed once per row)."""
    return _greeks(GREEKS, flag, S, K, t, r, sigma, q, model, return_as, dtype, backend, return_native)


def _one_greek(name):
    def fn(flag, S, K, t, r, sigma, q=None, *, model="black_scholes", return_as="dataframe",
           dtype=np.float64, backend=None, return_native=False):
        return _greeks((name,), flag, S, K, t, r, sigma, q, model, return_as, dtype, backend, return_native)
    fn.__name__ = fn.__qualname__ = "vectorized_" + name
    fn.__doc__ = f"{name} of every row (one fused Greeks call; greeks.py:45-98)."
    return fn


vectorized_delta = _one_greek("delta")
vectorized_gamma = _one_greek("gamma")
vectorized_theta = _one_greek("theta")
vectorized_rho = _one_greek("rho")
vectorized_vega = _one_greek("vega")


# ---------------------------------------------------------------------------
# drop-in patching
# ---------------------------------------------------------------------------
from ._patch import patch_py_vollib, patch_py_vollib_vectorized  # noqa: E402

__all__ = [
    "fast_black", "fast_black_scholes", "fast_black_scholes_merton", "fast_implied_volatility",
    "fast_implied_volatility_black", "get_all_greeks", "vectorized_delta", "vectorized_gamma",
    "vectorized_theta", "vectorized_rho", "vectorized_vega", "set_backend", "get_backend",
    "resolve_backend", "BackendUnavailable", "patch_py_vollib", "patch_py_vollib_vectorized", "jackel",
]
