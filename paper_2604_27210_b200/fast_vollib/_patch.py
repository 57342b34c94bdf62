"""``patch_py_vollib`` / ``patch_py_vollib_vectorized``:
point the upstream namespaces at the B200 functions so existing user code
dispatches here unchanged.  Each returns an ``undo()`` callable; a missing
upstream package raises ImportError (nothing is patched).

py_vollib's scalar API (``py_vollib.black.black(flag, F, K, t, r, sigma)``,
``...black_scholes.implied_volatility.implied_volatility(price, S, K, t, r,
flag)``, ``...greeks.analytical.delta(flag, S, K, t, r, sigma)``, ...) gets
wrappers that accept scalars or arrays and return a float for scalar inputs,
an ndarray otherwise.  py_vollib_vectorized's names map one to one onto this
package's (``vectorized_implied_volatility`` -> fast_implied_volatility, ...).
"""

import importlib

import numpy as np

GREEKS = ("delta", "gamma", "theta", "rho", "vega")


def _import(name):
    try:
        return importlib.import_module(name)
    except ImportError as exc:
        raise ImportError(f"{name} is not installed; nothing to patch") from exc


def _scalar_or_array(out, *inputs):
    arr = np.asarray(out, dtype=np.float64).reshape(-1)
    if all(np.ndim(x) == 0 for x in inputs if not isinstance(x, str)) and arr.size == 1:
        return float(arr[0])
    return arr


def _setattrs(saved, mod, mapping):
    for name, fn in mapping.items():
        saved.append((mod, name, getattr(mod, name, None), hasattr(mod, name)))
        setattr(mod, name, fn)


def _undo(saved):
    def undo():
        for mod, name, old, had in reversed(saved):
            if had:
                setattr(mod, name, old)
            else:
                delattr(mod, name)
    return undo


def patch_py_vollib():
    from . import (fast_black, fast_black_scholes, fast_black_scholes_merton, fast_implied_volatility,
                   fast_implied_volatility_black, get_all_greeks)
    _import("py_vollib")
    saved = []
    kw = {"return_as": "numpy"}

    def black(flag, F, K, t, r, sigma):
        return _scalar_or_array(fast_black(flag, F, K, t, r, sigma, **kw), F, K, t, r, sigma)

    def black_scholes(flag, S, K, t, r, sigma):
        return _scalar_or_array(fast_black_scholes(flag, S, K, t, r, sigma, **kw), S, K, t, r, sigma)

    def black_scholes_merton(flag, S, K, t, r, sigma, q):
        return _scalar_or_array(fast_black_scholes_merton(flag, S, K, t, r, sigma, q, **kw), S, K, t, r, sigma, q)

    def iv_black(discounted_option_price, F, K, r, t, flag):
        return _scalar_or_array(fast_implied_volatility_black(discounted_option_price, F, K, r, t, flag,
                                                              on_error="ignore", **kw),
                                discounted_option_price, F, K, r, t)

    def iv_bs(price, S, K, t, r, flag):
        return _scalar_or_array(fast_implied_volatility(price, S, K, t, r, flag, on_error="ignore",
                                                        model="black_scholes", **kw), price, S, K, t, r)

    def iv_bsm(price, S, K, t, r, q, flag):
        return _scalar_or_array(fast_implied_volatility(price, S, K, t, r, flag, q, on_error="ignore",
                                                        model="black_scholes_merton", **kw), price, S, K, t, r, q)

    def greek_fn(name, model, with_q):
        if with_q:
            def fn(flag, S, K, t, r, sigma, q):
                g = get_all_greeks(flag, S, K, t, r, sigma, q, model=model, return_as="dict")
                return _scalar_or_array(g[name], S, K, t, r, sigma, q)
        else:
            def fn(flag, S, K, t, r, sigma):
                g = get_all_greeks(flag, S, K, t, r, sigma, model=model, return_as="dict")
                return _scalar_or_array(g[name], S, K, t, r, sigma)
        fn.__name__ = name
        return fn

    targets = [
        ("py_vollib.black", {"black": black}),
        ("py_vollib.black_scholes", {"black_scholes": black_scholes}),
        ("py_vollib.black_scholes_merton", {"black_scholes_merton": black_scholes_merton}),
        ("py_vollib.black.implied_volatility", {"implied_volatility": iv_black}),
        ("py_vollib.black_scholes.implied_volatility", {"implied_volatility": iv_bs}),
        ("py_vollib.black_scholes_merton.implied_volatility", {"implied_volatility": iv_bsm}),
        ("py_vollib.black.greeks.analytical", {g: greek_fn(g, "black", False) for g in GREEKS}),
        ("py_vollib.black_scholes.greeks.analytical", {g: greek_fn(g, "black_scholes", False) for g in GREEKS}),
        ("py_vollib.black_scholes_merton.greeks.analytical",
         {g: greek_fn(g, "black_scholes_merton", True) for g in GREEKS}),
    ]
    for modname, mapping in targets:
        try:
            mod = importlib.import_module(modname)
        except ImportError:
            continue
        _setattrs(saved, mod, mapping)
    return _undo(saved)


def patch_py_vollib_vectorized():
    from . import (fast_black, fast_black_scholes, fast_black_scholes_merton, fast_implied_volatility,
                   fast_implied_volatility_black, get_all_greeks, vectorized_delta, vectorized_gamma,
                   vectorized_rho, vectorized_theta, vectorized_vega)
    mod = _import("py_vollib_vectorized")
    saved = []
    _setattrs(saved, mod, {
        "vectorized_black": fast_black,
        "vectorized_black_scholes": fast_black_scholes,
        "vectorized_black_scholes_merton": fast_black_scholes_merton,
        "vectorized_implied_volatility": fast_implied_volatility,
        "vectorized_implied_volatility_black": fast_implied_volatility_black,
        "get_all_greeks": get_all_greeks,
        "vectorized_delta": vectorized_delta, "vectorized_gamma": vectorized_gamma,
        "vectorized_theta": vectorized_theta, "vectorized_rho": vectorized_rho,
        "vectorized_vega": vectorized_vega,
    })
    return _undo(saved)
