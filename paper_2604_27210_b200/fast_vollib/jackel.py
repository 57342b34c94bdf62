"""``fast_vollib.jackel``: "Let's Be Rational"-style implied volatility for
Black-76 quotes (Table 1 rows at :167-170) on the B200 LBR
pipeline -- the reference is fastvol's ``implied_vol_lbr`` through
``batch_iv(BLACK76, "lbr", ...)`` (lbr.py:410-486, batch.py:206-247), which
this path reproduces bit for bit.

The paper ships four engines for this function (NumPy+Numba, torch.compile,
JAX, a single-pass Triton kernel).  This build has one: hand-written sm_100a
kernels (normalize + first anchor, lazy remaining anchors, region-uniform
straight-line Householder(3) solves).  ``jackel_iv_black_torch`` and
``jackel_iv_triton`` are the same engine taking / returning CUDA tensors
device-resident; ``jackel_iv_black_jax`` raises (no JAX engine).

Like the paper's Jäckel functions these take no ``return_as`` / ``backend``
keywords: they return the implied vols as an array (NaN where the quote has
no solution: below intrinsic, above the upper bound, max iterations), and
``return_status=True`` adds the reference's per-row status strings (or int8
codes for CUDA-tensor inputs).
"""

import numpy as np

from .. import _native
from ..batch import batch_iv
from ..models import Model
from ._device import device_call_iv, is_cuda_tensor


def jackel_iv_black(price, F, K, t, r, flag, *, return_status=False):
    """LBR implied volatility of Black-76 quotes (price, forward F, strike K,
    maturity t, rate r, flag 'c'/'p')."""
    if is_cuda_tensor(price, F, K, t, r):
        return jackel_iv_black_torch(price, F, K, t, r, flag, return_status=return_status)
    tb = batch_iv(Model.BLACK76, "lbr", flag, F, K, t, r, price=price)
    return (tb["iv"], tb["status"]) if return_status else tb["iv"]


def jackel_iv_black_torch(price, F, K, t, r, flag, *, return_status=False):
    """Device-resident form: CUDA tensors (or scalars) in, CUDA tensors out;
    no host round trip."""
    lib = _native.lib_for_compute()
    iv, st = device_call_iv(lib, Model.BLACK76, "lbr", flag, F, K, t, r, 0.0, price)
    return (iv, st) if return_status else iv


jackel_iv_triton = jackel_iv_black_torch


def jackel_iv_black_jax(*args, **kwargs):
    from . import BackendUnavailable
    raise BackendUnavailable("no JAX engine in this build; use jackel_iv_black (B200) instead")


__all__ = ["jackel_iv_black", "jackel_iv_black_torch", "jackel_iv_triton", "jackel_iv_black_jax"]
