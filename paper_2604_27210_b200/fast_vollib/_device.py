"""Device-resident calls of the C ABI for torch CUDA tensor inputs: columns
stay in HBM (stride-0 columns for scalars), outputs are allocated on the
device, and the kernels run on the caller's current stream.  Validation,
BatchError / Python-exception semantics are those of the host path
(batch.py), raised from the same fv_error record."""

import numpy as np

from .. import _native
from ..batch import GREEK_COLUMNS, BatchError, _ok_or_raise, parse_flags


def is_cuda_tensor(*xs):
    for x in xs:
        if x is not None and hasattr(x, "is_cuda") and x.is_cuda:
            return True
    return False


def _dev_cols(flag, und, K, t, r, q, last, last_name):
    import torch
    dev = next(x.device for x in (und, K, t, r, q, last) if hasattr(x, "is_cuda") and x.is_cuda)
    if hasattr(flag, "is_cuda"):
        fl = flag.to(device=dev, dtype=torch.int8).reshape(-1)
    else:
        fl = torch.from_numpy(np.ascontiguousarray(parse_flags(flag))).to(dev)

    def f64(x):
        if hasattr(x, "is_cuda"):
            return x.to(device=dev, dtype=torch.float64).reshape(-1)
        return torch.as_tensor(np.atleast_1d(np.asarray(x, dtype=np.float64)), device=dev).reshape(-1)

    cols = [fl] + [f64(x) for x in (und, K, t, r, q, last)]
    lengths = [c.numel() for c in cols]
    n = max(lengths, default=1)
    if 0 in lengths:
        n = 0
    for i, ln in enumerate(lengths):
        if ln not in (1, n):
            raise BatchError("ShapeMismatch", i, f"length {ln} incompatible with batch size {n}")
    cols = [c.contiguous() if c.numel() > 1 else c for c in cols]
    table = {"flag": cols[0], "underlying": cols[1], "strike": cols[2], "t": cols[3], "r": cols[4],
             "q": cols[5], last_name: cols[6]}
    return dev, n, cols, table


def device_call_price(lib, model, flag, und, K, t, r, q, sigma):
    import torch
    dev, n, cols, table = _dev_cols(flag, und, K, t, r, q, sigma, "sigma")
    out = torch.empty(n, dtype=torch.float64, device=dev)
    if n:
        err = _native.fv_error()
        with _native.device_scope(lib, dev):
            rc = lib.fv_batch_price(model.code, *[_native.col(c) for c in cols], n, out.data_ptr(), err)
        _ok_or_raise(rc, err, table, model, "sigma")
    return out


def device_call_iv(lib, model, method, flag, und, K, t, r, q, price):
    import torch
    dev, n, cols, table = _dev_cols(flag, und, K, t, r, q, price, "price")
    iv = torch.empty(n, dtype=torch.float64, device=dev)
    st = torch.empty(n, dtype=torch.int8, device=dev)
    if n:
        err = _native.fv_error()
        with _native.device_scope(lib, dev):
            rc = lib.fv_batch_iv(model.code, 1 if method == "lbr" else 0, *[_native.col(c) for c in cols], n,
                                 iv.data_ptr(), st.data_ptr(), None, err)
        _ok_or_raise(rc, err, table, model, "price")
    return iv, st


def device_call_greeks(lib, model, flag, und, K, t, r, q, sigma):
    import torch
    dev, n, cols, table = _dev_cols(flag, und, K, t, r, q, sigma, "sigma")
    outs = {g: torch.empty(n, dtype=torch.float64, device=dev) for g in GREEK_COLUMNS}
    st = torch.empty(n, dtype=torch.int8, device=dev)
    if n:
        err = _native.fv_error()
        with _native.device_scope(lib, dev):
            rc = lib.fv_batch_greeks(model.code, *[_native.col(c) for c in cols], n,
                                     *[outs[g].data_ptr() for g in GREEK_COLUMNS], st.data_ptr(), err)
        _ok_or_raise(rc, err, table, model, "sigma")
    outs["status"] = st
    return outs
