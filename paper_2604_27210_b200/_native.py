"""ctypes binding of libfastvol_b200.so (the C ABI in include/fastvol_b200.h).

There is no CPU fallback: if the CUDA library is missing or no GPU is visible,
every compute entry point raises (the reference's CPU path lives in the
reference; this package is the GPU drop-in for it).
"""

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FV_LIB") or os.path.join(HERE, "libfastvol_b200.so")

FV_OK, FV_ERR_BATCH, FV_ERR_PYEXC, FV_ERR_CUDA, FV_ERR_ARG = 0, 1, 2, 3, 4


class fv_col(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("stride", ctypes.c_int64)]


class fv_error(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("kind", ctypes.c_int32), ("index", ctypes.c_int64),
                ("column", ctypes.c_int32), ("value_is_numpy", ctypes.c_int32),
                ("value", ctypes.c_double), ("message", ctypes.c_char * 256)]


class fv_shard(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("cols", fv_col * 7),
                ("n", ctypes.c_int64), ("outs", ctypes.c_void_p * 6), ("status", ctypes.c_void_p),
                ("region", ctypes.c_void_p)]


FV_KIND_PRICE, FV_KIND_IV, FV_KIND_GREEKS, FV_KIND_PRICE_GREEKS, FV_KIND_PRICE_IV = range(5)


class NativeUnavailable(RuntimeError):
    """The CUDA extension is not built or cannot run here."""


_lock = threading.Lock()
_lib = None

_COL = fv_col
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_ERR = ctypes.POINTER(fv_error)

SIGNATURES = {
    "fv_batch_price": ([ctypes.c_int] + [_COL] * 7 + [_I64, _P, _ERR], ctypes.c_int),
    "fv_batch_iv": ([ctypes.c_int, ctypes.c_int] + [_COL] * 7 + [_I64, _P, _P, _P, _ERR],
                    ctypes.c_int),
    "fv_batch_greeks": ([ctypes.c_int] + [_COL] * 7 + [_I64] + [_P] * 6 + [_ERR], ctypes.c_int),
    "fv_price_greeks": ([ctypes.c_int] + [_COL] * 7 + [_I64] + [_P] * 7 + [_ERR, _ERR],
                        ctypes.c_int),
    "fv_price_iv": ([ctypes.c_int, ctypes.c_int] + [_COL] * 7 + [_I64, _P, _P, _P, _P, _ERR, _ERR],
                    ctypes.c_int),
    "fv_set_stream": ([_P], ctypes.c_int),
    "fv_run_shards": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _ERR, _ERR], ctypes.c_int),
    "fv_gather": ([_P, ctypes.c_int, _P, ctypes.c_int, _P, _P, _P], ctypes.c_int),
    "fv_device_count": ([], ctypes.c_int),
    "fv_set_devices": ([_P, ctypes.c_int], ctypes.c_int),
    "fv_get_devices": ([_P, ctypes.c_int], ctypes.c_int),
    "fv_version": ([], ctypes.c_char_p),
    "fv_set_chunk_rows": ([_I64], ctypes.c_int),
    "fv_last_launch_count": ([], _I64),
    "fv_last_h2d_bytes": ([], _I64),
    "fv_host_find_runs": ([_P, ctypes.c_int, _I64, _I64, _P, _P, _P], ctypes.c_int),
    "fv_set_round_rows": ([_I64, _I64], ctypes.c_int),
    "fv_probe_fp64_peak": ([_P, _P], ctypes.c_int),
    "fv_last_outcome": ([_P, _P, _P], ctypes.c_int),
    "fv_selftest_div_const": ([_I64, ctypes.c_uint64, _P], ctypes.c_int),
    "fv_selftest_fast": ([_I64, ctypes.c_uint64, _P, _P], ctypes.c_int),
    "fv_selftest_qlo": ([_P, _P, _P], ctypes.c_int),
    "fv_set_kernel_timing": ([ctypes.c_int], ctypes.c_int),
    "fv_set_span_timing": ([ctypes.c_int], ctypes.c_int),
    "fv_last_span_ms": ([], ctypes.c_double),
    "fv_kernel_times": ([_P, _P], ctypes.c_int),
    "fv_kernel_name": ([ctypes.c_int], ctypes.c_char_p),
}


def load(path=LIB_PATH):
    """Load the shared library (no device needed); raises NativeUnavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `python -m paper_2604_27210_b200._build`")
        lib = ctypes.CDLL(path)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


ENV_DEVICES = "FASTVOL_DEVICES"     # e.g. "0,1,2,3": host-buffer calls shard over these GPUs
_env_applied = False


def lib_for_compute():
    """The library, after checking a CUDA device is present (fails loudly).
    The first call applies FASTVOL_DEVICES (see set_devices), the analogue of
    the reference's FASTVOL_THREADS worker count (batch.py:166-178)."""
    global _env_applied
    lib = load()
    if lib.fv_device_count() < 1:
        raise NativeUnavailable("no CUDA device visible: the fastvol B200 path has no CPU fallback")
    if not _env_applied:
        _env_applied = True
        spec = os.environ.get(ENV_DEVICES, "").strip()
        if spec:
            ids = [int(x) for x in spec.split(",") if x.strip()]
            arr = (ctypes.c_int * max(1, len(ids)))(*ids)
            if lib.fv_set_devices(arr, len(ids)):
                raise ValueError(f"{ENV_DEVICES}={spec!r}: not a list of visible device ids")
    return lib


def col(arr):
    """fv_col for a 1-D numpy array / torch tensor (stride in elements); a
    single-element column is a stride-0 broadcast (batch.py:95-96)."""
    if hasattr(arr, "data_ptr"):             # torch tensor
        stride = arr.stride(0) if (arr.dim() == 1 and arr.numel() > 1) else 0
        return fv_col(arr.data_ptr(), stride)
    a = np.asarray(arr)
    stride = a.strides[0] // a.dtype.itemsize if (a.ndim == 1 and a.size > 1) else 0
    return fv_col(a.ctypes.data, stride)


def ptr(arr):
    if arr is None:
        return None
    if hasattr(arr, "data_ptr"):
        return arr.data_ptr()
    return np.asarray(arr).ctypes.data


class NativeCallError(RuntimeError):
    """A C-ABI call failed for a runtime / argument reason (FV_ERR_CUDA,
    FV_ERR_ARG) -- not one of the reference's own errors."""


def check_runtime(rc, err):
    """Raise on FV_ERR_CUDA / FV_ERR_ARG (the outputs and fv_last_outcome of
    such a call are meaningless); the reference's errors pass through."""
    if rc in (FV_ERR_CUDA, FV_ERR_ARG):
        raise NativeCallError("fastvol_b200: " + err.message.decode(errors="replace"))
    return rc


class device_scope:
    """``with device_scope(lib, dev):`` -- a device-pointer call on ``dev``:
    that device current (torch does not switch it for tensors on another
    device) and the kernels ordered on its current torch stream."""

    def __init__(self, lib, dev):
        import torch
        self.lib = lib
        self.dev = torch.device(dev)
        self._guard = torch.cuda.device(self.dev)

    def __enter__(self):
        import torch
        self._guard.__enter__()
        self.lib.fv_set_stream(torch.cuda.current_stream(self.dev).cuda_stream)
        return self

    def __exit__(self, *exc):
        return self._guard.__exit__(*exc)


def last_outcome(lib):
    """(check_rows[12], exc_rows[2], exc_codes[2]) of this thread's last call."""
    cr = np.empty(12, np.int64)
    er = np.empty(2, np.int64)
    ec = np.empty(2, np.int32)
    lib.fv_last_outcome(cr.ctypes.data, er.ctypes.data, ec.ctypes.data)
    return cr, er, ec


NKERNEL = 14


def kernel_times(lib):
    """{kernel name: (ms, launches)} accumulated since the last call
    (fv_set_kernel_timing must have been on)."""
    ms = (ctypes.c_double * NKERNEL)()
    ln = (ctypes.c_int64 * NKERNEL)()
    if lib.fv_kernel_times(ms, ln) != 0:
        raise RuntimeError("fv_kernel_times failed")
    return {lib.fv_kernel_name(k).decode(): (ms[k], ln[k]) for k in range(NKERNEL) if ln[k]}


def set_devices(ids=()):
    """Devices for host-buffer batch calls (fv_set_devices): with two or more,
    a call of at least len(ids) * 2^20 rows is split into contiguous row
    shards, one host thread and one GPU each.  ``()`` restores the default."""
    lib = lib_for_compute()
    arr = (ctypes.c_int * max(1, len(ids)))(*ids)
    rc = lib.fv_set_devices(arr, len(ids))
    if rc:
        raise ValueError(f"invalid device list {list(ids)!r}")


def get_devices():
    lib = load()
    arr = (ctypes.c_int * 64)()
    k = lib.fv_get_devices(arr, 64)
    return list(arr[:min(k, 64)])
