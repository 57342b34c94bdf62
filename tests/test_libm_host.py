"""CPU check of the device libm restatement (paper_2604_27210_b200/csrc/
fv_libm.h, compiled for the host): bit-identical to the live glibc 2.39 libm
(exp, log, erfc, pow) and scipy.special.erfcx, and the Markstein constant
division identical to IEEE division.  The same header is what the kernels run;
tests/test_gpu_parity.py repeats the comparison on the B200."""
import ctypes
import sys

import numpy as np
import pytest

sys.path.insert(0, __file__.rsplit("/", 1)[0] + "/native")
import build as native_build  # noqa: E402

N = 300_000


@pytest.fixture(scope="module")
def L():
    return ctypes.CDLL(native_build.build("libm_hostcheck"))


def _call(L, fn, x, y=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    P = ctypes.c_void_p
    if y is None:
        getattr(L, fn)(P(x.ctypes.data), ctypes.c_int64(len(x)), P(out.ctypes.data))
    else:
        y = np.ascontiguousarray(y, dtype=np.float64)
        getattr(L, fn)(P(x.ctypes.data), P(y.ctypes.data), ctypes.c_int64(len(x)),
                       P(out.ctypes.data))
    return out


def _mism(a, b):
    same = (a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))
    return int((~same).sum())


RNG = np.random.default_rng(0)
RANGES = {
    "exp": [RNG.uniform(-750, 750, N), RNG.uniform(-1, 1, N), RNG.uniform(-745.2, -708, N),
            RNG.uniform(700, 709.8, N), RNG.normal(0, 1e-9, N)],
    "log": [RNG.integers(0, 2 ** 63, N, dtype=np.int64).view(np.float64), RNG.uniform(0.9, 1.1, N),
            10 ** RNG.uniform(-320, -300, N), RNG.uniform(0, 10, N)],
    "erfc": [RNG.uniform(-30, 30, N), RNG.uniform(-1.3, 1.3, N), RNG.uniform(-7, 7, N),
             RNG.uniform(25, 30, N)],
}


@pytest.mark.parametrize("fn", ["exp", "log", "erfc"])
def test_glibc_bit_exact(L, fn):
    for x in RANGES[fn]:
        assert _mism(_call(L, "fvh_" + fn, x), _call(L, "glibc_" + fn, x)) == 0


def test_erfcx_bit_exact_vs_scipy(L):
    from scipy.special import erfcx
    for x in [RNG.uniform(-30, 60, N), RNG.uniform(-7, 1, N), 10 ** RNG.uniform(-10, 9, N)]:
        assert _mism(_call(L, "fvh_erfcx", x), erfcx(x)) == 0


@pytest.mark.parametrize("n", [2.0, 3.0, 4.0])
def test_pow_bit_exact(L, n):
    for x in [RNG.uniform(0, 10, N), 10 ** RNG.uniform(-200, 200, N), 10 ** RNG.uniform(-320, -300, N)]:
        x = x[np.isfinite(x) & (x > 0)]
        y = np.full_like(x, n)
        assert _mism(_call(L, "fvh_pow", x, y), _call(L, "glibc_pow", x, y)) == 0


def test_constant_division_is_ieee(L):
    L.fvh_div_const_check.restype = ctypes.c_int64
    bits = RNG.integers(0, 2 ** 64, 2_000_000, dtype=np.uint64)
    exp_ = (1023 + (bits >> np.uint64(52)) % np.uint64(200)).astype(np.uint64) - np.uint64(100)
    x = ((bits & np.uint64(0x800FFFFFFFFFFFFF)) | (exp_ << np.uint64(52))).view(np.float64)
    x = np.concatenate([x, RNG.integers(0, 2 ** 64, 200_000, dtype=np.uint64).view(np.float64),
                        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e308])])
    assert L.fvh_div_const_check(ctypes.c_void_p(x.ctypes.data), ctypes.c_int64(len(x))) == 0
