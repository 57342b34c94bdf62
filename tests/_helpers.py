"""Shared parity helpers: bit-level comparison with a readable failure."""
import numpy as np


def bits_equal(a, b):
    """True where a and b are the same IEEE double (any NaN matches any NaN)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    same = a.view(np.int64) == b.view(np.int64)
    return same | (np.isnan(a) & np.isnan(b))


def assert_bits(got, want, what, ctx=None):
    ok = bits_equal(got, want)
    if not ok.all():
        idx = np.flatnonzero(~ok)
        i = int(idx[0])
        extra = ""
        if ctx is not None:
            extra = " inputs: " + ", ".join(f"{k}={np.asarray(v)[i]!r}" for k, v in ctx.items())
        raise AssertionError(
            f"{what}: {idx.size}/{ok.size} rows differ; first row {i}: "
            f"got {np.asarray(got)[i]!r} want {np.asarray(want)[i]!r}{extra}")


def load(path):
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}
