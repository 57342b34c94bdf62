"""Synthetic quote workloads C1-C5.

Inputs only -- prices are produced by whichever pricer the caller trusts
(the reference / oracle on CPU, the product kernel on the GPU; they are
bit-identical).  Draw orders restate the reference generator
``fastvol.bench.synthetic_chain`` (/root/reference/pkg/src/fastvol/bench.py:19-31):
flag, K, t, r, q, sigma from ``numpy.random.default_rng(seed)``.

Flags are returned as int8 +1 (call) / -1 (put); ``flag_chars`` gives the
'c'/'p' strings the reference API takes.
"""

import numpy as np

C4_FLAGS = 2
C4_MATURITIES = 1000
C4_STRIKES = 50_000
C4_ROWS = C4_FLAGS * C4_MATURITIES * C4_STRIKES      # 100,000,000


def flag_chars(flag):
    return np.where(np.asarray(flag) > 0, "c", "p")


def chain_draws(rows, seed=0):
    """bench.py:21-28: (flag, S, K, t, r, q, sigma) with S = 100."""
    rng = np.random.default_rng(seed)
    flag = np.where(rng.random(rows) < 0.5, 1, -1).astype(np.int8)
    S = np.full(rows, 100.0)
    K = S * np.exp(rng.uniform(-0.6, 0.6, rows))
    t = rng.uniform(0.1, 2.0, rows)
    r = rng.uniform(-0.01, 0.05, rows)
    q = rng.uniform(0.0, 0.03, rows)
    sigma = rng.uniform(0.1, 0.8, rows)
    return flag, S, K, t, r, q, sigma


def c4_params(start, stop):
    """Rows [start, stop) of the C4 chain: 2 flags x 1,000 maturities x
    50,000 strikes, row = (f*1000 + j)*50000 + i.  Returns
    (flag, F, K, t, r, sigma) as numpy arrays (F = 100, r = 0.03)."""
    return c4_rows(np.arange(start, stop, dtype=np.int64))


def c4_rows(row):
    """The C4 chain's rows at the given (int64) row indices."""
    row = np.asarray(row, dtype=np.int64)
    i = row % C4_STRIKES
    j = (row // C4_STRIKES) % C4_MATURITIES
    f = row // (C4_STRIKES * C4_MATURITIES)
    x = -2.0 + 4.0 * i / (C4_STRIKES - 1)
    K = 100.0 * np.exp(-x)
    t = (1.0 / 365.0) * (5.0 * 365.0) ** (j / (C4_MATURITIES - 1))
    sigma = np.minimum(0.2 + 0.1 * x * x / np.sqrt(t), 2.0)
    flag = np.where(f == 0, 1, -1).astype(np.int8)
    n = row.shape[0]
    return flag, np.full(n, 100.0), K, t, np.full(n, 0.03), sigma


def c5_params(rows, seed=5):
    """Wing-stress set (C5).  kind = row % 4:
    0 deep wings x ~ U(-10, 10); 1 tiny maturity t ~ 10^U(-8, -3);
    2 out-of-bounds price (below intrinsic or above cap);
    3 exact boundary price (discounted intrinsic or cap).
    Base draws: x ~ U(-3, 3), t ~ U(0.01, 3), sigma ~ 10^U(-3, log10 5),
    r ~ U(-0.02, 0.08), F = 100.  Rows with |r t| > 50 or |x| > 10 are
    dropped (they only exercise Python exceptions; see exception sets).

    Returns (flag, F, K, t, r, sigma, kind, side) where ``side`` picks the
    below(0)/above(1) variant for kinds 2 and 3.  Prices are set by
    ``c5_prices``.
    """
    rng = np.random.default_rng(seed)
    kind = np.arange(rows) % 4
    flag = np.where(rng.random(rows) < 0.5, 1, -1).astype(np.int8)
    x = rng.uniform(-3.0, 3.0, rows)
    t = rng.uniform(0.01, 3.0, rows)
    sigma = 10.0 ** rng.uniform(-3.0, np.log10(5.0), rows)
    r = rng.uniform(-0.02, 0.08, rows)
    xw = rng.uniform(-10.0, 10.0, rows)
    tw = 10.0 ** rng.uniform(-8.0, -3.0, rows)
    side = (rng.random(rows) < 0.5).astype(np.int8)
    x = np.where(kind == 0, xw, x)
    t = np.where(kind == 1, tw, t)
    keep = (np.abs(r * t) <= 50.0) & (np.abs(x) <= 10.0)
    F = np.full(rows, 100.0)
    K = F * np.exp(-x)
    return (flag[keep], F[keep], K[keep], t[keep], r[keep], sigma[keep],
            kind[keep], side[keep])


def c5_prices(flag, F, K, t, r, kind, side, model_price):
    """Final C5 price column: ``model_price`` (Black-76 prices of the sigma
    column) for kinds 0/1, bound-violating or exact-bound prices for 2/3."""
    disc = np.exp(-r * t)
    intrinsic = disc * np.maximum(flag * (F - K), 0.0)
    cap = disc * np.where(flag > 0, F, K)
    below = np.maximum(intrinsic * (1.0 - 1e-3) - 1e-3, 0.0)
    above = cap * (1.0 + 1e-3) + 1e-3
    px = np.array(model_price, dtype=np.float64, copy=True)
    px = np.where(kind == 2, np.where(side == 0, below, above), px)
    px = np.where(kind == 3, np.where(side == 0, intrinsic, cap), px)
    return px
