"""paper_2604_27210_b200: a B200 (sm_100a) drop-in for the batched pricing,
Greeks and implied-volatility path of fast-vollib / ``fastvol``.

Public names mirror ``fastvol`` (/root/reference/pkg/src/fastvol/__init__.py:9-41)
for the batch path: batch_price / batch_iv / batch_greeks return the same
ChainTable, statuses and errors, computed by hand-written CUDA kernels
(csrc/) behind the C ABI in include/fastvol_b200.h.  The paper's names
(fast_black_scholes_merton, fast_implied_volatility, jackel_iv_black,
get_all_greeks, jackel.jackel_iv_black, set_backend, patch_py_vollib, ...,
with return_as containers) live in ``paper_2604_27210_b200.fast_vollib``; the
chain CSV reader of the reference's CLI (cli.py:140-173) in ``chain_csv``.
"""

from . import bench, chain_csv
from .batch import (BatchError, ChainTable, batch_greeks, batch_iv, batch_price, broadcast,
                    format_output, parse_flags, price_iv, validate)
from .errors import AboveUpperBoundError, BelowIntrinsicError, DomainError, StepFunctionEdge
from .models import Model, PricingInputs, parse_flag
from .solver import SolverResult, SolverStatus
from ._native import get_devices, set_devices

__version__ = "0.1.0"

__all__ = [
    "BatchError", "ChainTable", "batch_greeks", "batch_iv", "batch_price", "broadcast",
    "format_output", "parse_flags", "price_iv", "validate",
    "AboveUpperBoundError", "BelowIntrinsicError", "DomainError", "StepFunctionEdge",
    "Model", "PricingInputs", "parse_flag", "SolverResult", "SolverStatus", "chain_csv", "bench",
    "set_devices", "get_devices",
]
