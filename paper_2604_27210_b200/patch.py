"""Route an installed reference ``fastvol`` package's batch entry points to
the B200 path (the analogue of the paper's ``patch_py_vollib``).

    from paper_2604_27210_b200.patch import patch_fastvol
    undo = patch_fastvol()        # fastvol.batch.batch_* now run on the GPU
    ...
    undo()

The reference's callers keep working unchanged:
  * errors are raised as the TARGET package's classes -- ``vol``'s
    ``except (DataError, BatchError, DomainError, StepFunctionEdge)``
    (cli.py:247, :281) catches them and exits 1 -- with the same arguments
    and message (BatchError(kind, index, detail), batch.py:33-40);
  * results are the target's ``ChainTable`` (batch.py:43-62);
  * every already-imported ``fastvol.*`` module that bound an entry point by
    name (``fastvol.bench`` does ``from .batch import batch_iv, batch_price``,
    bench.py:15) is rebound too, and ``fastvol.bench`` / ``fastvol.cli`` are
    imported first so a later import cannot pick up the CPU originals.
"""

import functools
import importlib
import sys

from . import batch as _gpu
from . import errors as _gpu_errors

ENTRY_POINTS = ("batch_price", "batch_iv", "batch_greeks")
_SUBMODULES = ("batch", "bench", "cli")
_ERROR_NAMES = ("DomainError", "StepFunctionEdge", "BelowIntrinsicError", "AboveUpperBoundError")


def _translator(module_name):
    """Exception / result translation into the target package's types."""
    bmod = importlib.import_module(module_name + ".batch")
    try:
        emod = importlib.import_module(module_name + ".errors")
    except ImportError:
        emod = None
    t_batch_error = getattr(bmod, "BatchError", None)
    t_table = getattr(bmod, "ChainTable", None)
    err_map = {}
    for name in _ERROR_NAMES:
        ours = getattr(_gpu_errors, name)
        theirs = getattr(emod, name, None) if emod is not None else None
        if theirs is not None and theirs is not ours:
            err_map[ours] = theirs

    def wrap(fn):
        @functools.wraps(fn)
        def entry(*args, **kwargs):
            try:
                res = fn(*args, **kwargs)
            except _gpu.BatchError as exc:
                if t_batch_error is None or t_batch_error is _gpu.BatchError:
                    raise
                raise t_batch_error(exc.kind, exc.index, exc.detail) from None
            except tuple(err_map) as exc:
                raise err_map[type(exc)](*exc.args) from None
            if t_table is not None and t_table is not _gpu.ChainTable and isinstance(res, _gpu.ChainTable):
                res = t_table(dict(res.columns))
            return res
        entry.__fastvol_b200__ = fn
        return entry

    return wrap


def patch_fastvol(module_name="fastvol"):
    """Swap ``module_name``'s batch entry points for the B200 ones; returns an
    ``undo()`` that restores every rebinding."""
    pkg = importlib.import_module(module_name)
    bmod = importlib.import_module(module_name + ".batch")
    for sub in _SUBMODULES[1:]:            # import now: later imports would bind the originals
        try:
            importlib.import_module(module_name + "." + sub)
        except ImportError:
            pass
    wrap = _translator(module_name)
    originals = {name: getattr(bmod, name) for name in ENTRY_POINTS if hasattr(bmod, name)}
    replacement = {name: wrap(getattr(_gpu, name)) for name in originals}
    targets = [pkg] + [m for k, m in list(sys.modules.items())
                       if m is not None and k.startswith(module_name + ".")]
    saved = []
    for target in targets:
        for name, orig in originals.items():
            cur = getattr(target, name, None)
            # the package and its batch module by name; any other module that
            # bound the original object
            if cur is orig or (target in (pkg, bmod) and cur is not None):
                saved.append((target, name, cur))
                setattr(target, name, replacement[name])

    def undo():
        for target, name, fn in saved:
            setattr(target, name, fn)

    return undo
