"""Route an installed reference ``fastvol`` package's batch entry points to
the B200 path (the analogue of the paper's ``patch_py_vollib``).

    from paper_2604_27210_b200.patch import patch_fastvol
    undo = patch_fastvol()        # fastvol.batch.batch_* now run on the GPU
    ...
    undo()
"""

import importlib

from . import batch as _gpu

ENTRY_POINTS = ("batch_price", "batch_iv", "batch_greeks")


def patch_fastvol(module_name="fastvol"):
    pkg = importlib.import_module(module_name)
    bmod = importlib.import_module(module_name + ".batch")
    saved = []
    for name in ENTRY_POINTS:
        for target in (pkg, bmod):
            if hasattr(target, name):
                saved.append((target, name, getattr(target, name)))
                setattr(target, name, getattr(_gpu, name))

    def undo():
        for target, name, fn in saved:
            setattr(target, name, fn)

    return undo
