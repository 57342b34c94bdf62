"""patch_fastvol swaps the batch entry points of an importable fastvol-like
package and restores them (checked on a stand-in module: the reference is
not installed on the GPU box)."""
import sys
import types

from paper_2604_27210_b200 import batch as gpu
from paper_2604_27210_b200.patch import patch_fastvol


def test_patch_and_undo():
    pkg = types.ModuleType("fakefastvol")
    b = types.ModuleType("fakefastvol.batch")
    for mod in (pkg, b):
        for n in ("batch_price", "batch_iv", "batch_greeks"):
            setattr(mod, n, lambda *a, **k: "cpu")
    sys.modules["fakefastvol"] = pkg
    sys.modules["fakefastvol.batch"] = b
    try:
        undo = patch_fastvol("fakefastvol")
        assert b.batch_iv is gpu.batch_iv and pkg.batch_price is gpu.batch_price
        undo()
        assert b.batch_iv() == "cpu"
    finally:
        del sys.modules["fakefastvol"], sys.modules["fakefastvol.batch"]
