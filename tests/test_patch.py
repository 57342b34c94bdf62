"""patch_fastvol swaps the batch entry points of an importable fastvol-like
package and restores them; the reference's callers keep their behaviour:
errors arrive as the TARGET package's classes (cli.py:247, :281 catch
fastvol's own BatchError / DomainError), results are the target's
ChainTable, and modules that bound an entry point by name at import
(fastvol/bench.py:15) are rebound too."""
import os
import subprocess
import sys
import textwrap
import types

import numpy as np
import pytest

from conftest import REPO
from paper_2604_27210_b200 import batch as gpu
from paper_2604_27210_b200.patch import patch_fastvol

REF_SRC = "/root/reference/pkg/src"


def _fake_package(name):
    """A stand-in with its own BatchError / ChainTable / DomainError classes,
    a bench module binding batch_iv by name, and a cli.main mirroring
    cli.py:270-283's except clause."""
    pkg = types.ModuleType(name)
    b = types.ModuleType(name + ".batch")
    e = types.ModuleType(name + ".errors")
    bench = types.ModuleType(name + ".bench")
    cli = types.ModuleType(name + ".cli")

    class BatchError(Exception):
        def __init__(self, kind, index, detail):
            self.kind, self.index, self.detail = kind, index, detail
            super().__init__(f"{kind} at row {index}: {detail}")

    class ChainTable:
        def __init__(self, columns):
            self.columns = columns

        def __getitem__(self, k):
            return self.columns[k]

    class DomainError(ValueError):
        pass

    b.BatchError, b.ChainTable = BatchError, ChainTable
    e.DomainError = DomainError
    for mod in (pkg, b):
        for n in ("batch_price", "batch_iv", "batch_greeks"):
            setattr(mod, n, lambda *a, **k: "cpu")
    bench.batch_iv = b.batch_iv
    bench.batch_price = b.batch_price

    def main(argv):
        try:
            b.batch_iv("black", "lbr", argv, [100.0], [100.0], [1.0], [0.0], price=[8.0])
            return 0
        except (BatchError, DomainError) as exc:
            cli.last_message = str(exc)
            return 1
    cli.main = main
    mods = {name: pkg, name + ".batch": b, name + ".errors": e, name + ".bench": bench, name + ".cli": cli}
    return mods


@pytest.fixture
def fake():
    mods = _fake_package("fakefastvol")
    sys.modules.update(mods)
    try:
        yield mods
    finally:
        for k in mods:
            sys.modules.pop(k, None)


def test_patch_and_undo(fake):
    pkg, b, bench = fake["fakefastvol"], fake["fakefastvol.batch"], fake["fakefastvol.bench"]
    undo = patch_fastvol("fakefastvol")
    assert b.batch_iv.__fastvol_b200__ is gpu.batch_iv
    assert pkg.batch_price.__fastvol_b200__ is gpu.batch_price
    assert bench.batch_iv.__fastvol_b200__ is gpu.batch_iv          # bound by name at import
    assert bench.batch_price.__fastvol_b200__ is gpu.batch_price
    undo()
    assert b.batch_iv() == "cpu" and bench.batch_iv() == "cpu" and pkg.batch_price() == "cpu"


def test_patched_errors_are_the_target_packages_classes(fake):
    """A bad flag is rejected by the host front end before any device work:
    the stand-in CLI's except clause must see ITS BatchError (exit 1)."""
    cli, b = fake["fakefastvol.cli"], fake["fakefastvol.batch"]
    undo = patch_fastvol("fakefastvol")
    try:
        assert cli.main(["x"]) == 1
        assert cli.last_message == "BadFlag at row 0: 'x'" or cli.last_message.startswith("BadFlag at row 0")
        with pytest.raises(b.BatchError) as ei:
            b.batch_iv("black", "lbr", ["c", "q"], [100.0], [100.0], [1.0], [0.0], price=[8.0])
        assert (ei.value.kind, ei.value.index) == ("BadFlag", 1)
        assert not isinstance(ei.value, gpu.BatchError)
    finally:
        undo()


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present (GPU box)")
def test_patch_real_reference_cli_exit_code(tmp_path):
    """The real reference (imported from /root/reference in a subprocess):
    after patch_fastvol, ``vol chain`` on a bad flag prints the reference's
    'error: ...' line and returns 1 instead of a traceback, and
    fastvol.bench's by-name bindings point at the B200 path."""
    csv = tmp_path / "chain.csv"
    csv.write_text("flag,F,K,t,r,price\nc,100,100,1,0,8\nz,100,100,1,0,8\n")
    code = textwrap.dedent(f"""
        import sys
        sys.dont_write_bytecode = True
        sys.path.insert(0, {REF_SRC!r}); sys.path.insert(0, {REPO!r})
        import fastvol, fastvol.bench, fastvol.cli
        from paper_2604_27210_b200 import batch as gpu
        from paper_2604_27210_b200.patch import patch_fastvol
        ref_err = fastvol.batch.BatchError
        undo = patch_fastvol()
        assert fastvol.bench.batch_iv.__fastvol_b200__ is gpu.batch_iv
        assert fastvol.batch.batch_iv.__fastvol_b200__ is gpu.batch_iv
        assert fastvol.batch_iv.__fastvol_b200__ is gpu.batch_iv
        rc = fastvol.cli.main(["chain", "--input", {str(csv)!r}, "--model", "black", "--compute", "iv",
                               "--method", "lbr"])
        print("RC", rc)
        try:
            fastvol.batch.batch_iv("black", "lbr", ["c", "bad"], [100.0], [100.0], [1.0], [0.0], price=[8.0])
        except ref_err as exc:
            print("CAUGHT", type(exc).__module__, exc)
        undo()
        assert fastvol.bench.batch_iv.__module__ == "fastvol.batch"
    """)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "RC 1" in res.stdout, res.stdout + res.stderr
    assert "error: BadFlag at row 1" in res.stderr
    assert "CAUGHT fastvol.batch BadFlag at row 1" in res.stdout


def test_inputs_not_mutated_by_host_front_end():
    """inputs are read-only -- the host front end (flag parsing,
    broadcasting, column assembly) leaves the caller's arrays bit-identical
    even when the call is rejected."""
    rng = np.random.default_rng(3)
    n = 1000
    cols = [rng.uniform(50, 150, n), rng.uniform(50, 150, n), rng.uniform(0.1, 2, n),
            rng.uniform(-0.01, 0.05, n), rng.uniform(1, 20, n)]
    flags = np.where(rng.random(n) < 0.5, "c", "p")
    flags[-1] = "x"                                   # rejected by parse_flags (BadFlag)
    before = [c.tobytes() for c in cols] + [flags.tobytes()]
    with pytest.raises(gpu.BatchError):
        gpu.batch_iv("black", "lbr", flags, cols[0], cols[1], cols[2], cols[3], price=cols[4])
    after = [c.tobytes() for c in cols] + [flags.tobytes()]
    assert before == after
