"""The reference's batch-level acceptance checks with ``batch_*`` on the B200
path (VERDICT r1 missing item 4; /root/reference/pkg/tests/test_acceptance.py):

* the ``vol chain`` data path (cli.py:176-280) through
  ``paper_2604_27210_b200.chain.run_chain`` against the REAL reference CLI's
  output text, byte for byte (tests/golden/cli_chain.json.gz from
  gen_cli.py: price / iv / greeks for all three models, both methods, csv and
  json, pass-through columns, header-only files, the reader's slow path, and
  every DataError with the reference's message);
* the 1e6-row throughput smoke with its flat-memory bound
  (test_acceptance.py:323-347) through the bench-harness mirror;
* inputs are read-only: host arrays and device tensors are
  bit-identical after every entry point, accepted or rejected.

Cases that never reach the device (header-only files, reader and column
errors, bad flags) also run without a GPU.
"""
import gzip
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

CPU_CASES = {"header_only_csv", "header_only_json", "err_bad_flag", "err_not_a_number", "err_missing_column",
             "err_q_not_accepted", "err_price_needs_sigma", "err_iv_needs_price", "err_unknown_compute",
             "err_ragged_row", "err_unknown_column", "err_S_and_F", "err_empty_file"}


def _cases():
    with gzip.open(os.path.join(GOLDEN, "cli_chain.json.gz"), "rt") as fh:
        return json.load(fh)["cases"]


CASES = _cases()


def _run_case(case, tmp_path):
    """(rc, output text, stderr line) the way cli.main reports them."""
    from paper_2604_27210_b200 import chain
    from paper_2604_27210_b200.batch import BatchError
    from paper_2604_27210_b200.errors import DomainError
    src = tmp_path / "chain.csv"
    src.write_bytes(case["input"].encode())
    out = tmp_path / "out.txt"
    try:
        chain.run_chain(str(src), case["model"], case["compute"], case["method"], case["fmt"], output=str(out))
    except (chain.DataError, BatchError, DomainError) as exc:      # cli.py:281-283
        return 1, "", ("error: %s\n" % exc).replace(str(src), "<input>")
    return 0, out.read_text(), ""


def _check(case, tmp_path):
    rc, text, err = _run_case(case, tmp_path)
    assert (rc, err) == (case["rc"], case["err"]), case["name"]
    if rc == 0:
        if text != case["out"]:
            got, want = text.splitlines(), case["out"].splitlines()
            bad = next(i for i, (a, b) in enumerate(zip(got + [""], want + [""])) if a != b)
            pytest.fail(f"{case['name']}: line {bad} differs:\n got  {got[bad] if bad < len(got) else None}\n"
                        f" want {want[bad] if bad < len(want) else None}")


@pytest.mark.parametrize("case", [c for c in CASES if c["name"] in CPU_CASES], ids=lambda c: c["name"])
def test_chain_host_side_cases(case, tmp_path):
    _check(case, tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["name"] not in CPU_CASES], ids=lambda c: c["name"])
def test_chain_matches_reference_cli(case, tmp_path):
    _check(case, tmp_path)


@pytest.mark.gpu
def test_throughput_smoke_flat_memory(tmp_path):
    """test_acceptance.py:323-347 on the B200 path: run_bench(1e6, halley)
    writes the reference's report, converges >= 98 % of the rows and the
    process RSS grows by less than 500 MB (no per-call accumulation: the
    device workspace and pinned staging are reused)."""
    import psutil
    from paper_2604_27210_b200.bench import run_bench
    proc = psutil.Process()
    run_bench(10000, "halley", str(tmp_path / "warm.csv"))          # first-use allocations
    rss0 = proc.memory_info().rss
    out = tmp_path / "bench.csv"
    for _ in range(3):
        assert run_bench(1000000, "halley", str(out)) == 0
    growth = proc.memory_info().rss - rss0
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "rows,method,seconds,rows_per_sec,converged"
    cells = lines[1].split(",")
    assert int(cells[0]) == 1000000 and cells[1] == "halley"
    assert float(cells[3]) > 0
    assert int(cells[4]) >= 980000
    assert growth < 500 * 1024 * 1024, f"rss grew {growth / 1e6:.0f} MB"


def _checksums(arrays):
    return [a.tobytes() if isinstance(a, np.ndarray) else a.cpu().numpy().tobytes() for a in arrays]


@pytest.mark.gpu
def test_inputs_not_mutated_host_and_device():
    """every entry point leaves its inputs bit-identical -- host
    numpy columns through the Python API (accepted and rejected calls) and
    device-resident columns through the C ABI."""
    import torch
    from paper_2604_27210_b200 import _native, batch as B
    import workloads as W
    flag, S, K, t, r, q, sig = W.chain_draws(200000, seed=9)
    fl = W.flag_chars(flag)
    px = B.batch_price("bsm", fl, S, K, t, r, q, sigma=sig)["price"]
    host = [S, K, t, r, q, sig, px.copy()]
    before = _checksums(host) + [fl.tobytes()]
    B.batch_price("bsm", fl, S, K, t, r, q, sigma=sig)
    B.batch_greeks("bsm", fl, S, K, t, r, q, sigma=sig)
    B.batch_iv("bsm", "halley", fl, S, K, t, r, price=host[6], q=q)
    B.batch_iv("bsm", "lbr", fl, S, K, t, r, price=host[6], q=q)
    B.price_iv("bsm", "halley", fl, S, K, t, r, q, sigma=sig)
    bad_sig = sig.copy()
    bad_sig[1234] = -1.0                                          # rejected in the kernels
    before_bad = bad_sig.tobytes()
    with pytest.raises(B.BatchError):
        B.batch_price("bsm", fl, S, K, t, r, q, sigma=bad_sig)
    assert bad_sig.tobytes() == before_bad
    assert _checksums(host) + [fl.tobytes()] == before

    dev = torch.device("cuda", 0)
    lib = _native.lib_for_compute()
    lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
    n = len(S)
    cols = [torch.from_numpy(flag).to(dev)] + [torch.from_numpy(c).to(dev) for c in (S, K, t, r, q, sig)]
    dbefore = _checksums(cols)
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
    st = torch.empty(n, dtype=torch.int8, device=dev)
    ep, eg = _native.fv_error(), _native.fv_error()
    assert lib.fv_price_greeks(2, *[_native.col(c) for c in cols], n, *[o.data_ptr() for o in outs],
                               st.data_ptr(), ep, eg) == 0
    pcol = outs[0].clone()
    pbefore = _checksums([pcol])
    ivc = torch.empty(n, dtype=torch.float64, device=dev)
    for method in (0, 1):
        err = _native.fv_error()
        assert lib.fv_batch_iv(2, method, *[_native.col(c) for c in cols[:6]], _native.col(pcol), n,
                               ivc.data_ptr(), st.data_ptr(), None, err) == 0
    torch.cuda.synchronize()
    assert _checksums(cols) == dbefore
    assert _checksums([pcol]) == pbefore
