"""Multi-process (world_size 2, gloo, CPU) test of the quote-sharding layer
(paper_2604_27210_b200/distributed.py): contiguous shards, one MIN
all-reduce that reproduces the single-process reference's first error
(check order first, then lowest raising row), and the optional all-gather.
The per-shard compute is a stand-in here (no GPU); on the box the same
``run_sharded`` wraps the CUDA C ABI (batch_iv_sharded)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_27210_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, scenario, q, gather=True):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def compute(lo, hi):
            out = {"iv": np.arange(lo, hi, dtype=np.float64) * 0.5,
                   "status": (np.arange(lo, hi) % 5).astype(np.int8)}
            checks = np.full(12, -1, np.int64)
            exc_row, exc_code = -1, 0
            for (g_row, kind, code) in scenario:
                if lo <= g_row < hi:
                    if kind == "check":
                        if checks[code] < 0 or g_row - lo < checks[code]:
                            checks[code] = g_row - lo
                    elif exc_row < 0 or g_row - lo < exc_row:
                        exc_row, exc_code = g_row - lo, code
            return out, checks, exc_row, exc_code
        outputs, outcome = D.run_sharded(compute, n, gather=gather)
        q.put((rank, outcome, None if outputs is None else {k: np.asarray(v) for k, v in outputs.items()}))
    finally:
        dist.destroy_process_group()


def _run(n, scenario, gather=True, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, scenario, q, gather)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=60) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda t: t[0])


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 100, 10_001):
        for w in (1, 2, 3, 8):
            spans = [D.shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_clean_run_gathers_full_result():
    n = 1001
    res = _run(n, [])
    for rank, outcome, out in res:
        assert outcome is None
        assert np.array_equal(out["iv"], np.arange(n) * 0.5)
        assert np.array_equal(out["status"], (np.arange(n) % 5).astype(np.int8))


def test_gather_to_one_rank_only():
    """gather=<rank>: the full result lands on that rank only (point-to-point
    sends; NCCL over NVLink on a GPU box), the others keep nothing -- the
    north star's "NVLink only to gather results when the caller asks for
    them on one device"."""
    n = 1001
    for dst in (0, 1):
        res = _run(n, [], gather=dst)
        for rank, outcome, out in res:
            assert outcome is None
            if rank == dst:
                assert np.array_equal(out["iv"], np.arange(n) * 0.5)
                assert np.array_equal(out["status"], (np.arange(n) % 5).astype(np.int8))
            else:
                assert out is None


def test_gather_to_one_rank_world3_uneven():
    n = 1000                                  # 334 / 333 / 333 rows
    for rank, outcome, out in _run(n, [], gather=2, world=3):
        if rank == 2:
            assert np.array_equal(out["iv"], np.arange(n) * 0.5)
        else:
            assert out is None


def test_first_error_is_global_reference_order():
    # rank 1 holds an earlier check (kind 2 < 5) at a later row; rank 0 holds
    # exceptions: the batch error wins (validation precedes the kernel), and
    # within a check the lowest global row wins.
    n = 1000
    scen = [(100, "exc", 1), (700, "check", 2), (900, "check", 2), (300, "check", 5)]
    for rank, outcome, _ in _run(n, scen):
        assert outcome == ("batch", 2, 700)
    scen = [(800, "exc", 3), (550, "exc", 1), (20, "exc", 2)]
    for rank, outcome, _ in _run(n, scen):
        assert outcome == ("exc", 2, 20)


def _worker_staged(rank, world, port, n, scenario, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def compute(lo, hi):
            stages = []
            for stage in (0, 1):
                checks = np.full(12, -1, np.int64)
                exc_row, exc_code = -1, 0
                for (g_row, st, kind, code) in scenario:
                    if st != stage or not (lo <= g_row < hi):
                        continue
                    if kind == "check":
                        if checks[code] < 0 or g_row - lo < checks[code]:
                            checks[code] = g_row - lo
                    elif exc_row < 0 or g_row - lo < exc_row:
                        exc_row, exc_code = g_row - lo, code
                stages.append((checks, exc_row, exc_code))
            return {"price": np.arange(lo, hi, dtype=np.float64)}, stages
        outputs, outcome = D.run_sharded_stages(compute, n, 2)
        q.put((rank, outcome, {}))
    finally:
        dist.destroy_process_group()


def _run_staged(n, scenario):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_staged, args=(r, 2, port, n, scenario, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=60) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_price_iv_stages_price_failure_wins():
    """fv_price_iv sharded (distributed.price_iv_sharded): a price-stage
    exception on rank 1 beats an IV-stage check on rank 0 at an earlier row
    (the reference raises in batch_price before batch_iv runs); with no price
    failure anywhere, the IV stage's first error in the reference's order."""
    n = 1000
    scen = [(10, 1, "check", 6), (900, 0, "exc", 1), (950, 0, "exc", 2)]
    for rank, outcome, _ in _run_staged(n, scen):
        assert outcome == (0, ("exc", 1, 900))
    scen = [(10, 1, "exc", 2), (600, 1, "check", 6)]
    for rank, outcome, _ in _run_staged(n, scen):
        assert outcome == (1, ("batch", 6, 600))
    for rank, outcome, _ in _run_staged(n, []):
        assert outcome is None
