"""The bench's one-process-per-GPU path (torchrun, N = 2) on a 1-GPU box: the
two ranks share the visible GPU over gloo (FV_BENCH_SHARE_GPUS=1), so the
sharding, the barriers, the max-over-ranks timing, the per-rank parity check
and rank 0's single JSON line run exactly as on a multi-GPU node (with NCCL
there).  Its timings are not scaling numbers."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("workload,extra", [("c4", ["--rows", "4000000"]), ("c2", ["--rows", "2000000"])])
def test_bench_two_ranks_one_line(workload, extra):
    env = dict(os.environ, FV_BENCH_SHARE_GPUS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--workload", workload, "--steps", "3", "--warmup", "3", "--no-kernel-timing", *extra]
    res = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]            # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["parity"]["mismatches"] == 0
    assert d["parity"]["rows_checked"] == int(extra[1])
    assert "paper_2604_27210_b200/libfastvol_b200.so" in d["repo_libs_loaded"]
