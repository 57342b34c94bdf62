#!/usr/bin/env python3
"""Benchmark: fp64 LBR implied-vol solves/sec on the C4 100M-quote option chain.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c1|c2|c3|c5|rt] [--rows R]
                    [--scaling strong|weak] [--shard-scheme contiguous|cyclic]
                    [--shard g/G]

Metric (BASELINE.json): "fp64 IV solves/sec (LBR, 100M quotes) at 1/2/4/8 B200
vs host-CPU ref".  One step = one ``fv_batch_iv(BLACK76, LBR, ...)`` call per
rank over that rank's quotes of the C4 chain (2 flags x 1,000
maturities x 50,000 strikes = 100M quotes).

Multi-GPU (one process per GPU, torchrun):
  * ``--scaling strong`` (default): ONE 100M-quote chain sharded across the N
    ranks -- rank g solves its rows: 1M-row blocks dealt round-robin
    (``--shard-scheme cyclic``, default) or one contiguous range [g N/G,
    (g+1) N/G) (``contiguous``; the chain's (flag, maturity, strike) order
    gives contiguous shards different region mixes: 7.6 / 8.4 % imbalance at
    G = 4 / 8 against 1.1 / 2.3 % cyclic, profiles/r2/shard_times_c4.json),
    no collective on the data path; ``value`` = 100M / the max over ranks of
    the per-step time;
  * ``--scaling weak``: every rank solves its own full chain (F_r = 100 *
    1.01^r), ``value`` = N x rows / max time.
``--shard g/G`` runs shard g of a G-way strong split on this one GPU (the
per-shard times predict the strong-scaling imbalance on a 1-GPU pool).

``value`` is device-resident throughput (inputs already in HBM; CUDA events on
the launching stream, max over ranks).  ``e2e`` is the same call through the C
ABI with pinned HOST buffers (chunked H2D / kernel / D2H inside the timed
region, wall clock).  ``cpu_baseline`` is the oracle (oracle/fvoracle.cpp -- the
reference restated in C++ on glibc + scipy, all host threads) timed on ALL rows
of the workload; the same pass compares every row bit for bit with the GPU's
output (``parity``).  The inputs (2.5 GB per step) are larger than the 126 MB
L2, so no flush is needed between steps.

``--impl reference`` times the reference's CPU path on the same workload and
config (the oracle port, all host threads; /root/reference itself does not
exist on the GPU box) without importing the product package.
"""

import argparse
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import workloads as W  # noqa: E402  (numpy only; no product import)

# Weighted distinct FP64 ops per quote the reference executes (SURVEY.md 8(d),
# Appendix B.3): the algorithmic work per unit for the roofline.
# rt (the reference's bench harness: synthetic_chain's BSM pricing + run_bench's
# Halley inversion, one fused fv_price_iv call): price 200 + C2 Halley 1476.
W_OPS = {"c4": 1443.0, "c1": 1405.0, "c2": 1476.0, "c3": 298.0, "c5": 347.0, "rt": 1676.0}
METRIC = "fp64 IV solves/sec (LBR, 100M quotes) at 1/2/4/8 B200 vs host-CPU ref"
CYCLIC_BLOCK = 1 << 20
WL_NAMES = {"c4": "C4: jackel_iv_black (LBR) on the 100M-quote Black-76 chain "
                  "(2 flags x 1000 maturities x 50000 strikes)",
            "c1": "C1: LBR Black-76 1M synthetic quotes (synthetic_chain seed 0)",
            "c2": "C2: Halley BSM with dividend yield, 10M quotes (synthetic_chain seed 0)",
            "c3": "C3: fused BSM price + all Greeks, 10M quotes (synthetic_chain seed 0)",
            "c5": "C5: wing-stress set, LBR Black-76 (seed 5)",
            "rt": "RT: the reference bench harness's round trip (bench.py:19-40) on 10M C2 draws: "
                  "BSM price -> Halley IV in one fused fv_price_iv call"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c4", "c1", "c2", "c3", "c5", "rt"])
    ap.add_argument("--rows", type=int, default=0,
                    help="rows of the logical batch (default: the workload's size; fewer C4 rows = an "
                         "evenly strided sub-chain, for profiling)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--shard-scheme", default="cyclic", choices=["contiguous", "cyclic"])
    ap.add_argument("--shard", default="", help="g/G: run shard g of a G-way strong split on this GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle pass (cpu_baseline + parity)")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="skip the per-kernel event-timing and device-span passes (ncu traffic captures: "
                         "only the timed calls run)")
    return ap.parse_args(argv)


def default_rows(workload):
    return {"c4": W.C4_ROWS, "c1": 1_000_000, "c2": 10_000_000, "c3": 10_000_000,
            "c5": 10_000_000, "rt": 10_000_000}[workload]


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# sharding (every output row depends on its input row only)
# ---------------------------------------------------------------------------
def shard_ranges(n, nshard, g, scheme="contiguous", block=CYCLIC_BLOCK):
    """Row ranges [(lo, hi), ...] of shard g of n rows split nshard ways:
    one contiguous range, or blocks of ``block`` rows dealt round-robin."""
    if scheme == "contiguous":
        lo, hi = n * g // nshard, n * (g + 1) // nshard
        return [(lo, hi)] if hi > lo else []
    nb = (n + block - 1) // block
    return [(b * block, min(n, (b + 1) * block)) for b in range(g, nb, nshard)]


def plan(args, world, rank):
    """(logical rows, this process's row ranges, shard label, F, scaling)."""
    n_total = args.rows or default_rows(args.workload)
    if args.shard:
        g, G = (int(x) for x in args.shard.split("/"))
        assert 0 <= g < G and world == 1, "--shard g/G runs one shard in one process"
        return n_total, shard_ranges(n_total, G, g, args.shard_scheme), f"{g}/{G}", 100.0, "strong"
    if args.scaling == "weak":
        return n_total, [(0, n_total)], f"{rank}/{world}", 100.0 * (1.01 ** rank), "weak"
    return n_total, shard_ranges(n_total, world, rank, args.shard_scheme), f"{rank}/{world}", 100.0, "strong"


def c4_row_index(ranges, n_total):
    """Chain row indices of the given logical rows (an evenly strided
    sub-chain when the logical batch is smaller than the chain)."""
    stride = max(1, W.C4_ROWS // n_total) if n_total < W.C4_ROWS else 1
    return [(lo, hi, stride) for lo, hi in ranges]


# ---------------------------------------------------------------------------
# workload construction
# ---------------------------------------------------------------------------
def c4_device(rows, rank, dev, ranges=None, n_total=None, F=None):
    """C4 chain rows built on the GPU: returns the column
    tensors of a Black-76 LBR batch (F, r, q are broadcast scalars).  Default:
    rows [0, rows) of rank ``rank``'s weak-scaling chain (F = 100 * 1.01^rank)."""
    import torch
    F = (100.0 * (1.01 ** rank)) if F is None else F
    n_total = rows if n_total is None else n_total
    ranges = [(0, rows)] if ranges is None else ranges
    m = sum(hi - lo for lo, hi in ranges)
    flag = torch.empty(m, dtype=torch.int8, device=dev)
    K = torch.empty(m, dtype=torch.float64, device=dev)
    t = torch.empty(m, dtype=torch.float64, device=dev)
    sig = torch.empty(m, dtype=torch.float64, device=dev)
    step = 1 << 24
    o = 0
    for lo, hi, stride in c4_row_index(ranges, n_total):
        for s0 in range(lo, hi, step):
            s1 = min(hi, s0 + step)
            row = (torch.arange(s0, s1, device=dev, dtype=torch.int64) * stride) % W.C4_ROWS
            i = (row % W.C4_STRIKES).double()
            j = ((row // W.C4_STRIKES) % W.C4_MATURITIES).double()
            f = row // (W.C4_STRIKES * W.C4_MATURITIES)
            x = -2.0 + 4.0 * i / (W.C4_STRIKES - 1)
            k = s1 - s0
            K[o:o + k] = F * torch.exp(-x)
            tt = (1.0 / 365.0) * torch.pow(torch.tensor(5.0 * 365.0, dtype=torch.float64, device=dev),
                                           j / (W.C4_MATURITIES - 1))
            t[o:o + k] = tt
            sig[o:o + k] = torch.clamp(0.2 + 0.1 * x * x / torch.sqrt(tt), max=2.0)
            flag[o:o + k] = torch.where(f == 0, 1, -1).to(torch.int8)
            o += k
    return {"flag": flag, "strike": K, "t": t, "sigma": sig,
            "underlying": torch.full((1,), F, dtype=torch.float64, device=dev),
            "r": torch.full((1,), 0.03, dtype=torch.float64, device=dev),
            "q": torch.zeros(1, dtype=torch.float64, device=dev)}


def c4_host(ranges, n_total, F=100.0):
    """The same rows on the host (numpy; the reference arm / oracle)."""
    parts = []
    for lo, hi, stride in c4_row_index(ranges, n_total):
        parts.append((np.arange(lo, hi, dtype=np.int64) * stride) % W.C4_ROWS)
    row = np.concatenate(parts) if parts else np.zeros(0, np.int64)
    flag, _, K, t, _, sig = W.c4_rows(row)
    if F != 100.0:
        K = K * (F / 100.0)
    return {"flag": flag, "underlying": np.array([F]), "strike": K, "t": t, "r": np.array([0.03]),
            "q": np.zeros(1), "sigma": sig}


def draws_host(workload, n_total, ranges, rank_seed=0):
    """C1/C2/C3/C5/rt columns (numpy generators of the whole logical batch,
    sliced to this process's rows)."""
    if workload == "c5":
        flag, F, K, t, r, s, kind, side = W.c5_params(n_total, seed=5 + rank_seed)
        q = np.zeros_like(F)
        cols = {"flag": flag, "underlying": F, "strike": K, "t": t, "r": r, "q": q, "sigma": s,
                "kind": kind, "side": side}
    else:
        flag, F, K, t, r, q, s = W.chain_draws(n_total, seed=rank_seed)
        if workload == "c1":
            q = np.zeros_like(F)
        cols = {"flag": flag, "underlying": F, "strike": K, "t": t, "r": r, "q": q, "sigma": s}
    n = len(cols["flag"])
    idx = np.concatenate([np.arange(lo, min(hi, n)) for lo, hi in ranges]) if ranges else np.zeros(0, np.int64)
    return {k: np.ascontiguousarray(v[idx]) for k, v in cols.items()}


def draws_device(workload, rows, rank, dev, ranges=None):
    import torch
    h = draws_host(workload, rows, ranges if ranges is not None else [(0, rows)], rank_seed=rank)
    out = {k: torch.from_numpy(v).to(dev) for k, v in h.items() if k not in ("kind", "side")}
    out["kind"], out["side"] = h.get("kind"), h.get("side")
    return out


def cpu_sample_c4(rows):
    """``rows`` evenly strided rows of the C4 chain (numpy):
    (flag, F, K, t, r, sigma, stride)."""
    stride = max(1, W.C4_ROWS // rows)
    idx = np.arange(0, W.C4_ROWS, stride, dtype=np.int64)[:rows]
    flag, F, K, t, r, sig = W.c4_rows(idx)
    return flag, F, K, t, r, sig, stride


def native_cols(cols, last):
    from paper_2604_27210_b200 import _native
    return [_native.col(cols[k]) for k in ("flag", "underlying", "strike", "t", "r", "q", last)]


def price_on_device(lib, model, cols, n):
    import torch
    from paper_2604_27210_b200 import _native
    px = torch.empty(n, dtype=torch.float64, device=cols["strike"].device)
    err = _native.fv_error()
    rc = lib.fv_batch_price(model, *native_cols(cols, "sigma"), n, px.data_ptr(), err)
    if rc:
        raise RuntimeError(err.message)
    return px


def workload_call(workload):
    """(model code, method code: 1 LBR / 0 Halley / -1 price+Greeks, price->IV round trip?)"""
    if workload in ("c4", "c1", "c5"):
        return 0, 1, False
    if workload == "c2":
        return 2, 0, False
    if workload == "rt":
        return 2, 0, True
    return 2, -1, False


L2_FLUSH_BELOW = 256 << 20      # step bytes (inputs + outputs) under which L2 is flushed between steps
L2_SCRATCH_BYTES = 256 << 20


def config_for(args, world, n_total, scaling, shard_label, step_bytes=None):
    if step_bytes is not None and step_bytes < L2_FLUSH_BELOW:
        l2 = ("L2 flushed between timed steps: a %d MB write outside the per-step events (the step's "
              "%.0f MB of inputs + outputs would fit in the 126 MB L2); ms_per_step = mean of the "
              "per-step event pairs" % (L2_SCRATCH_BYTES >> 20, step_bytes / 1e6))
    else:
        l2 = ("inputs + outputs (%s per step per GPU) exceed twice the 126 MB L2; no flush needed"
              % ("%.2f GB" % (step_bytes / 1e9) if step_bytes else ">= 0.5 GB"))
    cfg = {"workload": WL_NAMES[args.workload], "rows_total": n_total,
           "parallelism": f"quote-sharded x{world} ({scaling} scaling"
                          + (f", {args.shard_scheme} shards" if scaling == "strong" else "") + ")",
           "l2": l2}
    if args.shard:
        cfg["shard"] = shard_label
    return cfg


# ---------------------------------------------------------------------------
# clocks (sampled DURING the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(REPO, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        # the sampler must be live before the timed region starts (nvidia-smi
        # takes a few hundred ms to print its first line)
        t0 = time.time()
        while time.time() - t0 < 5.0 and self.proc.poll() is None:
            self.fh.flush()
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.05)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# the oracle pass: CPU baseline timing + parity of every row
# ---------------------------------------------------------------------------
def host_info(threads):
    info = {"cores": threads, "host_cpus": os.cpu_count(), "cpu_model": None,
            "glibc": "-".join(platform.libc_ver()), "numpy": np.__version__}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import scipy
        info["scipy"] = scipy.__version__
    except ImportError:
        info["scipy"] = None
    return info


def oracle_run(workload, h, threads):
    """Run the oracle (reference restated on glibc + scipy) over the host
    columns ``h`` of one workload: returns (seconds, outputs dict).  The
    price column of the IV workloads is an input (given in ``h``)."""
    from oracle import fvoracle as O
    O.lib()
    O.set_threads(threads)
    model, method, rt = workload_call(workload)
    mname = {0: "black", 2: "bsm"}[model]
    a = [h[k] for k in ("flag", "underlying", "strike", "t", "r", "q")]
    t0 = time.perf_counter()
    if method == -1:
        p = O.rows_price(mname, *a, h["sigma"])
        g = O.rows_greeks(mname, *a, h["sigma"])
        out = {"price": p["price"], "delta": g["delta"], "gamma": g["gamma"], "theta": g["theta"],
               "rho": g["rho"], "vega": g["vega"], "status": g["status_code"],
               "exc": p["exc"].astype(np.int32) + g["exc"]}
    elif rt:
        p = O.rows_price(mname, *a, h["sigma"])
        w = O.rows_iv(mname, "halley" if method == 0 else "lbr", *a, p["price"])
        out = {"price": p["price"], "iv": w["iv"], "status": w["status_code"],
               "exc": p["exc"].astype(np.int32) + w["exc"]}
    else:
        w = O.rows_iv(mname, "lbr" if method == 1 else "halley", *a, h["price"])
        out = {"iv": w["iv"], "status": w["status_code"], "exc": w["exc"].astype(np.int32)}
    return time.perf_counter() - t0, out


def parity_count(got, want):
    """Rows whose outputs differ bit for bit (any NaN equals any NaN) or where
    the reference would have raised."""
    bad = np.asarray(want["exc"]) != 0
    for k, v in got.items():
        w = want[k]
        v = np.asarray(v)
        if v.dtype == np.float64:
            same = (v.view(np.int64) == w.view(np.int64)) | (np.isnan(v) & np.isnan(w))
        else:
            same = v.astype(np.int64) == np.asarray(w).astype(np.int64)
        bad |= ~same
    return int(bad.sum())


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------
def run_reference(args):
    """The reference's CPU path on the same workload and config: the oracle
    port (reference restated in C++ on glibc + scipy) on all host threads, no
    product code imported.  Rank 0 only under torchrun."""
    world, rank, local = dist_setup()
    if rank != 0:
        return 0
    assert "paper_2604_27210_b200" not in sys.modules
    n_total = args.rows or default_rows(args.workload)
    scaling = "weak" if args.scaling == "weak" else "strong"
    threads = os.cpu_count() or 1
    model, method, rt = workload_call(args.workload)
    # the whole logical batch (strong scaling's chain; the reference has one host)
    if args.workload == "c4":
        h = c4_host([(0, n_total)], n_total)
    else:
        h = draws_host(args.workload, n_total, [(0, n_total)])
    if method != -1 and not rt:
        from oracle import fvoracle as O
        O.lib()
        O.set_threads(threads)
        mname = {0: "black", 2: "bsm"}[model]
        h["price"] = O.rows_price(mname, *[h[k] for k in ("flag", "underlying", "strike", "t", "r", "q")],
                                  h["sigma"])["price"]
        if args.workload == "c5":
            F = np.broadcast_to(h["underlying"], h["strike"].shape)
            h["price"] = W.c5_prices(h["flag"], F, h["strike"], h["t"], h["r"], h["kind"], h["side"], h["price"])
    m = len(h["flag"])
    warm = min(m, 1_000_000)
    hw = {k: (v[:warm] if (isinstance(v, np.ndarray) and v.shape[0] == m) else v) for k, v in h.items()}
    for _ in range(args.warmup):
        oracle_run(args.workload, hw, threads)
    times = []
    for _ in range(args.steps):
        dt, _ = oracle_run(args.workload, h, threads)
        times.append(dt)
    ms = 1e3 * float(np.mean(times))
    value = m / (ms * 1e-3)
    sample = (f"all {m} rows of the workload per step; warm-up steps on its first {warm} rows; "
              f"oracle/fvoracle.cpp (the reference restated in C++ on glibc + scipy) on {threads} host threads")
    cpu = dict(host_info(threads), value=value, unit="quotes/s", kind="port", sample=sample)
    line = {"impl": "reference",
            "metric": METRIC if args.workload == "c4" else f"fp64 quotes/sec ({args.workload})",
            "value": value, "unit": "quotes/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (same generator and rows as the GPU arm)",
            "config": config_for(args, args.gpus, n_total, scaling, ""),
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "quotes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "repo_libs_loaded": repo_libs_loaded()}
    print(json.dumps(line), flush=True)
    return 0


def repo_libs_loaded():
    """The repo's shared objects mapped into this process (/proc/self/maps):
    the evidence of which native code a line's numbers came from -- the
    product library and host extension for our arm, oracle/ for the reference
    arm."""
    libs = set()
    try:
        with open("/proc/self/maps") as fh:
            for ln in fh:
                path = ln.split()[-1] if ln.strip() else ""
                if path.endswith(".so") and os.path.realpath(path).startswith(os.path.realpath(REPO)):
                    libs.add(os.path.relpath(os.path.realpath(path), os.path.realpath(REPO)))
    except OSError:
        return None
    return sorted(libs)


def run_ours(args):
    import torch
    from paper_2604_27210_b200 import _native
    world, rank, local = dist_setup()
    # FV_BENCH_SHARE_GPUS=1 (tests only): ranks share the visible GPUs (local
    # rank mod device count) over gloo, so the N > 1 code path runs on a
    # 1-GPU box; its timings are not scaling numbers
    share = os.environ.get("FV_BENCH_SHARE_GPUS") == "1"
    if share:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        pg = dist
    lib = _native.lib_for_compute()
    n_total, ranges, shard_label, Fr, scaling = plan(args, world, rank)
    stream = torch.cuda.current_stream(dev)
    lib.fv_set_stream(ctypes_ptr(stream.cuda_stream))
    model, method, roundtrip = workload_call(args.workload)

    # ---- inputs resident in HBM ------------------------------------------
    if args.workload == "c4":
        cols = c4_device(0, rank, dev, ranges=ranges, n_total=n_total, F=Fr)
        last = "price"
        n = cols["flag"].numel()
        cols["price"] = price_on_device(lib, 0, cols, n)
        extra = {}
    else:
        cols = draws_device(args.workload, n_total, 0 if scaling == "strong" else rank, dev, ranges)
        extra = {"kind": cols.pop("kind"), "side": cols.pop("side")}
        n = cols["flag"].numel()
        last = "sigma" if (method == -1 or roundtrip) else "price"
        if method != -1 and not roundtrip:
            cols["price"] = price_on_device(lib, model, cols, n)
            if args.workload == "c5":
                hh = {k: cols[k].cpu().numpy() for k in ("flag", "underlying", "strike", "t", "r", "price")}
                px = W.c5_prices(hh["flag"], hh["underlying"], hh["strike"], hh["t"], hh["r"],
                                 extra["kind"], extra["side"], hh["price"])
                cols["price"] = torch.from_numpy(px).to(dev)
    torch.cuda.synchronize(dev)

    out_iv = torch.empty(n, dtype=torch.float64, device=dev)
    out_st = torch.empty(n, dtype=torch.int8, device=dev)
    out_px = torch.empty(n, dtype=torch.float64, device=dev) if roundtrip else None
    greeks = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)] if method < 0 else []
    ncols = native_cols(cols, last)
    launches = [0]
    # L2 rule: a step whose inputs + outputs fit in twice the 126 MB L2 (C1's
    # 1M rows: ~42 MB) could run from a warm L2, so a 256 MB scratch buffer
    # is written between timed steps (outside the per-step events) and the
    # step time is the sum of the per-step event pairs; larger steps stream
    # from HBM anyway.
    step_bytes = sum(cols[k].numel() * cols[k].element_size()
                     for k in ("flag", "underlying", "strike", "t", "r", "q", last) if cols[k].numel() > 1)
    step_bytes += n * (9 + (8 if roundtrip else 0) + (40 if method < 0 else 0))
    l2_flush = step_bytes < L2_FLUSH_BELOW
    scratch = torch.empty(L2_SCRATCH_BYTES // 4, dtype=torch.int32, device=dev) if l2_flush else None

    def step():
        err = _native.fv_error()
        if roundtrip:
            err2 = _native.fv_error()
            rc = lib.fv_price_iv(model, method, *ncols, n, out_px.data_ptr(), out_iv.data_ptr(),
                                 out_st.data_ptr(), None, err, err2)
            if rc and not err.code:
                err = err2
        elif method >= 0:
            rc = lib.fv_batch_iv(model, method, *ncols, n, out_iv.data_ptr(), out_st.data_ptr(),
                                 None, err)
        else:
            err2 = _native.fv_error()
            rc = lib.fv_price_greeks(model, *ncols, n, *[g.data_ptr() for g in greeks],
                                     out_st.data_ptr(), err, err2)
        if rc:
            raise RuntimeError(f"fv call failed rc={rc}: {err.message}")
        launches[0] += lib.fv_last_launch_count()

    # the clock sampler starts first: the warm-up steps then also bring the
    # GPU back from the idle of the sampler's start-up (a first call right
    # after an idle period runs ~15 % slow)
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if pg:
        pg.barrier()
    launches[0] = 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    if pg:
        pg.barrier()
    t_all0 = torch.cuda.Event(enable_timing=True)
    t_all1 = torch.cuda.Event(enable_timing=True)
    t_all0.record(stream)
    for k in range(args.steps):
        if l2_flush:
            scratch.fill_(k)                       # evicts the previous step's lines
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    t_all1.record(stream)
    torch.cuda.synchronize(dev)
    if pg:
        pg.barrier()
    clk = clocks.stop()
    total_ms = t_all0.elapsed_time(t_all1)
    per_call_ms = [a.elapsed_time(b) for a, b in ev]
    if l2_flush:
        total_ms = float(sum(per_call_ms))        # the flushes are not part of a step
    own_ms = total_ms
    if pg:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / args.steps
    units = world * n if scaling == "weak" else (n_total if not args.shard else n)
    value = units / (ms_step * 1e-3)
    st = torch.bincount(out_st.to(torch.int64), minlength=5).cpu().tolist()

    # ---- per-kernel split of a step (CUDA events around each launch; the
    # timing pass serialises the side-stream branches, so the shares are of
    # the serialised call and each event pair brackets one kernel alone)
    kernels, n_far_low, serial_ms = None, None, None
    try:
        if args.no_kernel_timing:
            raise RuntimeError("skipped (--no-kernel-timing)")
        lib.fv_set_kernel_timing(1)
        _native.kernel_times(lib)
        nk = max(1, min(args.steps, 3))
        region = torch.empty(n, dtype=torch.int8, device=dev) if (method == 1 and not roundtrip) else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(nk):
            if region is not None:     # LBR: also record each quote's region (far-low count)
                err = _native.fv_error()
                rc = lib.fv_batch_iv(model, method, *ncols, n, out_iv.data_ptr(), out_st.data_ptr(),
                                     region.data_ptr(), err)
                if rc:
                    raise RuntimeError(err.message)
            else:
                step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        serial_ms = e0.elapsed_time(e1) / nk
        if region is not None:
            n_far_low = int((region == 0).sum().item())
        kt = _native.kernel_times(lib)
        lib.fv_set_kernel_timing(0)
        tot = sum(v[0] for v in kt.values()) or 1.0
        kernels = {k: {"ms_per_step": v[0] / nk, "launches_per_step": v[1] / nk, "share": v[0] / tot}
                   for k, v in sorted(kt.items(), key=lambda kv: -kv[1][0])}
    except Exception as exc:  # noqa: BLE001
        lib.fv_set_kernel_timing(0)
        kernels = {"error": repr(exc)}

    # ---- device span of a call (events around its launches, nothing
    # serialised): per_call_ms - span = host overhead of the synchronous call
    span_ms = None
    try:
        if args.no_kernel_timing:
            raise RuntimeError("skipped (--no-kernel-timing)")
        lib.fv_set_span_timing(1)
        spans = []
        for _ in range(max(1, min(args.steps, 5))):
            step()
            spans.append(lib.fv_last_span_ms())
        lib.fv_set_span_timing(0)
        span_ms = float(np.mean(spans)) if min(spans) >= 0 else None
    except Exception:  # noqa: BLE001
        lib.fv_set_span_timing(0)

    # ---- the dominant kernel's own roofline --------------------------------
    # algorithmic work per launch = the reference's weighted distinct fp64 ops
    # of the kernel's phase per quote (profiles/w_phases_*.json, tools/w_count*.py)
    # x the quotes it processes; time = its mean launch duration (event pass)
    dominant = None
    wp = {}
    try:
        wp = json.load(open(os.path.join(REPO, "profiles", "w_phases_%s.json" % args.workload)))
    except (OSError, ValueError):
        pass
    try:
        kname = "k_lbr_far_low_fast"
        if n_far_low and kernels and kname in kernels:
            w_solve = wp["by_region"]["FAR_LOW"]["W_solve"]
            t_k = kernels[kname]["ms_per_step"] * 1e-3
            dominant = {"kernel": kname, "share_of_call": kernels[kname]["share"], "units": n_far_low,
                        "W_per_unit": w_solve, "ms_per_launch": t_k * 1e3,
                        "achieved": w_solve * n_far_low / t_k / 1e12}
        kname = "k_halley_iter"
        if args.workload == "c2" and kernels and kname in kernels:
            ph = wp["phases"]["halley"]
            units_h = int(round(n * ph["share_reaching"]))
            t_k = kernels[kname]["ms_per_step"] * 1e-3
            dominant = {"kernel": kname, "share_of_call": kernels[kname]["share"], "units": units_h,
                        "W_per_unit": ph["W_per_reaching_quote"], "ms_per_launch": t_k * 1e3,
                        "achieved": ph["W_per_reaching_quote"] * units_h / t_k / 1e12,
                        "units_source": "rows x share of quotes reaching the Halley loop in a %d-row "
                                        "reference sample (profiles/w_phases_c2.json)" % wp["rows"]}
    except (KeyError, TypeError, ZeroDivisionError):
        pass

    # ---- e2e: same call with pinned host buffers ---------------------------
    e2e = None
    if not args.no_e2e:
        hcols = {}
        for k, v in cols.items():
            hcols[k] = v.cpu().pin_memory() if v.numel() > 1 else v.cpu()
        h_iv = torch.empty(n, dtype=torch.float64).pin_memory()
        h_st = torch.empty(n, dtype=torch.int8).pin_memory()
        h_px = torch.empty(n, dtype=torch.float64).pin_memory() if roundtrip else None
        h_g = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(6)] if method < 0 else []
        hn = native_cols(hcols, last)
        h2d = sum(hcols[k].numel() * hcols[k].element_size()
                  for k in ("flag", "underlying", "strike", "t", "r", "q", last) if hcols[k].numel() > 1)
        d2h = n * (17 if roundtrip else (9 if method >= 0 else 49))

        def estep():
            err = _native.fv_error()
            if roundtrip:
                err2 = _native.fv_error()
                rc = lib.fv_price_iv(model, method, *hn, n, h_px.data_ptr(), h_iv.data_ptr(),
                                     h_st.data_ptr(), None, err, err2)
            elif method >= 0:
                rc = lib.fv_batch_iv(model, method, *hn, n, h_iv.data_ptr(), h_st.data_ptr(), None, err)
            else:
                err2 = _native.fv_error()
                rc = lib.fv_price_greeks(model, *hn, n, *[g.data_ptr() for g in h_g], h_st.data_ptr(),
                                         err, err2)
            if rc:
                raise RuntimeError(err.message)
        estep()
        h2d_logical = h2d
        h2d = int(lib.fv_last_h2d_bytes())          # what crossed the link (runs for piecewise-constant columns)
        if pg:
            pg.barrier()
        times = []
        for _ in range(max(2, min(args.steps, 5))):
            torch.cuda.synchronize(dev)
            if pg:
                pg.barrier()
            t0 = time.perf_counter()
            estep()
            times.append(time.perf_counter() - t0)
        e_ms = 1e3 * float(np.mean(times))
        if pg:
            tt = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            pg.all_reduce(tt, op=pg.ReduceOp.MAX)
            e_ms = float(tt.item())
        if method >= 0:
            same = bool(torch.equal(h_iv.to(dev).view(torch.int64), out_iv.view(torch.int64)))
            if roundtrip:
                same = same and bool(torch.equal(h_px.to(dev).view(torch.int64), out_px.view(torch.int64)))
        else:
            same = all(bool(torch.equal(h.to(dev).view(torch.int64), g.view(torch.int64)))
                       for h, g in zip(h_g, greeks))
        h2d_gbs = None
        try:
            hb = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
            db = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
            db.copy_(hb, non_blocking=True)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for _ in range(3):
                db.copy_(hb, non_blocking=True)
            torch.cuda.synchronize(dev)
            h2d_gbs = 3 * (1 << 30) / (time.perf_counter() - t0) / 1e9
            del hb, db
        except Exception:  # noqa: BLE001
            pass
        e2e = {"value": units / (e_ms * 1e-3), "unit": "quotes/s", "h2d_bytes_per_step": int(h2d),
               "h2d_bytes_per_step_logical": int(h2d_logical),
               "h2d_note": "h2d_bytes_per_step = bytes the call moved host -> device (fv_last_h2d_bytes): "
                           "streamed columns, piecewise-constant columns as (first row, value) runs "
                           "rebuilt on the device, broadcast scalars; _logical = the input arrays' bytes",
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms,
               "timing": "wall clock around the synchronous C-ABI call (host buffers pinned), max over ranks",
               "bit_identical_to_device_resident": same, "pcie_h2d_gbs": h2d_gbs,
               "h2d_ceiling_quotes_s": (n * h2d_gbs * 1e9 / h2d * (units / n)) if h2d_gbs and h2d else None}

    # ---- oracle pass: CPU baseline (rank 0, N=1) + parity of every row ------
    parity, cpu = None, None
    if not args.no_cpu:
        try:
            hcpu = {k: v.cpu().numpy() for k, v in cols.items()}
            threads = max(1, (os.cpu_count() or 1) // world)
            dt, want = oracle_run(args.workload, hcpu, threads)
            if method == -1:
                got = {"price": greeks[0], "delta": greeks[1], "gamma": greeks[2], "theta": greeks[3],
                       "rho": greeks[4], "vega": greeks[5], "status": out_st}
            else:
                got = {"iv": out_iv, "status": out_st}
                if roundtrip:
                    got["price"] = out_px
            got = {k: v.cpu().numpy() for k, v in got.items()}
            bad = parity_count(got, want)
            rows_checked = n
            if pg:
                tt = torch.tensor([bad, rows_checked], dtype=torch.int64, device=dev)
                pg.all_reduce(tt, op=pg.ReduceOp.SUM)
                bad, rows_checked = (int(x) for x in tt.tolist())
            parity = {"rows_checked": rows_checked, "mismatches": bad,
                      "against": "oracle/fvoracle.cpp (pinned to the live reference by tests/golden/)",
                      "compared": sorted(got) + ["reference exception rows"],
                      "rule": "bit-identical doubles (any NaN = any NaN), identical status codes"}
            if world == 1:
                cpu = dict(host_info(threads), value=n / dt, unit="quotes/s", kind="port",
                           sample=f"all {n} rows of this run's workload, oracle/fvoracle.cpp (the reference "
                                  f"restated in C++ on glibc + scipy), OpenMP {threads} threads, {dt:.2f} s")
        except Exception as exc:  # noqa: BLE001
            parity = {"error": repr(exc)}

    # ---- roofline ------------------------------------------------------------
    peak = ctypes_double()
    secs = ctypes_double()
    lib.fv_probe_fp64_peak(ctypes_addr(peak), ctypes_addr(secs))
    peak_tops = peak.value / 1e12
    call_s = float(np.mean(per_call_ms)) * 1e-3
    achieved = W_OPS[args.workload] * n / call_s / 1e12
    w_read = wp.get("W_read_mean") if args.workload == "c4" else None
    w_done = wp.get("W_done_mean") if args.workload == "c4" else None
    in_bytes = sum(cols[k].numel() * cols[k].element_size()
                   for k in ("flag", "underlying", "strike", "t", "r", "q", last) if cols[k].numel() > 1)
    out_bytes = n * (17 if roundtrip else (9 if method >= 0 else 49))
    hbm_gbs = (in_bytes + out_bytes) / call_s / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = None
    try:
        prof = json.load(open(os.path.join(REPO, "profiles", "roofline_traffic.json")))
        bpq = prof.get(args.workload, {}).get("dram_bytes_per_quote")
        traffic = bpq * n if bpq else None
    except (OSError, ValueError, AttributeError):
        pass
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak_tops, "unit": "T weighted-fp64-ops/s",
                "frac": achieved / peak_tops if peak_tops else None, "traffic": traffic,
                "note": "kernel = one C-ABI call (its kernels in sequence on the call's stream, side-stream "
                        "branches overlapping); achieved = W=%.0f weighted distinct fp64 ops/quote (SURVEY 8(d)) "
                        "x rows per call / mean call duration (CUDA events on the launching stream); peak = "
                        "measured DFMA issue rate (fv_probe_fp64_peak, this run; MEASURED_PEAKS.json has no fp64 "
                        "entry); traffic = ncu DRAM read+write bytes per call (profiles/roofline_traffic.json)"
                        % W_OPS[args.workload]}
    if w_read:
        roofline["achieved_read"] = w_read * n / call_s / 1e12
        roofline["frac_read"] = roofline["achieved_read"] / peak_tops if peak_tops else None
        roofline["W_read"] = w_read
        roofline["note_read"] = ("frac_read counts only the W the GPU path must evaluate: the reference's "
                                 "anchors that _region never reads (b_c, b_hi of far-low quotes, b_hi of "
                                 "near-low ones; %.0f of W=%.0f on a 30k-row C4 sample, tools/w_count.py) "
                                 "are skipped by the lazy-anchor passes" % (W_OPS["c4"] - w_read, W_OPS["c4"]))
    if w_done:
        roofline["frac_done"] = w_done * n / call_s / 1e12 / peak_tops if peak_tops else None
        roofline["W_done"] = w_done
        roofline["note_done"] = ("frac_done also leaves out the first anchor b_lo of every far-low quote "
                                 "(%.0f of W per quote on average): the normalize pass's table bound proves "
                                 "beta < b_lo without it for whole warps of the chain, so this is a lower "
                                 "bound of the work done" % (w_read - w_done))
    if args.workload == "c2":
        roofline["note"] += ("; C2: the bracket pass decides f(10)'s sign in fp32 instead of evaluating it "
                             "(~8 % of W counted but not executed)")

    if rank == 0:
        line = {
            "metric": METRIC if args.workload == "c4" else f"fp64 quotes/sec ({args.workload})",
            "value": value, "unit": "quotes/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded chain generated on device; prices from the pricing kernel)",
            "config": config_for(args, world, n_total, scaling, shard_label, step_bytes),
            "rows_this_rank": n,
            "roofline": roofline,
            "kernels": kernels,
            "kernels_note": "per-kernel CUDA events in a separate pass that runs the side-stream branches in "
                            "sequence on the call's stream (fv_set_kernel_timing): shares are of the serialised "
                            "call (serial_ms_per_call); the timed calls overlap those branches",
            "serial_ms_per_call": serial_ms,
            "device_span_ms_per_call": span_ms,
            "device_span_note": "CUDA events on the call's stream before its first and after its last launch "
                                "(fv_set_span_timing); mean per-call time minus this = host overhead of the "
                                "synchronous C-ABI call",
            "dominant_kernel": (dict(dominant, peak=peak_tops, unit="T weighted-fp64-ops/s",
                                     frac=dominant["achieved"] / peak_tops if peak_tops else None)
                                if dominant else None),
            "roofline_hbm": {"bound": "hbm", "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                             "frac": hbm_gbs / hbm_peak, "bytes_per_quote": (in_bytes + out_bytes) / max(n, 1),
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": e2e,
            "gpu_launches": launches[0],
            "clocks": clk,
            "status_counts": dict(zip(["converged", "fell_back", "below_intrinsic", "above_upper",
                                       "max_iterations"], st)),
            "per_call_ms": per_call_ms,
            "rank0_ms_per_step": own_ms / args.steps,
            "repo_libs_loaded": repo_libs_loaded(),
        }
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def ctypes_ptr(v):
    import ctypes
    return ctypes.c_void_p(v)


def ctypes_double():
    import ctypes
    return ctypes.c_double(0.0)


def ctypes_addr(x):
    import ctypes
    return ctypes.cast(ctypes.pointer(x), ctypes.c_void_p)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
