#!/usr/bin/env python3
"""Benchmark: fp64 LBR implied-vol solves/sec on the C4 100M-quote option chain.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c1|c2|c3|c5] [--rows R]

Metric (BASELINE.json): "fp64 IV solves/sec (LBR, 100M quotes) at 1/2/4/8 B200
vs host-CPU ref".  One step = one ``fv_batch_iv(BLACK76, LBR, ...)`` call over
one rank's 100M-quote chain (2 flags x 1,000 maturities x
50,000 strikes).  Multi-GPU: one process per GPU (torchrun); rank r solves its
own 100M-quote chain (underlying F_r = 100 * 1.01^r, strikes scaled with it,
so every rank has the same normalized work) -- weak scaling, no collective
on the data path; ranks only barrier and max-reduce their timings.

``value`` is device-resident throughput (inputs already in HBM; CUDA events on
the launching stream, max over ranks).  ``e2e`` is the same call through the
C ABI with pinned HOST buffers (chunked H2D / kernel / D2H inside the timed
region).  The CPU baseline is the oracle port (oracle/fvoracle.cpp -- the
reference restated in C++ on glibc + scipy, all host threads) timed on a
bounded strided sample of the same chain.  The inputs (2.5 GB per step) are
larger than the 126 MB L2, so no flush is needed between steps.
"""

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# Weighted distinct FP64 ops per quote the reference executes (SURVEY.md 8(d),
# Appendix B.3): the algorithmic work per unit for the roofline.
# rt (the reference's bench harness: synthetic_chain's BSM pricing + run_bench's
# Halley inversion, one fused fv_price_iv call): price 200 + C2 Halley 1476.
W_OPS = {"c4": 1443.0, "c1": 1405.0, "c2": 1476.0, "c3": 298.0, "c5": 347.0, "rt": 1676.0}
METRIC = "fp64 IV solves/sec (LBR, 100M quotes) at 1/2/4/8 B200 vs host-CPU ref"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c4", "c1", "c2", "c3", "c5", "rt"])
    ap.add_argument("--rows", type=int, default=0, help="rows per rank (default: workload size)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="skip the per-kernel event-timing pass (ncu traffic captures)")
    return ap.parse_args()


def default_rows(workload):
    return {"c4": 100_000_000, "c1": 1_000_000, "c2": 10_000_000, "c3": 10_000_000,
            "c5": 10_000_000, "rt": 10_000_000}[workload]


# ---------------------------------------------------------------------------
# workload construction on the device
# ---------------------------------------------------------------------------
def c4_device(rows, rank, dev):
    """C4 chain for one rank, built on the GPU: returns the
    column tensors of a Black-76 LBR batch (F, r, q are broadcast scalars)."""
    import torch
    from paper_2604_27210_b200 import workloads as W
    F = 100.0 * (1.01 ** rank)
    out = {}
    flag = torch.empty(rows, dtype=torch.int8, device=dev)
    K = torch.empty(rows, dtype=torch.float64, device=dev)
    t = torch.empty(rows, dtype=torch.float64, device=dev)
    sig = torch.empty(rows, dtype=torch.float64, device=dev)
    step = 1 << 24
    # fewer rows than the chain: an evenly strided sub-chain (profiling runs)
    stride = max(1, W.C4_ROWS // rows) if rows < W.C4_ROWS else 1
    for s0 in range(0, rows, step):
        s1 = min(rows, s0 + step)
        row = (torch.arange(s0, s1, device=dev, dtype=torch.int64) * stride) % W.C4_ROWS
        i = (row % W.C4_STRIKES).double()
        j = ((row // W.C4_STRIKES) % W.C4_MATURITIES).double()
        f = row // (W.C4_STRIKES * W.C4_MATURITIES)
        x = -2.0 + 4.0 * i / (W.C4_STRIKES - 1)
        K[s0:s1] = F * torch.exp(-x)
        tt = (1.0 / 365.0) * torch.pow(torch.tensor(5.0 * 365.0, dtype=torch.float64, device=dev),
                                       j / (W.C4_MATURITIES - 1))
        t[s0:s1] = tt
        sig[s0:s1] = torch.clamp(0.2 + 0.1 * x * x / torch.sqrt(tt), max=2.0)
        flag[s0:s1] = torch.where(f == 0, 1, -1).to(torch.int8)
    out["flag"], out["strike"], out["t"], out["sigma"] = flag, K, t, sig
    out["underlying"] = torch.full((1,), F, dtype=torch.float64, device=dev)
    out["r"] = torch.full((1,), 0.03, dtype=torch.float64, device=dev)
    out["q"] = torch.zeros(1, dtype=torch.float64, device=dev)
    return out


def draws_device(workload, rows, rank, dev):
    """C1/C2/C3/C5 columns (numpy generators, moved to the device)."""
    import torch
    from paper_2604_27210_b200 import workloads as W
    if workload == "c5":
        flag, F, K, t, r, s, kind, side = W.c5_params(rows, seed=5 + rank)
        q = np.zeros_like(F)
        extra = {"kind": kind, "side": side}
    else:
        flag, F, K, t, r, q, s = W.chain_draws(rows, seed=rank)
        if workload == "c1":
            q = np.zeros_like(F)
        extra = {}
    cols = {"flag": flag, "underlying": F, "strike": K, "t": t, "r": r, "q": q, "sigma": s}
    out = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in cols.items()}
    out.update(extra)
    return out


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
        # takes a few hundred ms to print its first line; a short timed region
        # would otherwise end before any sample)
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
# CPU baseline: the oracle port on the host cores
# ---------------------------------------------------------------------------
def cpu_sample_c4(rows, stride_rows=None):
    from paper_2604_27210_b200 import workloads as W
    stride = max(1, W.C4_ROWS // rows)
    idx = np.arange(0, W.C4_ROWS, stride, dtype=np.int64)[:rows]
    i = idx % W.C4_STRIKES
    j = (idx // W.C4_STRIKES) % W.C4_MATURITIES
    f = idx // (W.C4_STRIKES * W.C4_MATURITIES)
    x = -2.0 + 4.0 * i / (W.C4_STRIKES - 1)
    K = 100.0 * np.exp(-x)
    t = (1.0 / 365.0) * (5.0 * 365.0) ** (j / (W.C4_MATURITIES - 1))
    sig = np.minimum(0.2 + 0.1 * x * x / np.sqrt(t), 2.0)
    flag = np.where(f == 0, 1, -1).astype(np.int8)
    n = len(idx)
    return flag, np.full(n, 100.0), K, t, np.full(n, 0.03), sig, stride


def cpu_baseline(seconds, workload="c4"):
    """Time the oracle (reference restated in C++, all host threads) on a
    strided sample of the chain sized to ~``seconds`` of CPU work."""
    from oracle import fvoracle as O
    O.lib()
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    flag, F, K, t, r, sig, stride = cpu_sample_c4(200_000)
    px = O.rows_price("black", flag, F, K, t, r, 0.0, sig)["price"]
    t0 = time.perf_counter()
    O.rows_iv("black", "lbr", flag, F, K, t, r, 0.0, px)
    rate = len(flag) / (time.perf_counter() - t0)
    rows = int(min(max(rate * seconds, 200_000), 50_000_000))
    flag, F, K, t, r, sig, stride = cpu_sample_c4(rows)
    px = O.rows_price("black", flag, F, K, t, r, 0.0, sig)["price"]
    t0 = time.perf_counter()
    O.rows_iv("black", "lbr", flag, F, K, t, r, 0.0, px)
    dt = time.perf_counter() - t0
    return {"value": len(flag) / dt, "unit": "quotes/s", "cores": cores, "kind": "port",
            "sample": f"{len(flag)} rows of the C4 chain (1 row in {stride}), "
                      f"oracle/fvoracle.cpp (reference restated on glibc+scipy), "
                      f"OpenMP {cores} threads, {dt:.2f} s"}


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    world, rank, local = dist_setup()
    if rank != 0:
        return 0
    from oracle import fvoracle as O
    O.lib()
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    # size one step to a few seconds of host work
    flag, F, K, t, r, sig, stride = cpu_sample_c4(100_000)
    px = O.rows_price("black", flag, F, K, t, r, 0.0, sig)["price"]
    t0 = time.perf_counter()
    O.rows_iv("black", "lbr", flag, F, K, t, r, 0.0, px)
    rate = len(flag) / (time.perf_counter() - t0)
    rows = int(min(max(rate * 4.0, 100_000), 50_000_000))
    flag, F, K, t, r, sig, stride = cpu_sample_c4(rows)
    px = O.rows_price("black", flag, F, K, t, r, 0.0, sig)["price"]
    for _ in range(args.warmup):
        O.rows_iv("black", "lbr", flag[:10000], F[:10000], K[:10000], t[:10000], r[:10000], 0.0,
                  px[:10000])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.rows_iv("black", "lbr", flag, F, K, t, r, 0.0, px)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    value = len(flag) / (ms * 1e-3)
    sample = (f"{len(flag)} rows of the C4 chain per step (1 row in {stride}), "
              f"oracle/fvoracle.cpp on {cores} host threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "quotes/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "C4 LBR Black-76 chain (strided sample)"},
            "cpu_baseline": {"value": value, "unit": "quotes/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "quotes/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    from paper_2604_27210_b200 import _native
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    lib = _native.lib_for_compute()
    rows = args.rows or default_rows(args.workload)
    stream = torch.cuda.current_stream(dev)
    lib.fv_set_stream(ctypes_ptr(stream.cuda_stream))

    # ---- inputs resident in HBM ------------------------------------------
    roundtrip = False
    if args.workload == "c4":
        cols = c4_device(rows, rank, dev)
        model, method, last = 0, 1, "price"
        cols["price"] = price_on_device(lib, 0, cols, rows)
    else:
        cols = draws_device(args.workload, rows, rank, dev)
        if args.workload in ("c1", "c5"):
            model, method = 0, 1
        elif args.workload in ("c2", "rt"):
            model, method = 2, 0
        else:
            model, method = 2, -1
        roundtrip = args.workload == "rt"
        last = "sigma" if (method == -1 or roundtrip) else "price"
        if method != -1 and not roundtrip:
            cols["price"] = price_on_device(lib, model, cols, rows)
            if args.workload == "c5":
                from paper_2604_27210_b200 import workloads as W
                h = {k: cols[k].cpu().numpy() for k in ("flag", "underlying", "strike", "t", "r", "price")}
                px = W.c5_prices(h["flag"], h["underlying"], h["strike"], h["t"], h["r"],
                                 cols["kind"], cols["side"], h["price"])
                cols["price"] = torch.from_numpy(px).to(dev)
    torch.cuda.synchronize(dev)

    n = rows
    out_iv = torch.empty(n, dtype=torch.float64, device=dev)
    out_st = torch.empty(n, dtype=torch.int8, device=dev)
    out_px = torch.empty(n, dtype=torch.float64, device=dev) if roundtrip else None
    greeks = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]

    ncols = native_cols(cols, last)
    launches = [0]

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

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if pg:
        pg.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
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
    if pg:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / args.steps
    value = world * n / (ms_step * 1e-3)

    # ---- per-kernel split of a step (CUDA events around each launch, on the
    # launching stream; a separate pass so the headline timing has no events)
    kernels = None
    n_far_low = None
    try:
        if args.no_kernel_timing:
            raise RuntimeError("skipped (--no-kernel-timing)")
        lib.fv_set_kernel_timing(1)
        _native.kernel_times(lib)
        nk = max(1, min(args.steps, 3))
        region = torch.empty(n, dtype=torch.int8, device=dev) if (method == 1 and not roundtrip) else None
        for _ in range(nk):
            if region is not None:     # LBR: also record each quote's region (far-low count)
                err = _native.fv_error()
                rc = lib.fv_batch_iv(model, method, *ncols, n, out_iv.data_ptr(), out_st.data_ptr(),
                                     region.data_ptr(), err)
                if rc:
                    raise RuntimeError(err.message)
            else:
                step()
        torch.cuda.synchronize(dev)
        if region is not None:
            n_far_low = int((region == 0).sum().item())
        kt = _native.kernel_times(lib)
        lib.fv_set_kernel_timing(0)
        tot = sum(v[0] for v in kt.values()) or 1.0
        kernels = {k: {"ms_per_step": v[0] / nk, "launches_per_step": v[1] / nk, "share": v[0] / tot}
                   for k, v in sorted(kt.items(), key=lambda kv: -kv[1][0])}
    except Exception as exc:  # noqa: BLE001
        kernels = {"error": repr(exc)}

    # ---- the dominant kernel's own roofline (C4: k_lbr_far_low_fast) --------
    # algorithmic work per launch = the reference's weighted distinct fp64 ops
    # of the far-low solve phase per far-low quote (profiles/w_phases_c4.json,
    # tools/w_count.py) x the far-low quotes of the call; time = its mean
    # launch duration from the CUDA-event pass above
    dominant = None
    try:
        wp = json.load(open(os.path.join(REPO, "profiles", "w_phases_%s.json" % args.workload)))
        kname = "k_lbr_far_low_fast"
        if n_far_low and kernels and kname in kernels:
            w_solve = wp["by_region"]["FAR_LOW"]["W_solve"]
            t_k = kernels[kname]["ms_per_step"] * 1e-3
            dominant = {"kernel": kname, "share_of_call": kernels[kname]["share"], "units": n_far_low,
                        "W_per_unit": w_solve, "ms_per_launch": t_k * 1e3,
                        "achieved": w_solve * n_far_low / t_k / 1e12}
        kname = "k_halley_iter"
        if args.workload == "c2" and kernels and kname in kernels:
            # the Halley-step phase (solver.py:115-144) of the reference, per quote
            # that reaches it (tools/w_count_halley.py on the C2 generator);
            # units = rows x the sample's share of such quotes
            ph = wp["phases"]["halley"]
            units = int(round(n * ph["share_reaching"]))
            t_k = kernels[kname]["ms_per_step"] * 1e-3
            dominant = {"kernel": kname, "share_of_call": kernels[kname]["share"], "units": units,
                        "W_per_unit": ph["W_per_reaching_quote"], "ms_per_launch": t_k * 1e3,
                        "achieved": ph["W_per_reaching_quote"] * units / t_k / 1e12,
                        "units_source": "rows x share of quotes reaching the Halley loop in a %d-row "
                                        "reference sample (profiles/w_phases_c2.json)" % wp["rows"]}
    except (OSError, ValueError, KeyError):
        pass

    # ---- status mix of the solved chain (for the record) --------------------
    st = torch.bincount(out_st.to(torch.int64) + 0, minlength=5).cpu().tolist()

    # ---- e2e: same call with pinned host buffers ---------------------------
    e2e = None
    if not args.no_e2e:
        hcols = {}
        for k, v in cols.items():
            if not torch.is_tensor(v):
                continue
            hcols[k] = v.cpu().pin_memory() if v.numel() > 1 else v.cpu()
        h_iv = torch.empty(n, dtype=torch.float64).pin_memory()
        h_st = torch.empty(n, dtype=torch.int8).pin_memory()
        h_px = torch.empty(n, dtype=torch.float64).pin_memory() if roundtrip else None
        h_g = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(6)] if method < 0 else []
        hn = native_cols(hcols, last)
        h2d = sum(hcols[k].numel() * hcols[k].element_size()
                  for k in ("flag", "underlying", "strike", "t", "r", "q", last)
                  if hcols[k].numel() > 1)
        d2h = n * (17 if roundtrip else (9 if method >= 0 else 49))   # (price +) iv + status | price + 5 Greeks + status

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
        if pg:
            pg.barrier()
        times = []
        for _ in range(max(2, min(args.steps, 5))):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            estep()
            times.append(time.perf_counter() - t0)
        e_ms = 1e3 * float(np.mean(times))
        if pg:
            tt = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            pg.all_reduce(tt, op=pg.ReduceOp.MAX)
            e_ms = float(tt.item())
        # bit-identical to the device-resident result
        if method >= 0:
            same = bool(torch.equal(h_iv.to(dev).view(torch.int64), out_iv.view(torch.int64)))
            if roundtrip:
                same = same and bool(torch.equal(h_px.to(dev).view(torch.int64), out_px.view(torch.int64)))
        else:
            same = all(bool(torch.equal(h.to(dev).view(torch.int64), g.view(torch.int64)))
                       for h, g in zip(h_g, greeks))
        # the link's own ceiling: a plain pinned 1 GB host->device copy
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
        e2e = {"value": world * n / (e_ms * 1e-3), "unit": "quotes/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms,
               "timing": "wall clock around the synchronous C-ABI call (host buffers pinned)",
               "bit_identical_to_device_resident": same,
               "pcie_h2d_gbs": h2d_gbs,
               "h2d_ceiling_quotes_s": (world * n * h2d_gbs * 1e9 / h2d) if h2d_gbs and h2d else None}

    # ---- roofline ------------------------------------------------------------
    peak = ctypes_double()
    secs = ctypes_double()
    lib.fv_probe_fp64_peak(ctypes_addr(peak), ctypes_addr(secs))
    peak_tops = peak.value / 1e12
    per_gpu_qps = n / (float(np.mean(per_call_ms)) * 1e-3)
    achieved = W_OPS[args.workload] * per_gpu_qps / 1e12
    in_bytes = sum(cols[k].numel() * cols[k].element_size()
                   for k in ("flag", "underlying", "strike", "t", "r", "q", last)
                   if torch.is_tensor(cols[k]) and cols[k].numel() > 1)
    out_bytes = n * (17 if roundtrip else (9 if method >= 0 else 49))
    hbm_gbs = (in_bytes + out_bytes) / (float(np.mean(per_call_ms)) * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # DRAM bytes (read + write) per launch of the call, from the committed
    # `ncu --set full` capture (profiles/roofline_traffic.json: bytes per
    # quote summed over the call's kernels) scaled to this launch's rows
    traffic = None
    try:
        prof = json.load(open(os.path.join(REPO, "profiles", "roofline_traffic.json")))
        bpq = prof.get(args.workload, {}).get("dram_bytes_per_quote")
        traffic = bpq * n if bpq else None
    except (OSError, ValueError, AttributeError):
        pass

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            try:
                cpu = cpu_baseline(args.cpu_seconds, args.workload)
            except Exception as exc:  # noqa: BLE001
                cpu = {"error": repr(exc)}
        wl_name = {"c4": "C4: jackel_iv_black (LBR) on a 100M-quote Black-76 chain "
                         "(2 flags x 1000 maturities x 50000 strikes) per GPU",
                   "c1": "C1: LBR Black-76 1M synthetic quotes",
                   "c2": "C2: Halley BSM with dividend yield, 10M quotes",
                   "c3": "C3: fused BSM price + all Greeks, 10M quotes",
                   "c5": "C5: wing-stress set, LBR Black-76",
                   "rt": "RT: the reference bench harness's round trip (bench.py:19-40) on 10M C2 draws: "
                         "BSM price -> Halley IV in one fused fv_price_iv call"}[args.workload]
        line = {
            "metric": METRIC if args.workload == "c4" else f"fp64 quotes/sec ({args.workload})",
            "value": value, "unit": "quotes/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded chain generated on device; prices from the pricing kernel)",
            "config": {"workload": wl_name, "rows_per_gpu": n, "parallelism": f"quote-sharded x{world}",
                       "l2": "inputs (%.1f GB/step) exceed the 126 MB L2; no flush needed" % (in_bytes / 1e9)},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak_tops,
                         "unit": "T weighted-fp64-ops/s", "frac": achieved / peak_tops if peak_tops else None,
                         "traffic": traffic,
                         "note": "kernel = one fv_batch_iv/fv_price_greeks call (its kernels in sequence on one "
                                 "stream); achieved = W=%.0f weighted distinct fp64 ops/quote (SURVEY 8(d)) x rows per "
                                 "call / mean call duration (CUDA events on the launching stream); peak = measured "
                                 "DFMA issue rate (fv_probe_fp64_peak, this run); traffic = ncu DRAM read+write bytes "
                                 "per call (profiles/roofline_traffic.json)" % W_OPS[args.workload]
                                 + ("; C2: the bracket pass decides f(10)'s sign in fp32 instead of evaluating "
                                    "it (~8 % of W counted but not executed)" if args.workload == "c2" else "")},
            "kernels": kernels,
            "kernels_note": "CUDA events around each launch on its own stream; the LBR far-low branch and the "
                            "Halley careful pass over the bracket's hand-backs run on a second stream beside the "
                            "other passes, so those kernels' times overlap and shares are of the summed time",
            "dominant_kernel": (dict(dominant, peak=peak_tops, unit="T weighted-fp64-ops/s",
                                     frac=dominant["achieved"] / peak_tops if peak_tops else None)
                                if dominant else None),
            "roofline_hbm": {"bound": "hbm", "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                             "frac": hbm_gbs / hbm_peak, "bytes_per_quote": (in_bytes + out_bytes) / n,
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches[0],
            "clocks": clk,
            "status_counts": dict(zip(["converged", "fell_back", "below_intrinsic", "above_upper",
                                       "max_iterations"], st)),
            "per_call_ms": per_call_ms,
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
