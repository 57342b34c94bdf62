#!/usr/bin/env python3
"""Strong-scaling prediction on a 1-GPU pool:
time every shard of a G-way split of the 100M-quote C4 chain on this one GPU,
for G = 2, 4, 8 and the contiguous and 1M-row block-cyclic schemes.  With no
exchange between shards, a G-GPU run takes max over shards of these times, so

    predicted strong-scaling efficiency(G) = T(whole chain) / (G * max_g T_g)
    imbalance(G) = max_g T_g / mean_g T_g - 1

Each shard: inputs built on the device (bench.c4_device), one warm-up call,
then K timed fv_batch_iv calls (CUDA events on the launching stream).

    python tools/shard_times.py [--steps K] [--out profiles/rN_shard_times.json]
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--workload", default="c4", choices=["c4", "c2"])
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "shard_times.json"))
    args = ap.parse_args()
    import torch
    import bench
    import workloads as W
    from paper_2604_27210_b200 import _native
    lib = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    lib.fv_set_stream(stream.cuda_stream)
    model, method, _ = bench.workload_call(args.workload)
    n_total = W.C4_ROWS if args.workload == "c4" else 10_000_000

    def time_ranges(ranges):
        if args.workload == "c4":
            cols = bench.c4_device(0, 0, dev, ranges=ranges, n_total=n_total, F=100.0)
        else:
            cols = bench.draws_device("c2", n_total, 0, dev, ranges)
            cols.pop("kind"), cols.pop("side")
        n = cols["flag"].numel()
        cols["price"] = bench.price_on_device(lib, model, cols, n)
        iv = torch.empty(n, dtype=torch.float64, device=dev)
        st = torch.empty(n, dtype=torch.int8, device=dev)
        nc = bench.native_cols(cols, "price")
        err = _native.fv_error()

        def call():
            rc = lib.fv_batch_iv(model, method, *nc, n, iv.data_ptr(), st.data_ptr(), None, err)
            assert rc == 0, err.message
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            call()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        counts = torch.bincount(st.to(torch.int64), minlength=5).cpu().tolist()
        del cols, iv, st
        torch.cuda.empty_cache()
        return ms, n, counts

    whole_ms, _, _ = time_ranges([(0, n_total)])
    out = {"workload": args.workload, "rows": n_total, "steps": args.steps, "whole_ms": whole_ms,
           "gpu": torch.cuda.get_device_name(0), "splits": {}}
    print(f"whole chain: {whole_ms:.3f} ms")
    for scheme in ("contiguous", "cyclic"):
        for G in (2, 4, 8):
            shards = []
            for g in range(G):
                ms, n, counts = time_ranges(bench.shard_ranges(n_total, G, g, scheme))
                shards.append({"shard": g, "rows": n, "ms": ms, "status_counts": counts})
            t = [s["ms"] for s in shards]
            rec = {"shards": shards, "max_ms": max(t), "min_ms": min(t), "mean_ms": sum(t) / G,
                   "imbalance": max(t) / (sum(t) / G) - 1.0,
                   "predicted_efficiency": whole_ms / (G * max(t)),
                   "predicted_quotes_per_s": n_total / (max(t) * 1e-3)}
            out["splits"][f"{scheme}_{G}"] = rec
            print(f"{scheme:10s} G={G}: max {max(t):.3f} min {min(t):.3f} ms, imbalance {rec['imbalance'] * 100:.1f} %, "
                  f"predicted efficiency {rec['predicted_efficiency'] * 100:.1f} %, "
                  f"{rec['predicted_quotes_per_s'] / 1e9:.2f} G quotes/s")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
