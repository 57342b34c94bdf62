#!/usr/bin/env python3
"""Workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the library on small batches -- LBR and
Halley IV (all passes: normalize, replay, anchors, far-low / near / far-high
solves on three streams; bracket / iter / bisect / careful), price, Greeks,
fused price + Greeks, the price -> IV round trip, host-pointer (chunked,
3-slot pipeline) and device-pointer calls, odd sizes around the warp and claim
granularities, wing rows that take the careful replay paths, host calls split
over two shards, and device shards + gather.  Each result is checked against
the oracle so a sanitizer run also proves the instrumented run computed the
right thing.

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch
    import bench
    import workloads as W
    from oracle import fvoracle as O
    from paper_2604_27210_b200 import _native
    from paper_2604_27210_b200 import distributed as D
    lib = _native.lib_for_compute()
    O.lib()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
    lib.fv_set_chunk_rows(4096)                # several chunks through the host pipeline
    checked = 0

    def same(a, b):
        a = np.asarray(a)
        b = np.asarray(b)
        if a.dtype == np.float64:
            return bool(((a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))).all())
        return bool((a.astype(np.int64) == b.astype(np.int64)).all())

    # C2-like draws + C5 wing rows (careful replays, boundary prices)
    f1, S1, K1, t1, r1, q1, s1 = W.chain_draws(6000, seed=3)
    f5, F5, K5, t5, r5, s5, kind, side = W.c5_params(6000, seed=5)
    p5 = O.rows_price("black", f5, F5, K5, t5, r5, 0.0, s5)["price"]
    p5 = W.c5_prices(f5, F5, K5, t5, r5, kind, side, p5)
    sets = [("bsm", 2, f1, S1, K1, t1, r1, q1, s1, None),
            ("black", 0, f5, F5, K5, t5, r5, np.zeros_like(F5), s5, p5)]
    for mname, mcode, fl, un, k, t, r, q, sg, px in sets:
        if px is None:
            px = O.rows_price(mname, fl, un, k, t, r, q, sg)["price"]
        for n in (1, 33, 257, 4097, len(fl)):
            cols_h = [np.ascontiguousarray(c[:n]) for c in (fl, un, k, t, r, q)]
            for method, mc in (("lbr", 1), ("halley", 0)):
                want = O.rows_iv(mname, method, *cols_h, px[:n])
                for device in (False, True):
                    cols = cols_h + [np.ascontiguousarray(px[:n])]
                    if device:
                        cols = [torch.from_numpy(c).to(dev) for c in cols]
                        iv = torch.empty(n, dtype=torch.float64, device=dev)
                        st = torch.empty(n, dtype=torch.int8, device=dev)
                        reg = torch.empty(n, dtype=torch.int8, device=dev)
                    else:
                        iv, st, reg = np.empty(n), np.empty(n, np.int8), np.empty(n, np.int8)
                    err = _native.fv_error()
                    rc = lib.fv_batch_iv(mcode, mc, *[_native.col(c) for c in cols], n, _native.ptr(iv),
                                         _native.ptr(st), _native.ptr(reg), err)
                    assert rc == 0, err.message
                    ivn = iv.cpu().numpy() if device else iv
                    stn = st.cpu().numpy() if device else st
                    assert same(ivn, want["iv"]) and same(stn, want["status_code"]), (mname, method, n, device)
                    checked += n
            # price, Greeks, fused, round trip (device)
            dc = [torch.from_numpy(c).to(dev) for c in cols_h] + [torch.from_numpy(np.ascontiguousarray(sg[:n])).to(dev)]
            outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
            st = torch.empty(n, dtype=torch.int8, device=dev)
            ep, eg = _native.fv_error(), _native.fv_error()
            assert lib.fv_price_greeks(mcode, *[_native.col(c) for c in dc], n, *[o.data_ptr() for o in outs],
                                       st.data_ptr(), ep, eg) in (0, 2)
            g = O.rows_greeks(mname, *cols_h, sg[:n])
            if not g["exc"].any():
                assert same(outs[1].cpu().numpy(), g["delta"]) and same(outs[5].cpu().numpy(), g["vega"])
            pxo = torch.empty(n, dtype=torch.float64, device=dev)
            assert lib.fv_batch_price(mcode, *[_native.col(c) for c in dc], n, pxo.data_ptr(), ep) == 0
            ivo = torch.empty(n, dtype=torch.float64, device=dev)
            ei = _native.fv_error()
            rc = lib.fv_price_iv(mcode, 0, *[_native.col(c) for c in dc], n, pxo.data_ptr(), ivo.data_ptr(),
                                 st.data_ptr(), None, ep, ei)
            assert rc in (0, 2)
            checked += n
    # run-length transport: piecewise-constant host columns (flag, S, t, r, q,
    # sigma) shipped as runs and rebuilt by k_expand_runs, three chunks
    lib.fv_set_chunk_rows(20_000)
    n = 60_000
    fl = np.where(np.arange(n) < 30_000, 1, -1).astype(np.int8)
    S, r, q = np.full(n, 100.0), np.full(n, 0.01), np.zeros(n)
    t = np.repeat([0.25, 0.5, 1.0], 20_000)
    K = 100.0 * np.exp(np.linspace(-0.3, 0.3, n))
    sg = np.repeat([0.2, 0.35], 30_000)
    px = O.rows_price("bsm", fl, S, K, t, r, q, sg)["price"]
    want = O.rows_iv("bsm", "lbr", fl, S, K, t, r, q, px)
    iv, st = np.empty(n), np.empty(n, np.int8)
    err = _native.fv_error()
    assert lib.fv_batch_iv(2, 1, *[_native.col(c) for c in (fl, S, K, t, r, q, px)], n, iv.ctypes.data,
                           st.ctypes.data, None, err) == 0, err.message
    assert same(iv, want["iv"]) and same(st, want["status_code"])
    assert lib.fv_last_h2d_bytes() < n * 17, lib.fv_last_h2d_bytes()      # K and price whole, the rest as runs
    checked += n
    # host call split into shards; device shards + gather
    _native.set_devices((0, 0))
    lib.fv_set_chunk_rows(1 << 20)
    try:
        n = 2_200_000
        fl, S, K, t, r, q, sg = W.chain_draws(n, seed=8)
        px = O.rows_price("bsm", fl, S, K, t, r, q, sg)["price"]
        iv, st = np.empty(n), np.empty(n, np.int8)
        err = _native.fv_error()
        assert lib.fv_batch_iv(2, 1, *[_native.col(np.ascontiguousarray(c)) for c in (fl, S, K, t, r, q, px)], n,
                               iv.ctypes.data, st.ctypes.data, None, err) == 0
    finally:
        _native.set_devices(())
    cols = {"flag": torch.from_numpy(f1).to(dev), "underlying": torch.from_numpy(S1).to(dev),
            "strike": torch.from_numpy(K1).to(dev), "t": torch.from_numpy(t1).to(dev),
            "r": torch.from_numpy(r1).to(dev), "q": torch.from_numpy(q1).to(dev)}
    cols["price"] = bench.price_on_device(lib, 2, dict(cols, sigma=torch.from_numpy(s1).to(dev)), len(f1))
    shards = [{k: v[a:b].clone() for k, v in cols.items()} for a, b in ((0, 2500), (2500, len(f1)))]
    outs, rc, e1, e2 = D.run_device_shards(_native.FV_KIND_IV, "bsm", "halley", shards)
    assert rc == 0
    full = D.gather_device([o["iv"] for o in outs], dev)
    want = O.rows_iv("bsm", "halley", f1, S1, K1, t1, r1, q1, cols["price"].cpu().numpy())
    assert same(full.cpu().numpy(), want["iv"])
    torch.cuda.synchronize()
    print(f"sanitize workload ok: {checked} rows checked against the oracle")


if __name__ == "__main__":
    main()
