"""Quote-sharded execution across GPUs (one process per GPU, torch.distributed).

Every output row of the reference batch is a pure function of its input row
(batch.py:4-7), so a chain shards by contiguous row ranges with no exchange
on the data path.  The only cross-rank traffic is
  * one small all-reduce (MIN) of each shard's first-failure rows, so every
    rank raises exactly the error the single-process reference would
    (validation checks in the reference's order first, then the lowest
    raising row -- batch.py:104-148, :166-178), and
  * optionally, an all-gather of the result shards when the caller asks for
    the whole result on every rank (NCCL over NVLink / NVSwitch).

``run_sharded`` holds the merge logic and is backend-agnostic (tested on CPU
with gloo); ``batch_iv_sharded`` binds it to the CUDA C ABI.  ``gather_to``
brings the shards to ONE rank only (point-to-point sends, NCCL over NVLink /
NVSwitch on a GPU box) when the caller asks for the result on one device.

Inside one process, ``run_device_shards`` drives several GPUs from one call
(``fv_run_shards``: one host thread per device-resident shard, outcome merged
in C) and ``gather_device`` copies the shards' results into one device's
memory (``fv_gather``: peer copies over NVLink).
"""

import numpy as np

NCHECK = 12
NO_ROW = np.iinfo(np.int64).max


def shard_bounds(n, world, rank):
    """Contiguous shard [lo, hi) of n rows for ``rank`` of ``world`` (the
    first n % world ranks get one extra row)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def _status_vector(check_rows, exc_row, exc_code, offset):
    """Local outcome -> global keys: per-check first global row, then the
    first raising global row packed with its code (row * 256 + code)."""
    v = np.full(NCHECK + 1, NO_ROW, dtype=np.int64)
    for c in range(NCHECK):
        if check_rows[c] >= 0:
            v[c] = offset + int(check_rows[c])
    if exc_row >= 0:
        v[NCHECK] = (offset + int(exc_row)) * 256 + int(exc_code)
    return v


def merge_status(vec):
    """Global outcome from the MIN-reduced status vector:
    ('batch', check, row) | ('exc', code, row) | None."""
    for c in range(NCHECK):
        if vec[c] != NO_ROW:
            return ("batch", c, int(vec[c]))
    if vec[NCHECK] != NO_ROW:
        return ("exc", int(vec[NCHECK] % 256), int(vec[NCHECK] // 256))
    return None


def gather_to(shard, n, dst=0, group=None):
    """The full n-row result on rank ``dst`` only (None elsewhere): rank r's
    ``shard`` holds rows shard_bounds(n, world, r).  Point-to-point: every
    other rank sends its shard once (NCCL: over NVLink / NVSwitch), so the
    traffic is the gathered bytes, not world x them as an all-gather."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    t = shard if torch.is_tensor(shard) else torch.from_numpy(np.ascontiguousarray(shard))
    if world == 1:
        return t
    if rank != dst:
        dist.send(t.contiguous(), dst=dist.get_global_rank(group, dst) if group is not None else dst,
                  group=group)
        return None
    full = torch.empty(n, dtype=t.dtype, device=t.device)
    reqs = []
    for r in range(world):
        lo, hi = shard_bounds(n, world, r)
        if r == rank:
            full[lo:hi] = t
        elif hi > lo:
            src = dist.get_global_rank(group, r) if group is not None else r
            reqs.append(dist.irecv(full[lo:hi], src=src, group=group))
    for q in reqs:
        q.wait()
    return full


def run_sharded(compute, n, group=None, device=None, gather=False):
    """Run ``compute(lo, hi) -> (outputs: dict of 1-D arrays/tensors,
    check_rows[12], exc_row, exc_code)`` on this rank's shard, agree on the
    global outcome with one MIN all-reduce, and optionally all-gather the
    outputs.  Returns (outputs, outcome) where outputs are this rank's shard
    (or the full arrays with ``gather=True``)."""
    def one_stage(lo, hi):
        outputs, check_rows, exc_row, exc_code = compute(lo, hi)
        return outputs, [(check_rows, exc_row, exc_code)]
    outputs, staged = run_sharded_stages(one_stage, n, 1, group=group, device=device, gather=gather)
    return outputs, (staged[1] if staged else None)


def run_sharded_stages(compute, n, nstage, group=None, device=None, gather=False):
    """``run_sharded`` for a call made of ``nstage`` stages run in sequence by
    the reference, each with its own checks and exception stream (fv_price_iv:
    batch_price, then batch_iv on its prices).  ``compute(lo, hi) ->
    (outputs, [(check_rows[12], exc_row, exc_code)] * nstage)``.  One MIN
    all-reduce over the stages' status vectors; the first stage with an
    outcome anywhere decides, as the reference raises in the first call that
    fails.  ``gather``: False (each rank keeps its shard), True / "all" (every
    rank gets the full arrays: all-gather), or an int rank (only that rank
    gets them, ``gather_to``; the others get None).  Returns (outputs,
    (stage, outcome) | None)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(n, world, rank)
    outputs, stages = compute(lo, hi)
    assert len(stages) == nstage
    vec = torch.from_numpy(np.concatenate([_status_vector(cr, er, ec, lo) for cr, er, ec in stages]))
    if device is not None:
        vec = vec.to(device)
    if world > 1:
        dist.all_reduce(vec, op=dist.ReduceOp.MIN, group=group)
    v = vec.cpu().numpy()
    outcome = None
    for s in range(nstage):
        o = merge_status(v[s * (NCHECK + 1):(s + 1) * (NCHECK + 1)])
        if o is not None:
            outcome = (s, o)
            break
    if gather is not False and gather is not None and not isinstance(gather, bool) and gather != "all" \
            and world > 1 and outcome is None:
        dst = int(gather)
        outputs = {name: gather_to(shard if device is None or not torch.is_tensor(shard) else shard.to(device),
                                   n, dst=dst, group=group)
                   for name, shard in outputs.items()}
        if rank != dst:
            outputs = None
    elif gather and world > 1 and outcome is None:
        full = {}
        for name, shard in outputs.items():
            t = shard if torch.is_tensor(shard) else torch.from_numpy(np.ascontiguousarray(shard))
            if device is not None:
                t = t.to(device)
            sizes = [shard_bounds(n, world, r)[1] - shard_bounds(n, world, r)[0] for r in range(world)]
            m = max(sizes)
            padded = torch.zeros(m, dtype=t.dtype, device=t.device)
            padded[:t.numel()] = t
            parts = [torch.empty(m, dtype=t.dtype, device=t.device) for _ in sizes]
            dist.all_gather(parts, padded, group=group)        # equal-size collective
            full[name] = torch.cat([p[:sz] for p, sz in zip(parts, sizes)])
        outputs = full
    return outputs, outcome


def batch_iv_sharded(model, method, cols, n, group=None, gather=False):
    """Sharded ``batch_iv`` on device-resident torch columns (each rank holds
    the full logical columns or at least its shard's rows; broadcast
    columns are 1-element tensors).  Returns ((iv, status) or gathered
    dict, outcome) -- outcome as in ``merge_status``."""
    import torch
    from . import _native
    from .models import as_model
    lib = _native.lib_for_compute()
    m = as_model(model).code
    dev = cols["strike"].device

    def compute(lo, hi):
        sl = {k: (v if v.numel() == 1 else v[lo:hi]) for k, v in cols.items()}
        k = hi - lo
        iv = torch.empty(k, dtype=torch.float64, device=dev)
        st = torch.empty(k, dtype=torch.int8, device=dev)
        err = _native.fv_error()
        with _native.device_scope(lib, dev):
            rc = lib.fv_batch_iv(m, 1 if method == "lbr" else 0,
                                 *[_native.col(sl[c]) for c in ("flag", "underlying", "strike", "t", "r", "q",
                                                               "price")],
                                 k, iv.data_ptr(), st.data_ptr(), None, err)
        _native.check_runtime(rc, err)
        cr, er, ec = _native.last_outcome(lib)
        return {"iv": iv, "status": st}, cr, int(er[0]), int(ec[0])

    return run_sharded(compute, n, group=group, device=dev, gather=gather)


def price_iv_sharded(model, method, cols, n, group=None, gather=False):
    """Sharded ``price_iv`` (fv_price_iv) on device-resident torch columns
    (``sigma`` instead of ``price``).  Returns ((price, iv, status) or the
    gathered dict, (stage, outcome) | None) with stage 0 = batch_price, 1 =
    batch_iv: the price stage's failure on any shard is the call's."""
    import torch
    from . import _native
    from .models import as_model
    lib = _native.lib_for_compute()
    m = as_model(model).code
    dev = cols["strike"].device
    none = np.full(NCHECK, -1, np.int64)

    def compute(lo, hi):
        sl = {k: (v if v.numel() == 1 else v[lo:hi]) for k, v in cols.items()}
        k = hi - lo
        px = torch.empty(k, dtype=torch.float64, device=dev)
        iv = torch.empty(k, dtype=torch.float64, device=dev)
        st = torch.empty(k, dtype=torch.int8, device=dev)
        ep, ei = _native.fv_error(), _native.fv_error()
        with _native.device_scope(lib, dev):
            rc = lib.fv_price_iv(m, 1 if method == "lbr" else 0,
                                 *[_native.col(sl[c]) for c in ("flag", "underlying", "strike", "t", "r", "q",
                                                               "sigma")],
                                 k, px.data_ptr(), iv.data_ptr(), st.data_ptr(), None, ep, ei)
        _native.check_runtime(rc, ep)
        cr, er, ec = _native.last_outcome(lib)
        price_checks = ep.code == _native.FV_ERR_BATCH      # fv_last_outcome: the deciding stage's rows
        stages = [(cr if price_checks else none, int(er[0]), int(ec[0])),
                  (none if price_checks else cr, int(er[1]), int(ec[1]))]
        return {"price": px, "iv": iv, "status": st}, stages

    return run_sharded_stages(compute, n, 2, group=group, device=dev, gather=gather)


# ---------------------------------------------------------------------------
# several GPUs from one process (fv_run_shards / fv_gather)
# ---------------------------------------------------------------------------
_KIND_LAST = {0: "sigma", 1: "price", 2: "sigma", 3: "sigma", 4: "sigma"}


def run_device_shards(kind, model, method, shards):
    """One logical batch whose row ranges live on several devices (``shards``:
    list, in row order, of dicts of device-resident torch columns -- flag,
    underlying, strike, t, r, q and sigma | price -- all on one device each).
    Runs every shard on its own device from its own host thread (one
    ``fv_run_shards`` call), on each device's current torch stream.  Returns
    (per-shard output dicts, rc, err1, err2): outputs are allocated on each
    shard's device; rc / err1 / err2 as the single-device entry point (the
    merged outcome in GLOBAL rows; ``_native.last_outcome`` likewise)."""
    import torch
    from . import _native
    from .models import as_model
    lib = _native.lib_for_compute()
    m = as_model(model).code
    last = _KIND_LAST[kind]
    arr = (_native.fv_shard * len(shards))()
    outs = []
    for g, cols in enumerate(shards):
        dev = cols["strike"].device
        n = cols["flag"].numel() if cols["flag"].numel() > 1 else max(
            c.numel() for c in cols.values())
        sh = arr[g]
        sh.device = dev.index
        sh.stream = torch.cuda.current_stream(dev).cuda_stream
        for i, k in enumerate(("flag", "underlying", "strike", "t", "r", "q", last)):
            sh.cols[i] = _native.col(cols[k])
        sh.n = n
        o = {}
        if kind in (_native.FV_KIND_PRICE, _native.FV_KIND_PRICE_GREEKS, _native.FV_KIND_PRICE_IV):
            o["price"] = torch.empty(n, dtype=torch.float64, device=dev)
        if kind in (_native.FV_KIND_IV, _native.FV_KIND_PRICE_IV):
            o["iv"] = torch.empty(n, dtype=torch.float64, device=dev)
        if kind in (_native.FV_KIND_GREEKS, _native.FV_KIND_PRICE_GREEKS):
            for name in ("delta", "gamma", "theta", "rho", "vega"):
                o[name] = torch.empty(n, dtype=torch.float64, device=dev)
        if kind != _native.FV_KIND_PRICE:
            o["status"] = torch.empty(n, dtype=torch.int8, device=dev)
        slots = {"price": 0, "delta": 1, "gamma": 2, "theta": 3, "rho": 4, "vega": 5}
        if kind == _native.FV_KIND_IV:
            slots = {"iv": 0}
        elif kind == _native.FV_KIND_PRICE_IV:
            slots = {"price": 0, "iv": 1}
        for name, j in slots.items():
            if name in o:
                sh.outs[j] = o[name].data_ptr()
        if "status" in o:
            sh.status = o["status"].data_ptr()
        outs.append(o)
    e1, e2 = _native.fv_error(), _native.fv_error()
    rc = lib.fv_run_shards(kind, m, 1 if method == "lbr" else 0, len(shards), arr, e1, e2)
    _native.check_runtime(rc, e1)
    return outs, rc, e1, e2


def gather_device(tensors, dst_device):
    """Concatenate per-device 1-D tensors (in order) into one tensor on
    ``dst_device`` with peer copies (``fv_gather``: NVLink / NVSwitch P2P)."""
    import ctypes
    import torch
    from . import _native
    lib = _native.lib_for_compute()
    dst_device = torch.device(dst_device)
    dtype = tensors[0].dtype
    n = sum(t.numel() for t in tensors)
    out = torch.empty(n, dtype=dtype, device=dst_device)
    k = len(tensors)
    src = (ctypes.c_void_p * k)(*[t.data_ptr() for t in tensors])
    sdev = (ctypes.c_int * k)(*[t.device.index for t in tensors])
    nb = (ctypes.c_int64 * k)(*[t.numel() * t.element_size() for t in tensors])
    for t in tensors:                     # the shards' producers are done before the copies start
        torch.cuda.current_stream(t.device).synchronize()
    rc = lib.fv_gather(out.data_ptr(), dst_device.index, torch.cuda.current_stream(dst_device).cuda_stream,
                       k, src, sdev, nb)
    if rc:
        raise _native.NativeCallError(f"fv_gather failed (rc={rc})")
    return out
