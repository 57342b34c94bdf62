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
with gloo); ``batch_iv_sharded`` binds it to the CUDA C ABI.
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
    fails.  Returns (outputs, (stage, outcome) | None)."""
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
    if gather and world > 1 and outcome is None:
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
