// fv_kernels.cu -- sm_100a kernels + the C ABI (include/fastvol_b200.h) for
// the batched pricing / Greeks / implied-vol path.
//
// Execution model (one quote = one unit of independent fp64 work, one quote
// per thread, no tensor cores -- the path is scalar fp64 transcendentals):
//   * every hot pass runs the straight-line routines of fv_fast.h (main paths
//     of the glibc / scipy restatements, branch-free, with range flags); a
//     quote they flag is recomputed from scratch by the careful routines of
//     fv_quote.h -- through a replay queue (LBR passes, Halley) or an
//     out-of-line careful row (pricing, anchors) -- so results never depend
//     on which path ran;
//   * LBR: normalize + first anchor (k_lbr_normalize: a 16-byte pair of rows
//     per thread), remaining anchors only for non-far-low quotes
//     (k_lbr_anchors), then region-uniform solves over dense row queues
//     (k_lbr_far_low_fast, k_lbr_near_fast, k_lbr_solve<FAR_HIGH>); work is
//     handed out per warp by atomic counters (dynamic load balance);
//   * Halley: a setup pass, then a persistent per-lane state machine with
//     refill whose shared step is one black_kernel evaluation (its two CDFs
//     through a warp's range-bucketed erfc);
//   * pricing / Greeks: one row per thread, 8-byte coalesced column access;
//   * the reference's batch validation (batch.py:104-124, :144-147) is fused
//     into the first pass: each row's failed checks go to a per-check
//     atomicMin, so the first failing row per check comes out of the same HBM
//     read that feeds the solver; rows whose reference execution would raise
//     a Python exception publish (row << 8 | code) through one atomicMin --
//     the lowest raising row wins, exactly as _run_chunked surfaces it
//     (batch.py:166-178);
//   * host-pointer calls stream through chunked H2D -> kernels -> D2H on
//     NSLOT streams (pageable buffers via pinned staging with threaded host
//     copies) so copies overlap compute.
// All arithmetic is bit-faithful to the reference; compile with -fmad=false.
#include <cuda_runtime.h>
#include <sched.h>
#include <stdint.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "fv_fast.h"
#include "../../include/fastvol_b200.h"

#define FV_VERSION "fastvol_b200 0.1.0 (sm_100a)"
// tuning knobs (occupancy hints; see profiles/README.md for the sweep)
#ifndef FV_SOLVE_MINB
#define FV_SOLVE_MINB 4
#endif
#ifndef FV_ANCH_MINB
#define FV_ANCH_MINB 3
#endif
#ifndef FV_NORM_CLAIM
#define FV_NORM_CLAIM 128
#endif
#ifndef FV_NORM_MINB
#define FV_NORM_MINB 3
#endif
#ifndef FV_NORM_MINB_BIG
#define FV_NORM_MINB_BIG 4
#endif
#ifndef FV_NORM_BIG_ROWS
#define FV_NORM_BIG_ROWS (1 << 23)
#endif
#ifndef FV_PG_MINB
#define FV_PG_MINB 3
#endif
#ifndef FV_FAST_MINB
#define FV_FAST_MINB 4
#endif
#define FV_NSLOT 3

// ---------------------------------------------------------------------------
// device-side column access
// ---------------------------------------------------------------------------
struct DCol {
  const double* p;
  int64_t stride;
  int mode;  // 0 broadcast, 1 contiguous + 16B aligned (double2), 2 generic strided
};
struct DFlag {
  const int8_t* p;
  int64_t stride;
  int mode;  // 0 broadcast, 1 contiguous + 2B aligned (char2), 2 generic
};

__device__ __forceinline__ void ld2(const DCol& c, int64_t i, bool two, double& a, double& b) {
  if (c.mode == 0) {
    a = __ldg(c.p);
    b = a;
  } else if (c.mode == 1 && two) {
    double2 v = __ldg(reinterpret_cast<const double2*>(c.p + i));
    a = v.x;
    b = v.y;
  } else {
    a = __ldg(c.p + i * c.stride);
    b = two ? __ldg(c.p + (i + 1) * c.stride) : 0.0;
  }
}
__device__ __forceinline__ void ldf2(const DFlag& c, int64_t i, bool two, int& a, int& b) {
  if (c.mode == 0) {
    a = c.p[0];
    b = a;
  } else if (c.mode == 1 && two) {
    char2 v = *reinterpret_cast<const char2*>(c.p + i);
    a = v.x;
    b = v.y;
  } else {
    a = c.p[i * c.stride];
    b = two ? c.p[(i + 1) * c.stride] : 0;
  }
}
// ---------------------------------------------------------------------------
// status block shared by all kernels of one call
// ---------------------------------------------------------------------------
struct FvDevStatus {
  unsigned long long check_first[FV_NCHECK];
  unsigned long long exc_first;    // (row << 8) | code: price / iv / greeks
  unsigned long long exc2_first;   // second stream (fused greeks)
  unsigned long long pad[2];
};

struct KArgs {
  int model;
  int has_sigma;       // last column is sigma (price/greeks) rather than price (iv)
  uint32_t check_mask; // checks evaluated per row (broadcast columns are host-checked)
  DFlag flag;
  DCol un, k, t, r, q, last;
  int64_t n;           // rows in this launch
  int64_t row0;        // global index of local row 0
  double* o0;          // price | iv
  double* o1;          // delta
  double* o2;          // gamma
  double* o3;          // theta
  double* o4;          // rho
  double* o5;          // vega
  int8_t* status;
  int8_t* region;
  FvDevStatus* st;
};

__device__ __forceinline__ uint32_t row_checks(const KArgs& a, int fl, double un, double k,
                                               double t, double r, double q, double last) {
  uint32_t b = 0;
  b |= (uint32_t)(fl != 1 && fl != -1) << FV_CHECK_BAD_FLAG;
  b |= (uint32_t)(!fv_isfinite(un)) << FV_CHECK_NONFINITE_UNDERLYING;
  b |= (uint32_t)(!fv_isfinite(k)) << FV_CHECK_NONFINITE_STRIKE;
  b |= (uint32_t)(!fv_isfinite(t)) << FV_CHECK_NONFINITE_T;
  b |= (uint32_t)(!fv_isfinite(r)) << FV_CHECK_NONFINITE_R;
  b |= (uint32_t)(!fv_isfinite(q)) << FV_CHECK_NONFINITE_Q;
  b |= (uint32_t)(!fv_isfinite(last)) << FV_CHECK_NONFINITE_LAST;
  b |= (uint32_t)(!(un > 0.0)) << FV_CHECK_POSITIVE_UNDERLYING;
  b |= (uint32_t)(!(k > 0.0)) << FV_CHECK_POSITIVE_STRIKE;
  b |= (uint32_t)(t < 0.0) << FV_CHECK_NONNEG_T;
  b |= (uint32_t)(a.has_sigma && last < 0.0) << FV_CHECK_NONNEG_SIGMA;
  b |= (uint32_t)(a.model != FV_MODEL_BLACK_SCHOLES_MERTON && q != 0.0) << FV_CHECK_DIVIDEND;
  return b & a.check_mask;
}

__device__ __noinline__ void publish_checks(FvDevStatus* st, uint32_t bits, int64_t row) {
  while (bits) {
    int c = __ffs(bits) - 1;
    bits &= bits - 1;
    atomicMin(&st->check_first[c], (unsigned long long)row);
  }
}
__device__ __forceinline__ void publish_exc(unsigned long long* slot, int code, int64_t row) {
  if (code) atomicMin(slot, ((unsigned long long)row << 8) | (unsigned long long)code);
}

__device__ __forceinline__ double ld1(const DCol& c, int64_t i) {
  return c.mode == 0 ? __ldg(c.p) : __ldg(c.p + i * c.stride);
}
__device__ __forceinline__ int ldf1(const DFlag& c, int64_t i) {
  return c.mode == 0 ? c.p[0] : c.p[i * c.stride];
}

// Loads the pair (i, i+1) of every input column.
struct Pair {
  int fl[2];
  double un[2], k[2], t[2], r[2], q[2], last[2];
};
__device__ __forceinline__ void load_pair(const KArgs& a, int64_t i, bool two, Pair& p) {
  ldf2(a.flag, i, two, p.fl[0], p.fl[1]);
  ld2(a.un, i, two, p.un[0], p.un[1]);
  ld2(a.k, i, two, p.k[0], p.k[1]);
  ld2(a.t, i, two, p.t[0], p.t[1]);
  ld2(a.r, i, two, p.r[0], p.r[1]);
  ld2(a.q, i, two, p.q[0], p.q[1]);
  ld2(a.last, i, two, p.last[0], p.last[1]);
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// Careful rows (fv_quote.h) for the rows the straight-line forms flag; out of
// line so the kernels keep the fast path's small footprint.
__device__ __noinline__ double price_row_careful(const KArgs& a, int64_t row, int fl, double un, double k,
                                                 double t, double r, double q, double sig) {
  FvExc e = {0, 0, 0.0};
  const double v = fv_price_row(a.model, (double)fl, un, k, t, r, q, sig, e);
  publish_exc(&a.st->exc_first, e.code, a.row0 + row);
  return v;
}
template <bool kPrice, bool kGreeks>
__device__ __noinline__ FvGreeks price_greeks_row_careful(const KArgs& a, int64_t row, int fl, double un,
                                                          double k, double t, double r, double q, double sig) {
  FvExc ep = {0, 0, 0.0}, eg = {0, 0, 0.0};
  FvGreeks g = fv_price_greeks_row(a.model, (double)fl, un, k, t, r, q, sig, kPrice, kGreeks, ep, eg);
  if (kPrice) publish_exc(&a.st->exc_first, ep.code, a.row0 + row);
  if (kGreeks) publish_exc(&a.st->exc2_first, eg.code, a.row0 + row);
  return g;
}

// Pricing (batch_price): straight-line row (fx_price_row), careful row where
// it flags.  One row per thread: 8-byte loads and stores, 256 B per warp per
// column, fully coalesced.  (A 16-byte pair per thread held both rows' state
// across the row loop -- 128 registers, 16 warps/SM; one row per thread fits
// 80 registers and runs 19 % faster on C3, profiles/README.md.)
__global__ void __launch_bounds__(256, FV_PG_MINB) k_price(KArgs a) {
  __shared__ double sm_x[8][64], sm_r[8][64];      // range-bucketed erfc staging
  __shared__ unsigned char sm_f[8][64];
  const int wib = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nloop = (a.n + stride - 1) / stride;
  for (int64_t it = 0; it < nloop; ++it) {          // warp-uniform trip count (bucketed erfc)
    const int64_t r0 = it * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = r0 < a.n;
    const int64_t row = valid ? r0 : 0;
    const int fl = ldf1(a.flag, row);
    const double un = ld1(a.un, row), k = ld1(a.k, row), t = ld1(a.t, row), r = ld1(a.r, row);
    const double q = ld1(a.q, row), sg = ld1(a.last, row);
    const uint32_t bad = valid ? row_checks(a, fl, un, k, t, r, q, sg) : 0u;
    FxBad flagged;
    double v = fx_price_row(a.model, (double)fl, un, k, t, r, q, sg, flagged, valid && !bad,
                            sm_x[wib], sm_r[wib], sm_f[wib]);
    if (!valid) continue;
    if (bad) {
      publish_checks(a.st, bad, a.row0 + row);
      v = __builtin_nan("");
    } else if (flagged) {
      v = price_row_careful(a, row, fl, un, k, t, r, q, sg);
    }
    a.o0[row] = v;
  }
}

// Fused price + Greeks (batch_price and/or batch_greeks in one pass):
// straight-line row (fx_price_greeks_row), careful row where it flags.
// One row per thread (see k_price).
template <bool kPrice, bool kGreeks>
__global__ void __launch_bounds__(256, FV_PG_MINB) k_price_greeks(KArgs a) {
  __shared__ double sm_x[8][64], sm_r[8][64];      // range-bucketed erfc staging
  __shared__ unsigned char sm_f[8][64];
  const int wib = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nloop = (a.n + stride - 1) / stride;
  for (int64_t it = 0; it < nloop; ++it) {          // warp-uniform trip count
    const int64_t r0 = it * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = r0 < a.n;
    const int64_t row = valid ? r0 : 0;
    const int fl = ldf1(a.flag, row);
    const double un = ld1(a.un, row), k = ld1(a.k, row), t = ld1(a.t, row), r = ld1(a.r, row);
    const double q = ld1(a.q, row), sg = ld1(a.last, row);
    const uint32_t bad = valid ? row_checks(a, fl, un, k, t, r, q, sg) : 0u;
    FxBad flagged;
    FvGreeks g = fx_price_greeks_row(a.model, (double)fl, un, k, t, r, q, sg, kGreeks, flagged,
                                     valid && !bad, sm_x[wib], sm_r[wib], sm_f[wib]);
    if (!valid) continue;
    if (bad) {
      publish_checks(a.st, bad, a.row0 + row);
      g.price = g.delta = g.gamma = g.theta = g.rho = g.vega = __builtin_nan("");
      g.status = 0;
    } else if (flagged) {
      g = price_greeks_row_careful<kPrice, kGreeks>(a, row, fl, un, k, t, r, q, sg);
    }
    if (kPrice) a.o0[row] = g.price;
    if (kGreeks) {
      a.o1[row] = g.delta; a.o2[row] = g.gamma; a.o3[row] = g.theta; a.o4[row] = g.rho; a.o5[row] = g.vega;
      if (a.status) a.status[row] = (int8_t)g.status;
    }
  }
}

// Programmatic dependent launch (FV_PDL): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in the
// stream is still running; it waits here -- griddepcontrol.wait returns once
// the predecessor grid has completed and its writes are visible -- before it
// reads anything the predecessor wrote.  Every kernel also lets its own
// dependents launch right away (launch_dependents): their CTAs fill the SM
// slots this grid's tail frees instead of waiting for the launch after it.
// Both are no-ops for kernels launched without the attribute.  The early
// trigger is off (FV_PDL_TRIGGER): dependents parked in the draining grid's
// freed slots measured slower (C2 -2.5 %, C5 -3.5 %); with the implicit
// trigger at completion the dependent launch is still prepared ahead (C1
// 3.405 -> 3.46, C5 12.17 -> 12.26, C2 3.305 -> 3.308 G quotes/s).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifndef FV_PDL_TRIGGER
#define FV_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_trigger() {
#if FV_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

__device__ __forceinline__ unsigned int warp_append(unsigned int* counter, bool want) {
  unsigned mask = __ballot_sync(0xffffffffu, want);
  unsigned int base = 0;
  int lane = threadIdx.x & 31;
  int leader = __ffs(mask) - 1;
  if (mask) {
    if (lane == leader) base = atomicAdd(counter, (unsigned int)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
  }
  return base + __popc(mask & ((1u << lane) - 1));
}

// LBR as classify + region-uniform solve passes.  k_lbr_classify normalizes
// every quote, finishes the ones that need no iteration (bounds, ATM,
// exceptions) and sorts the rest into three queues (far-low, near, far-high)
// with their anchors; each k_lbr_solve<R> then runs one region's guess +
// Householder(3) code over a dense queue, so warps are region-uniform and
// each kernel's instruction footprint stays small.
struct LbrQueues {
  // per-local-row state, structure of arrays (each pass writes / reads whole
  // 32-byte sectors of the fields it touches)
  // sqrt(t) and s_c = sqrt(2|x|) are not stored: the solves recompute them
  // (one sqrt each, the same IEEE expression) instead of a 16-byte write +
  // read per quote
  double* sx;      double* sbeta;
  double* sb0;     double* sb1;    double* sE0;     double* sE1;
  int32_t* q[7];         // 0..2: local rows per region class; 3: rows pending anchors;
                         // 4: far-low rows the straight-line solver handed back;
                         // 5: rows the straight-line normalize pass handed back;
                         // 6: near rows the straight-line near solver handed back
  unsigned int* count;   // [16]: queue lengths [0..6], work counters of the far-low
                         // solve [7], the normalize pass [8] and the near solve [9]
  unsigned int norm_claim;  // pairs per work claim of the normalize pass (32 | 64 | 128)
};

__device__ __forceinline__ int region_class(int region) {
  return region == FV_FAR_LOW ? 0 : (region == FV_FAR_HIGH ? 2 : 1);
}

// Warp-aggregated append of up to two entries per lane, in lane order
// (lane 0's two, lane 1's two, ...) so a queue segment follows row order.
__device__ __forceinline__ unsigned int warp_append2(unsigned int* counter, bool p0, bool p1) {
  const unsigned m0 = __ballot_sync(0xffffffffu, p0);
  const unsigned m1 = __ballot_sync(0xffffffffu, p1);
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  const unsigned total = __popc(m0) + __popc(m1);
  unsigned int base = 0;
  if (total) {
    if (lane == 0) base = atomicAdd(counter, total);
    base = __shfl_sync(0xffffffffu, base, 0);
  }
  return base + __popc(m0 & lt) + __popc(m1 & lt);
}

// One row of pass 1 on the careful routines (fv_quote.h): normalize_quote +
// bounds + ATM + the first anchor, outputs and state written, *far_low /
// *pending say which queue the row belongs in.  Validation is the caller's.
__device__ __forceinline__ void lbr_norm_row_careful(const KArgs& a, const LbrQueues& lq, int64_t row,
                                                     int fl, double un, double k, double t, double r,
                                                     double q, double px, bool* far_low_out,
                                                     bool* pending_out) {
  bool pending = false, far_low = false;
  double ivu = __builtin_nan("");
  int stu = FV_IV_MAX_ITER;
  FvLbrState st;
  st.x = 0.0; st.beta = 0.0; st.sqrt_t = 0.0; st.s_c = 0.0; st.b0 = 0.0; st.E0 = 0.0;
  FvExc e = {0, 0, 0.0};
  FvLbrOut o;
  o.sigma = __builtin_nan(""); o.status = FV_IV_MAX_ITER; o.region = -1; o.iterations = 0;
  double Fw = un;
  bool done = true;
  if (a.model != 0) Fw = un * py_exp((r - q) * t, e);     // batch.py:229
  if (e.code) {
  } else if (!(t > 0.0)) {
    o.status = FV_IV_BELOW_INTRINSIC;                      // batch.py:230-236
  } else {
    done = fv_lbr_normalize((double)fl, Fw, k, t, r, px, st, o, e) != 0;
  }
  if (!(done || e.code)) {
    const int cls = fv_lbr_anchor_lo(st, e);      // s_c, b_lo, far-low test
    if (cls < 0) { o.sigma = __builtin_nan(""); o.status = FV_IV_MAX_ITER; }
    else if (cls == FV_FAR_LOW) far_low = true;
    else pending = true;
  }
  publish_exc(&a.st->exc_first, e.code, a.row0 + row);
  if (!(far_low || pending)) {
    ivu = (o.status == FV_IV_CONVERGED) ? o.sigma : __builtin_nan("");
    stu = o.status;
  }
  if (far_low || pending) {
    lq.sx[row] = st.x; lq.sbeta[row] = st.beta;
    if (pending) { lq.sb0[row] = st.b0; lq.sE0[row] = st.E0; }   // read by pass 2
  } else {
    a.o0[row] = ivu;
    a.status[row] = (int8_t)stu;
  }
  if (a.region) a.region[row] = (int8_t)(far_low ? FV_FAR_LOW : -1);
  *far_low_out = far_low;
  *pending_out = pending;
}

// Pass 1: validation + normalize_quote + bounds + the first anchor (one pass
// over the input columns), on the straight-line routines (fv_fast.h).
// Finished quotes are written out; the rest get (x, beta, sqrt_t, s_c) in the
// state arrays and their row in the far-low queue (beta < b_lo: no further
// anchor is needed, see fv_lbr_anchor_lo) or in the pending queue with (b_lo,
// E_lo) for pass 2.  Rows the straight-line routines flag (ATM shortcut,
// exceptions, range edges) go to queue 5 for k_lbr_normalize_replay.
// MINB: blocks per SM the register budget is cut for.  Large batches run the
// 4-block form (64 registers, ~110 B of spills; C4 13.70 -> 13.61 ms), small
// ones the 3-block form (80 registers; C1 is latency-bound and 2.5 % slower
// at 4) -- see FV_NORM_BIG_ROWS.
#ifndef FV_NORM_DEFER_FL
#define FV_NORM_DEFER_FL 1
#endif
// One queue append for a whole normalize claim (warp-collective): bits =
// this lane's rows of the claim (bit 2 sub + u for row 2 (claim + 32 sub +
// lane) + u); entries in (sub, lane, u) order, row * mul each.
__device__ __forceinline__ void claim_append(unsigned bits, unsigned int* counter, int32_t* q, unsigned claim,
                                             int mul, int lane) {
  const unsigned lt = (1u << lane) - 1;
  unsigned m[8];
  unsigned total = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) { m[b] = __ballot_sync(0xffffffffu, (bits >> b) & 1u); total += __popc(m[b]); }
  if (!total) return;
  unsigned int base0 = 0;
  if (lane == 0) base0 = atomicAdd(counter, total);
  base0 = __shfl_sync(0xffffffffu, base0, 0);
  unsigned off = 0;
#pragma unroll
  for (int sb = 0; sb < 4; ++sb) {
    unsigned slot = base0 + off + __popc(m[2 * sb] & lt) + __popc(m[2 * sb + 1] & lt);
    const int64_t ii = 2 * ((int64_t)claim + 32 * sb + lane);
    if ((bits >> (2 * sb)) & 1u) q[slot++] = (int32_t)(mul * ii);
    if ((bits >> (2 * sb + 1)) & 1u) q[slot] = (int32_t)(mul * (ii + 1));
    off += __popc(m[2 * sb]) + __popc(m[2 * sb + 1]);
  }
}
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_lbr_normalize(KArgs a, LbrQueues lq) {
  pdl_wait();
  pdl_trigger();
  const int64_t npair = (a.n + 1) >> 1;
  const int lane = threadIdx.x & 31;
  // dynamic distribution: each warp takes the next 32 pairs (see
  // k_lbr_far_low_fast: per-row cost depends on the strike band)
  // (FV_NORM_CLAIM pairs per atomic, processed 32 at a time)
  for (;;) {
    unsigned int claim = 0;
    if (lane == 0) claim = atomicAdd(lq.count + 8, lq.norm_claim);
    claim = __shfl_sync(0xffffffffu, claim, 0);
    if ((int64_t)claim >= npair) break;
#if FV_NORM_DEFER_FL
    unsigned flbits = 0, pdbits = 0;   // far-low / pending rows of the claim: bit 2 sub + u
#endif
#pragma unroll 1
  for (int sub = 0; sub < (int)(lq.norm_claim / 32); ++sub) {
    const unsigned int base = claim + 32u * sub;
    if ((int64_t)base >= npair) break;
    const int64_t j = (int64_t)base + lane;
    const bool active = j < npair;
    const int64_t i = 2 * j;
    const bool two = active && (i + 1 < a.n);
    bool pend[2] = {false, false}, flow[2] = {false, false}, rep[2] = {false, false};
    Pair p;
    if (active) load_pair(a, i, two, p);
#pragma unroll 1
    for (int u = 0; u < 2; ++u) {
      const bool valid = active && (u == 0 || two);
      if (!valid) continue;
      const int64_t row = i + u;
      bool pending = false, far_low = false;
      FxBad flagged;
      double ivu = __builtin_nan("");
      int stu = FV_IV_MAX_ITER;
      FvLbrState st;
      st.x = 0.0; st.beta = 0.0; st.sqrt_t = 0.0; st.s_c = 0.0; st.b0 = 0.0; st.E0 = 0.0;
      const int fl = u ? p.fl[1] : p.fl[0];
      const double un = u ? p.un[1] : p.un[0], k = u ? p.k[1] : p.k[0];
      const double t = u ? p.t[1] : p.t[0], r = u ? p.r[1] : p.r[0];
      const double q = u ? p.q[1] : p.q[0], px = u ? p.last[1] : p.last[0];
      uint32_t badc = row_checks(a, fl, un, k, t, r, q, px);
      if (badc) {
        publish_checks(a.st, badc, a.row0 + row);
      } else {
        FvLbrOut o;
        const int cls = fx_lbr_classify_lo<MINB == FV_NORM_MINB_BIG>(a.model, (double)fl, un, k, t, r, q, px,
                                                                    st, o, flagged);
        if (!flagged) {
          if (cls == FV_FAR_LOW) far_low = true;
          else if (cls == FV_NEAR_LOW) pending = true;
          else { ivu = (o.status == FV_IV_CONVERGED) ? o.sigma : __builtin_nan(""); stu = o.status; }
        }
      }
      if (far_low || pending) {
        lq.sx[row] = st.x; lq.sbeta[row] = st.beta;
        if (pending) { lq.sb0[row] = st.b0; lq.sE0[row] = st.E0; }   // read by pass 2
      }
      // outputs of finished rows only: far-low / pending rows get theirs from
      // the solve that finishes them (one writer per row, no placeholder
      // write of 9 B per quote), flagged rows from the replay pass
      if (!(flagged || far_low || pending)) {
        a.o0[row] = ivu;
        a.status[row] = (int8_t)stu;
      }
      if (a.region && !flagged) a.region[row] = (int8_t)(far_low ? FV_FAR_LOW : -1);
      if (u) { pend[1] = pending; flow[1] = far_low; rep[1] = (bool)flagged; }
      else { pend[0] = pending; flow[0] = far_low; rep[0] = (bool)flagged; }
    }
    // queue appends in row order (lane 0's pair, lane 1's pair, ...); far-low
    // entries are 2 * row (the solve's entry format), the others plain rows
#if FV_NORM_DEFER_FL
    flbits |= ((unsigned)flow[0] | ((unsigned)flow[1] << 1)) << (2 * sub);
    pdbits |= ((unsigned)pend[0] | ((unsigned)pend[1] << 1)) << (2 * sub);
    unsigned int slot;
#else
    unsigned int slot = warp_append2(lq.count + 0, flow[0], flow[1]);
    if (flow[0]) { lq.q[0][slot++] = (int32_t)(2 * i); }
    if (flow[1]) { lq.q[0][slot] = (int32_t)(2 * (i + 1)); }
    slot = warp_append2(lq.count + 3, pend[0], pend[1]);
    if (pend[0]) { lq.q[3][slot++] = (int32_t)i; }
    if (pend[1]) { lq.q[3][slot] = (int32_t)(i + 1); }
#endif
    if (__any_sync(0xffffffffu, rep[0] || rep[1])) {
      slot = warp_append2(lq.count + 5, rep[0], rep[1]);
      if (rep[0]) { lq.q[5][slot++] = (int32_t)i; }
      if (rep[1]) { lq.q[5][slot] = (int32_t)(i + 1); }
    }
  }
#if FV_NORM_DEFER_FL
    // the claim's far-low and pending rows, one append each (one atomic ->
    // shfl -> store chain per claim instead of one per 32 pairs); far-low
    // entries are 2 * row (the solve's entry format), pending ones plain rows
    claim_append(flbits, lq.count + 0, lq.q[0], claim, 2, lane);
    claim_append(pdbits, lq.count + 3, lq.q[3], claim, 1, lane);
#endif
  }
}


// Pass 1b: the rows pass 1 flagged, on the careful routines.
__global__ void __launch_bounds__(256) k_lbr_normalize_replay(KArgs a, LbrQueues lq) {
  pdl_wait();
  pdl_trigger();
  const unsigned int n = lq.count[5];
  const unsigned int stride = gridDim.x * blockDim.x;
  const unsigned int nloop = (n + stride - 1) / stride;
  for (unsigned int it = 0; it < nloop; ++it) {
    const unsigned int j = it * stride + blockIdx.x * blockDim.x + threadIdx.x;
    bool far_low = false, pending = false;
    int32_t row = 0;
    if (j < n) {
      row = lq.q[5][j];
      lbr_norm_row_careful(a, lq, row, ldf1(a.flag, row), ld1(a.un, row), ld1(a.k, row), ld1(a.t, row),
                           ld1(a.r, row), ld1(a.q, row), ld1(a.last, row), &far_low, &pending);
    }
    unsigned int slot = warp_append(lq.count + 0, far_low);
    if (far_low) lq.q[0][slot] = 2 * row;
    slot = warp_append(lq.count + 3, pending);
    if (pending) lq.q[3][slot] = row;
  }
}

// Pass 2: the remaining anchors + region (fv_lbr_anchor_rest) over the
// pending queue (row order); appends each quote to its region class queue.
__device__ __noinline__ int anchor_rest_careful(FvLbrState& st, FvExc& e) { return fv_lbr_anchor_rest(st, e); }

__global__ void __launch_bounds__(256, FV_ANCH_MINB) k_lbr_anchors(KArgs a, LbrQueues lq) {
  pdl_wait();
  pdl_trigger();
  const unsigned int n = lq.count[3];
  const unsigned int stride = gridDim.x * blockDim.x;
  const unsigned int nloop = (n + stride - 1) / stride;
  for (unsigned int it = 0; it < nloop; ++it) {
    const unsigned int j = it * stride + blockIdx.x * blockDim.x + threadIdx.x;
    int cls = -1, region = -1;
    int32_t row = 0;
    FvLbrState st;
    if (j < n) {
      row = lq.q[3][j];
      st.x = lq.sx[row]; st.beta = lq.sbeta[row];
      { FvExc e0 = {0, 0, 0.0}; st.s_c = py_sqrt(2.0 * fv_fabs(st.x), e0); }
      st.b0 = lq.sb0[row]; st.E0 = lq.sE0[row];
      FvExc e = {0, 0, 0.0};
      FxBad flagged;
      FvLbrState sf = st;
      region = fx_lbr_anchor_rest(sf, flagged);            // straight-line form
      if (flagged) region = anchor_rest_careful(st, e);   // range edge: careful form
      else st = sf;
      if (region < 0) {
        publish_exc(&a.st->exc_first, e.code, a.row0 + row);
        a.o0[row] = __builtin_nan("");
        a.status[row] = (int8_t)FV_IV_MAX_ITER;
      } else {
        cls = region_class(region);
        if (region != FV_FAR_HIGH) {
          if (region == FV_NEAR_HIGH) { lq.sb0[row] = st.b0; lq.sE0[row] = st.E0; }
          lq.sb1[row] = st.b1; lq.sE1[row] = st.E1;
        }
      }
    }
#pragma unroll
    for (int c = 1; c < 3; ++c) {
      unsigned int slot = warp_append(lq.count + c, cls == c);
      // entry = local row * 2 + near-high bit (the near class holds both)
      if (cls == c) lq.q[c][slot] = (int32_t)(2 * row + (region == FV_NEAR_HIGH ? 1 : 0));
    }
    if (j < n && a.region && cls >= 0) a.region[row] = (int8_t)region;
  }
}

// Far-low solve on the straight-line fx_* routines (fv_fast.h) over queue 0;
// a quote that leaves their domain is appended to queue 4 for the careful
// solver (k_lbr_solve<FV_FAR_LOW>), which recomputes it from scratch.
__global__ void __launch_bounds__(256, FV_FAST_MINB) k_lbr_far_low_fast(KArgs a, LbrQueues lq) {
  pdl_wait();
  pdl_trigger();
  const unsigned int n = lq.count[0];
  const int32_t* q = lq.q[0];
  // dynamic distribution: each warp takes the next 32 queue entries (one
  // atomic per warp per 32 quotes).  A static grid stride hands each block a
  // fixed strike band of every stride window, and per-quote cost depends on
  // the strike, so blocks finished unevenly (ncu: 25 of 32 warps/SM active).
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned int base = 0;
    if (lane == 0) base = atomicAdd(lq.count + 7, 32u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    const unsigned int j = base + lane;
    FxBad bad;
    int32_t ent = 0;
    if (j < n) {
      ent = q[j];
      const int32_t row = ent >> 1;
      FvLbrState st;
      st.x = lq.sx[row]; st.beta = lq.sbeta[row];
      st.sqrt_t = fx_sqrt(ld1(a.t, row), bad);
      st.s_c = fx_sqrt(2.0 * fv_fabs(st.x), bad);
      st.b0 = st.b1 = st.E0 = st.E1 = 0.0;
      FvLbrOut o = fx_lbr_far_low(st, bad);
      if (!bad) {
        a.o0[row] = (o.status == FV_IV_CONVERGED) ? o.sigma : __builtin_nan("");
        a.status[row] = (int8_t)o.status;
      }
    }
    const unsigned int slot = warp_append(lq.count + 4, (bool)bad);
    if (bad) lq.q[4][slot] = ent;
  }
}

// Near-region solve on the straight-line routines (fx_lbr_near) over queue
// 1; a quote that leaves their domain goes to queue 6 for the careful solver.
__global__ void __launch_bounds__(256, FV_FAST_MINB) k_lbr_near_fast(KArgs a, LbrQueues lq) {
  pdl_wait();
  pdl_trigger();
  const unsigned int n = lq.count[1];
  const int32_t* q = lq.q[1];
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned int base = 0;
    if (lane == 0) base = atomicAdd(lq.count + 9, 32u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    const unsigned int j = base + lane;
    FxBad bad;
    int32_t ent = 0;
    if (j < n) {
      ent = q[j];
      const int32_t row = ent >> 1;
      FvLbrState st;
      st.x = lq.sx[row]; st.beta = lq.sbeta[row];
      st.sqrt_t = fx_sqrt(ld1(a.t, row), bad);
      st.s_c = fx_sqrt(2.0 * fv_fabs(st.x), bad);
      st.b0 = lq.sb0[row]; st.b1 = lq.sb1[row]; st.E0 = lq.sE0[row]; st.E1 = lq.sE1[row];
      FvLbrOut o = fx_lbr_near((ent & 1) ? FV_NEAR_HIGH : FV_NEAR_LOW, st, bad);
      if (!bad) {
        a.o0[row] = (o.status == FV_IV_CONVERGED) ? o.sigma : __builtin_nan("");
        a.status[row] = (int8_t)o.status;
      }
    }
    const unsigned int slot = warp_append(lq.count + 6, (bool)bad);
    if (bad) lq.q[6][slot] = ent;
  }
}

template <int R>
__global__ void __launch_bounds__(256, FV_SOLVE_MINB) k_lbr_solve(KArgs a, LbrQueues lq) {
  pdl_wait();
  pdl_trigger();
  // far-low: the careful solver over the quotes the straight-line one handed back
  // near: the careful solver over the quotes the straight-line one handed back
  const int c = R == FV_FAR_LOW ? 4 : (R == FV_FAR_HIGH ? 2 : 6);
  const unsigned int n = lq.count[c];
  const int32_t* q = lq.q[c];
  for (unsigned int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int32_t ent = q[j];
    const int32_t row = ent >> 1;
    FvLbrState st;
    st.x = lq.sx[row]; st.beta = lq.sbeta[row];
    st.sqrt_t = sqrt(ld1(a.t, row));
    { FvExc e0 = {0, 0, 0.0}; st.s_c = py_sqrt(2.0 * fv_fabs(st.x), e0); }
    if (R == FV_NEAR_LOW) { st.b0 = lq.sb0[row]; st.b1 = lq.sb1[row]; st.E0 = lq.sE0[row]; st.E1 = lq.sE1[row]; }
    else { st.b0 = st.b1 = st.E0 = st.E1 = 0.0; }
    const int region = (R == FV_NEAR_LOW) ? ((ent & 1) ? FV_NEAR_HIGH : FV_NEAR_LOW) : R;
    FvExc e = {0, 0, 0.0};
    FvLbrOut o = (R == FV_FAR_LOW) ? fv_lbr_far_low_fused(st, e) : fv_lbr_solve<R>(region, st, e);
    publish_exc(&a.st->exc_first, e.code, a.row0 + row);
    a.o0[row] = (o.status == FV_IV_CONVERGED) ? o.sigma : __builtin_nan("");
    a.status[row] = (int8_t)o.status;
  }
}

// ---- Halley + bisection (solver.py:49-161) in three passes ------------------
// The reference's sequence of f evaluations per quote is f(SIGMA_LO), f(hi)
// (doubling while negative), f(guess), up to 16 Halley steps (candidate, or
// the midpoint when the candidate leaves the bracket / does not improve), and
// for ~4 % of quotes a bisection tail of up to 128 steps.  The passes follow
// that shape so each one runs a short, nearly branch-free loop:
//   k_halley_bracket  one row per thread: validation + :60-86, then the three
//                     fixed evaluations f(SIGMA_LO), f(10), f(guess) (:91-112);
//                     quotes still open get a HalRec in a dense queue;
//   k_halley_iter     per-lane loop with refill over that queue: the Halley
//                     steps (:115-144); quotes reaching 16 steps are re-queued;
//   k_halley_bisect   per-lane loop with refill over the re-queued ones (:146-161);
//   k_halley_careful  a row per thread over the quotes any pass handed back:
//                     the whole careful solver from the inputs (fv_halley_row_sm).
// The fast passes evaluate f on the straight-line routines (range-bucketed
// erfc); anything they flag -- range edges, F/K <= 0, exceptions, the rare
// f(10) < 0 doubling -- is handed back, so every value is the careful
// solver's.
struct HalRec {            // 96 bytes, 16-byte aligned: a quote between passes
  double Fw, K, disc, sqrt_t, lnFK, target, tol, pad;
  double lo, hi, sigma, fval;
};
struct HalRecRow { int64_t rowbits; };   // row | (call << 62), parallel array

#define FV_HAL_CALL (1ll << 62)
// rowbits = row | k << 56 | midp << 61 | call << 62: the record also carries
// the Halley step count and the pending-midpoint flag of a quote whose first
// steps ran in the bracket pass (FV_HAL_BRACKET_TRIPS)
#define FV_HAL_ROWMASK ((1ll << 56) - 1)
#define FV_HAL_KSHIFT 56
#define FV_HAL_MIDP (1ll << 61)

// The record's spare slot (p[3].y) carries the row bits (row | call << 62):
// a refill then issues the record's six 16-byte loads straight after the
// claim, instead of a dependent load of a separate row array first (the
// refill's load -> test chain was the top stall of k_halley_iter).
// FV_HAL_RROW keeps the separate array (A/B).
__device__ __forceinline__ void hal_store(HalRec* r, const FvHalleyCtx& c, double lo, double hi,
                                          double sigma, double fval, int64_t rowbits) {
  double2* p = reinterpret_cast<double2*>(r);
  p[0] = make_double2(c.Fw, c.K);
  p[1] = make_double2(c.disc, c.sqrt_t);
  p[2] = make_double2(c.lnFK, c.target);
  p[3] = make_double2(c.tol_price, __longlong_as_double(rowbits));
  p[4] = make_double2(lo, hi);
  p[5] = make_double2(sigma, fval);
}
__device__ __forceinline__ void hal_load(const HalRec* r, FvHalleyCtx& c, double& lo, double& hi,
                                         double& sigma, double& fval, int64_t& rowbits) {
  const double2* p = reinterpret_cast<const double2*>(r);
  const double2 v0 = p[0], v1 = p[1], v2 = p[2], v3 = p[3], v4 = p[4], v5 = p[5];
  c.Fw = v0.x; c.K = v0.y; c.disc = v1.x; c.sqrt_t = v1.y; c.lnFK = v2.x; c.target = v2.y;
  c.tol_price = v3.x;
  rowbits = __double_as_longlong(v3.y);
  c.th = (rowbits & FV_HAL_CALL) ? 1.0 : -1.0;
  c.fk_bad = false;                        // such quotes never enter the queues
  lo = v4.x; hi = v4.y; sigma = v5.x; fval = v5.y;
}

// One trip of the Halley loop (solver.py:115-144) for the lanes with `busy`
// (warp-collective: all 32 lanes call it): the next evaluation point -- the
// Halley candidate, or the midpoint after a rejected candidate (`midp`) --
// f there, and the bracket / iterate update.  fin >= 0: the quote finished
// with that status at `sigma`; to_bis: the 16 Halley steps are spent
// (bisection next); hb: a straight-line routine flagged (careful pass).
// busy is cleared for all three.
__device__ __forceinline__ void hal_trip(bool& busy, bool& midp, int& k, const FvHalleyCtx& c, double& lo,
                                         double& hi, double& sigma, double& fval, int& fin, bool& to_bis,
                                         bool& hb, double* sm_x, double* sm_r, unsigned char* sm_f) {
  double x = 0.5 * (lo + hi);
  bool chk = false;
  hb = false;
  fin = -1;
  to_bis = false;
  if (busy && !midp) {
    FxBad vb;
    const double s = sigma * c.sqrt_t;
    double vega = 0.0, d1 = 0.0;
    if (!(s < FV_K_1EM12)) {
      d1 = fx_div0(c.lnFK + 0.5 * s * s, s, vb);
      vega = c.disc * c.Fw * fx_norm_pdf(d1, vb) * c.sqrt_t;
    }
    double cn = __builtin_nan("");
    if (vega > 0.0) {
      const double d2 = d1 - s;
      const double vomma = fx_div0(vega * d1 * d2, sigma, vb);
      const double denom = 2.0 * vega * vega - fval * vomma;
      if (denom != 0.0) cn = sigma - fx_div0(2.0 * fval * vega, denom, vb);
    }
    if (fv_isfinite(cn) && lo < cn && cn < hi) { x = cn; chk = true; }
    if (vb) hb = true;
  }
  if (hb) busy = false;
  __syncwarp();
  FxBad fb;
  const double fx = fx_halley_f_warp(busy, c, x, fb, sm_x, sm_r, sm_f);
  __syncwarp();
  if (busy && fb) { hb = true; busy = false; }
  if (busy) {
    if (chk && !(fv_fabs(fx) < fv_fabs(fval))) {          // :129-135: rejected -> f(mid) next
      midp = true;
    } else {                                               // :136-144
      midp = false;
      if (fx > 0.0) hi = x;
      else if (fx < 0.0) lo = x;
      const double step = x - sigma;
      sigma = x; fval = fx;
      if (fv_fabs(step) <= FV_K_1EM12 * py_max(1.0, sigma)) fin = FV_IV_CONVERGED;
      else if (++k == 16) to_bis = true;
      else if (fv_fabs(fval) <= c.tol_price) fin = FV_IV_CONVERGED;   // :116-117 of the next step
    }
  }
  if (fin >= 0 || to_bis) busy = false;
}

#ifndef FV_HAL_SIGN32
#define FV_HAL_SIGN32 1
#endif
// Halley trips run by the bracket pass itself, one row per thread, before a
// quote is queued: nearly every quote needs its first steps (C2: 99.3 % reach
// the loop, mode 3 steps), and here they run with all lanes of a warp busy and
// no claim / record reload, against ~24 of 32 lanes in the refill loop.
#ifndef FV_HAL_BRACKET_TRIPS
#define FV_HAL_BRACKET_TRIPS 0
#endif
#ifndef FV_HSET_MINB
#define FV_HSET_MINB 3
#endif
// kPrice (fv_price_iv): the row's price is computed here from the sigma
// column of the price stage's arguments `pa` (its checks, status block and
// price output) -- batch_price's row, straight-line with the careful row where
// it flags -- written out and inverted in the same thread, instead of a
// pricing kernel writing the column and this pass reading it back.
template <bool kPrice>
__global__ void __launch_bounds__(256, FV_HSET_MINB) k_halley_bracket(KArgs a, KArgs pa, HalRec* recs,
                                                                  int64_t* rrow, unsigned int* count,
                                                                  int32_t* hrow) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sm_x[8][64], sm_r[8][64];
  __shared__ unsigned char sm_f[8][64];
  const int wib = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nloop = (a.n + stride - 1) / stride;
  for (int64_t it = 0; it < nloop; ++it) {
    const int64_t row = it * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool active = row < a.n;
    double px_fused = 0.0;
    if (kPrice) {                                  // batch_price's row (warp-collective erfc)
      const int64_t prow = active ? row : 0;
      const int fl = ldf1(pa.flag, prow);
      const double un = ld1(pa.un, prow), k = ld1(pa.k, prow), t = ld1(pa.t, prow), r = ld1(pa.r, prow);
      const double q = ld1(pa.q, prow), sg = ld1(pa.last, prow);
      const uint32_t pbad = active ? row_checks(pa, fl, un, k, t, r, q, sg) : 0u;
      FxBad pflag;
      double v = fx_price_row(pa.model, (double)fl, un, k, t, r, q, sg, pflag, active && !pbad,
                              sm_x[wib], sm_r[wib], sm_f[wib]);
      __syncwarp();
      if (active) {
        if (pbad) {
          publish_checks(pa.st, pbad, pa.row0 + row);
          v = __builtin_nan("");
        } else if (pflag) {
          v = price_row_careful(pa, row, fl, un, k, t, r, q, sg);
        }
        pa.o0[row] = v;
      }
      px_fused = v;
    }
    bool open = false, hb = false;
    FvHalleySM m;
    m.c.th = 1.0; m.c.Fw = m.c.K = m.c.disc = m.c.sqrt_t = m.c.lnFK = m.c.target = m.c.tol_price = 0.0;
    m.c.fk_bad = false; m.guess = 0.0;
    if (active) {
      const int fl = ldf1(a.flag, row);
      const double un = ld1(a.un, row), k = ld1(a.k, row), t = ld1(a.t, row), r = ld1(a.r, row);
      const double q = ld1(a.q, row), px = kPrice ? px_fused : ld1(a.last, row);
      const uint32_t bad = row_checks(a, fl, un, k, t, r, q, px);
      if (bad) {
        publish_checks(a.st, bad, a.row0 + row);
        a.o0[row] = __builtin_nan("");
        a.status[row] = (int8_t)FV_IV_MAX_ITER;
      } else {
        FvExc e = {0, 0, 0.0};
        if (fv_hsm_setup(a.model, (double)fl, un, k, t, r, q, px, m, e)) {
          publish_exc(&a.st->exc_first, e.code, a.row0 + row);
          a.o0[row] = (m.status == FV_IV_CONVERGED || m.status == FV_IV_FELL_BACK) ? m.out_sigma : __builtin_nan("");
          a.status[row] = (int8_t)m.status;
        } else if (m.c.fk_bad) {
          hb = true;                                         // log(F/K) raises: careful pass
        } else {
          open = true;
        }
      }
      if (a.region) a.region[row] = -1;
    }
    // f(SIGMA_LO) (:91-96)
    __syncwarp();
    FxBad f1;
    const double flo = fx_halley_f_warp(open, m.c, FV_K_1EM9, f1, sm_x[wib], sm_r[wib], sm_f[wib]);
    __syncwarp();
    if (open && f1) { open = false; hb = true; }
    if (open && flo >= 0.0) {
      const bool conv = fv_fabs(flo) <= m.c.tol_price;
      a.o0[row] = conv ? FV_K_1EM9 : __builtin_nan("");
      a.status[row] = (int8_t)(conv ? FV_IV_CONVERGED : FV_IV_BELOW_INTRINSIC);
      open = false;
    }
    // f(10) (:97-102): only its sign is consumed -- fp32 with a rigorous margin
    // (fx_halley_sign); f(10) < 0 (doubling) and undecided signs are left to
    // the careful pass
#if FV_HAL_SIGN32
    if (open && fx_halley_sign(m.c, 10.0) <= 0) { open = false; hb = true; }
#else
    FxBad f2;
    const double fhi = fx_halley_f_warp(open, m.c, 10.0, f2, sm_x[wib], sm_r[wib], sm_f[wib]);
    __syncwarp();
    if (open && (f2 || fhi < 0.0)) { open = false; hb = true; }
#endif
    // f(guess) (:104-112)
    const double sigma = py_min(py_max(py_min(py_max(m.guess, FV_K_0P05), 2.0), FV_K_1EM9), 10.0);
    FxBad f3;
    const double fval = fx_halley_f_warp(open, m.c, sigma, f3, sm_x[wib], sm_r[wib], sm_f[wib]);
    __syncwarp();
    if (open && f3) { open = false; hb = true; }
    double lo = FV_K_1EM9, hi = 10.0;
    if (fval > 0.0) hi = py_min(hi, sigma);
    else if (fval < 0.0) lo = py_max(lo, sigma);
    if (open && fv_fabs(fval) <= m.c.tol_price) {            // :116-117 of the first step
      a.o0[row] = sigma;
      a.status[row] = (int8_t)FV_IV_CONVERGED;
      open = false;
    }
    // the first Halley trips, row per thread (all lanes call: f is warp-collective)
    double sg = sigma, fv = fval;
    int kst = 0;
    bool midp = false;
#pragma unroll 1
    for (int trip = 0; trip < FV_HAL_BRACKET_TRIPS; ++trip) {
      if (!__any_sync(0xffffffffu, open)) break;
      int fin;
      bool to_bis, hbt;
      hal_trip(open, midp, kst, m.c, lo, hi, sg, fv, fin, to_bis, hbt, sm_x[wib], sm_r[wib], sm_f[wib]);
      if (fin >= 0) {
        a.o0[row] = sg;
        a.status[row] = (int8_t)fin;
      }
      if (hbt) hb = true;
    }
    const unsigned int slot = warp_append(count, open);
    if (open) {
      const int64_t rb = row | (m.c.th > 0.0 ? FV_HAL_CALL : 0) | ((int64_t)kst << FV_HAL_KSHIFT) |
                         (midp ? FV_HAL_MIDP : 0);
      hal_store(recs + slot, m.c, lo, hi, sg, fv, rb);
#ifdef FV_HAL_RROW
      rrow[slot] = rb;
#endif
    }
    const unsigned int hs = warp_append(count + 1, hb);
    if (hb) hrow[hs] = (int32_t)row;
  }
}

// Warp-aggregated claim of queue entries for the lanes in `need`: returns the
// lane's entry index (>= n: queue exhausted).
__device__ __forceinline__ unsigned long long claim(bool need, unsigned long long* next, int lane) {
  const unsigned mask = __ballot_sync(0xffffffffu, need);
  unsigned long long base = 0;
  if (mask) {
    if (lane == __ffs(mask) - 1) base = atomicAdd(next, (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
  }
  return base + __popc(mask & ((1u << lane) - 1));
}

#ifndef FV_HSM_MINB
#define FV_HSM_MINB 3
#endif
#ifndef FV_HAL_PREFETCH
#define FV_HAL_PREFETCH 0
#endif

// One-record-ahead prefetch for the Halley passes' refill: each lane claims
// its NEXT record while it still works on the current one and copies it into
// its shared-memory slot with cp.async (16-byte, L2-only), so a lane whose
// quote finishes takes the next one from shared memory instead of waiting on
// the claim atomic and a dependent HBM load (the refill's load -> test chain
// was the top stall of k_halley_iter).
__device__ __forceinline__ void hal_prefetch(double* slot, const HalRec* r) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(slot);
  const char* g = reinterpret_cast<const char*>(r);
#pragma unroll
  for (int k = 0; k < 6; ++k)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa + 16 * k), "l"(g + 16 * k) : "memory");
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void hal_take(const double* slot, FvHalleyCtx& c, double& lo, double& hi, double& sigma,
                                         double& fval, int64_t& rowbits) {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  hal_load(reinterpret_cast<const HalRec*>(slot), c, lo, hi, sigma, fval, rowbits);
}
// Halley steps (:115-144) over the bracket pass's queue.  One f evaluation
// per loop trip: at the Halley candidate when it lies inside the bracket,
// else (and after a candidate that did not improve |f|) at the midpoint.
__global__ void __launch_bounds__(256, FV_HSM_MINB) k_halley_iter(KArgs a, HalRec* recs, const int64_t* rrow,
                                                              const unsigned int* count,
                                                              unsigned long long* next, int32_t* bis,
                                                              unsigned int* nbis, int32_t* hrow,
                                                              unsigned int* nhb) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const unsigned long long n = *count;
  __shared__ double sm_x[8][64], sm_r[8][64];
  __shared__ unsigned char sm_f[8][64];
  const int wib = threadIdx.x >> 5;
  FvHalleyCtx c;
  c.th = 1.0; c.Fw = c.K = c.disc = c.sqrt_t = c.lnFK = c.target = c.tol_price = 0.0; c.fk_bad = false;
  double lo = 0.0, hi = 0.0, sigma = 0.0, fval = 0.0;
  int k = 0;
  int64_t row = 0;
  int32_t rec = 0;
  bool busy = false, exhausted = false, midp = false;
#if FV_HAL_PREFETCH
  // 12 doubles of record + the record index per lane (14 x 8 B: the slot
  // holds the index too, so it does not occupy a register across the trip)
  __shared__ __align__(16) double sm_next[256 * 14];
  bool has_next = false;
#endif
  for (;;) {
#if FV_HAL_PREFETCH
    const bool need = !has_next && !exhausted;
    const unsigned long long jq = claim(need, next, lane);
    if (need) {
      if (jq >= n) {
        exhausted = true;
      } else {
        double* my_next = sm_next + 14 * threadIdx.x;   // 16-byte aligned 112-byte slot
        reinterpret_cast<int32_t*>(my_next + 12)[0] = (int32_t)jq;
        hal_prefetch(my_next, recs + jq);
        has_next = true;
      }
    }
    if (!busy && has_next) {
      const double* my_next = sm_next + 14 * threadIdx.x;
      rec = reinterpret_cast<const int32_t*>(my_next + 12)[0];
      int64_t rb;
      hal_take(my_next, c, lo, hi, sigma, fval, rb);
      row = rb & FV_HAL_ROWMASK;
      has_next = false;
      k = (int)((rb >> FV_HAL_KSHIFT) & 31);
      midp = (rb & FV_HAL_MIDP) != 0;
      busy = true;
    }
#else
    const bool need = !busy && !exhausted;
    const unsigned long long jq = claim(need, next, lane);
    if (need) {
      if (jq >= n) {
        exhausted = true;
      } else {
        rec = (int32_t)jq;
#ifdef FV_HAL_RROW
        const int64_t rb0 = rrow[rec];
        row = rb0 & FV_HAL_ROWMASK;
#endif
        int64_t rb;
        hal_load(recs + rec, c, lo, hi, sigma, fval, rb);
#ifndef FV_HAL_RROW
        row = rb & FV_HAL_ROWMASK;
#endif
        k = (int)((rb >> FV_HAL_KSHIFT) & 31);
        midp = (rb & FV_HAL_MIDP) != 0;
        busy = true;
      }
    }
#endif
#if FV_ERFC_CTA
    if (!__syncthreads_or(busy)) break;          // the block's warps share the erfc rounds
#else
    if (!__any_sync(0xffffffffu, busy)) break;
#endif
    int fin;
    bool to_bis, hb;
    hal_trip(busy, midp, k, c, lo, hi, sigma, fval, fin, to_bis, hb, sm_x[wib], sm_r[wib], sm_f[wib]);
    if (fin >= 0) {
      a.o0[row] = sigma;
      a.status[row] = (int8_t)fin;
    }
    if (to_bis) {
      double2* p = reinterpret_cast<double2*>(recs + rec);
      p[4] = make_double2(lo, hi);
      p[5] = make_double2(sigma, fval);
    }
    const unsigned int bs = warp_append(nbis, to_bis);
    if (to_bis) bis[bs] = rec;
    const unsigned int hs = warp_append(nhb, hb);
    if (hb) hrow[hs] = (int32_t)row;
  }
}

// Bisection tail (:146-161) over the quotes the Halley pass re-queued.
__global__ void __launch_bounds__(256, FV_HSM_MINB) k_halley_bisect(KArgs a, const HalRec* recs,
                                                                const int64_t* rrow, const int32_t* bis,
                                                                const unsigned int* nbis,
                                                                unsigned long long* next, int32_t* hrow,
                                                                unsigned int* nhb) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const unsigned long long n = *nbis;
  __shared__ double sm_x[8][64], sm_r[8][64];
  __shared__ unsigned char sm_f[8][64];
  const int wib = threadIdx.x >> 5;
  FvHalleyCtx c;
  c.th = 1.0; c.Fw = c.K = c.disc = c.sqrt_t = c.lnFK = c.target = c.tol_price = 0.0; c.fk_bad = false;
  double lo = 0.0, hi = 0.0, sigma = 0.0, fval = 0.0;
  int k = 0;
  int64_t row = 0;
  bool busy = false, exhausted = false;
  for (;;) {
    const bool need = !busy && !exhausted;
    const unsigned long long jq = claim(need, next, lane);
    if (need) {
      if (jq >= n) {
        exhausted = true;
      } else {
        const int32_t rec = bis[jq];
#ifdef FV_HAL_RROW
        const int64_t rb0 = rrow[rec];
        row = rb0 & FV_HAL_ROWMASK;
#endif
        int64_t rb;
        hal_load(recs + rec, c, lo, hi, sigma, fval, rb);
#ifndef FV_HAL_RROW
        row = rb & FV_HAL_ROWMASK;
#endif
        k = 0; busy = true;
      }
    }
#if FV_ERFC_CTA
    if (!__syncthreads_or(busy)) break;          // the block's warps share the erfc rounds
#else
    if (!__any_sync(0xffffffffu, busy)) break;
#endif
    if (busy && (fv_fabs(fval) <= c.tol_price || (hi - lo) <= FV_K_1EM12 * py_max(1.0, sigma))) {
      a.o0[row] = sigma;                                     // :147-149
      a.status[row] = (int8_t)FV_IV_FELL_BACK;
      busy = false;
    }
    const double x = 0.5 * (lo + hi);
    __syncwarp();
    FxBad fb;
    const double fx = fx_halley_f_warp(busy, c, x, fb, sm_x[wib], sm_r[wib], sm_f[wib]);
    __syncwarp();
    const bool hb = busy && fb;
    if (hb) busy = false;
    if (busy) {                                              // :150-157
      sigma = x; fval = fx;
      if (fx > 0.0) hi = x;
      else lo = x;
      if (++k == 128) {                                      // :158-161
        const bool ok = fv_fabs(fval) <= c.tol_price || (hi - lo) <= FV_K_1EM12 * py_max(1.0, sigma);
        a.o0[row] = ok ? sigma : __builtin_nan("");
        a.status[row] = (int8_t)(ok ? FV_IV_FELL_BACK : FV_IV_MAX_ITER);
        busy = false;
      }
    }
    const unsigned int hs = warp_append(nhb, hb);
    if (hb) hrow[hs] = (int32_t)row;
  }
}

// Handed-back quotes: the careful solver from the row's inputs.
__global__ void __launch_bounds__(256) k_halley_careful(KArgs a, const int32_t* hrow, const unsigned int* nhb) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = *nhb;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = hrow[j];
    const int fl = ldf1(a.flag, row);
    const double un = ld1(a.un, row), k = ld1(a.k, row), t = ld1(a.t, row), r = ld1(a.r, row);
    const double q = ld1(a.q, row), px = ld1(a.last, row);
    FvExc e = {0, 0, 0.0};
    int status;
    double sig;
    fv_halley_row_sm(a.model, (double)fl, un, k, t, r, q, px, &status, &sig, e);
    if (e.code) publish_exc(&a.st->exc_first, e.code, a.row0 + row);
    a.o0[row] = (status == FV_IV_CONVERGED || status == FV_IV_FELL_BACK) ? sig : __builtin_nan("");
    a.status[row] = (int8_t)status;
  }
}

// One-row re-run that records the full exception (value + numpy-ness) for
// DomainError messages that quote a value.
struct ExplainOut { int code; int np; double val; };
__global__ void k_explain(KArgs a, int method, int64_t local_row, ExplainOut* out) {
  Pair p;
  load_pair(a, local_row, false, p);
  FvExc e = {0, 0, 0.0};
  if (method == FV_METHOD_LBR) {
    fv_lbr_batch_row(a.model, (double)p.fl[0], p.un[0], p.k[0], p.t[0], p.r[0], p.q[0], p.last[0], e);
  } else {
    int status; double sig;
    fv_halley_row_sm(a.model, (double)p.fl[0], p.un[0], p.k[0], p.t[0], p.r[0], p.q[0], p.last[0],
                     &status, &sig, e);
  }
  out->code = e.code; out->np = e.np; out->val = e.val;
}

// FP64-pipe peak probe: 8 independent DFMA chains per thread (the roofline
// denominator for this FP64-bound path; MEASURED_PEAKS.json has no fp64 entry).
__global__ void __launch_bounds__(256) k_fp64_probe(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b);
      x3 = __fma_rn(x3, a, b); x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b);
      x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keep live
}

// Self-test: fv_div_const against the hardware IEEE division on the device
// for every constant divisor the path uses (random 64-bit patterns, biased
// to moderate exponents, plus the full range).
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void k_selftest_div_const(int64_t n, uint64_t seed, unsigned long long* bad) {
  const double cs[9] = {FV_DIV_SQRT2_C, 6.0, 120.0, 5040.0, 362880.0, 39916800.0, 6227020800.0, 365.0, 100.0};
  const double yh[9] = {FV_DIV_SQRT2_YH, FV_DIV_6_YH, FV_DIV_120_YH, FV_DIV_5040_YH, FV_DIV_362880_YH,
                        FV_DIV_39916800_YH, FV_DIV_6227020800_YH, FV_DIV_365_YH, FV_DIV_100_YH};
  const double yl[9] = {FV_DIV_SQRT2_YL, FV_DIV_6_YL, FV_DIV_120_YL, FV_DIV_5040_YL, FV_DIV_362880_YL,
                        FV_DIV_39916800_YL, FV_DIV_6227020800_YL, FV_DIV_365_YL, FV_DIV_100_YL};
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t u = splitmix64(seed + (uint64_t)i);
    uint64_t e = (i & 7) ? (uint64_t)(1023 + (int)((u >> 52) % 128) - 64) : ((u >> 52) & 0x7ff);
    uint64_t bits = (u & 0x800fffffffffffffull) | (e << 52);
    double x = __longlong_as_double((long long)bits);
#pragma unroll 1
    for (int k = 0; k < 9; ++k) {
      double a = fv_div_const(x, cs[k], yh[k], yl[k]);
      double b = __ddiv_rn(x, cs[k]);
      if (__double_as_longlong(a) != __double_as_longlong(b) && !(a != a && b != b)) ++local;
    }
  }
  if (local) atomicAdd(bad, local);
}

// fx_* (fv_fast.h) against the careful routines on random inputs; counts,
// per routine, unflagged mismatches and flagged inputs.
__device__ __forceinline__ double st_uniform(uint64_t u) { return (double)(u >> 11) * 0x1p-53; }
__device__ __forceinline__ double st_bits(uint64_t u, int e_lo, int e_hi) {
  // random sign-less mantissa, exponent uniform in [e_lo, e_hi]
  const int span = e_hi - e_lo + 1;
  const uint64_t e = (uint64_t)(1023 + e_lo + (int)((u >> 52) % (uint64_t)span));
  uint64_t m = u & 0x000fffffffffffffull;
  // every 8th input: mantissa near all-zeros / all-ones (division/rounding edges)
  if (((u >> 40) & 7) == 0) m = (u & 1) ? (0x000fffffffffffffull - ((u >> 1) & 0xff)) : ((u >> 1) & 0xff);
  return __longlong_as_double((long long)((e << 52) | m));
}
__device__ __forceinline__ bool st_same(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b) || (a != a && b != b);
}
#define FX_NTEST 11
__global__ void k_selftest_fast(int64_t n, uint64_t seed, unsigned long long* mism, unsigned long long* flg) {
  unsigned long long lm[FX_NTEST] = {}, lf[FX_NTEST] = {};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u1 = splitmix64(seed + 7919ull * (uint64_t)i);
    const uint64_t u2 = splitmix64(u1 ^ 0x9e3779b97f4a7c15ull);
    const uint64_t u3 = splitmix64(u2 + 12345ull);
    FxBad bad;
    // 0: a / b, exponents spanning the whole range (incl. slow-path ones)
    {
      const int wide = (int)(u3 & 3) == 0;
      double a = st_bits(u1, wide ? -1074 + 52 : -600, wide ? 1023 : 600);
      double b = st_bits(u2, wide ? -1022 : -600, wide ? 1023 : 600);
      if (u3 & 16) a = -a;
      if (u3 & 32) b = -b;
      bad = FxBad();
      const bool z = (u3 & 0xf00) == 0;             // 1/16: zero numerators through fx_div0
      if (z) a = (u3 & 16) ? -0.0 : 0.0;
      const double f = z ? fx_div0(a, b, bad) : fx_div(a, b, bad);
      if (bad) ++lf[0]; else if (!st_same(f, __ddiv_rn(a, b))) ++lm[0];
    }
    // 1: exp over [-800, 800] and tiny arguments
    {
      double x = ((u3 >> 8) & 3) ? (st_uniform(u1) * 1600.0 - 800.0) : st_bits(u1, -70, 10);
      if (u3 & 64) x = -x;
      bad = FxBad();
      const double f = fx_exp(x, bad);
      if (bad) ++lf[1]; else if (!st_same(f, fv_exp(x))) ++lm[1];
    }
    // 2: log of positives, half of them in [0.5, 2]
    {
      const double x = ((u3 >> 10) & 1) ? st_bits(u2, -1, 0) : st_bits(u2, -1000, 1000);
      bad = FxBad();
      const double f = fx_log(x, bad);
      if (bad) ++lf[2]; else if (!st_same(f, fv_log_i(x))) ++lm[2];
    }
    // 3: x ** n, n in {2, 3, 4}
    {
      const int nn = 2 + (int)((u3 >> 12) % 3);
      double x = ((u3 >> 14) & 1) ? st_bits(u1 ^ u2, -2, 1) : st_bits(u1 ^ u2, -300, 300);
      if (u3 & 128) x = -x;
      bad = FxBad();
      const double f = fx_powi(x, nn, bad);
      FvExc e = {0, 0, 0.0};
      if (bad) ++lf[3]; else if (!st_same(f, py_powi_t<true>(x, nn, false, e)) || e.code) ++lm[3];
    }
    // 4: erfcx over [0, 1e8] (log-uniform), [0, 60] (uniform) and tiny x
    //    (where 4 + x rounds to 4: erfcx's y100 == 100 branch)
    {
      const int sel = (int)((u3 >> 16) & 3);
      const double x = sel == 0 ? st_uniform(u2) * 60.0
                     : (sel == 1 ? st_bits(u2, -64, -30) : exp10(st_uniform(u2) * 11.0 - 3.0));
      bad = FxBad();
      const double f = fx_erfcx_pos(x, bad);
      if (bad) ++lf[4]; else if (!st_same(f, fv_erfcx_i(x))) ++lm[4];
    }
    // 5: normalized_black_log(h, s) on far-low-like arguments
    {
      const double s = exp10(st_uniform(u1) * 8.5 - 8.0);
      const double h = -exp10(st_uniform(u3) * 7.0 - 2.0);
      bad = FxBad();
      const double f = fx_nbl_h(h, s, bad);
      FvExc e = {0, 0, 0.0};
      const double c = fv_nbl_h<true>(h, s, e);
      if (bad) ++lf[5]; else if (!st_same(f, c) || e.code) ++lm[5];
    }
    // 6: x / sqrt(2) by the constant-division product
    {
      const double x = st_bits(u3, -1000, 1000);
      bad = FxBad();
      const double f = FX_DIV_SQRT2(x, bad);
      if (bad) ++lf[6]; else if (!st_same(f, __ddiv_rn(x, FV_DIV_SQRT2_C))) ++lm[6];
    }
    // 7: sqrt over the whole positive range (and some negatives)
    {
      double x = st_bits(u1 ^ u3, -1074 + 52, 1023);
      if ((u2 & 63) == 0) x = -x;
      bad = FxBad();
      const double f = fx_sqrt(x, bad);
      if (bad) ++lf[7]; else if (!st_same(f, __dsqrt_rn(x))) ++lm[7];
    }
    // 9: erfc over [-30, 30] (and a few wider)
    {
      double x = st_uniform(u1 ^ (u3 << 7)) * 60.0 - 30.0;
      if ((u2 & 15) == 0) x = st_bits(u2, -60, 8) * ((u2 & 16) ? -1.0 : 1.0);
      bad = FxBad();
      const double f = fx_erfc(x, bad);
      if (bad) ++lf[9]; else if (!st_same(f, fv_erfc(x))) ++lm[9];
    }
    // 10: erfcx over [-6.2, 60], tiny |x| (incl. +-0: y100 == 100) and wide x
    {
      const int sel = (int)((u3 >> 24) & 3);
      double x = sel == 0 ? st_uniform(u1) * 66.2 - 6.2
               : (sel == 1 ? st_bits(u1, -70, -30) : (sel == 2 ? 0.0 : exp10(st_uniform(u1) * 11.0 - 3.0)));
      if ((u3 >> 26) & 1) x = -x;
      bad = FxBad();
      const double f = fx_erfcx_any(x, bad);
      if (bad) ++lf[10]; else if (!st_same(f, fv_erfcx_i(x))) ++lm[10];
    }
    // 8: log, both paths (half of the inputs within 2^-4 of 1)
    {
      const double x = ((u3 >> 20) & 1) ? 1.0 + (st_uniform(u2) - 0.5) * 0.13 : st_bits(u2 ^ u3, -1000, 1000);
      bad = FxBad();
      const double f = fx_log_any(x, bad);
      if (bad) ++lf[8]; else if (!st_same(f, fv_log_i(x))) ++lm[8];
    }
  }
#pragma unroll
  for (int k = 0; k < FX_NTEST; ++k) {
    if (lm[k]) atomicAdd(mism + k, lm[k]);
    if (lf[k]) atomicAdd(flg + k, lf[k]);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

thread_local cudaStream_t t_user_stream = nullptr;
thread_local bool t_user_stream_set = false;   // fv_set_stream called (NULL = legacy default stream)
thread_local int64_t t_launches = 0;
thread_local int64_t t_h2d_bytes = 0;       // host calls: bytes this thread's last call moved host -> device
#ifndef FV_CALL_TRACE
#define FV_CALL_TRACE 0
#endif
#if FV_CALL_TRACE
thread_local std::chrono::steady_clock::time_point t_ct0;
thread_local double t_ct[16];
thread_local int t_ctn = 0;
#define CT_MARK() do { if (t_ctn < 16) t_ct[t_ctn++] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_ct0).count(); } while (0)
#else
#define CT_MARK() ((void)0)
#endif

// Optional per-kernel timing (fv_set_kernel_timing): CUDA events around every
// launch on the launching stream, summed per kernel by fv_kernel_times.
const char* const kKernelNames[FV_NKERNEL] = {
    "k_price", "k_price_greeks", "k_lbr_normalize", "k_lbr_normalize_replay", "k_lbr_anchors",
    "k_lbr_far_low_fast", "k_lbr_solve<FAR_LOW>", "k_lbr_solve<NEAR>", "k_lbr_solve<FAR_HIGH>",
    "k_halley_bracket", "k_halley_iter", "k_halley_careful", "k_lbr_near_fast", "k_halley_bisect"};
struct TimedLaunch { int id; cudaEvent_t a, b; };
thread_local bool t_timing = false;
// Device span of a device-pointer call (fv_set_span_timing): events around
// its launches on the call's stream, without serialising anything -- the
// difference to the caller's own per-call time is host overhead.
thread_local bool t_span = false;
thread_local float t_span_ms = -1.0f;
thread_local std::vector<TimedLaunch> t_timed;
inline void time_begin(int id, cudaStream_t s) {
  if (!t_timing) return;
  TimedLaunch tl;
  tl.id = id;
  cudaEventCreate(&tl.a);
  cudaEventCreate(&tl.b);
  cudaEventRecord(tl.a, s);
  t_timed.push_back(tl);
}
inline void time_end(cudaStream_t s) {
  if (!t_timing || t_timed.empty()) return;
  cudaEventRecord(t_timed.back().b, s);
}
#define FV_LAUNCH(id, s, ...) do { time_begin((id), (s)); __VA_ARGS__; time_end(s); ++t_launches; } while (0)
// A kernel launch with programmatic dependent launch (see pdl_wait): the
// kernel may begin while the previous kernel of its stream drains.  Off in the
// per-kernel timing mode (events must bracket each kernel alone).
#ifndef FV_PDL
#define FV_PDL 1
#endif
template <typename... Exp, typename... Act>
cudaError_t launch_pdl(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (FV_PDL && !t_timing) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}
// raw outcome of this thread's last call (for sharded callers that merge
// the first-failure rows of several shards)
thread_local int64_t t_check_rows[FV_NCHECK];
thread_local int64_t t_exc_row[2] = {-1, -1};
thread_local int32_t t_exc_code[2] = {0, 0};
int64_t g_chunk_rows = 1 << 22;

struct DevWork {
  int dev = -1;
  int sm_count = 0;
  cudaStream_t streams[FV_NSLOT] = {};
  // per slot: a second stream and fork / join events -- the LBR far-low
  // branch runs beside the anchors -> near -> far-high branch
  cudaStream_t aux[FV_NSLOT] = {}, aux2[FV_NSLOT] = {};
  cudaEvent_t fork_ev[FV_NSLOT] = {}, join_ev[FV_NSLOT] = {};
  cudaEvent_t fork2_ev[FV_NSLOT] = {}, join2_ev[FV_NSLOT] = {};   // LBR far-high solve
  FvDevStatus* st = nullptr;            // device, [2]: call (or price stage), IV stage of fv_price_iv
  FvDevStatus* st_host = nullptr;       // pinned mirror [2]
  bool st_armed = false;                // st holds the all-ones "nothing failed" state
  // chunk buffers for host-pointer calls
  char* chunk[FV_NSLOT] = {};
  int64_t chunk_cap_rows[FV_NSLOT] = {};
  char* stage[FV_NSLOT] = {};              // pinned host staging (pageable callers)
  int64_t stage_cap[FV_NSLOT] = {};
  char* rle_host[FV_NSLOT] = {};           // pinned: a chunk's column runs (run-length transport)
  char* rle_dev[FV_NSLOT] = {};
  int64_t rle_cap[FV_NSLOT] = {};
  ExplainOut* explain = nullptr;
  double* scal = nullptr;               // device copies of a host call's broadcast scalars
  // LBR classify -> solve workspace (per slot)
  double* lbr_state[FV_NSLOT] = {};     // 8 SoA fields x lbr_cap
  int32_t* lbr_q[FV_NSLOT] = {};        // 6 queues of lbr_cap entries each
  unsigned int* lbr_count = nullptr;    // [FV_NSLOT][8]
  int64_t lbr_cap[FV_NSLOT] = {};
  int blocks_price = 0, blocks_greeks = 0, blocks_hiter = 0, blocks_hbis = 0, blocks_hcare = 0;
  unsigned long long* work_ctr = nullptr;   // [FV_NSLOT][2]: Halley / bisection claims
  unsigned int* hsm_count = nullptr;        // [FV_NSLOT][4]: records, handed back, bisection queue
  HalRec* hsm_recs[FV_NSLOT] = {};
  int64_t* hsm_rrow[FV_NSLOT] = {};         // row | call bit per record
  int32_t* hsm_ridx[FV_NSLOT] = {};         // [cap] rows handed back by the bracket pass, [cap]
                                            // bisection queue, [cap] handed back later
  int64_t hsm_cap[FV_NSLOT] = {};
  int blocks_hset = 0, blocks_hset_p = 0;
  int blocks_lbr_nfast = 0;
  int blocks_lbr_norm_big = 0;
  int blocks_lbr_norm = 0, blocks_lbr_nrep = 0, blocks_lbr_anch = 0, blocks_lbr_fast = 0, blocks_lbr_fl = 0, blocks_lbr_near = 0, blocks_lbr_fh = 0;
  std::mutex mu;
};

std::mutex g_mu;
std::vector<DevWork*> g_work;

#define CK(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return _e; } while (0)

// The quick far-low table (fv_fast.h g_qlo_tab): one thread per bin.
__device__ double qlo_b_lo(double ax) {       // the exact first anchor at x = -ax
  FvExc e = {0, 0, 0.0};
  const double x = -ax;
  const double s_c = py_sqrt(2.0 * ax, e);
  double E = 0.0;
  return py_max(fv_normalized_black(x, s_c * 0.5, false, e, &E, nullptr), 0.0);
}
__global__ void k_qlo_table() {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= FV_QLO_NBIN) return;
  const int oct = k / FV_QLO_PER, m = k % FV_QLO_PER;
  const double base = ldexp(1.0, oct - 13);
  const double lo = base * (1.0 + (double)m / FV_QLO_PER), hi = base * (1.0 + (double)(m + 1) / FV_QLO_PER);
  double mn = 1e300;
  for (int j = 0; j <= 16; ++j) mn = fmin(mn, qlo_b_lo(lo + (hi - lo) * j / 16.0));
  const double D = 17.0 / 16.0 + 0.5 / lo;
  const double L = mn * exp(-D * (hi - lo) / 32.0) * (1.0 - 1e-4);
  g_qlo_tab[k] = (L > 0.0 && L == L) ? __double2float_rd(L) : 0.0f;
}
cudaError_t qlo_table_init() {
  k_qlo_table<<<(FV_QLO_NBIN + 127) / 128, 128>>>();
  return cudaDeviceSynchronize();
}
int occupancy_blocks(const void* fn, int sm) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
  if (per_sm < 1) per_sm = 1;
  return per_sm * sm;
}

cudaError_t get_work(DevWork** out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(g_mu);
  if ((int)g_work.size() <= dev) g_work.resize(dev + 1, nullptr);
  if (!g_work[dev]) {
    DevWork* w = new DevWork();
    w->dev = dev;
    CK(cudaDeviceGetAttribute(&w->sm_count, cudaDevAttrMultiProcessorCount, dev));
    for (int s = 0; s < FV_NSLOT; ++s) {
      CK(cudaStreamCreateWithFlags(&w->streams[s], cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&w->aux[s], cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&w->aux2[s], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&w->fork2_ev[s], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&w->join2_ev[s], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&w->fork_ev[s], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&w->join_ev[s], cudaEventDisableTiming));
    }
    CK(cudaMalloc(&w->st, 2 * sizeof(FvDevStatus)));
    CK(cudaMallocHost(&w->st_host, 2 * sizeof(FvDevStatus)));
    CK(cudaMalloc(&w->explain, sizeof(ExplainOut)));
    CK(cudaMalloc(&w->scal, 8 * sizeof(double)));
    w->blocks_price = occupancy_blocks((const void*)k_price, w->sm_count);
    w->blocks_greeks = occupancy_blocks((const void*)k_price_greeks<true, true>, w->sm_count);
    CK(cudaMalloc(&w->lbr_count, sizeof(unsigned int) * 16 * FV_NSLOT));
    w->blocks_lbr_norm = occupancy_blocks((const void*)k_lbr_normalize<FV_NORM_MINB>, w->sm_count);
    w->blocks_lbr_norm_big = occupancy_blocks((const void*)k_lbr_normalize<FV_NORM_MINB_BIG>, w->sm_count);
    w->blocks_lbr_nrep = occupancy_blocks((const void*)k_lbr_normalize_replay, w->sm_count);
    w->blocks_lbr_anch = occupancy_blocks((const void*)k_lbr_anchors, w->sm_count);
    w->blocks_lbr_fast = occupancy_blocks((const void*)k_lbr_far_low_fast, w->sm_count);
    w->blocks_lbr_fl = occupancy_blocks((const void*)k_lbr_solve<FV_FAR_LOW>, w->sm_count);
    w->blocks_lbr_near = occupancy_blocks((const void*)k_lbr_solve<FV_NEAR_LOW>, w->sm_count);
    w->blocks_lbr_nfast = occupancy_blocks((const void*)k_lbr_near_fast, w->sm_count);
    w->blocks_lbr_fh = occupancy_blocks((const void*)k_lbr_solve<FV_FAR_HIGH>, w->sm_count);
    w->blocks_hiter = occupancy_blocks((const void*)k_halley_iter, w->sm_count);
    w->blocks_hbis = occupancy_blocks((const void*)k_halley_bisect, w->sm_count);
    w->blocks_hcare = occupancy_blocks((const void*)k_halley_careful, w->sm_count);
    CK(cudaMalloc(&w->work_ctr, sizeof(unsigned long long) * 2 * FV_NSLOT));
    CK(cudaMalloc(&w->hsm_count, sizeof(unsigned int) * 4 * FV_NSLOT));
    w->blocks_hset = occupancy_blocks((const void*)k_halley_bracket<false>, w->sm_count);
    w->blocks_hset_p = occupancy_blocks((const void*)k_halley_bracket<true>, w->sm_count);
    CK(qlo_table_init());                     // the quick far-low bounds (fv_fast.h)
    g_work[dev] = w;
  }
  *out = g_work[dev];
  return cudaSuccess;
}


// rows per LBR classify/solve round.  The workspace is 64 B of state + 24 B
// of queues per row: 2^27 rows = 11.8 GB, a small slice of the B200's 180 GB,
// so a 100M-quote chain is one round (fewer kernel boundaries and tails than
// 2^25-row rounds, and one dynamic work pool per kernel).
#ifndef FV_LBR_ROUND_LOG2
#define FV_LBR_ROUND_LOG2 27
#endif
// Runtime-settable (fv_set_round_rows) so tests can force multi-round calls
// on small batches and check them against single-round ones.
int64_t g_lbr_round = 1ll << FV_LBR_ROUND_LOG2;
int64_t g_halley_round = 1ll << 26;

cudaError_t ensure_lbr(DevWork* w, int slot, int64_t rows) {
  if (w->lbr_cap[slot] >= rows) return cudaSuccess;
  if (w->lbr_state[slot]) cudaFree(w->lbr_state[slot]);
  if (w->lbr_q[slot]) cudaFree(w->lbr_q[slot]);
  w->lbr_state[slot] = nullptr;
  w->lbr_q[slot] = nullptr;
  w->lbr_cap[slot] = 0;
  int64_t cap = rows < 4096 ? 4096 : ((rows + 255) / 256) * 256;   // keeps every SoA field 16B-aligned
  CK(cudaMalloc(&w->lbr_state[slot], sizeof(double) * 6 * cap));
  CK(cudaMalloc(&w->lbr_q[slot], sizeof(int32_t) * 7 * cap));
  w->lbr_cap[slot] = cap;
  return cudaSuccess;
}

// Rows [off, off + len) of a launch as a launch of its own.
DCol dcol_at(DCol c, int64_t off) { if (c.mode != 0) c.p += off * c.stride; return c; }
DFlag dflag_at(DFlag c, int64_t off) { if (c.mode != 0) c.p += off * c.stride; return c; }
KArgs sub_args(const KArgs& a, int64_t off, int64_t len) {
  KArgs b = a;
  b.flag = dflag_at(a.flag, off);
  b.un = dcol_at(a.un, off); b.k = dcol_at(a.k, off); b.t = dcol_at(a.t, off);
  b.r = dcol_at(a.r, off); b.q = dcol_at(a.q, off); b.last = dcol_at(a.last, off);
  double** outs[6] = {&b.o0, &b.o1, &b.o2, &b.o3, &b.o4, &b.o5};
  for (double** o : outs) if (*o) *o += off;
  if (b.status) b.status += off;
  if (b.region) b.region += off;
  b.n = len;
  b.row0 = a.row0 + off;
  return b;
}

cudaError_t ensure_hsm(DevWork* w, int slot, int64_t rows) {
  if (w->hsm_cap[slot] >= rows) return cudaSuccess;
  if (w->hsm_recs[slot]) cudaFree(w->hsm_recs[slot]);
  if (w->hsm_rrow[slot]) cudaFree(w->hsm_rrow[slot]);
  if (w->hsm_ridx[slot]) cudaFree(w->hsm_ridx[slot]);
  w->hsm_recs[slot] = nullptr;
  w->hsm_rrow[slot] = nullptr;
  w->hsm_ridx[slot] = nullptr;
  w->hsm_cap[slot] = 0;
  int64_t cap = rows < 4096 ? 4096 : rows;
  CK(cudaMalloc(&w->hsm_recs[slot], sizeof(HalRec) * cap));
  CK(cudaMalloc(&w->hsm_rrow[slot], sizeof(int64_t) * cap));
  CK(cudaMalloc(&w->hsm_ridx[slot], sizeof(int32_t) * 3 * cap));
  w->hsm_cap[slot] = cap;
  return cudaSuccess;
}

enum Kind { KIND_PRICE, KIND_IV, KIND_GREEKS, KIND_PRICE_GREEKS, KIND_PRICE_IV };

struct Call {
  Kind kind;
  int model, method;
  fv_col cols[7];      // flag, under, strike, t, r, q, last
  int64_t n;
  double* outs[6];     // price|iv, delta, gamma, theta, rho, vega
  int8_t* status;
  int8_t* region;
  bool want_price, want_greeks;
  uint32_t bbits_iv;   // KIND_PRICE_IV: host-checked broadcast-column bits of the IV stage
  bool bcast_dev;      // device call: broadcast columns are checked by the kernels (row 0 wins)
};

// fv_price_iv's IV stage: batch_iv over the price column the price stage
// wrote (outs[0]), reading the same input columns; its own check mask (the
// IV checks: no sigma check, price never broadcast) and status block.
KArgs iv_stage_args(const KArgs& a, DevWork* w) {
  KArgs b = a;
  b.has_sigma = 0;
  b.check_mask = a.check_mask & ~((1u << FV_CHECK_NONNEG_SIGMA) | (1u << FV_CHECK_NONFINITE_LAST));
  b.check_mask |= 1u << FV_CHECK_NONFINITE_LAST;
  b.last.p = a.o0;
  b.last.stride = 1;
  b.last.mode = (((uintptr_t)a.o0) & 15) == 0 ? 1 : 2;
  b.o0 = a.o1;
  b.o1 = nullptr;
  b.st = w->st + 1;
  return b;
}

int64_t blocks_for(int64_t max_blocks, int64_t n) {
  int64_t need = ((n + 1) / 2 + 255) / 256;
  if (need < 1) need = 1;
  return need < max_blocks ? need : max_blocks;
}

// The IV passes of one launch (LBR or Halley) over rows [0, a.n).
cudaError_t launch_iv(DevWork* w, int method, const KArgs& a, int slot, cudaStream_t s,
                      const KArgs* price = nullptr) {
  if (a.n <= 0) return cudaSuccess;
  if (method == FV_METHOD_LBR) {
    const int64_t kLbrChunk = g_lbr_round;
    const int64_t chunk = a.n < kLbrChunk ? a.n : kLbrChunk;
    CK(ensure_lbr(w, slot, chunk));
    for (int64_t off = 0; off < a.n; off += chunk) {
      KArgs b = sub_args(a, off, (a.n - off) < chunk ? (a.n - off) : chunk);
      LbrQueues lq;
      double* sb = w->lbr_state[slot];
      const int64_t cp = w->lbr_cap[slot];
      lq.sx = sb; lq.sbeta = sb + cp;
      lq.sb0 = sb + 2 * cp; lq.sb1 = sb + 3 * cp; lq.sE0 = sb + 4 * cp; lq.sE1 = sb + 5 * cp;
      for (int c3 = 0; c3 < 7; ++c3) lq.q[c3] = w->lbr_q[slot] + c3 * w->lbr_cap[slot];
      lq.count = w->lbr_count + 16 * slot;
      // claims as large as FV_NORM_CLAIM pairs while every warp still gets
      // >= 4 of them: a small batch (C1: 1M rows = 141 pairs per warp) with
      // 128-pair claims leaves a tenth of the warps a second claim to run
      // alone after the rest are done
      {
        const int64_t npair = (b.n + 1) / 2, warps = (int64_t)w->blocks_lbr_norm * 8;
        unsigned cl = FV_NORM_CLAIM;
        while (cl > 32 && npair < warps * (int64_t)cl * 4) cl /= 2;
        lq.norm_claim = cl;
      }
      CK(cudaMemsetAsync(lq.count, 0, 16 * sizeof(unsigned int), s));
      const int64_t cap1 = (b.n + 255) / 256;
      auto g = [cap1](int blocks) { return (int)(cap1 < blocks ? cap1 : blocks); };
      if (b.n >= FV_NORM_BIG_ROWS)
        FV_LAUNCH(FV_KID_LBR_NORM, s, k_lbr_normalize<FV_NORM_MINB_BIG><<<blocks_for(w->blocks_lbr_norm_big, b.n), 256, 0, s>>>(b, lq));
      else
        FV_LAUNCH(FV_KID_LBR_NORM, s, k_lbr_normalize<FV_NORM_MINB><<<blocks_for(w->blocks_lbr_norm, b.n), 256, 0, s>>>(b, lq));
      // the three replay passes usually find an empty queue: one CTA per SM
      // keeps their launch + drain short (a full occupancy grid costs ~7 us)
      FV_LAUNCH(FV_KID_LBR_NREP, s, launch_pdl(k_lbr_normalize_replay, g(w->sm_count), 256, 0, s, b, lq));
      // Two independent branches after the normalize passes: the far-low
      // solve (queue 0 -> queue 4) and anchors -> near / far-high solves
      // (queue 3 -> queues 1, 2 -> 6); disjoint queues, counters, state rows
      // and output rows.  Run concurrently, each fills the other's tail (a
      // 1M-row batch is a few quotes per lane per pass).
#ifdef FV_LBR_SERIAL
      cudaStream_t s2 = s;                       // A/B: the branches in sequence
#else
      // the per-kernel timing pass (fv_set_kernel_timing) serialises the
      // branches so each kernel's events bracket it alone
      cudaStream_t s2 = t_timing ? s : w->aux[slot];
#endif
      CK(cudaEventRecord(w->fork_ev[slot], s));
      CK(cudaStreamWaitEvent(s2, w->fork_ev[slot], 0));
      FV_LAUNCH(FV_KID_LBR_FAST, s2, k_lbr_far_low_fast<<<g(w->blocks_lbr_fast), 256, 0, s2>>>(b, lq));
      FV_LAUNCH(FV_KID_LBR_FL, s2, launch_pdl(k_lbr_solve<FV_FAR_LOW>, g(w->sm_count), 256, 0, s2, b, lq));
      FV_LAUNCH(FV_KID_LBR_ANCH, s, launch_pdl(k_lbr_anchors, g(w->blocks_lbr_anch), 256, 0, s, b, lq));
      // the far-high solve (queue 2) depends on the anchors pass only: a third
      // stream, beside the near solve (queues 1 -> 6)
#if defined(FV_LBR_SERIAL) || defined(FV_LBR_FH_SERIAL)
      cudaStream_t s3 = s;
#else
      cudaStream_t s3 = t_timing ? s : w->aux2[slot];
#endif
      CK(cudaEventRecord(w->fork2_ev[slot], s));
      CK(cudaStreamWaitEvent(s3, w->fork2_ev[slot], 0));
      FV_LAUNCH(FV_KID_LBR_FH, s3, k_lbr_solve<FV_FAR_HIGH><<<g(w->blocks_lbr_fh), 256, 0, s3>>>(b, lq));
      FV_LAUNCH(FV_KID_LBR_NEAR_FAST, s, launch_pdl(k_lbr_near_fast, g(w->blocks_lbr_nfast), 256, 0, s, b, lq));
      FV_LAUNCH(FV_KID_LBR_NEAR, s, launch_pdl(k_lbr_solve<FV_NEAR_LOW>, g(w->sm_count), 256, 0, s, b, lq));
      CK(cudaEventRecord(w->join_ev[slot], s2));
      CK(cudaStreamWaitEvent(s, w->join_ev[slot], 0));
      CK(cudaEventRecord(w->join2_ev[slot], s3));
      CK(cudaStreamWaitEvent(s, w->join2_ev[slot], 0));
    }
  } else {
    // chunks of <= 2^26 rows: int32 row indices in the queues, bounded buffers
    const int64_t kHalleyChunk = g_halley_round;
    const int64_t chunk = a.n < kHalleyChunk ? a.n : kHalleyChunk;
    CK(ensure_hsm(w, slot, chunk));
    for (int64_t off = 0; off < a.n; off += chunk) {
      KArgs b = sub_args(a, off, (a.n - off) < chunk ? (a.n - off) : chunk);
      unsigned long long* ctr = w->work_ctr + 2 * slot;   // [0] Halley, [1] bisection claims
      unsigned int* cnt = w->hsm_count + 4 * slot;         // [0] records, [1] handed back by the
                                                           // bracket pass, [2] bisection, [3] handed back later
      int32_t* hrow = w->hsm_ridx[slot];
      int32_t* bis = w->hsm_ridx[slot] + w->hsm_cap[slot];
      int32_t* hrow2 = w->hsm_ridx[slot] + 2 * w->hsm_cap[slot];
      CK(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), s));
      CK(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned int), s));
      const int64_t need = (b.n + 255) / 256;
      auto g = [need](int blocks) { return (int)(need < blocks ? need : blocks); };
      if (price) {                    // fv_price_iv: prices computed in the bracket pass
        const KArgs pb = sub_args(*price, off, b.n);
        FV_LAUNCH(FV_KID_HALLEY_SETUP, s, k_halley_bracket<true><<<blocks_for(w->blocks_hset_p, b.n), 256, 0, s>>>(
            b, pb, w->hsm_recs[slot], w->hsm_rrow[slot], cnt, hrow));
      } else {
        FV_LAUNCH(FV_KID_HALLEY_SETUP, s, k_halley_bracket<false><<<blocks_for(w->blocks_hset, b.n), 256, 0, s>>>(
            b, b, w->hsm_recs[slot], w->hsm_rrow[slot], cnt, hrow));
      }
      // The bracket pass's hand-backs (f(10) sign undecided or doubling, log(F/K)
      // raising, range flags) are final once it ends: their careful pass runs
      // on the second stream beside the Halley / bisection passes, which hand
      // back into a queue of their own, drained after them.  (A careful row is
      // long -- the whole solver on the careful routines -- and ~1 per lane.)
#ifdef FV_HAL_SERIAL
      cudaStream_t s2 = s;
#else
      cudaStream_t s2 = t_timing ? s : w->aux[slot];
#endif
      CK(cudaEventRecord(w->fork_ev[slot], s));
      CK(cudaStreamWaitEvent(s2, w->fork_ev[slot], 0));
      FV_LAUNCH(FV_KID_HALLEY_SM2, s2, k_halley_careful<<<g(w->sm_count), 256, 0, s2>>>(b, hrow, cnt + 1));
      FV_LAUNCH(FV_KID_HALLEY_SM, s, launch_pdl(k_halley_iter, g(w->blocks_hiter), 256, 0, s, 
          b, w->hsm_recs[slot], w->hsm_rrow[slot], cnt, ctr, bis, cnt + 2, hrow2, cnt + 3));
      FV_LAUNCH(FV_KID_HALLEY_BISECT, s, launch_pdl(k_halley_bisect, g(w->blocks_hbis), 256, 0, s, 
          b, w->hsm_recs[slot], w->hsm_rrow[slot], bis, cnt + 2, ctr + 1, hrow2, cnt + 3));
      FV_LAUNCH(FV_KID_HALLEY_SM2, s, launch_pdl(k_halley_careful, g(w->sm_count), 256, 0, s, b, hrow2, cnt + 3));
      CK(cudaEventRecord(w->join_ev[slot], s2));
      CK(cudaStreamWaitEvent(s, w->join_ev[slot], 0));
    }
  }
  return cudaGetLastError();
}

cudaError_t launch(DevWork* w, const Call& c, const KArgs& a, int slot, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  switch (c.kind) {
    case KIND_PRICE:
      FV_LAUNCH(FV_KID_PRICE, s, k_price<<<blocks_for(w->blocks_price, a.n), 256, 0, s>>>(a));
      break;
    case KIND_GREEKS:
      FV_LAUNCH(FV_KID_PRICE_GREEKS, s, k_price_greeks<false, true><<<blocks_for(w->blocks_greeks, a.n), 256, 0, s>>>(a));
      break;
    case KIND_PRICE_GREEKS:
      if (c.want_price && c.want_greeks)
        FV_LAUNCH(FV_KID_PRICE_GREEKS, s, k_price_greeks<true, true><<<blocks_for(w->blocks_greeks, a.n), 256, 0, s>>>(a));
      else if (c.want_greeks)
        FV_LAUNCH(FV_KID_PRICE_GREEKS, s, k_price_greeks<false, true><<<blocks_for(w->blocks_greeks, a.n), 256, 0, s>>>(a));
      else
        FV_LAUNCH(FV_KID_PRICE_GREEKS, s, k_price_greeks<true, false><<<blocks_for(w->blocks_greeks, a.n), 256, 0, s>>>(a));
      break;
    case KIND_IV:
      CK(launch_iv(w, c.method, a, slot, s));
      break;
    case KIND_PRICE_IV:
#ifdef FV_RT_FUSED
      // price computed inside the bracket pass: measured SLOWER on the rt
      // workload (3.59 vs 3.48 ms per 10M rows, profiles/README.md) -- the
      // pass is FP64-latency-bound either way and the pricing row's extra
      // live state costs more than the 57 B/row of HBM traffic it saves
      if (c.method == FV_METHOD_HALLEY) {
        CK(launch_iv(w, c.method, iv_stage_args(a, w), slot, s, &a));
        break;
      }
#endif
      FV_LAUNCH(FV_KID_PRICE, s, k_price<<<blocks_for(w->blocks_price, a.n), 256, 0, s>>>(a));
      CK(launch_iv(w, c.method, iv_stage_args(a, w), slot, s));
      break;
  }
  return cudaGetLastError();
}

// Device pointer? (*dev: its device)
bool is_device_ptr(const void* p, int* dev = nullptr) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  if (dev) *dev = at.device;
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Restores the calling thread's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

const char* check_name(int c, bool has_sigma, char* buf, size_t len) {
  static const char* cols[] = {"underlying", "strike", "t", "r", "q"};
  switch (c) {
    case FV_CHECK_BAD_FLAG: snprintf(buf, len, "option flag must be +1 (call) or -1 (put)"); break;
    case FV_CHECK_NONFINITE_UNDERLYING: case FV_CHECK_NONFINITE_STRIKE: case FV_CHECK_NONFINITE_T:
    case FV_CHECK_NONFINITE_R: case FV_CHECK_NONFINITE_Q:
      snprintf(buf, len, "column %s is not finite", cols[c - 1]); break;
    case FV_CHECK_NONFINITE_LAST:
      snprintf(buf, len, "column %s is not finite", has_sigma ? "sigma" : "price"); break;
    case FV_CHECK_POSITIVE_UNDERLYING: snprintf(buf, len, "column underlying must be positive"); break;
    case FV_CHECK_POSITIVE_STRIKE: snprintf(buf, len, "column strike must be positive"); break;
    case FV_CHECK_NONNEG_T: snprintf(buf, len, "column t must be >= 0"); break;
    case FV_CHECK_NONNEG_SIGMA: snprintf(buf, len, "column sigma must be >= 0"); break;
    case FV_CHECK_DIVIDEND: snprintf(buf, len, "model does not accept a dividend yield"); break;
    default: snprintf(buf, len, "check %d", c);
  }
  return buf;
}

const int kCheckColumn[FV_NCHECK] = {0, 1, 2, 3, 4, 5, 6, 1, 2, 3, 6, 5};

void fill_exc_message(fv_error* e) {
  const char* txt = "";
  switch (e->kind) {
    case FV_EXC_MATH_RANGE: txt = "OverflowError: math range error"; break;
    case FV_EXC_MATH_DOMAIN: txt = "ValueError: math domain error"; break;
    case FV_EXC_ZERO_DIV: txt = "ZeroDivisionError: float division by zero"; break;
    case FV_EXC_POW_RANGE: txt = "OverflowError: (34, 'Numerical result out of range')"; break;
    case FV_EXC_DOM_FK: txt = "DomainError: F and K must be positive"; break;
    case FV_EXC_DOM_ATM_BETA: txt = "DomainError: atm_inverse requires beta in (0, 1)"; break;
    case FV_EXC_DOM_INVCDF_P: txt = "DomainError: inv_norm_cdf requires p in (0, 1)"; break;
    case FV_EXC_DOM_NB_X: txt = "DomainError: normalized_black requires x <= 0"; break;
    case FV_EXC_DOM_NB_S: txt = "DomainError: normalized_black requires s > 0"; break;
    case FV_EXC_DOM_OBJ_S: txt = "DomainError: objective_branch requires s > 0"; break;
  }
  snprintf(e->message, sizeof(e->message), "%s (row %lld)", txt, (long long)e->index);
}

void set_ok(fv_error* e) {
  if (!e) return;
  memset(e, 0, sizeof(*e));
  e->index = -1;
}
int set_cuda_err(fv_error* e, cudaError_t ce) {
  if (e) {
    memset(e, 0, sizeof(*e));
    e->code = FV_ERR_CUDA;
    e->index = -1;
    snprintf(e->message, sizeof(e->message), "CUDA error: %s", cudaGetErrorString(ce));
  }
  return FV_ERR_CUDA;
}
int set_arg_err(fv_error* e, const char* msg) {
  if (e) {
    memset(e, 0, sizeof(*e));
    e->code = FV_ERR_ARG;
    e->index = -1;
    snprintf(e->message, sizeof(e->message), "%s", msg);
  }
  return FV_ERR_ARG;
}

// Host-side checks for broadcast columns (row 0 is their only row).
uint32_t bcast_checks(const Call& c, const double vals[7], int flag_val, const bool bc[7]) {
  uint32_t b = 0;
  bool has_sigma = c.kind != KIND_IV;
  if (bc[0]) b |= (uint32_t)(flag_val != 1 && flag_val != -1) << FV_CHECK_BAD_FLAG;
  for (int col = 1; col <= 6; ++col)
    if (bc[col]) b |= (uint32_t)(!fv_isfinite(vals[col])) << (FV_CHECK_NONFINITE_UNDERLYING + col - 1);
  if (bc[1]) b |= (uint32_t)(!(vals[1] > 0.0)) << FV_CHECK_POSITIVE_UNDERLYING;
  if (bc[2]) b |= (uint32_t)(!(vals[2] > 0.0)) << FV_CHECK_POSITIVE_STRIKE;
  if (bc[3]) b |= (uint32_t)(vals[3] < 0.0) << FV_CHECK_NONNEG_T;
  if (bc[6] && has_sigma) b |= (uint32_t)(vals[6] < 0.0) << FV_CHECK_NONNEG_SIGMA;
  if (bc[5]) b |= (uint32_t)(c.model != FV_MODEL_BLACK_SCHOLES_MERTON && vals[5] != 0.0) << FV_CHECK_DIVIDEND;
  return b;
}

// Resolve the device status into the two fv_error records.
int finish(DevWork* w, const Call& c, const KArgs& a0, uint32_t bcast_bits, cudaStream_t s,
           fv_error* e1, fv_error* e2, const FvDevStatus& st) {
  bool has_sigma = c.kind != KIND_IV;
  for (int ck = 0; ck < FV_NCHECK; ++ck) {
    unsigned long long row = st.check_first[ck];
    if (bcast_bits & (1u << ck)) row = 0;
    t_check_rows[ck] = row == ~0ull ? -1 : (int64_t)row;
  }
  for (int k = 0; k < 2; ++k) {
    unsigned long long ex = k ? st.exc2_first : st.exc_first;
    t_exc_row[k] = ex == ~0ull ? -1 : (int64_t)(ex >> 8);
    t_exc_code[k] = ex == ~0ull ? 0 : (int32_t)(ex & 0xff);
  }
  // BatchError: first check in order that failed anywhere
  for (int ck = 0; ck < FV_NCHECK; ++ck) {
    unsigned long long row = st.check_first[ck];
    if (bcast_bits & (1u << ck)) row = 0;
    if (row != ~0ull) {
      fv_error* outs[2] = {e1, e2};
      for (fv_error* e : outs) {
        if (!e) continue;
        memset(e, 0, sizeof(*e));
        e->code = FV_ERR_BATCH;
        e->kind = ck;
        e->index = (int64_t)row;
        e->column = kCheckColumn[ck];
        char detail[128];
        check_name(ck, has_sigma, detail, sizeof(detail));
        const char* kindname = ck == FV_CHECK_BAD_FLAG ? "BadFlag"
                               : (ck <= FV_CHECK_NONFINITE_LAST ? "NonFiniteInput" : "DomainError");
        snprintf(e->message, sizeof(e->message), "%s at row %lld: %s", kindname, (long long)row, detail);
      }
      return FV_ERR_BATCH;
    }
  }
  int rc = FV_OK;
  unsigned long long ex[2] = {st.exc_first, st.exc2_first};
  fv_error* outs[2] = {e1, e2};
  for (int k = 0; k < 2; ++k) {
    fv_error* e = outs[k];
    if (e) set_ok(e);
    if (ex[k] == ~0ull) continue;
    rc = FV_ERR_PYEXC;
    if (!e) continue;
    e->code = FV_ERR_PYEXC;
    e->kind = (int)(ex[k] & 0xff);
    e->index = (int64_t)(ex[k] >> 8);
    if (e->kind >= FV_EXC_DOM_ATM_BETA && c.kind == KIND_IV && a0.n > 0) {
      // re-run the row once to recover the value the message quotes
      k_explain<<<1, 1, 0, s>>>(a0, c.method, e->index - a0.row0, w->explain);
      ++t_launches;
      ExplainOut eo;
      cudaMemcpyAsync(&eo, w->explain, sizeof(eo), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      e->value = eo.val;
      e->value_is_numpy = eo.np;
    }
    fill_exc_message(e);
  }
  return rc;
}

// fv_price_iv: the price stage's outcome (st_host[0]) is the call's when it
// failed -- the reference's batch_price raises before batch_iv runs; else the
// IV stage's (st_host[1]).  fv_last_outcome: check rows of the stage that
// decides, exception stream [0] price, [1] IV.
int finish_price_iv(DevWork* w, const Call& c, const KArgs& ap, const KArgs& ai, uint32_t bbits,
                    cudaStream_t s, fv_error* ep, fv_error* ei) {
  Call cp = c, ci = c;
  cp.kind = KIND_PRICE;
  ci.kind = KIND_IV;
  const int rci = finish(w, ci, ai, c.bbits_iv, s, ei, nullptr, w->st_host[1]);
  int64_t rows_i[FV_NCHECK];
  for (int k = 0; k < FV_NCHECK; ++k) rows_i[k] = t_check_rows[k];
  const int64_t xr = t_exc_row[0];
  const int32_t xc = t_exc_code[0];
  const int rcp = finish(w, cp, ap, bbits, s, ep, nullptr, w->st_host[0]);
  if (rcp == FV_OK)
    for (int k = 0; k < FV_NCHECK; ++k) t_check_rows[k] = rows_i[k];
  t_exc_row[1] = xr;
  t_exc_code[1] = xc;
  return rcp != FV_OK ? rcp : rci;
}

DCol make_dcol(const fv_col& c, const void* base_override) {
  DCol d;
  d.p = (const double*)(base_override ? base_override : c.data);
  d.stride = c.stride;
  if (c.stride == 0) d.mode = 0;
  else if (c.stride == 1 && (((uintptr_t)d.p) & 15) == 0) d.mode = 1;
  else d.mode = 2;
  return d;
}
DFlag make_dflag(const fv_col& c, const void* base_override) {
  DFlag d;
  d.p = (const int8_t*)(base_override ? base_override : c.data);
  d.stride = c.stride;
  if (c.stride == 0) d.mode = 0;
  else if (c.stride == 1 && (((uintptr_t)d.p) & 1) == 0) d.mode = 1;
  else d.mode = 2;
  return d;
}

KArgs base_args(const Call& c, DevWork* w) {
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.model = c.model;
  a.has_sigma = c.kind != KIND_IV;
  uint32_t mask = (1u << FV_NCHECK) - 1;
  if (!a.has_sigma) mask &= ~(1u << FV_CHECK_NONNEG_SIGMA);
  // broadcast columns are checked on the host (once), not per row
  const int col_checks[7][3] = {{FV_CHECK_BAD_FLAG, -1, -1},
                                {FV_CHECK_NONFINITE_UNDERLYING, FV_CHECK_POSITIVE_UNDERLYING, -1},
                                {FV_CHECK_NONFINITE_STRIKE, FV_CHECK_POSITIVE_STRIKE, -1},
                                {FV_CHECK_NONFINITE_T, FV_CHECK_NONNEG_T, -1},
                                {FV_CHECK_NONFINITE_R, -1, -1},
                                {FV_CHECK_NONFINITE_Q, FV_CHECK_DIVIDEND, -1},
                                {FV_CHECK_NONFINITE_LAST, FV_CHECK_NONNEG_SIGMA, -1}};
  for (int col = 0; col < 7; ++col)
    if (c.cols[col].stride == 0 && !c.bcast_dev)
      for (int j = 0; j < 3; ++j)
        if (col_checks[col][j] >= 0) mask &= ~(1u << col_checks[col][j]);
  a.check_mask = mask;
  a.st = w->st;
  a.status = c.status;
  a.region = c.region;
  return a;
}


// A call's outcome block: every pass folds its first failing rows into w->st
// (atomicMin on all-ones), and the call reads it back at the end.
// FV_STATUS_KERNEL: one warp copies the block into the pinned host mirror
// through its UVA address and re-arms it for the next call (which then skips
// its reset), instead of a D2H copy at the end and a memset at the start.
#ifndef FV_STATUS_KERNEL
#define FV_STATUS_KERNEL 1
#endif
__global__ void k_publish_status(unsigned long long* st, unsigned long long* host) {
  constexpr int kWords = (int)(2 * sizeof(FvDevStatus) / 8);
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) {
    host[i] = st[i];
    st[i] = ~0ull;
  }
}
cudaError_t arm_status(DevWork* w, cudaStream_t s) {
  cudaError_t ce = cudaSuccess;
  if (!(FV_STATUS_KERNEL && w->st_armed)) ce = cudaMemsetAsync(w->st, 0xff, 2 * sizeof(FvDevStatus), s);
  w->st_armed = false;                     // re-armed only by a call that completes
  return ce;
}
cudaError_t read_status(DevWork* w, cudaStream_t s) {
#if FV_STATUS_KERNEL
  k_publish_status<<<1, 32, 0, s>>>((unsigned long long*)w->st, (unsigned long long*)w->st_host);
  ++t_launches;
  return cudaGetLastError();
#else
  return cudaMemcpyAsync(w->st_host, w->st, 2 * sizeof(FvDevStatus), cudaMemcpyDeviceToHost, s);
#endif
}

int run_device(DevWork* w, const Call& c, cudaStream_t s, uint32_t bcast_bits, fv_error* e1,
               fv_error* e2) {
  cudaError_t ce;
  KArgs a = base_args(c, w);
  a.flag = make_dflag(c.cols[0], nullptr);
  a.un = make_dcol(c.cols[1], nullptr);
  a.k = make_dcol(c.cols[2], nullptr);
  a.t = make_dcol(c.cols[3], nullptr);
  a.r = make_dcol(c.cols[4], nullptr);
  a.q = make_dcol(c.cols[5], nullptr);
  a.last = make_dcol(c.cols[6], nullptr);
  a.n = c.n;
  a.row0 = 0;
  a.o0 = c.outs[0]; a.o1 = c.outs[1]; a.o2 = c.outs[2];
  a.o3 = c.outs[3]; a.o4 = c.outs[4]; a.o5 = c.outs[5];
  cudaEvent_t sp0 = nullptr, sp1 = nullptr;
  if (t_span) {
    cudaEventCreate(&sp0);
    cudaEventCreate(&sp1);
    cudaEventRecord(sp0, s);
  }
  CT_MARK();                                   // [2] run_device entered
  if ((ce = arm_status(w, s)) != cudaSuccess) return set_cuda_err(e1, ce);
  if ((ce = launch(w, c, a, 0, s)) != cudaSuccess) return set_cuda_err(e1, ce);
  CT_MARK();                                   // [3] kernels launched
  if (t_span) cudaEventRecord(sp1, s);
  if ((ce = read_status(w, s)) != cudaSuccess) return set_cuda_err(e1, ce);
  CT_MARK();                                   // [4] status kernel launched
  if ((ce = cudaStreamSynchronize(s)) != cudaSuccess) return set_cuda_err(e1, ce);
  CT_MARK();                                   // [5] synchronised
  w->st_armed = true;
  if (t_span) {
    t_span_ms = -1.0f;
    cudaEventElapsedTime(&t_span_ms, sp0, sp1);
    cudaEventDestroy(sp0);
    cudaEventDestroy(sp1);
  }
  if (c.kind == KIND_PRICE_IV) return finish_price_iv(w, c, a, iv_stage_args(a, w), bcast_bits, s, e1, e2);
  return finish(w, c, a, bcast_bits, s, e1, e2, w->st_host[0]);
}

// Host-pointer path: chunked H2D -> kernel -> D2H, FV_NSLOT streams.
// Host memcpy split over threads: pageable caller buffers are moved through
// pinned staging slots, and one thread's memcpy (~11 GB/s) would otherwise
// cap the pipeline far below the link (~55 GB/s pinned).
// A persistent pool of host copy workers (created on first use): a pageable
// call's staging copies are split into 8 MB+ parts spread over the workers and
// the calling thread, without creating threads per copy (thread start-up was
// ~50 us per thread per column per chunk).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool();      // never destroyed: workers outlive static teardown
    return *pool;
  }
  int workers() const { return (int)th_.size(); }
  // runs fn(0..parts-1), part 0 on the caller; returns when all are done.
  // Workers spin (yielding) for a while after each job and the caller spins
  // on the completion count before sleeping: a host call hands the pool one
  // job per chunk, and a futex wake-up per job and per join showed up as
  // host-side gaps in the pipeline.
  void run(int parts, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> lk(mu_);
    job_ = &fn;
    next_ = 1;
    parts_ = parts;
    pending_.store(parts - 1, std::memory_order_relaxed);
    ++gen_;
    agen_.store(gen_, std::memory_order_release);
    cv_.notify_all();
    lk.unlock();
    fn(0);
    const auto t0 = std::chrono::steady_clock::now();
    while (pending_.load(std::memory_order_acquire) != 0 &&
           std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(5))
      cpu_relax();
    lk.lock();
    done_.wait(lk, [&] { return pending_.load(std::memory_order_acquire) == 0; });
    job_ = nullptr;
  }

 private:
  // a yielding spin: a pause-only spin starved the calling thread for whole
  // scheduler slices (~3.5 ms per job) whenever the box had other runnable
  // threads (tools: the pool harness in profiles/r2/ab_session3.txt item 7)
  static void cpu_relax() { std::this_thread::yield(); }
  // threads: the cores this process may run on (its affinity mask, not the
  // machine's count), shared with the other ranks on this host when launched
  // one process per GPU (LOCAL_WORLD_SIZE, set by torchrun), at most 16
  static unsigned host_threads() {
    unsigned nt = std::thread::hardware_concurrency();
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0 && CPU_COUNT(&set) > 0) nt = (unsigned)CPU_COUNT(&set);
    if (const char* e = getenv("LOCAL_WORLD_SIZE")) {
      const long k = atol(e);
      if (k > 1) nt = nt / (unsigned)k;
    }
    if (nt < 2) nt = 2;
    return nt > 16 ? 16 : nt;
  }
  CopyPool() {
    const unsigned nt = host_threads();
    for (unsigned k = 1; k < nt; ++k) th_.emplace_back([this] { loop(); });
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      const auto t0 = std::chrono::steady_clock::now();
      while (agen_.load(std::memory_order_acquire) == seen &&
             std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(500))
        cpu_relax();
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      while (job_ && next_ < parts_) {
        const int part = next_++;
        const std::function<void(int)>* fn = job_;
        lk.unlock();
        (*fn)(part);
        lk.lock();
        if (pending_.fetch_sub(1, std::memory_order_acq_rel) == 1) done_.notify_all();
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int next_ = 0, parts_ = 0;
  std::atomic<int> pending_{0};
  unsigned long long gen_ = 0;
  std::atomic<unsigned long long> agen_{0};
};
std::mutex g_copy_mu;     // one pooled copy at a time (calls on several devices share the pool)

// A batch of copies (the staged columns of one chunk) as one pool job: every
// segment is cut into ~2 MB parts and all parts share the workers, so a chunk's
// columns are copied together instead of one fork / join per column.
struct CopySeg { char* dst; const char* src; size_t bytes; };
void par_memcpy_batch(const std::vector<CopySeg>& segs) {
  const size_t kPart = (size_t)2 << 20;
  struct Part { char* dst; const char* src; size_t bytes; };
  std::vector<Part> parts;
  size_t total = 0;
  for (const CopySeg& g : segs) {
    total += g.bytes;
    for (size_t o = 0; o < g.bytes; o += kPart)
      parts.push_back({g.dst + o, g.src + o, (o + kPart <= g.bytes) ? kPart : g.bytes - o});
  }
  if (parts.empty()) return;
  if (total < ((size_t)4 << 20) || parts.size() < 2) {
    for (const Part& q : parts) memcpy(q.dst, q.src, q.bytes);
    return;
  }
  CopyPool& pool = CopyPool::get();
  const int nw = pool.workers() + 1;
  const int nparts = (int)parts.size();
  const int ntask = nparts < nw ? nparts : nw;
  std::lock_guard<std::mutex> g(g_copy_mu);
  pool.run(ntask, [&](int k) {                       // task k: parts k, k + ntask, ...
    for (int i = k; i < nparts; i += ntask) memcpy(parts[i].dst, parts[i].src, parts[i].bytes);
  });
}


std::vector<std::pair<int64_t, int64_t>> chunk_plan(int64_t n, int64_t chunk) {
  std::vector<std::pair<int64_t, int64_t>> plan;
  if (n <= 0) return plan;
  if (n <= 3 * chunk) {                        // small calls: plain chunks
    for (int64_t r0 = 0; r0 < n; r0 += chunk) plan.push_back({r0, (r0 + chunk < n) ? chunk : n - r0});
    return plan;
  }
  const int64_t q = chunk / 4, h = chunk / 2;
  int64_t r0 = 0;
  plan.push_back({r0, q}); r0 += q;
  plan.push_back({r0, h}); r0 += h;
  const int64_t tail = h + q;                  // the last two chunks: 1/2 and 1/4
  while (n - r0 - tail > chunk) { plan.push_back({r0, chunk}); r0 += chunk; }
  const int64_t mid = n - r0 - tail;           // 0 < mid <= chunk
  if (mid > 0) { plan.push_back({r0, mid}); r0 += mid; }
  plan.push_back({r0, h}); r0 += h;
  plan.push_back({r0, n - r0});
  return plan;
}

// ---- run-length transport of piecewise-constant host columns ---------------
// A host call's input column whose chunk is a few runs of one value (an option
// chain's maturity column, a flag column sorted by side, one value repeated as
// an array) crosses the link as (first row, value) runs and k_expand_runs
// rebuilds the chunk's column in HBM: the kernels read the same bits, the link
// carries 12 bytes per run instead of 8 per row (C4's chain: t and flag, 9 of
// its 25 bytes per quote).  A chunk uses it when it has at most
// rows / kRleRowsPerRun runs; the scan runs on the copy pool, each part giving
// up past its share of that budget, so a column of distinct values costs about
// 1/kRleRowsPerRun of a pass over it.
#ifndef FV_HOST_RLE
#define FV_HOST_RLE 1
#endif
const int64_t kRleRowsPerRun = 64;
// pageable columns: staging copy made in the scan's pass (1) or after it, for
// the columns that did not go as runs (0)
#ifndef FV_SCAN_COPY
#define FV_SCAN_COPY 0
#endif
const int64_t kRleMinRows = 1 << 14;

// bytes of one column's runs area for a chunk of `rows` rows: int32 starts
// [budget + 1] then the values [budget], 256-byte aligned
size_t rle_starts_bytes(int64_t rows) {
  const int64_t b = rows / kRleRowsPerRun + 1;
  return (4 * (size_t)(b + 1) + 255) & ~(size_t)255;
}
size_t rle_col_bytes(int64_t rows, size_t elem) {
  const int64_t b = rows / kRleRowsPerRun + 1;
  return rle_starts_bytes(rows) + ((elem * (size_t)b + 255) & ~(size_t)255);
}

// row i of the chunk takes the value of the last run starting at or before i;
// each block covers a contiguous tile, so a thread searches only the runs
// that meet its block's tile
template <typename T>
__global__ void __launch_bounds__(256) k_expand_runs(const int32_t* __restrict__ starts, const T* __restrict__ vals,
                                                     int nruns, T* __restrict__ out, int64_t n) {
  const int64_t tile = (int64_t)blockDim.x * 8;
  __shared__ int s_r0, s_r1;
  for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < n; t0 += (int64_t)gridDim.x * tile) {
    const int64_t t1 = (t0 + tile < n ? t0 + tile : n) - 1;
    if (threadIdx.x < 2) {
      const int64_t row = threadIdx.x ? t1 : t0;
      int lo = 0, hi = nruns - 1;                 // last run with starts[r] <= row
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (starts[mid] <= row) lo = mid; else hi = mid - 1;
      }
      if (threadIdx.x) s_r1 = lo; else s_r0 = lo;
    }
    __syncthreads();
    const int r0 = s_r0, r1 = s_r1;
    for (int64_t i = t0 + threadIdx.x; i <= t1; i += blockDim.x) {
      int lo = r0, hi = r1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (starts[mid] <= i) lo = mid; else hi = mid - 1;
      }
      out[i] = vals[lo];
    }
    __syncthreads();
  }
}

// One chunk's candidate columns scanned for runs in ONE pool job (a fork /
// join per column cost ~40 us each): every column is cut into parts of >= 32K
// rows (a thread scans ~10 GB/s), each part gives up past its share of the
// column's budget.  Per column: nr runs into starts / vals (starts[nr] = n),
// or nr = -1 when the column has more than `budget` runs.
struct RunScan {
  const void* p;
  int elem;                 // 8 (double bits) or 1 (flag)
  int64_t n, budget;
  int32_t* starts;
  void* vals;
  int64_t nr;
  char* copy_to;            // pageable column: also copied here (pinned staging) in the same pass
};

// rows [lo, hi) of one column: its runs (the first entry may continue the
// previous part's last run; the merge drops it).  Runs that start in this
// part are published to the column's total 64 at a time, and the scan stops
// once that total passes the budget (a lower bound of the true count, so
// stopping is always right; the exact count is checked after the join).
template <typename T>
void scan_part(const T* p, int64_t lo, int64_t hi, int64_t budget, std::atomic<int64_t>& total,
               std::atomic<bool>& over, std::vector<std::pair<int64_t, uint64_t>>& v, int64_t& mine) {
  T cur = p[lo];
  v.push_back({lo, (uint64_t)cur});
  int64_t counted = (lo == 0 || p[lo - 1] != cur) ? 1 : 0, pending = counted;
  for (int64_t i = lo + 1; i < hi;) {
    if (i + 8 <= hi) {                           // eight rows of the current run at a time
      T acc = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) acc |= (T)(p[i + u] ^ cur);
      if (acc == 0) { i += 8; continue; }
    }
    if (p[i] == cur) { ++i; continue; }
    ++counted;
    if (++pending == 64) {
      if (total.fetch_add(pending, std::memory_order_relaxed) + pending > budget ||
          over.load(std::memory_order_relaxed)) {
        over.store(true, std::memory_order_relaxed);
        return;
      }
      pending = 0;
    }
    cur = p[i];
    v.push_back({i, (uint64_t)cur});
    ++i;
  }
  total.fetch_add(pending, std::memory_order_relaxed);
  mine = counted;
}

void find_runs_batch(std::vector<RunScan>& jobs) {
  if (jobs.empty()) return;
  CopyPool& pool = CopyPool::get();
  const int nw = pool.workers() + 1;
  struct Task { int job; int64_t lo, hi; };
  std::vector<Task> tasks;
  for (int j = 0; j < (int)jobs.size(); ++j) {
    const RunScan& r = jobs[j];
    int parts = (int)(r.n >> 15);                // >= 32K rows per part (a thread scans ~10 GB/s)
    if (parts > nw) parts = nw;
    if (parts < 1) parts = 1;
    for (int k = 0; k < parts; ++k) tasks.push_back({j, r.n * k / parts, r.n * (k + 1) / parts});
  }
  const int nt = (int)tasks.size();
  // the parts' run lists keep their capacity from call to call: fresh vectors
  // page-faulted on every call (~0.5 ms per 2.5M-row column that gives up)
  std::lock_guard<std::mutex> g(g_copy_mu);
  static std::vector<std::vector<std::pair<int64_t, uint64_t>>> found;
  if ((int)found.size() < nt) found.resize(nt);
  for (int t = 0; t < nt; ++t) found[t].clear();
  std::vector<int64_t> counted(nt, 0);
  std::unique_ptr<std::atomic<bool>[]> over(new std::atomic<bool>[jobs.size()]);
  std::unique_ptr<std::atomic<int64_t>[]> total(new std::atomic<int64_t>[jobs.size()]);
  for (size_t j = 0; j < jobs.size(); ++j) {
    over[j].store(jobs[j].budget < 1 || jobs[j].n <= 0);
    total[j].store(0);
  }
  auto run_task = [&](int t) {
    const Task& k = tasks[t];
    const RunScan& r = jobs[k.job];
    if (r.copy_to)
      memcpy(r.copy_to + k.lo * r.elem, (const char*)r.p + k.lo * r.elem, (size_t)((k.hi - k.lo) * r.elem));
    if (over[k.job].load(std::memory_order_relaxed)) return;
    if (r.elem == 8)
      scan_part((const uint64_t*)r.p, k.lo, k.hi, r.budget, total[k.job], over[k.job], found[t], counted[t]);
    else
      scan_part((const uint8_t*)r.p, k.lo, k.hi, r.budget, total[k.job], over[k.job], found[t], counted[t]);
  };
  const int ntask = nt < nw ? nt : nw;
  if (ntask <= 1) {
    for (int t = 0; t < nt; ++t) run_task(t);
  } else {
    pool.run(ntask, [&](int w) { for (int t = w; t < nt; t += ntask) run_task(t); });
  }
  std::vector<int64_t> exact(jobs.size(), 0);
  for (int t = 0; t < nt; ++t) exact[tasks[t].job] += counted[t];
  for (size_t j = 0; j < jobs.size(); ++j)
    jobs[j].nr = (over[j].load() || exact[j] > jobs[j].budget) ? -1 : 0;
  for (int t = 0; t < nt; ++t) {                 // tasks are in row order within a column
    RunScan& r = jobs[tasks[t].job];
    if (r.nr < 0) continue;
    for (const auto& run : found[t]) {
      if (r.nr > 0) {                             // the previous part's last run continues here
        const uint64_t last = r.elem == 8 ? ((const uint64_t*)r.vals)[r.nr - 1] : ((const uint8_t*)r.vals)[r.nr - 1];
        if (last == run.second) continue;
      }
      r.starts[r.nr] = (int32_t)run.first;
      if (r.elem == 8) ((uint64_t*)r.vals)[r.nr] = run.second;
      else ((uint8_t*)r.vals)[r.nr] = (uint8_t)run.second;
      ++r.nr;
    }
  }
  for (RunScan& r : jobs)
    if (r.nr >= 0) r.starts[r.nr] = (int32_t)r.n;
}

bool is_pageable(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return true; }
  return at.type == cudaMemoryTypeUnregistered;
}

// Rows per chunk of a host-buffer call: the configured size (2^22 by default,
// fv_set_chunk_rows), but at least 8 chunks when the call is smaller than 8 of
// them, down to 2^18 rows: the first chunk's H2D and the last chunk's kernels
// + D2H overlap nothing, so a 10M-row call in three 4M-row chunks spent a
// third of its time filling and draining the pipeline.
#ifndef FV_HOST_AUTO_CHUNK
#define FV_HOST_AUTO_CHUNK 1
#endif
// FV_CAP_BY_CALL: size a host call's chunk / staging buffers by this call's
// chunk instead of the configured one (A/B: a 1M-row first call 27 -> 20 ms,
// but the first large call after small ones then grows them again)
#ifndef FV_CAP_BY_CALL
#define FV_CAP_BY_CALL 0
#endif
#ifndef FV_HOST_CHUNK_DIV
#define FV_HOST_CHUNK_DIV 8
#endif
#ifndef FV_HOST_CHUNK_MIN_LOG2
#define FV_HOST_CHUNK_MIN_LOG2 18
#endif
// FV_HOST_TRACE (diagnostic builds only): per-call host timestamps and a
// device timeline of each chunk's H2D / kernels / D2H on stderr
#ifndef FV_HOST_TRACE
#define FV_HOST_TRACE 0
#endif
#if FV_HOST_TRACE
__device__ unsigned long long g_stamps[512];
__global__ void k_stamp(int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_stamps[i] = t;
}
struct HostTrace {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  std::vector<std::pair<const char*, double>> marks;
  std::vector<const char*> names;
  std::vector<std::pair<int64_t, int>> ev_chunk;
  void mark(const char* m) {
    marks.push_back({m, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count()});
  }
  void ev(const char* name, int64_t ci, int slot, cudaStream_t s) {
    if (names.size() >= 512) return;
    k_stamp<<<1, 1, 0, s>>>((int)names.size());
    names.push_back(name);
    ev_chunk.push_back({ci, slot});
  }
  ~HostTrace() {
    mark("trace_end");
    for (auto& m : marks) fprintf(stderr, "host %-14s %9.1f us\n", m.first, m.second);
    if (names.empty()) return;
    cudaDeviceSynchronize();
    unsigned long long st[512];
    cudaMemcpyFromSymbol(st, g_stamps, sizeof(st));
    for (size_t i = 0; i < names.size(); ++i)
      fprintf(stderr, "dev  chunk %3lld slot %d %-10s %9.1f us\n", (long long)ev_chunk[i].first, ev_chunk[i].second,
              names[i], 1e-3 * (double)(st[i] - st[0]));
  }
};
#define TR_MARK(x) tr.mark(x)
#define TR_EV(n, ci, sl, st) tr.ev(n, ci, sl, st)
#else
#define TR_MARK(x) ((void)0)
#define TR_EV(n, ci, sl, st) ((void)0)
#endif
// Pageable callers: chunks of at least 2^19 rows -- each chunk's staging copies
// are pool jobs on the host, and a 1M-row pageable call in 7 ramped chunks spent
// 3.2 ms against 1.9 ms in two (pinned callers: 0.82 vs 0.81 G quotes/s, even)
#ifndef FV_HOST_CHUNK_MIN_LOG2_PAGEABLE
#define FV_HOST_CHUNK_MIN_LOG2_PAGEABLE 19
#endif
int64_t host_chunk_rows(int64_t n, bool pageable = false) {
  int64_t c = g_chunk_rows;
#if FV_HOST_AUTO_CHUNK
  const int64_t floor_rows = 1ll << (pageable ? FV_HOST_CHUNK_MIN_LOG2_PAGEABLE : FV_HOST_CHUNK_MIN_LOG2);
  const int64_t eighth = ((n / FV_HOST_CHUNK_DIV + 65535) / 65536) * 65536;
  const int64_t want = eighth > floor_rows ? eighth : floor_rows;
  if (want < c) c = want;
#endif
  (void)n;
  (void)pageable;
  return c;
}

int run_host(DevWork* w, const Call& c, uint32_t bcast_bits, fv_error* e1, fv_error* e2) {
  cudaError_t ce;
#if FV_HOST_TRACE
  HostTrace tr;
#endif
  bool any_pageable = false;
  for (int col = 0; col < 7; ++col)
    if (c.cols[col].stride != 0 && is_pageable(c.cols[col].data)) any_pageable = true;
  for (int i = 0; i < 6; ++i)
    if (c.outs[i] && is_pageable(c.outs[i])) any_pageable = true;
  if (c.status && is_pageable(c.status)) any_pageable = true;
  const int64_t chunk = host_chunk_rows(c.n, any_pageable);
  const int64_t n = c.n;
  // column element sizes and whether each is streamed
  const size_t in_sz[7] = {1, 8, 8, 8, 8, 8, 8};
  int nout = 0;
  for (int i = 0; i < 6; ++i) if (c.outs[i]) ++nout;
  bool has_status = c.status != nullptr, has_region = c.region != nullptr;
  // per-slot layout: [inputs (streamed cols)] [outputs] [status] [region], 256B aligned
  auto align = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t slot_bytes = 0;
  size_t off_in[7], off_out[6], off_status = 0, off_region = 0;
  for (int col = 0; col < 7; ++col) {
    off_in[col] = slot_bytes;
    if (c.cols[col].stride != 0) slot_bytes += align(in_sz[col] * chunk);
  }
  for (int i = 0; i < 6; ++i) { off_out[i] = slot_bytes; if (c.outs[i]) slot_bytes += align(8 * chunk); }
  off_status = slot_bytes; if (has_status) slot_bytes += align(chunk);
  off_region = slot_bytes; if (has_region) slot_bytes += align(chunk);
  // buffers grow to the largest layout of this chunk size at once (every
  // column streamed, six outputs, status, region): a call with more streamed
  // columns than the last one must not pay another pinned allocation (~0.4 s
  // for the three staging slots of 2^22 rows)
  // (sized for the configured chunk, so smaller auto-sized chunks of a
  // mid-size call never shrink the buffers a large call needs)
#if FV_CAP_BY_CALL
  const int64_t cap_rows = chunk;
#else
  const int64_t cap_rows = g_chunk_rows > chunk ? g_chunk_rows : chunk;
#endif
  const size_t max_slot = align(cap_rows) + 6 * align(8 * cap_rows) + 6 * align(8 * cap_rows) + 2 * align(cap_rows);
  for (int s = 0; s < FV_NSLOT; ++s) {
    if (w->chunk_cap_rows[s] < (int64_t)slot_bytes) {
      if (w->chunk[s]) cudaFree(w->chunk[s]);
      w->chunk[s] = nullptr;
      if ((ce = cudaMalloc(&w->chunk[s], max_slot)) != cudaSuccess) return set_cuda_err(e1, ce);
      w->chunk_cap_rows[s] = (int64_t)max_slot;
    }
  }
  // pageable caller buffers go through pinned staging (parallel host copies)
  bool stage_in[7] = {}, stage_out[6] = {}, stage_status = false, stage_region = false, any_stage = false;
  for (int col = 0; col < 7; ++col)
    if (c.cols[col].stride != 0) any_stage |= (stage_in[col] = is_pageable(c.cols[col].data));
  for (int i = 0; i < 6; ++i) if (c.outs[i]) any_stage |= (stage_out[i] = is_pageable(c.outs[i]));
  if (has_status) any_stage |= (stage_status = is_pageable(c.status));
  if (has_region) any_stage |= (stage_region = is_pageable(c.region));
  if (any_stage) {
    for (int s = 0; s < FV_NSLOT; ++s) {
      if (w->stage_cap[s] < (int64_t)slot_bytes) {
        if (w->stage[s]) cudaFreeHost(w->stage[s]);
        w->stage[s] = nullptr;
        if ((ce = cudaMallocHost(&w->stage[s], max_slot)) != cudaSuccess) return set_cuda_err(e1, ce);
        w->stage_cap[s] = (int64_t)max_slot;
      }
    }
  }
  // run-length transport: candidate columns (the streamed ones) and each
  // slot's runs areas, pinned and on the device
  bool rle_cand[7] = {};
  size_t off_rle[7] = {};
  bool any_rle_cand = false;
#if FV_HOST_RLE
  if (n >= kRleMinRows && cap_rows < ((int64_t)1 << 31)) {
    size_t rle_bytes = 0;
    for (int col = 0; col < 7; ++col) {
      off_rle[col] = rle_bytes;
      rle_bytes += rle_col_bytes(cap_rows, in_sz[col]);
      any_rle_cand |= (rle_cand[col] = c.cols[col].stride != 0);
    }
    for (int s = 0; any_rle_cand && s < FV_NSLOT; ++s) {
      if (w->rle_cap[s] < (int64_t)rle_bytes) {
        if (w->rle_host[s]) cudaFreeHost(w->rle_host[s]);
        if (w->rle_dev[s]) cudaFree(w->rle_dev[s]);
        w->rle_host[s] = nullptr;
        w->rle_dev[s] = nullptr;
        w->rle_cap[s] = 0;
        if ((ce = cudaMallocHost(&w->rle_host[s], rle_bytes)) != cudaSuccess) return set_cuda_err(e1, ce);
        if ((ce = cudaMalloc(&w->rle_dev[s], rle_bytes)) != cudaSuccess) return set_cuda_err(e1, ce);
        w->rle_cap[s] = (int64_t)rle_bytes;
      }
    }
  }
#endif
  TR_MARK("buffers_ready");
  struct SlotEvents {
    cudaEvent_t ev[FV_NSLOT];
    SlotEvents() { for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming); }
    ~SlotEvents() { for (auto& e : ev) cudaEventDestroy(e); }
  } sev, rev;
  cudaEvent_t* slot_done = sev.ev;
  cudaEvent_t* rle_sent = rev.ev;            // a slot's runs have left its pinned area
  bool rle_inflight[FV_NSLOT] = {};
  // chunk plan: full-size chunks in the middle, a ramp of 1/4- and 1/2-size
  // chunks at both ends -- the first chunk's H2D and the last chunk's kernels
  // + D2H are not overlapped with anything, so smaller end chunks shorten the
  // pipeline's fill and drain (C4 100M rows: ~3 ms of a ~49 ms call)
  std::vector<std::pair<int64_t, int64_t>> plan = chunk_plan(n, chunk);
  int64_t slot_chunk[FV_NSLOT];
  for (int s = 0; s < FV_NSLOT; ++s) slot_chunk[s] = -1;
  // results of chunk `ci` (in slot s) from pinned staging to the caller
  auto drain = [&](int s) {
    const int64_t ci = slot_chunk[s];
    if (ci < 0) return;
    cudaEventSynchronize(slot_done[s]);
    const int64_t r0 = plan[ci].first, rn = plan[ci].second;
    char* st = w->stage[s];
    std::vector<CopySeg> segs;
    for (int i = 0; i < 6; ++i)
      if (stage_out[i]) segs.push_back({(char*)(c.outs[i] + r0), st + off_out[i], (size_t)(8 * rn)});
    if (stage_status) segs.push_back({(char*)(c.status + r0), st + off_status, (size_t)rn});
    if (stage_region) segs.push_back({(char*)(c.region + r0), st + off_region, (size_t)rn});
    par_memcpy_batch(segs);
    slot_chunk[s] = -1;
  };
  if ((ce = arm_status(w, w->streams[0])) != cudaSuccess) return set_cuda_err(e1, ce);
  cudaEvent_t ready;
  cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  cudaEventRecord(ready, w->streams[0]);
  for (int s = 1; s < FV_NSLOT; ++s) cudaStreamWaitEvent(w->streams[s], ready, 0);
  KArgs a_first;
  memset(&a_first, 0, sizeof(a_first));
  const int64_t nchunks = (int64_t)plan.size();
  TR_MARK("setup_done");
  TR_EV("start", -1, 0, w->streams[0]);
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    int slot = (int)(ci % FV_NSLOT);
    cudaStream_t s = w->streams[slot];
    const int64_t r0 = plan[ci].first, rn = plan[ci].second;
    char* base = w->chunk[slot];
    char* stg = w->stage[slot];
    if (any_stage) drain(slot);               // the slot's previous chunk is done with staging
    // the chunk's piecewise-constant columns as runs
    bool rle[7] = {}, scanned[7] = {};
    int64_t nrun[7] = {};
    if (any_rle_cand && rn >= kRleMinRows) {
      if (rle_inflight[slot]) { cudaEventSynchronize(rle_sent[slot]); rle_inflight[slot] = false; }
      std::vector<RunScan> jobs;
      int jcol[7];
      for (int col = 0; col < 7; ++col) {
        if (!rle_cand[col]) continue;
        char* area = w->rle_host[slot] + off_rle[col];
        jcol[jobs.size()] = col;
        jobs.push_back({(const char*)c.cols[col].data + r0 * in_sz[col], (int)in_sz[col], rn,
                        rn / kRleRowsPerRun, (int32_t*)area, area + rle_starts_bytes(cap_rows), -1,
                        (FV_SCAN_COPY && stage_in[col]) ? stg + off_in[col] : nullptr});
        scanned[col] = true;
      }
      find_runs_batch(jobs);
      TR_MARK("runs_scanned");
      for (size_t j = 0; j < jobs.size(); ++j) {
        nrun[jcol[j]] = jobs[j].nr;
        rle[jcol[j]] = jobs[j].nr > 0;
      }
    }
    {                                         // the chunk's pageable input columns, one pool job
      std::vector<CopySeg> segs;
      for (int col = 0; col < 7; ++col)
        if (c.cols[col].stride != 0 && stage_in[col] && !(FV_SCAN_COPY ? scanned[col] : rle[col]))
          segs.push_back({stg + off_in[col], (const char*)c.cols[col].data + r0 * in_sz[col],
                          (size_t)(rn * in_sz[col])});
      par_memcpy_batch(segs);
    }
    void* dev_in[7];
    TR_EV("h2d_start", ci, slot, s);
    // runs first (a few KB), then the streamed columns, then the expansions:
    // an expansion waits for SMs the previous chunk's kernels still hold, and
    // a copy queued behind it on this stream would leave the link idle
    bool any_rle = false;
    const size_t vat = rle_starts_bytes(cap_rows);
    for (int col = 0; col < 7; ++col) {
      dev_in[col] = c.cols[col].stride == 0 ? nullptr : base + off_in[col];
      if (!rle[col]) continue;
      const char* hs = w->rle_host[slot] + off_rle[col];
      char* ds = w->rle_dev[slot] + off_rle[col];
      const size_t sb = 4 * (size_t)(nrun[col] + 1), vb = in_sz[col] * (size_t)nrun[col];
      if ((ce = cudaMemcpyAsync(ds, hs, sb, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
          (ce = cudaMemcpyAsync(ds + vat, hs + vat, vb, cudaMemcpyHostToDevice, s)) != cudaSuccess) {
        cudaEventDestroy(ready);
        return set_cuda_err(e1, ce);
      }
      t_h2d_bytes += (int64_t)(sb + vb);
      any_rle = true;
    }
    if (any_rle) { cudaEventRecord(rle_sent[slot], s); rle_inflight[slot] = true; }
    for (int col = 0; col < 7; ++col) {
      if (c.cols[col].stride == 0 || rle[col]) continue;
      const char* src = (const char*)c.cols[col].data + r0 * in_sz[col];
      if (stage_in[col]) src = stg + off_in[col];
      if ((ce = cudaMemcpyAsync(dev_in[col], src, rn * in_sz[col], cudaMemcpyHostToDevice, s)) != cudaSuccess) {
        cudaEventDestroy(ready);
        return set_cuda_err(e1, ce);
      }
      t_h2d_bytes += rn * (int64_t)in_sz[col];
    }
    for (int col = 0; col < 7; ++col) {
      if (!rle[col]) continue;
      const char* ds = w->rle_dev[slot] + off_rle[col];
      int64_t blocks = (rn + 2047) / 2048;
      if (blocks > 8 * (int64_t)w->sm_count) blocks = 8 * (int64_t)w->sm_count;
      if (in_sz[col] == 8)
        k_expand_runs<uint64_t><<<(unsigned)blocks, 256, 0, s>>>((const int32_t*)ds, (const uint64_t*)(ds + vat),
                                                                 (int)nrun[col], (uint64_t*)dev_in[col], rn);
      else
        k_expand_runs<uint8_t><<<(unsigned)blocks, 256, 0, s>>>((const int32_t*)ds, (const uint8_t*)(ds + vat),
                                                                (int)nrun[col], (uint8_t*)dev_in[col], rn);
      ++t_launches;
    }
    KArgs a = base_args(c, w);
    a.flag = make_dflag(c.cols[0], dev_in[0]);
    a.un = make_dcol(c.cols[1], dev_in[1]);
    a.k = make_dcol(c.cols[2], dev_in[2]);
    a.t = make_dcol(c.cols[3], dev_in[3]);
    a.r = make_dcol(c.cols[4], dev_in[4]);
    a.q = make_dcol(c.cols[5], dev_in[5]);
    a.last = make_dcol(c.cols[6], dev_in[6]);
    a.n = rn;
    a.row0 = r0;
    double* douts[6];
    for (int i = 0; i < 6; ++i) douts[i] = c.outs[i] ? (double*)(base + off_out[i]) : nullptr;
    a.o0 = douts[0]; a.o1 = douts[1]; a.o2 = douts[2]; a.o3 = douts[3]; a.o4 = douts[4]; a.o5 = douts[5];
    a.status = has_status ? (int8_t*)(base + off_status) : nullptr;
    a.region = has_region ? (int8_t*)(base + off_region) : nullptr;
    if (ci == 0) a_first = a;
    TR_EV("h2d_done", ci, slot, s);
    if ((ce = launch(w, c, a, slot, s)) != cudaSuccess) { cudaEventDestroy(ready); return set_cuda_err(e1, ce); }
    TR_EV("kern_done", ci, slot, s);
    for (int i = 0; i < 6; ++i)
      if (c.outs[i])
        cudaMemcpyAsync(stage_out[i] ? (void*)(stg + off_out[i]) : (void*)(c.outs[i] + r0), douts[i], 8 * rn,
                        cudaMemcpyDeviceToHost, s);
    if (has_status)
      cudaMemcpyAsync(stage_status ? (void*)(stg + off_status) : (void*)(c.status + r0), a.status, rn,
                      cudaMemcpyDeviceToHost, s);
    if (has_region)
      cudaMemcpyAsync(stage_region ? (void*)(stg + off_region) : (void*)(c.region + r0), a.region, rn,
                      cudaMemcpyDeviceToHost, s);
    if (any_stage) { cudaEventRecord(slot_done[slot], s); slot_chunk[slot] = ci; }
    TR_EV("d2h_done", ci, slot, s);
    TR_MARK("chunk_issued");
  }
  if (any_stage) for (int s = 0; s < FV_NSLOT; ++s) drain(s);
  for (int s = 1; s < FV_NSLOT; ++s) {
    cudaEventRecord(ready, w->streams[s]);
    cudaStreamWaitEvent(w->streams[0], ready, 0);
  }
  cudaEventDestroy(ready);
  cudaStream_t s0 = w->streams[0];
  if ((ce = read_status(w, s0)) != cudaSuccess) return set_cuda_err(e1, ce);
  if ((ce = cudaStreamSynchronize(s0)) != cudaSuccess) return set_cuda_err(e1, ce);
  for (int s = 1; s < FV_NSLOT; ++s)
    if ((ce = cudaStreamSynchronize(w->streams[s])) != cudaSuccess) return set_cuda_err(e1, ce);
  if ((ce = cudaGetLastError()) != cudaSuccess) return set_cuda_err(e1, ce);
  w->st_armed = true;
  TR_MARK("synced");
  // exceptions in later chunks: the explain kernel needs that chunk's inputs;
  // re-stage the offending row alone (fv_price_iv: the IV stage's row, its
  // price from the caller's price column).
  const bool piv = c.kind == KIND_PRICE_IV;
  const FvDevStatus& st = w->st_host[piv ? 1 : 0];
  unsigned long long ex = st.exc_first;
  KArgs ax = a_first;
  if (ex != ~0ull && (c.kind == KIND_IV || piv) && (int)(ex & 0xff) >= FV_EXC_DOM_ATM_BETA) {
    int64_t row = (int64_t)(ex >> 8);
    char* base = w->chunk[0];
    void* dev_in[7];
    for (int col = 0; col < 7; ++col) {
      if (c.cols[col].stride == 0 && !(piv && col == 6)) { dev_in[col] = nullptr; continue; }
      dev_in[col] = base + off_in[col];
      const void* src = (piv && col == 6) ? (const void*)(c.outs[0] + row)
                                          : (const void*)((const char*)c.cols[col].data + row * in_sz[col]);
      cudaMemcpyAsync(dev_in[col], src, in_sz[col], cudaMemcpyHostToDevice, s0);   // ordered before the
                                                                                // explain kernel on s0
    }
    ax.flag = make_dflag(c.cols[0], dev_in[0]);
    ax.un = make_dcol(c.cols[1], dev_in[1]);
    ax.k = make_dcol(c.cols[2], dev_in[2]);
    ax.t = make_dcol(c.cols[3], dev_in[3]);
    ax.r = make_dcol(c.cols[4], dev_in[4]);
    ax.q = make_dcol(c.cols[5], dev_in[5]);
    if (piv) {
      ax = iv_stage_args(ax, w);
      ax.last.p = (const double*)dev_in[6];
      ax.last.mode = 2;
    } else {
      ax.last = make_dcol(c.cols[6], dev_in[6]);
    }
    ax.n = 1;
    ax.row0 = row;
  } else if (piv) {
    ax = iv_stage_args(a_first, w);
  }
  if (piv) return finish_price_iv(w, c, a_first, ax, bcast_bits, s0, e1, e2);
  return finish(w, c, ax, bcast_bits, s0, e1, e2, w->st_host[0]);
}

// ---- host calls over several devices -------------------------
// fv_set_devices(ids, n): host-pointer calls of at least n * kMinShardRows rows
// are split into n contiguous row shards, one host thread per shard, each
// driving its device's own chunked H2D -> kernels -> D2H pipeline into the
// caller's buffers (no exchange on the data path: every output row depends
// on its input row only).  The shards' outcomes merge to the single-device
// one: the first failing check in the reference's order at its lowest global
// row, else the lowest raising row per exception stream.
std::mutex g_dev_mu;
std::vector<int> g_devices;
const int64_t kMinShardRows = 1 << 20;

std::vector<int> devices_for_host_calls() {
  std::lock_guard<std::mutex> g(g_dev_mu);
  return g_devices;
}

int dispatch(Call c, fv_error* e1, fv_error* e2);

struct ShardOut {
  int rc = FV_OK;
  fv_error e1, e2;
  int64_t check_rows[FV_NCHECK];
  int64_t exc_row[2];
  int32_t exc_code[2];
  int64_t launches = 0;
  int64_t h2d_bytes = 0;
};

thread_local bool t_in_shard = false;

void shard_call(int dev, Call cs, ShardOut* out, bool set_stream = false, void* stream = nullptr) {
  t_in_shard = true;                           // a shard runs on its device only
  cudaError_t ce = cudaSetDevice(dev);
  if (ce != cudaSuccess) { out->rc = set_cuda_err(&out->e1, ce); return; }
  if (set_stream) { t_user_stream = (cudaStream_t)stream; t_user_stream_set = true; }
  out->rc = dispatch(cs, &out->e1, &out->e2);
  for (int k = 0; k < FV_NCHECK; ++k) out->check_rows[k] = t_check_rows[k];
  for (int k = 0; k < 2; ++k) { out->exc_row[k] = t_exc_row[k]; out->exc_code[k] = t_exc_code[k]; }
  out->launches = t_launches;
  out->h2d_bytes = t_h2d_bytes;
}

void shift_error(fv_error* e, int64_t off) {
  if (e->code == FV_ERR_PYEXC) {
    e->index += off;
    fill_exc_message(e);
  } else if (e->code == FV_ERR_BATCH) {
    const char* colon = strstr(e->message, ": ");
    char detail[200];
    snprintf(detail, sizeof(detail), "%s", colon ? colon + 2 : "");
    const char* kindname = e->kind == FV_CHECK_BAD_FLAG ? "BadFlag"
                           : (e->kind <= FV_CHECK_NONFINITE_LAST ? "NonFiniteInput" : "DomainError");
    e->index += off;
    snprintf(e->message, sizeof(e->message), "%s at row %lld: %s", kindname, (long long)e->index, detail);
  }
}

int merge_shards(Kind kind, const std::vector<ShardOut>& outs, const std::vector<int64_t>& off, fv_error* e1,
                 fv_error* e2);

int dispatch_sharded(const Call& c, const std::vector<int>& devs, fv_error* e1, fv_error* e2) {
  const int64_t G = (int64_t)devs.size();
  const size_t in_sz[7] = {1, 8, 8, 8, 8, 8, 8};
  std::vector<ShardOut> outs(G);
  std::vector<int64_t> off(G);
  std::vector<std::thread> th;
  for (int64_t g = 0; g < G; ++g) {
    const int64_t lo = c.n * g / G, hi = c.n * (g + 1) / G;
    off[g] = lo;
    Call cs = c;
    cs.n = hi - lo;
    for (int i = 0; i < 7; ++i)
      if (c.cols[i].stride != 0)
        cs.cols[i].data = (const char*)c.cols[i].data + lo * c.cols[i].stride * (int64_t)in_sz[i];
    for (int i = 0; i < 6; ++i) if (c.outs[i]) cs.outs[i] = c.outs[i] + lo;
    if (c.status) cs.status = c.status + lo;
    if (c.region) cs.region = c.region + lo;
    set_ok(&outs[g].e1);
    set_ok(&outs[g].e2);
    th.emplace_back(shard_call, devs[g], cs, &outs[g], false, nullptr);
  }
  for (auto& t : th) t.join();
  return merge_shards(c.kind, outs, off, e1, e2);
}

// The shards' outcomes (shards in row order, row offsets off[g]) merged into
// the single-call one, and into this thread's fv_last_outcome.
int merge_shards(Kind kind, const std::vector<ShardOut>& outs, const std::vector<int64_t>& off, fv_error* e1,
                 fv_error* e2) {
  const int64_t G = (int64_t)outs.size();
  int64_t launches = 0, h2d = 0;
  for (int k = 0; k < FV_NCHECK; ++k) t_check_rows[k] = -1;
  for (int k = 0; k < 2; ++k) { t_exc_row[k] = -1; t_exc_code[k] = 0; }
  for (int64_t g = 0; g < G; ++g) {
    const ShardOut& o = outs[g];
    launches += o.launches;
    h2d += o.h2d_bytes;
    for (int k = 0; k < FV_NCHECK; ++k)
      if (o.check_rows[k] >= 0 && t_check_rows[k] < 0) t_check_rows[k] = o.check_rows[k] + off[g];
    for (int k = 0; k < 2; ++k)
      if (o.exc_row[k] >= 0 && t_exc_row[k] < 0) { t_exc_row[k] = o.exc_row[k] + off[g]; t_exc_code[k] = o.exc_code[k]; }
  }
  t_launches = launches;
  t_h2d_bytes = h2d;
  // errors: runtime / argument failures first, then the reference's order
  for (int64_t g = 0; g < G; ++g)
    if (outs[g].rc == FV_ERR_CUDA || outs[g].rc == FV_ERR_ARG) {
      if (e1) *e1 = outs[g].e1;
      if (e2) *e2 = outs[g].e2;
      return outs[g].rc;
    }
  // each error record merges on its own: the first failing check in the
  // reference's order at its lowest global row, else the lowest raising row
  // (shards are in row order, so the earliest shard holding one wins)
  bool any_batch[2] = {false, false}, any_exc[2] = {false, false};
  fv_error* dst[2] = {e1, e2};
  for (int k = 0; k < 2; ++k) {
    int best = -1;
    for (int64_t g = 0; g < G; ++g) {
      const fv_error& e = k ? outs[g].e2 : outs[g].e1;
      if (e.code != FV_ERR_BATCH) continue;
      const fv_error& b = k ? outs[best < 0 ? 0 : best].e2 : outs[best < 0 ? 0 : best].e1;
      if (best < 0 || e.kind < b.kind) best = (int)g;
    }
    if (best < 0)
      for (int64_t g = 0; g < G && best < 0; ++g)
        if ((k ? outs[g].e2 : outs[g].e1).code == FV_ERR_PYEXC) best = (int)g;
    fv_error merged;
    set_ok(&merged);
    if (best >= 0) {
      merged = k ? outs[best].e2 : outs[best].e1;
      shift_error(&merged, off[best]);
      any_batch[k] = merged.code == FV_ERR_BATCH;
      any_exc[k] = merged.code == FV_ERR_PYEXC;
    }
    if (dst[k]) *dst[k] = merged;
  }
  if (kind == KIND_PRICE_IV) {            // the price stage's failure is the call's
    if (any_batch[0]) return FV_ERR_BATCH;
    if (any_exc[0]) return FV_ERR_PYEXC;
    return any_batch[1] ? FV_ERR_BATCH : (any_exc[1] ? FV_ERR_PYEXC : FV_OK);
  }
  if (any_batch[0] || any_batch[1]) return FV_ERR_BATCH;
  return (any_exc[0] || any_exc[1]) ? FV_ERR_PYEXC : FV_OK;
}

// For host calls, broadcast columns must be readable on the device.
int dispatch(Call c, fv_error* e1, fv_error* e2) {
#if FV_CALL_TRACE
  t_ct0 = std::chrono::steady_clock::now();
  t_ctn = 0;
#endif
  t_launches = 0;
  t_h2d_bytes = 0;
  // fv_last_outcome describes THIS call, even when it fails before finish()
  for (int k = 0; k < FV_NCHECK; ++k) t_check_rows[k] = -1;
  for (int k = 0; k < 2; ++k) { t_exc_row[k] = -1; t_exc_code[k] = 0; }
  set_ok(e1);
  set_ok(e2);
  if (c.n < 0) return set_arg_err(e1, "n must be >= 0");
  if (c.model < 0 || c.model > 2) return set_arg_err(e1, "unknown model");
  if ((c.kind == KIND_IV || c.kind == KIND_PRICE_IV) && c.method != FV_METHOD_HALLEY && c.method != FV_METHOD_LBR)
    return set_arg_err(e1, "unknown IV method");
  for (int i = 0; i < 7; ++i)
    if (!c.cols[i].data) return set_arg_err(e1, "null input column");
  // memory space: all device or all host
  // memory space: all device (one device) or all host
  int ndev = 0, nptr = 0, pdev = -1;
  bool mixed_dev = false;
  auto note = [&](const void* p) {
    int d = -1;
    ++nptr;
    if (is_device_ptr(p, &d)) {
      ++ndev;
      if (pdev < 0) pdev = d;
      else if (d != pdev) mixed_dev = true;
    }
  };
  for (int i = 0; i < 7; ++i) note(c.cols[i].data);
  for (int i = 0; i < 6; ++i) if (c.outs[i]) note(c.outs[i]);
  if (c.status) note(c.status);
  if (c.region) note(c.region);
  bool device = ndev == nptr;
  if (ndev != 0 && !device) return set_arg_err(e1, "all pointers of a call must be device pointers or all host pointers");
  if (mixed_dev) return set_arg_err(e1, "device pointers of a call must all be on one device");
  // device calls run on the device that owns the columns, whatever the
  // thread's current device is (restored on return)
  DeviceGuard guard;
  if (device) {
    int cur = -1;
    cudaError_t ce0 = cudaGetDevice(&cur);
    if (ce0 != cudaSuccess) return set_cuda_err(e1, ce0);
    if (cur != pdev) {
      if ((ce0 = cudaSetDevice(pdev)) != cudaSuccess) return set_cuda_err(e1, ce0);
      guard.prev = cur;
    }
    if (t_user_stream_set && t_user_stream) {
      int sdev = -1;
      if (cudaStreamGetDevice(t_user_stream, &sdev) != cudaSuccess) {
        cudaGetLastError();
        return set_arg_err(e1, "the stream set by fv_set_stream is not a valid CUDA stream");
      }
      if (sdev != pdev) {
        char msg[160];
        snprintf(msg, sizeof(msg), "the stream set by fv_set_stream belongs to device %d, the columns to device %d",
                 sdev, pdev);
        return set_arg_err(e1, msg);
      }
    }
  }
  if (!device && !t_in_shard) {
    std::vector<int> devs = devices_for_host_calls();
    if (devs.size() > 1 && c.n >= (int64_t)devs.size() * kMinShardRows) return dispatch_sharded(c, devs, e1, e2);
  }
  CT_MARK();                                   // [0] pointer classification done
  DevWork* w = nullptr;
  cudaError_t ce = get_work(&w);
  if (ce != cudaSuccess) return set_cuda_err(e1, ce);
  std::lock_guard<std::mutex> g(w->mu);
  CT_MARK();                                   // [1] work + lock
  // broadcast scalars of a host call: checked once on the host and copied
  // into the device's scalar slot.  A device call does not read them back
  // (a synchronous device -> host copy per column, ~10 us each, before any
  // launch): its kernels check them like any column, and every row failing
  // such a check puts the reported row at 0, as the host check does.
  bool bc[7];
  double vals[7] = {0, 0, 0, 0, 0, 0, 0};
  int flag_val = 0;
  for (int i = 0; i < 7; ++i) bc[i] = c.cols[i].stride == 0;
  c.bcast_dev = device;
  if (!device) {
    if (bc[0]) flag_val = *(const int8_t*)c.cols[0].data;
    for (int i = 1; i < 7; ++i)
      if (bc[i]) vals[i] = *(const double*)c.cols[i].data;
  }
  uint32_t bbits = (c.n > 0 && !device) ? bcast_checks(c, vals, flag_val, bc) : 0;
  if (c.kind == KIND_PRICE_IV && c.n > 0 && !device) {
    // the IV stage reads the same broadcast columns; its price column is the
    // price stage's n-row output (never broadcast)
    Call ci = c;
    ci.kind = KIND_IV;
    bool bci[7];
    for (int i = 0; i < 7; ++i) bci[i] = bc[i];
    bci[6] = false;
    c.bbits_iv = bcast_checks(ci, vals, flag_val, bci);
  }
  if (!device) {
    // device copies of the broadcast scalars (the DevWork's slot; host calls
    // are synchronous, so the slot is free again when the next one starts)
    double tmp[8] = {0};
    int8_t f8 = (int8_t)flag_val;
    memcpy(&tmp[7], &f8, 1);
    for (int i = 1; i < 7; ++i) tmp[i] = vals[i];
    // On the host pipeline's first stream, ahead of its status reset and the
    // `ready` event every slot stream waits on: a synchronous cudaMemcpy from
    // pageable memory may return before its DMA lands, and the library's
    // streams do not synchronise with the legacy default stream, so a
    // kernel could read the previous call's scalars (seen once in ~10^6 calls:
    // a 1-row batch_iv solving the preceding batch_price's sigma).
    if ((ce = cudaMemcpyAsync(w->scal, tmp, sizeof(tmp), cudaMemcpyHostToDevice, w->streams[0])) != cudaSuccess)
      return set_cuda_err(e1, ce);
    t_h2d_bytes += (int64_t)sizeof(tmp);
    const int8_t* dflag = (const int8_t*)(w->scal + 7);
    for (int i = 0; i < 7; ++i)
      if (bc[i]) c.cols[i].data = (i == 0) ? (const void*)dflag : (const void*)(w->scal + i);
  }
  int rc;
  if (device) {
    cudaStream_t s = t_user_stream_set ? t_user_stream : w->streams[0];
    rc = run_device(w, c, s, bbits, e1, e2);
  } else {
    rc = run_host(w, c, bbits, e1, e2);
  }
  return rc;
}

Call make_call(Kind kind, int model, int method, fv_col flag, fv_col un, fv_col k, fv_col t,
               fv_col r, fv_col q, fv_col last, int64_t n) {
  Call c;
  memset(&c, 0, sizeof(c));
  c.kind = kind; c.model = model; c.method = method;
  c.cols[0] = flag; c.cols[1] = un; c.cols[2] = k; c.cols[3] = t;
  c.cols[4] = r; c.cols[5] = q; c.cols[6] = last;
  c.n = n;
  return c;
}

}  // namespace

extern "C" {

FV_API int fv_batch_price(int model, fv_col flag, fv_col underlying, fv_col strike, fv_col t,
                          fv_col r, fv_col q, fv_col sigma, int64_t n, double* price,
                          fv_error* err) {
  Call c = make_call(KIND_PRICE, model, 0, flag, underlying, strike, t, r, q, sigma, n);
  c.outs[0] = price;
  if (!price && n > 0) return set_arg_err(err, "null output");
  return dispatch(c, err, nullptr);
}

FV_API int fv_batch_iv(int model, int method, fv_col flag, fv_col underlying, fv_col strike,
                       fv_col t, fv_col r, fv_col q, fv_col price, int64_t n, double* iv,
                       int8_t* status, int8_t* region, fv_error* err) {
  Call c = make_call(KIND_IV, model, method, flag, underlying, strike, t, r, q, price, n);
  c.outs[0] = iv;
  c.status = status;
  c.region = region;
  if ((!iv || !status) && n > 0) return set_arg_err(err, "null output");
  return dispatch(c, err, nullptr);
}

FV_API int fv_batch_greeks(int model, fv_col flag, fv_col underlying, fv_col strike, fv_col t,
                           fv_col r, fv_col q, fv_col sigma, int64_t n, double* delta,
                           double* gamma, double* theta, double* rho, double* vega,
                           int8_t* status, fv_error* err) {
  Call c = make_call(KIND_GREEKS, model, 0, flag, underlying, strike, t, r, q, sigma, n);
  c.outs[1] = delta; c.outs[2] = gamma; c.outs[3] = theta; c.outs[4] = rho; c.outs[5] = vega;
  c.status = status;
  c.want_greeks = true;
  if ((!delta || !gamma || !theta || !rho || !vega || !status) && n > 0)
    return set_arg_err(err, "null output");
  fv_error unused;
  return dispatch(c, &unused, err);
}

FV_API int fv_price_greeks(int model, fv_col flag, fv_col underlying, fv_col strike, fv_col t,
                           fv_col r, fv_col q, fv_col sigma, int64_t n, double* price,
                           double* delta, double* gamma, double* theta, double* rho,
                           double* vega, int8_t* status, fv_error* err_price,
                           fv_error* err_greeks) {
  Call c = make_call(KIND_PRICE_GREEKS, model, 0, flag, underlying, strike, t, r, q, sigma, n);
  c.outs[0] = price;
  c.outs[1] = delta; c.outs[2] = gamma; c.outs[3] = theta; c.outs[4] = rho; c.outs[5] = vega;
  c.status = status;
  c.want_price = price != nullptr;
  c.want_greeks = delta || gamma || theta || rho || vega || status;
  if (!c.want_price && !c.want_greeks) return set_arg_err(err_price, "no outputs requested");
  if (c.want_greeks && (!delta || !gamma || !theta || !rho || !vega || !status))
    return set_arg_err(err_price, "Greeks outputs must be all set or all NULL");
  fv_error ep, eg;
  int rc = dispatch(c, &ep, &eg);
  if (err_price) *err_price = ep;
  if (err_greeks) *err_greeks = eg;
  if (rc == FV_ERR_PYEXC) {
    bool any = (c.want_price && ep.code) || (c.want_greeks && eg.code);
    if (!any) rc = FV_OK;
    if (!c.want_price && err_price) set_ok(err_price);
    if (!c.want_greeks && err_greeks) set_ok(err_greeks);
  }
  return rc;
}

FV_API int fv_price_iv(int model, int method, fv_col flag, fv_col underlying, fv_col strike,
                       fv_col t, fv_col r, fv_col q, fv_col sigma, int64_t n, double* price,
                       double* iv, int8_t* status, int8_t* region, fv_error* err_price,
                       fv_error* err_iv) {
  Call c = make_call(KIND_PRICE_IV, model, method, flag, underlying, strike, t, r, q, sigma, n);
  c.outs[0] = price;
  c.outs[1] = iv;
  c.status = status;
  c.region = region;
  if ((!price || !iv || !status) && n > 0) return set_arg_err(err_price, "null output");
  fv_error ep, ei;
  const int rc = dispatch(c, &ep, &ei);
  if (rc == FV_ERR_CUDA || rc == FV_ERR_ARG) ei = ep;
  if (err_price) *err_price = ep;
  if (err_iv) *err_iv = ei;
  return rc;
}

FV_API int fv_run_shards(int kind, int model, int method, int nshard, const fv_shard* shards,
                         fv_error* err1, fv_error* err2) {
  set_ok(err1);
  set_ok(err2);
  for (int k = 0; k < FV_NCHECK; ++k) t_check_rows[k] = -1;
  for (int k = 0; k < 2; ++k) { t_exc_row[k] = -1; t_exc_code[k] = 0; }
  t_launches = 0;
  t_h2d_bytes = 0;
  if (kind < FV_KIND_PRICE || kind > FV_KIND_PRICE_IV) return set_arg_err(err1, "unknown call kind");
  if (nshard < 1 || !shards) return set_arg_err(err1, "no shards");
  int have = 0;
  if (cudaGetDeviceCount(&have) != cudaSuccess) { cudaGetLastError(); have = 0; }
  std::vector<ShardOut> outs(nshard);
  std::vector<int64_t> off(nshard);
  std::vector<Call> calls(nshard);
  int64_t row = 0;
  for (int g = 0; g < nshard; ++g) {
    const fv_shard& sh = shards[g];
    if (sh.device < 0 || sh.device >= have) return set_arg_err(err1, "shard device out of range");
    if (sh.n < 0) return set_arg_err(err1, "shard n must be >= 0");
    Call& c = calls[g];
    c = make_call((Kind)kind, model, method, sh.cols[0], sh.cols[1], sh.cols[2], sh.cols[3], sh.cols[4],
                  sh.cols[5], sh.cols[6], sh.n);
    for (int i = 0; i < 6; ++i) c.outs[i] = sh.outs[i];
    c.status = sh.status;
    c.region = (kind == FV_KIND_IV || kind == FV_KIND_PRICE_IV) ? sh.region : nullptr;
    bool ok = true;
    switch (kind) {
      case FV_KIND_PRICE: ok = sh.outs[0] != nullptr; break;
      case FV_KIND_IV: ok = sh.outs[0] && sh.status; break;
      case FV_KIND_GREEKS:
        c.outs[0] = nullptr;
        ok = sh.outs[1] && sh.outs[2] && sh.outs[3] && sh.outs[4] && sh.outs[5] && sh.status;
        c.want_greeks = true;
        break;
      case FV_KIND_PRICE_GREEKS:
        c.want_price = sh.outs[0] != nullptr;
        c.want_greeks = sh.outs[1] || sh.outs[2] || sh.outs[3] || sh.outs[4] || sh.outs[5] || sh.status;
        ok = (c.want_price || c.want_greeks) &&
             (!c.want_greeks || (sh.outs[1] && sh.outs[2] && sh.outs[3] && sh.outs[4] && sh.outs[5] && sh.status));
        break;
      case FV_KIND_PRICE_IV: ok = sh.outs[0] && sh.outs[1] && sh.status; break;
    }
    if (!ok && sh.n > 0) return set_arg_err(err1, "shard outputs missing for this call kind");
    off[g] = row;
    row += sh.n;
    set_ok(&outs[g].e1);
    set_ok(&outs[g].e2);
  }
  // one host thread per shard, each on its shard's device and stream (the
  // shards of one device run one after the other on it: DevWork's lock)
  std::vector<std::thread> th;
  for (int g = 0; g < nshard; ++g)
    th.emplace_back(shard_call, shards[g].device, calls[g], &outs[g], true, shards[g].stream);
  for (auto& t : th) t.join();
  fv_error m1, m2;
  int rc = merge_shards((Kind)kind, outs, off, &m1, &m2);
  if (kind == FV_KIND_PRICE_GREEKS && rc == FV_ERR_PYEXC) {
    const bool wp = calls[0].want_price, wg = calls[0].want_greeks;
    if (!((wp && m1.code) || (wg && m2.code))) rc = FV_OK;
    if (!wp) set_ok(&m1);
    if (!wg) set_ok(&m2);
  }
  if (kind == FV_KIND_PRICE_IV && (rc == FV_ERR_CUDA || rc == FV_ERR_ARG)) m2 = m1;
  if (err1) *err1 = m1;
  if (err2) *err2 = m2;
  return rc;
}

FV_API int fv_gather(void* dst, int dst_device, void* dst_stream, int nshard, const void* const* src,
                     const int* src_device, const int64_t* bytes) {
  if (nshard < 0 || (nshard > 0 && (!src || !src_device || !bytes)) || !dst) return FV_ERR_ARG;
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return FV_ERR_CUDA;
  DeviceGuard guard;
  guard.prev = prev;
  if (cudaSetDevice(dst_device) != cudaSuccess) { cudaGetLastError(); return FV_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)dst_stream;
  int64_t o = 0;
  for (int g = 0; g < nshard; ++g) {
    if (bytes[g] < 0) return FV_ERR_ARG;
    if (src_device[g] != dst_device) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, dst_device, src_device[g]);
      if (can) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(src_device[g], 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      }
    }
    if (bytes[g] && cudaMemcpyPeerAsync((char*)dst + o, dst_device, src[g], src_device[g], (size_t)bytes[g], s) !=
                        cudaSuccess)
      return FV_ERR_CUDA;
    o += bytes[g];
  }
  return cudaStreamSynchronize(s) == cudaSuccess ? FV_OK : FV_ERR_CUDA;
}

FV_API int fv_set_stream(void* stream) {
  t_user_stream = (cudaStream_t)stream;
  t_user_stream_set = true;
  return FV_OK;
}

FV_API int fv_set_devices(const int* ids, int n) {
  int have = 0;
  if (cudaGetDeviceCount(&have) != cudaSuccess) { cudaGetLastError(); have = 0; }
  if (n < 0 || (n > 0 && !ids)) return FV_ERR_ARG;
  for (int i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= have) return FV_ERR_ARG;
  std::lock_guard<std::mutex> g(g_dev_mu);
  g_devices.assign(ids, ids + n);
  return FV_OK;
}

FV_API int fv_get_devices(int* ids, int cap) {
  std::lock_guard<std::mutex> g(g_dev_mu);
  for (int i = 0; i < (int)g_devices.size() && i < cap; ++i) ids[i] = g_devices[i];
  return (int)g_devices.size();
}

FV_API int fv_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return 0; }
  return n;
}

FV_API const char* fv_version(void) { return FV_VERSION; }

FV_API int fv_set_chunk_rows(int64_t rows) {
  if (rows < 1024) return FV_ERR_ARG;
  g_chunk_rows = rows;
  return FV_OK;
}

FV_API int64_t fv_last_launch_count(void) { return t_launches; }

FV_API int64_t fv_last_h2d_bytes(void) { return t_h2d_bytes; }

#if FV_CALL_TRACE
// diagnostic builds only: the last device call's host-side stage timestamps (us)
FV_API int fv_call_trace(double* out, int cap) {
  for (int i = 0; i < t_ctn && i < cap; ++i) out[i] = t_ct[i];
  return t_ctn;
}
#endif

FV_API int fv_host_find_runs(const void* data, int elem, int64_t n, int64_t budget, int32_t* starts, void* vals,
                             int64_t* nruns) {
  if (!data || !starts || !vals || !nruns || (elem != 1 && elem != 8) || n < 1 || n >= ((int64_t)1 << 31))
    return FV_ERR_ARG;
  std::vector<RunScan> jobs(1);
  jobs[0] = {data, elem, n, budget, starts, vals, -1, nullptr};
  find_runs_batch(jobs);
  *nruns = jobs[0].nr;
  return FV_OK;
}

FV_API int fv_set_round_rows(int64_t lbr_rows, int64_t halley_rows) {
  if (lbr_rows < 0 || halley_rows < 0 || halley_rows > (1ll << 26)) return FV_ERR_ARG;   // int32 queue entries
  g_lbr_round = lbr_rows ? lbr_rows : (1ll << FV_LBR_ROUND_LOG2);
  g_halley_round = halley_rows ? halley_rows : (1ll << 26);
  return FV_OK;
}

FV_API int fv_set_span_timing(int on) {
  t_span = on != 0;
  return FV_OK;
}

FV_API double fv_last_span_ms(void) { return (double)t_span_ms; }

FV_API int fv_set_kernel_timing(int on) {
  t_timing = on != 0;
  return FV_OK;
}

FV_API int fv_kernel_times(double* ms, int64_t* launches) {
  for (int k = 0; k < FV_NKERNEL; ++k) { ms[k] = 0.0; launches[k] = 0; }
  int rc = FV_OK;
  for (TimedLaunch& tl : t_timed) {
    float e = 0.0f;
    if (cudaEventSynchronize(tl.b) != cudaSuccess || cudaEventElapsedTime(&e, tl.a, tl.b) != cudaSuccess)
      rc = FV_ERR_CUDA;
    ms[tl.id] += e;
    launches[tl.id] += 1;
    cudaEventDestroy(tl.a);
    cudaEventDestroy(tl.b);
  }
  t_timed.clear();
  return rc;
}

FV_API const char* fv_kernel_name(int id) {
  return (id >= 0 && id < FV_NKERNEL) ? kKernelNames[id] : "";
}

FV_API int fv_selftest_div_const(int64_t n, uint64_t seed, int64_t* mismatches) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) return FV_ERR_CUDA;
  cudaMemset(d, 0, sizeof(*d));
  k_selftest_div_const<<<148 * 8, 256>>>(n, seed, d);
  unsigned long long h = 0;
  cudaError_t ce = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (ce != cudaSuccess) return FV_ERR_CUDA;
  *mismatches = (int64_t)h;
  return FV_OK;
}

// Exhaustive check of the table: every fp32 |x| in [2^-13, 2^5): violations
// of b_lo(x) >= g_qlo_tab[bin(x)] -> out[0]; the smallest b_lo / bound ratio
// seen (as ordered bits of a positive double) -> out[1]; points -> out[2].
__global__ void k_selftest_qlo(uint32_t lo_bits, uint32_t hi_bits, unsigned long long* out) {
  unsigned long long bad = 0, cnt = 0;
  double worst = 1e300;
  for (uint64_t b = lo_bits + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < hi_bits;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const double ax = (double)__uint_as_float((uint32_t)b);
    const int k = fx_qlo_bin(ax);
    const double L = (k >= 0) ? (double)g_qlo_tab[k] : 0.0;
    const double ex = qlo_b_lo(ax);
    if (!(ex >= L)) ++bad;
    if (L > 0.0) worst = fmin(worst, ex / L);
    ++cnt;
  }
  atomicAdd(out, bad);
  atomicMin(out + 1, (unsigned long long)__double_as_longlong(worst));
  atomicAdd(out + 2, cnt);
}
FV_API int fv_selftest_qlo(int64_t* violations, double* min_ratio, int64_t* points) {
  DevWork* w = nullptr;
  if (get_work(&w) != cudaSuccess) return FV_ERR_CUDA;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 3 * sizeof(unsigned long long)) != cudaSuccess) return FV_ERR_CUDA;
  unsigned long long init[3] = {0, ~0ull, 0};
  cudaMemcpy(d, init, sizeof(init), cudaMemcpyHostToDevice);
  const float lo = 0x1p-13f, hi = 0x1p5f;
  uint32_t lob, hib;
  memcpy(&lob, &lo, 4);
  memcpy(&hib, &hi, 4);
  k_selftest_qlo<<<148 * 16, 256>>>(lob, hib, d);
  unsigned long long h[3] = {0, 0, 0};
  const cudaError_t ce = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (ce != cudaSuccess) return FV_ERR_CUDA;
  *violations = (int64_t)h[0];
  memcpy(min_ratio, &h[1], 8);
  *points = (int64_t)h[2];
  return 0;
}

FV_API int fv_selftest_fast(int64_t n, uint64_t seed, int64_t* mismatches, int64_t* flagged) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(*d) * 2 * FX_NTEST) != cudaSuccess) return FV_ERR_CUDA;
  cudaMemset(d, 0, sizeof(*d) * 2 * FX_NTEST);
  k_selftest_fast<<<148 * 8, 256>>>(n, seed, d, d + FX_NTEST);
  unsigned long long h[2 * FX_NTEST];
  cudaError_t ce = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (ce != cudaSuccess) return FV_ERR_CUDA;
  for (int k = 0; k < FX_NTEST; ++k) { mismatches[k] = (int64_t)h[k]; flagged[k] = (int64_t)h[FX_NTEST + k]; }
  return FV_OK;
}

FV_API int fv_last_outcome(int64_t* check_rows, int64_t* exc_rows, int32_t* exc_codes) {
  for (int c = 0; c < FV_NCHECK; ++c) check_rows[c] = t_check_rows[c];
  for (int k = 0; k < 2; ++k) { exc_rows[k] = t_exc_row[k]; exc_codes[k] = t_exc_code[k]; }
  return FV_OK;
}

// Measured FP64 DFMA issue rate of the current device (DFMA instructions per
// second across the chip), timed with CUDA events.
FV_API int fv_probe_fp64_peak(double* dfma_per_s, double* seconds) {
  int dev = 0, sm = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FV_ERR_CUDA;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_fp64_probe, 256, 0);
  if (per_sm < 1) per_sm = 1;
  int blocks = sm * per_sm;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * blocks * 256) != cudaSuccess) return FV_ERR_CUDA;
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  // alone on the device (work still draining on the library's non-blocking
  // streams would share the SMs), the fastest of three timed runs
  cudaError_t ce = cudaDeviceSynchronize();
  k_fp64_probe<<<blocks, 256>>>(out, 64, 0.999999, 1e-7);          // warm-up
  float ms = 0.f;
  for (int rep = 0; rep < 3 && ce == cudaSuccess; ++rep) {
    cudaEventRecord(e0);
    k_fp64_probe<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    ce = cudaEventSynchronize(e1);
    float m = 0.f;
    cudaEventElapsedTime(&m, e0, e1);
    if (rep == 0 || m < ms) ms = m;
  }
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cudaFree(out);
  if (ce != cudaSuccess) return FV_ERR_CUDA;
  double dfma = (double)blocks * 256.0 * iters * 16.0 * 8.0;
  if (dfma_per_s) *dfma_per_s = dfma / (ms * 1e-3);
  if (seconds) *seconds = ms * 1e-3;
  return FV_OK;
}

}  // extern "C"

