/* fastvol_b200.h -- C ABI of the B200 batched pricing / Greeks / implied-vol
 * library (libfastvol_b200.so, built from paper_2604_27210_b200/csrc).
 *
 * Drop-in boundary for the reference's batch engine (fastvol 0.1.0,
 * /root/reference/pkg/src/fastvol/batch.py).  Each entry point replaces one
 * `fill(start, stop)` loop + `_run_chunked(fill, n)` pair of the reference;
 * the SPEC's intended binding shape (bind_batch_price,
 * bind_batch_iv(model, method, buffers) -> (iv, status), bind_all_greeks ->
 * five buffers) maps onto:
 *
 *   fv_batch_price   <- batch.py:181-203  batch_price   (fill :195-198)
 *   fv_batch_iv      <- batch.py:206-247  batch_iv      (fill :223-241)
 *   fv_batch_greeks  <- batch.py:250-280  batch_greeks  (fill :263-274)
 *   fv_price_greeks  <- batch_price + batch_greeks on the same columns, one
 *                       fused pass (shared d1/d2/Phi/phi), two error records
 *   fv_price_iv      <- batch_price then batch_iv on the price column it
 *                       produced (bench.py:19-40 synthetic_chain + run_bench,
 *                       SURVEY 8(f) rank 3): one call, the price column stays
 *                       on the device between the stages, two error records
 *
 * Columns are structure-of-arrays: a column is a pointer
 * plus an element stride; stride 0 broadcasts element 0 (the reference's
 * length-1 columns, batch.py:91-101).  Flags are int8 +1 (call) / -1 (put)
 * (the result of batch.py:parse_flags).  All pointers of one call live in the
 * same memory space: either all device memory (kernels run in place on the
 * current device, on the stream set by fv_set_stream) or all host memory
 * (pinned or pageable; the library pipelines H2D / kernel / D2H in chunks).
 *
 * Semantics are the reference's, bit for bit:
 *   - validation (batch.py:104-124, :144-147): the first failing check in the
 *     reference's order, at its lowest row, is reported as FV_ERR_BATCH with
 *     fv_error.kind / index / column (BatchError(kind, index, detail));
 *   - per-row numeric failures stay in-band: NaN + status code;
 *   - a row whose reference execution raises a Python exception (e.g.
 *     OverflowError from math.exp) aborts the batch: FV_ERR_PYEXC with the
 *     lowest such row in fv_error.index and the exception in fv_error.kind.
 * Reentrant; no global mutable state besides the per-thread stream setting
 * and a per-device workspace cache (mutex-protected).
 */
#ifndef FASTVOL_B200_H
#define FASTVOL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FV_API __attribute__((visibility("default")))

/* models (fastvol/models.py:27-48) */
#define FV_MODEL_BLACK76 0
#define FV_MODEL_BLACK_SCHOLES 1
#define FV_MODEL_BLACK_SCHOLES_MERTON 2

/* IV methods (batch.py:212) */
#define FV_METHOD_HALLEY 0
#define FV_METHOD_LBR 1

/* IV status codes (fastvol/solver.py:14-19, in declaration order) */
#define FV_STATUS_CONVERGED 0
#define FV_STATUS_FELL_BACK_TO_BISECTION 1
#define FV_STATUS_BELOW_INTRINSIC 2
#define FV_STATUS_ABOVE_UPPER_BOUND 3
#define FV_STATUS_MAX_ITERATIONS 4
/* Greeks status codes (batch.py:270-274) */
#define FV_STATUS_OK 0
#define FV_STATUS_STEP_FUNCTION_EDGE 1

/* return codes */
#define FV_OK 0
#define FV_ERR_BATCH 1   /* BatchError: kind = FV_CHECK_*, index, column */
#define FV_ERR_PYEXC 2   /* reference raised: kind = FV_EXC_*, index = row */
#define FV_ERR_CUDA 3    /* CUDA runtime failure (message has the text) */
#define FV_ERR_ARG 4     /* bad arguments (mixed memory spaces, bad model...) */

/* validation checks, in the reference's evaluation order (fv_error.kind for
 * FV_ERR_BATCH).  BadFlag: a flag that is not +1/-1 (parse_flags). */
#define FV_CHECK_BAD_FLAG 0
#define FV_CHECK_NONFINITE_UNDERLYING 1
#define FV_CHECK_NONFINITE_STRIKE 2
#define FV_CHECK_NONFINITE_T 3
#define FV_CHECK_NONFINITE_R 4
#define FV_CHECK_NONFINITE_Q 5
#define FV_CHECK_NONFINITE_LAST 6     /* sigma (price/greeks) or price (iv) */
#define FV_CHECK_POSITIVE_UNDERLYING 7
#define FV_CHECK_POSITIVE_STRIKE 8
#define FV_CHECK_NONNEG_T 9
#define FV_CHECK_NONNEG_SIGMA 10
#define FV_CHECK_DIVIDEND 11          /* q != 0 with a non-BSM model */
#define FV_NCHECK 12

/* Python exceptions the reference can raise mid-batch (fv_error.kind for
 * FV_ERR_PYEXC) */
#define FV_EXC_MATH_RANGE 1     /* OverflowError('math range error') */
#define FV_EXC_MATH_DOMAIN 2    /* ValueError('math domain error') */
#define FV_EXC_ZERO_DIV 3       /* ZeroDivisionError('float division by zero') */
#define FV_EXC_POW_RANGE 4      /* OverflowError(34, 'Numerical result out of range') */
#define FV_EXC_DOM_FK 5         /* DomainError('F and K must be positive') */
#define FV_EXC_DOM_ATM_BETA 6   /* DomainError('atm_inverse requires beta in (0, 1), got <value>') */
#define FV_EXC_DOM_INVCDF_P 7   /* DomainError('inv_norm_cdf requires p in (0, 1), got <value>') */
#define FV_EXC_DOM_NB_X 8       /* DomainError('normalized_black requires x <= 0, got <value>') */
#define FV_EXC_DOM_NB_S 9       /* DomainError('normalized_black requires s > 0, got <value>') */
#define FV_EXC_DOM_OBJ_S 10     /* DomainError('objective_branch requires s > 0, got <value>') */

typedef struct fv_col {
  const void* data;   /* double* (flag column: int8_t*) */
  int64_t stride;     /* in elements; 0 = broadcast data[0] */
} fv_col;

typedef struct fv_error {
  int32_t code;        /* FV_OK / FV_ERR_* */
  int32_t kind;        /* FV_CHECK_* or FV_EXC_* */
  int64_t index;       /* first offending row */
  int32_t column;      /* FV_ERR_BATCH: 0 flag, 1 underlying, 2 strike, 3 t, 4 r, 5 q, 6 sigma/price */
  int32_t value_is_numpy; /* FV_EXC_DOM_* with a value: the reference value was a numpy.float64 */
  double value;        /* the value a DomainError message quotes */
  char message[256];   /* human-readable, reference wording where it exists */
} fv_error;

/* batch_price (batch.py:181-203): price[i] for every row. */
FV_API int fv_batch_price(int model, fv_col flag, fv_col underlying, fv_col strike, fv_col t,
                          fv_col r, fv_col q, fv_col sigma, int64_t n, double* price,
                          fv_error* err);

/* batch_iv (batch.py:206-247): iv[i] (NaN unless status is converged or
 * fell_back_to_bisection) and status[i] (FV_STATUS_*).  region may be NULL;
 * otherwise it receives the LBR region (0 far_low, 1 near_low, 2 near_high,
 * 3 far_high, -1 none: bounds/ATM/Halley) for diagnostics. */
FV_API int fv_batch_iv(int model, int method, fv_col flag, fv_col underlying, fv_col strike,
                       fv_col t, fv_col r, fv_col q, fv_col price, int64_t n, double* iv,
                       int8_t* status, int8_t* region, fv_error* err);

/* batch_greeks (batch.py:250-280): per-day theta, per-1% vega/rho
 * (greeks.py:93-96); status FV_STATUS_OK / FV_STATUS_STEP_FUNCTION_EDGE. */
FV_API int fv_batch_greeks(int model, fv_col flag, fv_col underlying, fv_col strike, fv_col t,
                           fv_col r, fv_col q, fv_col sigma, int64_t n, double* delta,
                           double* gamma, double* theta, double* rho, double* vega,
                           int8_t* status, fv_error* err);

/* Fused batch_price + batch_greeks over the same columns.  Any output may be
 * NULL (not computed).  err_price / err_greeks get the outcome each separate
 * reference call would have had; the return code is the worse of the two. */
FV_API int fv_price_greeks(int model, fv_col flag, fv_col underlying, fv_col strike, fv_col t,
                           fv_col r, fv_col q, fv_col sigma, int64_t n, double* price,
                           double* delta, double* gamma, double* theta, double* rho,
                           double* vega, int8_t* status, fv_error* err_price,
                           fv_error* err_greeks);

/* Price -> IV round trip (the reference's bench harness,
 * bench.py:19-40): price[i] = batch_price(model, ..., sigma)[i], then
 * iv[i] / status[i] / region[i] = batch_iv(model, method, ..., price=price)
 * on that column.  One call: the inputs are read (host calls: copied) once,
 * the price column goes from the pricing kernel to the IV passes in device
 * memory, and price + iv + status come back together.  err_price is
 * batch_price's outcome; err_iv is batch_iv's on the produced prices, which
 * the reference only reaches when batch_price succeeded -- the return code is
 * err_price's when it failed, else err_iv's.  region may be NULL. */
FV_API int fv_price_iv(int model, int method, fv_col flag, fv_col underlying, fv_col strike,
                       fv_col t, fv_col r, fv_col q, fv_col sigma, int64_t n, double* price,
                       double* iv, int8_t* status, int8_t* region, fv_error* err_price,
                       fv_error* err_iv);

/* ---- one logical batch over several devices, device-resident
 * Each shard is a contiguous row range of the logical batch (shards in row
 * order) whose columns and outputs live on `device`; every shard runs from
 * its own host thread on its device and stream (NULL = that device's legacy
 * default stream).  No exchange between shards: every output row depends on
 * its input row only.  The outcome is the single-call one -- the first
 * failing check in the reference's order at its lowest GLOBAL row, else the
 * lowest raising row -- with err1 = the price / IV (price stage of
 * FV_KIND_PRICE_IV) record and err2 = the Greeks (IV stage) record, as the
 * single-device entry points report them.  fv_last_outcome is the merged
 * one, in global rows. */
#define FV_KIND_PRICE 0          /* fv_batch_price:  outs[0] = price */
#define FV_KIND_IV 1             /* fv_batch_iv:     outs[0] = iv, status (+ region) */
#define FV_KIND_GREEKS 2         /* fv_batch_greeks: outs[1..5], status */
#define FV_KIND_PRICE_GREEKS 3   /* fv_price_greeks: outs[0] and/or outs[1..5] + status */
#define FV_KIND_PRICE_IV 4       /* fv_price_iv:     outs[0] = price, outs[1] = iv, status (+ region) */
typedef struct fv_shard {
  int device;          /* CUDA device owning this shard's pointers */
  void* stream;        /* cudaStream_t on that device (NULL = its legacy default stream) */
  fv_col cols[7];      /* flag, underlying, strike, t, r, q, sigma | price */
  int64_t n;           /* rows of this shard */
  double* outs[6];     /* price|iv, delta, gamma, theta, rho, vega (FV_KIND_PRICE_IV: price, iv) */
  int8_t* status;
  int8_t* region;      /* optional (IV kinds) */
} fv_shard;
FV_API int fv_run_shards(int kind, int model, int method, int nshard, const fv_shard* shards,
                         fv_error* err1, fv_error* err2);

/* Gather per-shard device buffers into one buffer on dst_device (NVLink /
 * NVSwitch peer copies where peer access is available, else staged by the
 * driver): src[g] (bytes[g] bytes on src_device[g]) lands at dst + the sum of
 * the previous bytes.  Ordered on dst_stream (a stream of dst_device, NULL =
 * its legacy default stream); returns when the data is in place. */
FV_API int fv_gather(void* dst, int dst_device, void* dst_stream, int nshard, const void* const* src,
                     const int* src_device, const int64_t* bytes);

/* Stream used by device-pointer calls made from the calling thread
 * (cudaStream_t; NULL = the device's legacy default stream, which is what
 * torch's default stream is).  A thread that never calls it uses the
 * library's own non-blocking stream (ordered with nothing else: the call is
 * synchronous, but inputs must be complete before it). */
FV_API int fv_set_stream(void* stream);

/* Number of CUDA devices visible; library version string. */
FV_API int fv_device_count(void);
/* Devices for host-pointer calls: with n >= 2, a host call of
 * at least n * 2^20 rows is split into n contiguous row shards, one host
 * thread and one device each (ids may repeat), results written straight into
 * the caller's buffers; errors and fv_last_outcome are the single-device
 * ones.  n = 0 restores the default (the calling thread's current device).
 * Device-pointer calls run on the device that owns the pointers (all on one
 * device, else FV_ERR_ARG); the thread's current device is restored after the
 * call.  A stream set by fv_set_stream must belong to that device. */
FV_API int fv_set_devices(const int* ids, int n);
FV_API int fv_get_devices(int* ids, int cap);
FV_API const char* fv_version(void);

/* Host-pointer calls: rows per pipelined chunk (default 1<<22). */
FV_API int fv_set_chunk_rows(int64_t rows);

/* Kernels launched by this thread's last call (instrumentation for the
 * bench's gpu_launches count). */
FV_API int64_t fv_last_launch_count(void);

/* Bytes this thread's last host-pointer call moved host -> device: streamed
 * columns, the run-length form of piecewise-constant ones (a chunk whose
 * column is at most rows/64 runs of one value travels as (first row, value)
 * runs and is rebuilt in device memory), broadcast scalars.  0 for
 * device-pointer calls. */
FV_API int64_t fv_last_h2d_bytes(void);

/* The host side of that transport on its own (no device needed): the runs of
 * data[0, n) (elem 8: 64-bit values compared bit for bit; elem 1: flags) into
 * starts[0..nr] (starts[nr] = n) and vals[0..nr), on the library's copy
 * threads.  *nruns = nr, or -1 when the column has more than `budget` runs. */
FV_API int fv_host_find_runs(const void* data, int elem, int64_t n, int64_t budget, int32_t* starts,
                             void* vals, int64_t* nruns);

/* Testing knob: rows per LBR classify/solve round and per Halley chunk of
 * one launch (0 = default: 2^27 and 2^26; Halley <= 2^26).  Results do not
 * depend on it; tests force multi-round calls on small batches with it. */
FV_API int fv_set_round_rows(int64_t lbr_rows, int64_t halley_rows);

/* Raw outcome of the calling thread's last batch call: per validation check
 * (FV_CHECK_* order) the first failing row or -1; the first raising row and
 * its FV_EXC_* code for the price/iv stream [0] and the Greeks stream [1]
 * (-1 / 0 when none).  After fv_price_iv: stream [0] is the price stage,
 * [1] the IV stage, and the check rows are the price stage's when one of its
 * checks failed, else the IV stage's.  Lets a caller that shards one logical batch over
 * several calls/devices reproduce the reference's single first error. */
FV_API int fv_last_outcome(int64_t* check_rows /*[FV_NCHECK]*/, int64_t* exc_rows /*[2]*/,
                           int32_t* exc_codes /*[2]*/);

/* Self-test: the exact constant-division used by the kernels against the
 * device's IEEE division on n random inputs x 9 divisors; mismatches out. */
FV_API int fv_selftest_div_const(int64_t n, uint64_t seed, int64_t* mismatches);

/* Self-test of the straight-line routines of the far-low solver (fv_fast.h)
 * against their careful forms on n random inputs each, for 11 routines
 * (division, exp, log, pow, erfcx, normalized_black_log, constant division,
 * sqrt, two-path log, erfc, erfcx incl. negative / zero arguments):
 * per routine, the inputs whose result differs although the routine did not
 * flag them (must be 0) and the inputs it flagged for the careful path. */
FV_API int fv_selftest_fast(int64_t n, uint64_t seed, int64_t* mismatches /*[11]*/,
                            int64_t* flagged /*[11]*/);

/* Exhaustive check of the lower-bound table behind the quick far-low
 * decision of the LBR normalize pass (fv_fast.h g_qlo_tab): over every fp32
 * |x| in [2^-13, 2^5), the points where the exact first anchor b_lo(x) is
 * below its bin's bound (must be 0), the smallest b_lo / bound ratio (>= 1:
 * the bound's tightness) and the number of points.  Diagnostics / tests. */
FV_API int fv_selftest_qlo(int64_t* violations, double* min_ratio, int64_t* points);

/* Per-kernel timing (diagnostics; off by default).  While on, every kernel
 * the calling thread launches is bracketed by CUDA events on its stream;
 * fv_kernel_times sums the elapsed milliseconds and launch counts per kernel
 * (FV_KID_* order, names from fv_kernel_name) since the previous call and
 * resets them.  While on, the passes that otherwise run concurrently on side
 * streams (LBR far-low / far-high branches, the Halley careful pass) run in
 * sequence on the call's stream, so each event pair brackets one kernel
 * alone and the shares add up to the serialised call. */
#define FV_KID_PRICE 0
#define FV_KID_PRICE_GREEKS 1
#define FV_KID_LBR_NORM 2
#define FV_KID_LBR_NREP 3
#define FV_KID_LBR_ANCH 4
#define FV_KID_LBR_FAST 5
#define FV_KID_LBR_FL 6
#define FV_KID_LBR_NEAR 7
#define FV_KID_LBR_FH 8
#define FV_KID_HALLEY_SETUP 9
#define FV_KID_HALLEY_SM 10
#define FV_KID_HALLEY_SM2 11
#define FV_KID_LBR_NEAR_FAST 12
#define FV_KID_HALLEY_BISECT 13
#define FV_NKERNEL 14
FV_API int fv_set_kernel_timing(int on);

/* Device span of this thread's last device-pointer call (diagnostics; off by
 * default): milliseconds between CUDA events recorded on the call's stream
 * before its first and after its last launch (side streams joined), nothing
 * serialised.  The caller's own per-call time minus this is host overhead
 * (argument checks, launches, the status read-back).  -1 when not recorded. */
FV_API int fv_set_span_timing(int on);
FV_API double fv_last_span_ms(void);
FV_API int fv_kernel_times(double* ms /*[FV_NKERNEL]*/, int64_t* launches /*[FV_NKERNEL]*/);
FV_API const char* fv_kernel_name(int id);

/* Diagnostics: measured DFMA instruction rate of the current device (the
 * FP64-pipe roofline denominator for this path). */
FV_API int fv_probe_fp64_peak(double* dfma_per_s, double* seconds);

#ifdef __cplusplus
}
#endif
#endif /* FASTVOL_B200_H */
