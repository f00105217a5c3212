/*
 * mertens_sm100.h — C ABI of the B200 (sm_100a) exact-Mertens engine.
 *
 * Drop-in boundary for the reference package `mertens` (pkg/src/mertens).
 * Plain pointers and sizes only; all buffers are HOST memory owned by the
 * caller (the library owns device memory for the duration of one call and
 * retains no pointer across calls).  Calls are synchronous; ctypes releases
 * the GIL around them.  Return codes map onto the reference exceptions
 * (errors.py:4-50) in the Python shim paper_1108_0135_b200/_lib.py.
 *
 * Two layers, mirroring the reference:
 *   1. Backend-protocol ops — exactly the functions the engine calls through
 *      `_kernels.get_backend(name)` (_kernels/__init__.py:15-33), with the
 *      same argument meaning; used for per-kernel parity tests.
 *   2. The job-level production entry mt_run(): one call per
 *      mertens_exact / mertens_exact_multi (engine.py:405-446), covering the
 *      whole sieve -> update -> resolve pipeline on the GPU.
 */
#ifndef MERTENS_SM100_H
#define MERTENS_SM100_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MT_ABI_VERSION 2

/* return codes */
#define MT_OK 0
#define MT_ERR_RESOURCE 1 /* -> ResourceLimitError  (errors.py:8)  */
#define MT_ERR_CONTRACT 2 /* -> ContractViolationError (errors.py:16) */
#define MT_ERR_CUDA 3     /* -> RuntimeError (device / driver failure) */
#define MT_ERR_VALUE 4    /* -> ValueError   */
#define MT_ERR_OVERFLOW 5 /* -> OverflowError (_native.pyx:308-309) */

/* mt_job.flags */
#define MT_FLAG_FORCE_WIDE 1u    /* tests: 64-bit remainders / 64-bit quotient walks everywhere */
#define MT_FLAG_FORCE_SLOWDIV 2u /* tests: exact 128/64 division in the counted walk            */
#define MT_FLAG_TIMING 4u        /* per-kernel-class CUDA-event timing into mt_stats.kernel_ms  */
#define MT_FLAG_CAP32 8u         /* cap_m_out / small_m_out are int32_t* (dense full quotient map) */

/* last error message of the calling thread ("" if none) */
const char* mt_last_error(void);
int mt_abi_version(void);
/* number of visible CUDA devices (0 when no GPU / no driver) */
int mt_device_count(void);
/* select the device for subsequent calls of this thread */
int mt_set_device(int device);

/* ---- 1. backend-protocol ops (host buffers) -------------------------------- */

/* replaces _native.pyx:127-160 sieve_logprime(y1, y2, primes, logs, wheel):
 * mu over [y1, y2], y1 >= 2.  Uses primes[i] with primes[i]^2 <= y2, logs[i]
 * added for p >= 11, 0x80 for p^2 | y, p >= 5, on top of wheel[13860]. */
int mt_sieve_logprime(uint64_t y1, uint64_t y2, const uint64_t* primes, const uint8_t* logs,
                      uint64_t nprimes, const uint8_t* wheel, int8_t* mu_out);

/* replaces _native.pyx:113-124 logprime_states(...): raw 8-bit states */
int mt_logprime_states(uint64_t y1, uint64_t y2, const uint64_t* primes, const uint8_t* logs,
                       uint64_t nprimes, const uint8_t* wheel, uint8_t* states_out);

/* replaces _native.pyx:163-206 sieve_naive(y1, y2, primes): mu over [y1, y2]
 * (y1 >= 1, y2 < 2^63).  Same mu; computed by the GPU log-prime sieve. */
int mt_sieve_naive(uint64_t y1, uint64_t y2, const uint64_t* primes, uint64_t nprimes,
                   int8_t* mu_out);

/* replaces _native.pyx:227-310 apply_block(acc, v, lo, xcut, mcut, dnext, ynext,
 * y1, y2, mprefix, divtable): folds one block's M values (mprefix[i] = M(y1+i))
 * into every element; acc/dnext/ynext updated in place; signed-128 partial sums
 * with the |acc| <= 2^62 guard (MT_ERR_OVERFLOW).  The divisor table argument
 * of the reference is not needed (exact fp64-reciprocal division on device). */
int mt_apply_block(uint64_t K, int64_t* acc, const uint64_t* v, const uint64_t* lo,
                   const uint64_t* xcut, const uint64_t* mcut, uint64_t* dnext, uint64_t* ynext,
                   uint64_t y1, uint64_t y2, const int64_t* mprefix, uint64_t* counted_out,
                   uint64_t* dense_out);

/* replaces _native.pyx:313-334 finalize_recursion(tails, D) */
int mt_finalize(uint64_t K, const int64_t* tails, const uint64_t* D, int64_t* final_out);

/* replaces _native.pyx:32-68 build_divisor_arrays(cap): arrays of cap+1 */
int mt_build_divisor_arrays(uint64_t cap, uint64_t* magic, uint8_t* shift, uint8_t* scheme);

/* M(y) for y in [y1, y2] (y1 >= 1): GPU sieve + scan from 1.  Backs the
 * direct path (engine.py:449-458) and the naive oracle (engine.py:553-603). */
int mt_mertens_range(uint64_t y1, uint64_t y2, int64_t* m_out);

/* M(y) at sorted points pts[0..npts) (each >= 1): one GPU sieve pass over
 * [1, max pts].  Backs mertens_naive(n, checkpoints) (engine.py:553-603). */
int mt_mertens_at(const uint64_t* pts, uint64_t npts, int64_t* m_out);

/* the engine's production sieve (mt_sieve2.cu: presieve patterns, in-tile
 * primes, bucketed large primes, look-back scan) over [y1, y2]: mu(y) into
 * mu_out and, if m_out is non-null, M(y) into m_out (either may be null) */
int mt_sieve_fast(uint64_t y1, uint64_t y2, int8_t* mu_out, int64_t* m_out);

/* the production sieve in wheel (tail) mode, the one the engine runs above the
 * head: mu of the y of [y1, y2] coprime to the wheel (2: odd y; 6: gcd(y, 6) = 1),
 * y1 >= one tile (2^18 or 3 * 2^17), into mu_out[i] for the i-th such y */
int mt_sieve_wheel(uint64_t y1, uint64_t y2, int wheel, int8_t* mu_out);
int mt_sieve_odd(uint64_t y1, uint64_t y2, int8_t* mu_out); /* wheel 2 */

/* profiling entry (tools/sieve_bench.py): the production sieve in tail mode
 * over nseg segments of 6 tiles per SM from Y0 (a multiple of the tile's y-span:
 * 2^17 x 1, 2 or 3 for wheel 1, 2, 6) with the primes of y_last; summed
 * CUDA-event ms per kernel class into ms_out[7] (sieve_tile, bucket_fill, -, -,
 * -, -, finish) */
int mt_sieve_bench2(uint64_t Y0, uint64_t nseg, uint64_t y_last, int wheel, double* ms_out);
int mt_sieve_bench(uint64_t Y0, uint64_t nseg, uint64_t y_last, double* ms_out); /* wheel 1 */

/* the engine's exact 128/64 division (reciprocal multiply + exact correction,
 * taken by the elements with v >= 2^64 at n >= 2^64) on a batch: q = v / m for
 * v = v_hi:v_lo < 2^120, m >= 1 (parity entry for tests) */
int mt_udiv128_batch(const uint64_t* v_lo, const uint64_t* v_hi, const uint64_t* m, uint64_t n,
                     uint64_t* q_lo, uint64_t* q_hi);

/* the engine keeps its device buffers in the current device's memory pool between
 * calls (a 1e19 plan maps several GB; re-mapping them per call costs ~0.1 s);
 * this returns the cached blocks to the driver (no reference counterpart) */
int mt_trim_device_memory(void);

/* the paper's approximate algorithm (Eq. 2):
 * out[j] = q_n = 2 sum_{i<n_terms} a[i] cos(z[i] * delta_j + b[i]) in fp64, over a
 * shifted table (b[i] = b'_i for the table's x0; delta = ln x - x0).
 * mt_q_batch: the grid delta_j = delta0 + j * step, j < count (rotation recurrence
 * re-seeded every 32 points); mt_q_points: arbitrary delta[j]. */
int mt_q_batch(const double* z, const double* a, const double* b, uint64_t n_terms, double delta0,
               double step, uint64_t count, double* out);
int mt_q_points(const double* z, const double* a, const double* b, uint64_t n_terms, const double* delta,
                uint64_t count, double* out);

/* ---- 2. job-level production entry ----------------------------------------- */

typedef struct {
  uint32_t n_targets;      /* N >= 1 (mertens_exact: 1; mertens_exact_multi: N) */
  const uint64_t* n_lo;    /* n_i mod 2^64, n_i >= 4 (any order, distinct)       */
  const uint64_t* n_hi;    /* n_i >> 64 (n_i < 2^75)                              */
  uint64_t u;              /* sieve bound, from choose_u (engine.py:116-131)     */
  /* quotient capture for target 0 (engine.py:242-252): M(floor(n0/c)) for
   * c in [cap_c_lo, cap_c_hi] (floor(n0/c) <= u) into cap_m_out, and M(y) for
   * y in [0, cap_small] into small_m_out.  Zero-length ranges disable. */
  uint64_t cap_c_lo, cap_c_hi;
  uint64_t cap_small;
  /* tuning (0 = default) */
  uint64_t q_budget_bytes; /* device bytes for the Q tables (default 48 GiB)       */
  uint32_t seg_log2_head;  /* head segment length 2^x (x >= 17; default: 2 tiles of
                              2^17 cells per SM, MT_SEG_TILES_PER_SM_HEAD overrides) */
  uint32_t seg_log2_tail;  /* tail segment length 2^x (x >= 17; default: 6 tiles of
                              2^17 cells per SM, MT_SEG_TILES_PER_SM overrides)    */
  int32_t device;          /* CUDA device ordinal (-1: current)                    */
  /* multi-GPU sharding: rank r of w sieves the head redundantly,
   * takes every w-th work unit of the head update and of the head part of the
   * Q-gather, and owns the r-th of w tail ranges balanced by sieve work (odd y of
   * [ya/2, yb/2) U [ya, yb)).  w <= 1: all. */
  uint32_t shard_rank, shard_world;
  uint32_t flags;          /* MT_FLAG_*                                          */
  void* stream;            /* cudaStream_t to run on (null: the engine's own)    */
} mt_job;

typedef struct {
  /* reference RunStats fields (engine.py:188-197), counters in closed form */
  uint64_t blocks, counted_items, dense_items;
  uint64_t divtable_cap, divtable_released_at, r4_block_len;
  /* engine-specific */
  uint64_t head_end, n_head_segments, n_tail_segments, kernel_launches;
  uint64_t max_mcut;
  uint64_t windowed_items, qgather_items; /* reserved (0) */
  uint64_t q_entries;
  double ms_total, ms_sieve_head, ms_update_head, ms_sieve_tail, ms_qgather, ms_finalize;
  double ms_counted_kernel, ms_dense_kernel;  /* event-timed (MT_FLAG_TIMING) */
  /* multi-GPU algebra: M(head_end - 1) and this rank's local tail total */
  int64_t m_head, tail_total;
  /* per kernel class (sieve_tile, sieve_large, counted, dwin, dsparse, qgather,
   * other): summed CUDA-event ms and launch counts (MT_FLAG_TIMING) */
  double kernel_ms[8];
  uint64_t kernel_count[8];
  uint64_t tail_seg_begin, tail_seg_end; /* this rank's tail range [ya, yb) (y values) */
  double ms_setup;                        /* mt_plan_create wall time      */
  uint64_t head_cells, tail_cells;        /* sieve cells of this execution: head (all y
                                             below head_end), tail (odd y only)          */
} mt_stats;

typedef struct {
  int64_t* finals;         /* concatenated: target i's M(floor(n_i/k)), k=1..K_i, K_i = n_i//u,
                              in the order of mt_job.n_lo                         */
  int64_t* cap_m_out;      /* cap_c_hi - cap_c_lo + 1 entries (or null); int32_t*
                              with MT_FLAG_CAP32                                  */
  int64_t* small_m_out;    /* cap_small + 1 entries (or null); int32_t* with CAP32 */
  uint64_t* acc_out;       /* optional: raw accumulators (ΣK_i) before resolve   */
  mt_stats stats;
} mt_result;

/* one exact job: sieve 1..u, update every element, resolve (shard_world <= 1) */
int mt_run(const mt_job* job, mt_result* out);

/* ---- 3. plan API: the same job split at its exchange points --------------------
 * mt_run == create, sieve_update, tail_offset(m_head), gather, resolve, destroy.
 * With shard_world = w > 1 every rank runs the phases and the caller performs
 * the collectives between them (paper_1108_0135_b200/distributed.py):
 *   after sieve_update : allgather tail_total -> offset_r = m_head + sum_{h<r} T_h
 *   after tail_offset  : (only when quotient captures are requested) sum-reduce
 *                        mt_plan_cap_window (device int32; each rank holds its
 *                        own entries and zeros elsewhere)
 *   after gather       : allreduce(sum, int64 two's complement) of mt_plan_acc
 * Rank r owns the tail range [ya_r, yb_r) (mt_stats.tail_seg_begin/end) and the
 * quotient-table slice mt_plan_q_slice(t, r) whose quotients fall in it; the
 * Q-gather of rank r reads only that slice and the replicated head part, so no
 * rank needs another rank's slice.  A plan is re-executable (sieve_update
 * re-initialises the accumulators), and all device memory of the job lives in
 * the plan. */
typedef struct mt_plan mt_plan;
int mt_plan_create(const mt_job* job, mt_plan** out);
int mt_plan_sieve_update(mt_plan* p, int64_t* m_head, int64_t* tail_total);
/* phase 1 in steps (checkpointing): the head on the first call, then at most
 * max_tail_segments tail segments per call; *done = 1 when the tail is
 * complete, and then m_head / tail_total are written as by sieve_update */
int mt_plan_sieve_step(mt_plan* p, uint64_t max_tail_segments, int* done, int64_t* m_head,
                       int64_t* tail_total);
/* checkpoint / resume of a single-target plan between sieve steps (one file per
 * rank): the reference's MERTCKP1 header (engine.py:646-680; version 3 = this
 * engine, flags = rank | world << 16) followed by the accumulators, M(mcut), the
 * quotient table, the tail-slice P2 table, the small captures and the running
 * prefixes.  Written to path.tmp, flushed, fsync'ed, then renamed; a failed write
 * removes path.tmp and leaves the previous checkpoint in place. */
int mt_plan_checkpoint(mt_plan* p, const char* path);
int mt_plan_restore(mt_plan* p, const char* path);
int mt_plan_tail_offset(mt_plan* p, int64_t offset);
int mt_plan_q_slice(mt_plan* p, uint32_t target, uint32_t rank, void** dptr, uint64_t* count);
/* target 0's quotient-capture window (M(floor(n0/c)), c in [cap_c_lo, cap_c_hi]) as
 * device int32; count = 0 when no capture was requested */
int mt_plan_cap_window(mt_plan* p, void** dptr, uint64_t* count);
int mt_plan_acc(mt_plan* p, void** dptr, uint64_t* count);
int mt_plan_gather(mt_plan* p);
/* finalize every target; copies into the non-null host pointers of out */
int mt_plan_resolve(mt_plan* p, mt_result* out);
void mt_plan_destroy(mt_plan* p);

#ifdef __cplusplus
}
#endif
#endif
