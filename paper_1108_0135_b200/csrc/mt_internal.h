// Internal (non-ABI) declarations shared by the engine's translation units.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/mertens_sm100.h"

// Device allocations of the engine: stream-ordered from the device's default memory
// pool with its release threshold raised, so a plan's buffers (several GB at 1e19)
// are reused by the next plan instead of being mapped and unmapped per call.
// MT_POOL=0 falls back to cudaMalloc / cudaFree.  mt_dfree waits for the device
// first (as cudaFree does), so no buffer is recycled while a kernel may use it.
cudaError_t mt_dmalloc_raw(void** p, size_t bytes);
void mt_dfree(void* p);
template <class T> inline cudaError_t mt_dmalloc(T** p, size_t bytes) { return mt_dmalloc_raw((void**)p, bytes); }

#define MT_TILE 65536u          // sieve tile: cells (bytes) held in shared memory
#define MT_SIEVE_THREADS 512    // threads per sieve tile (128 cells each)
#define MT_WHEEL 13860u
#define MT_WHEEL_WORDS (MT_WHEEL / 4)
#define MT_CT 256               // elements per counted-walk tile (threads per CTA)
#ifndef MT_CM
#define MT_CM 2736              // list capacity of a counted-walk work unit (the m coprime to 6 of MT_CU consecutive m)
#endif
#define MT_BLK 32768u           // M16 block: values stored relative to M(block start - 1)
#ifndef MT_WIN_SPLIT
#define MT_WIN_SPLIT 64         // d_sp = ceil(sqrt(v)/64): windowed walk up to y ~ 64 sqrt(v)
#endif

struct SieveTileArgs {
  uint64_t Y0;                   // segment start (multiple of MT_TILE)
  uint64_t y2;                   // prime bound rule: primes with p*p <= y2
  const uint32_t* wheel32x;      // 13860-periodic wheel as words, extended by MT_TILE/4 words
  const uint32_t* big;           // per-segment large-prime marks (or null)
  const uint32_t* primes;
  const double* rprimes;         // __drcp_rn(p)
  const uint8_t* logs;
  uint32_t p_first;              // first prime index sieved in-tile (prime 5)
  uint32_t p_warp_end;           // [p_first, p_warp_end): warp-per-prime
  uint32_t p_small_end;          // [p_warp_end, p_small_end): thread-per-prime
  uint32_t log_min;              // logs added for p >= log_min (11: reference wheel)
  int do_logs;
  int* tile_sum;                 // [ntiles]
  int8_t* mu_out;                // segment mu (or null)
  int* m_out;                    // segment partial M (in-tile prefix) (or null)
  int16_t* m16_out;              // M(y) - M(start of its 32K block - 1)   (or null)
  int* half_out;                 // [ntiles] in-tile prefix at the tile's 32K midpoint
  uint8_t* states_out;           // raw states (instrumented) or null
  const void* caps;              // CaptureTarget[n_cap] (device)
  int n_cap;
};

struct SieveSegment {
  uint64_t Y0, R, y2;
  uint32_t* big;                 // R bytes
  const uint32_t* primes;
  const double* rprimes;
  const uint8_t* logs;
  uint32_t p_large_begin, p_large_end;
  int do_logs_large;
  int64_t* running;              // device scalar M(Y0-1) (null: no scan)
  int64_t* tile_base;            // [ntiles]
  int64_t* bk;                   // [2*ntiles] absolute M(start of 32K block - 1) (or null)
  SieveTileArgs tile;
};

// Per-kernel-class device timing (MT_FLAG_TIMING): CUDA events around every
// launch of a class, on the launching stream, drained through a ring so that
// a long job does not hold one event pair per launch.
enum { KT_SIEVE_TILE = 0, KT_SIEVE_LARGE, KT_COUNTED, KT_DWIN, KT_DSPARSE, KT_QGATHER, KT_OTHER, KT_NCLASS };
struct KTimer {
  bool on = false;
  static const int RING = 1024;
  cudaEvent_t a[RING], b[RING];
  int cls[RING];
  bool busy[RING];
  int next = 0, open = -1;
  double ms[KT_NCLASS] = {0};
  uint64_t n[KT_NCLASS] = {0};
  void init(bool enable) {
    on = enable;
    if (!on) return;
    for (int i = 0; i < RING; i++) {
      cudaEventCreate(&a[i]); cudaEventCreate(&b[i]); busy[i] = false;
    }
  }
  void reset() {
    drain();
    for (int i = 0; i < KT_NCLASS; i++) { ms[i] = 0; n[i] = 0; }
  }
  void retire(int i) {
    if (!busy[i]) return;
    cudaEventSynchronize(b[i]);
    float f = 0.f;
    cudaEventElapsedTime(&f, a[i], b[i]);
    ms[cls[i]] += f; n[cls[i]]++;
    busy[i] = false;
  }
  void begin(int c, cudaStream_t st) {
    if (!on) return;
    retire(next);
    cls[next] = c; open = next;
    cudaEventRecord(a[next], st);
  }
  void end(cudaStream_t st) {
    if (!on || open < 0) return;
    cudaEventRecord(b[open], st);
    busy[open] = true; open = -1;
    next = (next + 1) % RING;
  }
  void drain() { if (on) for (int i = 0; i < RING; i++) retire(i); }
  ~KTimer() {
    if (!on) return;
    for (int i = 0; i < RING; i++) { cudaEventDestroy(a[i]); cudaEventDestroy(b[i]); }
  }
};

int mt_launch_sieve_segment(const SieveSegment& s, cudaStream_t st, KTimer* kt = nullptr);

// ---- production sieve (mt_sieve2.cu)
struct CaptureTarget2 {  // one exact target n for quotient captures (same layout as CaptureTarget)
  uint64_t n_lo, n_hi;
  double nd;
  int nbits;
  uint64_t jq0, jq1;  // capture j in [jq0, jq1]
  int* Q;             // Q[j - jq0] = M(floor(n/j))
};

struct Bucket2Args {
  uint64_t Y0;
  uint32_t ntiles, cap, nprod_grid;
  uint32_t bin;          // write-combining entries per tile in shared memory (0 = direct stores)
  const uint32_t* primes;
  const double* rprimes;
  const uint8_t* logs;
  uint32_t p_lo, p_hi;   // log marks of primes [p_lo, p_hi)  (p > 2^17)
  uint32_t q_lo, q_hi;   // square flags of primes [q_lo, q_hi) (p^2 > 2^17)
  const uint32_t* pperm; // producer-major bucket primes: [nprod][kp] log marks, [nprod][kq] squares
  const uint32_t* qperm;
  uint32_t kp, kq;
  uint32_t* buf;         // [nprod][ntiles][cap]
  uint32_t* counts;      // [nprod][ntiles]
};

struct Sieve2Args {
  uint64_t Y0;
  uint32_t ntiles;
  uint32_t* ticket;                 // tile order (zeroed per launch)
  unsigned long long* tstate;       // look-back words [ntiles] (zeroed per launch)
  int64_t* running;                 // M(Y0 - 1) in, M(Y0 + R - 1) out
  const uint32_t *w1, *w2;          // presieve patterns (words)
  uint64_t w1_period4, w2_period4;
  const uint32_t* primes;
  const double* rprimes;
  const uint8_t* logs;
  uint32_t p_first, p_warp_end, p_small_end;  // in-tile log primes
  uint32_t p_b2;                                // first in-tile prime of the plain-stream B2 range
  uint32_t sq_first, sq_end;                  // in-tile squares
  uint32_t nprod, cap;                        // bucket lists (nprod = 0: none)
  const uint32_t* counts;
  const uint32_t* buf;
  uint32_t p_lo, p_hi, q_lo, q_hi;            // bucket producers' prime ranges (overflow path)
  unsigned long long* overflow;
  uint8_t* states_out;                        // debug: raw states
  int8_t* mu_out;                             // head: mu
  int16_t* m16_out;                           // head: M(y) - M(32K block start - 1)
  int64_t* bk;                                // head: M(32K block start - 1)
  int* tile_sum;                              // [ntiles] tile totals
  int64_t* tile_base;                         // [ntiles] M(tile start - 1)
  int* bkrel;                                 // head: tile-relative 32K block starts [ntiles*4]
  uint32_t tiles_per_cta;                     // persistent CTAs: contiguous tiles each
  uint32_t wheel;                             // 1: cell c = y; 2: odd y (y = 2c + 1); 6: y coprime to 6
  const CaptureTarget2* caps;
  int n_cap;
};

struct Sieve2Segment {
  Bucket2Args bucket;
  Sieve2Args tile;
};
int mt_sieve2_segment(const Sieve2Segment& g, cudaStream_t st, KTimer* kt);

// host-side context of the production sieve: patterns, primes, bucket space
struct Sieve2Host;
int mt_sieve2_create(Sieve2Host** out, uint64_t y_last, uint32_t max_tiles, cudaStream_t st);
void mt_sieve2_destroy(Sieve2Host* h);
// one segment [Y0, Y0 + ntiles*2^17): outputs as requested (null = skip)
// wheel 2 / 6: the segment's cells are the odd y / the y coprime to 6 of
// [Y0, Y0 + ntiles * 2^17 * (2 or 3)) (tail mode: sums and captures of the
// wheel's prefix; mu_out gets mu of the cells)
int mt_sieve2_run(Sieve2Host* h, uint64_t Y0, uint32_t ntiles, int64_t* running, int8_t* mu_out,
                  int16_t* m16_out, int64_t* bk, uint8_t* states_out, const CaptureTarget2* caps,
                  int n_cap, cudaStream_t st, KTimer* kt, int wheel = 1);
uint64_t mt_sieve2_overflows(Sieve2Host* h);
uint64_t mt_sieve2_launches(Sieve2Host* h, bool reset);
#define MT_S2_TILE (1u << 17)

// element arrays (device, SoA), one entry per harmonic-array element of every target
struct ElemDev {
  const double* vd;      // double(v)
  const uint64_t* vlo;   // v mod 2^64
  const uint64_t* vhi;   // v >> 64
  const uint8_t* vbits;  // bit length of v
  const uint64_t* k;     // array index k (1-based, within its target)
  const uint32_t* tgt;   // target id
  const uint64_t* mcut;
  const uint64_t* xcut;
  const uint64_t* lo;    // max(2, D+1)
  const uint64_t* lo_w;  // first d of the windowed dense walk: max(lo, J/k + 1)
  const uint64_t* dq_hi; // last d of the Q-gather walk: min(xcut, J/k)
  const uint64_t* d_sp;  // windowed walk split: d >= d_sp in shared-memory windows, d < d_sp gathered from L2
  uint64_t n;            // total elements
};

struct TargetDev {       // per-target constants for Q lookups
  int* Q;                // Q[j - jq0]
  uint64_t jq0;
  uint64_t wlo, whi;     // Q-gather window of this pass: table indices [wlo, whi)
};

// update-side launchers (mt_update.cu)
struct UpdateCtx;
struct GroupDev {        // element groups for the shared-memory window walk
  const uint64_t* start; // [ng+1] first element of each group
  const uint64_t* ylo;   // [ng] min first window-walk quotient
  const uint64_t* yhi;   // [ng] max last window-walk quotient
  const uint8_t* wide;   // [ng] 1 if some member has xcut >= 2^30 (64-bit walk)
  uint64_t ng;
};
// work sharding across ranks: rank r of w takes work units u with u % w == r
struct Shard {
  uint32_t rank = 0, world = 1;
  uint32_t flags = 0;  // MT_FLAG_* (force-wide arithmetic paths for tests)
};
// counted-walk entries (mt_update.cu): the elements, then the virtual halves
// v = floor(v_k / 2) of the elements with 2k > K; each adds S_o(v, lim1) to acc[t1]
// and subtracts S_o(v, lim2) from acc[t2] (t = 0xFFFFFFFF: none)
// counted-walk entries: the elements and the virtual values floor(n/j),
// j = 2k, 3k, 6k > K.  Role r of an entry adds mu(d) S_6(v, lim[r]) to acc[tg[r]],
// d = 1, 2, 3, 6 for r = 0..3 (tg = 0xFFFFFFFF: no such role)
#define CE_ROLES 4
struct CountedEntries {
  double* vd;
  uint64_t* vlo;
  uint64_t* vhi;
  uint8_t* vbits;
  uint64_t* lim[CE_ROLES];
  uint32_t* tg[CE_ROLES];
  uint64_t n;
};
// Kt: K of every target (host), in element order
int mt_update_create(UpdateCtx** ctx, const ElemDev& E, uint64_t* acc, int32_t* Mmc, const uint64_t* Kt,
                     const TargetDev* tgts, int ntgt, const GroupDev& grp,
                     const Shard& sh, KTimer* kt, cudaStream_t st);
void mt_update_destroy(UpdateCtx* ctx);
int mt_update_head_segment(UpdateCtx* ctx, uint64_t Y0, uint64_t R, const int8_t* mu,
                           const int16_t* M16, const int64_t* bk, cudaStream_t st);
// dense items whose table index k*d - jq0 lies in the per-target window [wlo[t], whi[t]);
// interleave: this rank takes every world-th work chunk (else all of them)
int mt_update_qgather(UpdateCtx* ctx, const uint64_t* wlo, const uint64_t* whi, bool interleave, cudaStream_t st);
void mt_update_reset_launches(UpdateCtx* ctx);
int mt_update_finish(UpdateCtx* ctx, cudaStream_t st);  // acc -= M(mcut)*xcut
int mt_finalize_dev(const uint64_t* acc, const uint64_t* D, uint64_t K, int64_t* final_out,
                    cudaStream_t st, uint64_t* launches = nullptr);
int mt_apply_block_dev(uint64_t K, int64_t* acc, const uint64_t* v, const uint64_t* lo,
                       const uint64_t* xcut, const uint64_t* mcut, uint64_t* dnext,
                       uint64_t* ynext, uint64_t y1, uint64_t y2, const int64_t* mp,
                       uint64_t* counters /*[3]: counted, dense, overflow*/, cudaStream_t st);
int mt_divisor_arrays_dev(uint64_t cap, uint64_t* magic, uint8_t* shift, uint8_t* scheme,
                          cudaStream_t st);
uint64_t mt_update_launches(UpdateCtx* ctx);
