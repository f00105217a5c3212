// Host runtime of the B200 exact-Mertens engine and the C ABI
// (include/mertens_sm100.h).  Replaces the reference's job orchestration
// _ExactJob (engine.py:255-402): parameter setup, the y-block loop with its
// prefetch thread, the per-block apply, quotient capture and finalize — as one
// stream of device work with no host round trip per block.
//
// Phases of mt_run:
//   init    element parameters on device (engine.py:134-159 HarmonicArray),
//           per-target quotient-table extent J, head extent Y_H
//   head    y in [0, Y_H]: sieve segments of 2^25 cells writing mu and M,
//           counted walk, windowed dense walk, M(mcut) capture, Q capture
//   tail    y in (Y_H, u]: sieve segments of 2^27 cells, Q capture only
//   gather  dense items with k*d <= J from the Q table
//   resolve level-parallel finalize_recursion (engine.py:394-402)
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <unistd.h>

#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>

#include "mt_common.cuh"
#include "mt_internal.h"

#ifndef MT_XCUT_ALPHA_DEFAULT
#define MT_XCUT_ALPHA_DEFAULT 0.39  // xcut ~ 0.39 sqrt(v) (measured at 1e19: 0.38-0.40 best, -1.8 % vs the reference's split)
#endif

static thread_local char g_err[2048];

// ------------------------------------------------------------ device memory
namespace {
struct PoolState {
  bool init = false, on = false;
  cudaStream_t st = nullptr;
  cudaMemPool_t mp = nullptr;
};
PoolState g_pool[64];
std::mutex g_pool_mu;
PoolState& pool_for_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  PoolState& P = g_pool[dev & 63];
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!P.init) {
    P.init = true;
    const char* e = getenv("MT_POOL");
    int sup = 0;
    cudaDeviceGetAttribute(&sup, cudaDevAttrMemoryPoolsSupported, dev);
    if (sup && !(e && atoi(e) == 0)) {
      cudaMemPool_t mp;
      if (cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
        P.mp = mp;
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
        if (cudaStreamCreateWithFlags(&P.st, cudaStreamNonBlocking) == cudaSuccess) P.on = true;
      }
    }
    cudaGetLastError();
  }
  return P;
}
}  // namespace

cudaError_t mt_dmalloc_raw(void** p, size_t bytes) {
  PoolState& P = pool_for_device();
  if (!P.on) return cudaMalloc(p, bytes);
  cudaError_t e = cudaMallocAsync(p, bytes, P.st);
  if (e == cudaErrorMemoryAllocation) {  // the pool's cached blocks do not fit: return them, retry
    cudaGetLastError();
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(P.mp, 0);
    e = cudaMallocAsync(p, bytes, P.st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(P.st);  // usable from any stream
  return e;
}

extern "C" int mt_trim_device_memory(void) {
  PoolState& P = pool_for_device();
  if (!P.on) return MT_OK;
  cudaDeviceSynchronize();
  cudaMemPoolTrimTo(P.mp, 0);
  return cudaGetLastError() == cudaSuccess ? MT_OK : MT_ERR_CUDA;
}

void mt_dfree(void* p) {
  if (!p) return;
  PoolState& P = pool_for_device();
  if (!P.on) { cudaFree(p); return; }
  cudaDeviceSynchronize();
  cudaFreeAsync(p, P.st);
}

void mt_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* mt_last_error(void) { return g_err; }
extern "C" int mt_abi_version(void) { return MT_ABI_VERSION; }
extern "C" int mt_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return 0; }
  return n;
}
extern "C" int mt_set_device(int d) {
  MT_CUDA_CHECK(cudaSetDevice(d));
  return MT_OK;
}

#define RC(x)                 \
  do {                        \
    int _rc = (x);            \
    if (_rc != MT_OK) return _rc; \
  } while (0)

// ------------------------------------------------------------ host integer math
static u64 isqrt_u128(u128 x) {
  if (x == 0) return 0;
  long double d = sqrtl((long double)x);
  u64 s = (u64)d;
  while ((u128)s * s > x) s--;
  while ((u128)(s + 1) * (s + 1) <= x) s++;
  return s;
}
static u64 ceil_sqrt_u128(u128 x) {
  u64 s = isqrt_u128(x);
  return s + ((u128)s * s < x);
}

// ------------------------------------------------------------ device buffers
struct DevBuf {
  void* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
  ~DevBuf() { if (p) mt_dfree(p); }
  template <class T> T* as() { return (T*)p; }
};
static int dalloc(DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = mt_dmalloc(&b.p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    mt_set_error("device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    return MT_ERR_RESOURCE;
  }
  return MT_OK;
}

// ------------------------------------------------------------ primes (host)
struct PrimeTable {
  std::vector<uint32_t> p;
  std::vector<double> r;
  std::vector<uint8_t> lg;
};
static void build_primes(u64 limit, PrimeTable& t) {
  std::vector<uint8_t> f(limit + 1, 1);
  f[0] = 0;
  if (limit >= 1) f[1] = 0;
  for (u64 i = 2; i * i <= limit; i++)
    if (f[i]) for (u64 j = i * i; j <= limit; j += i) f[j] = 0;
  for (u64 i = 2; i <= limit; i++)
    if (f[i]) {
      t.p.push_back((uint32_t)i);
      t.r.push_back(1.0 / (double)i);  // correctly rounded on IEEE hosts
      int bl = 0;
      for (u64 x = i - 1; x; x >>= 1) bl++;
      t.lg.push_back((uint8_t)(bl | 1));  // ceil(log2 p)|1, sieve.py:111-121
    }
}
static void build_wheel_words(const uint8_t* wheel /*13860*/, std::vector<uint32_t>& w32x) {
  w32x.resize(MT_WHEEL_WORDS + MT_TILE / 4 + 4);
  for (size_t i = 0; i < w32x.size(); i++) {
    size_t base = (i % MT_WHEEL_WORDS) * 4;
    w32x[i] = (uint32_t)wheel[base] | ((uint32_t)wheel[base + 1] << 8) |
              ((uint32_t)wheel[base + 2] << 16) | ((uint32_t)wheel[base + 3] << 24);
  }
}
static void reference_wheel(uint8_t* w) {  // sieve.py:134-145
  memset(w, 0, MT_WHEEL);
  const int P[4] = {2, 3, 5, 7};
  for (int i = 0; i < 4; i++) {
    int bl = 0;
    for (int x = P[i] - 1; x; x >>= 1) bl++;
    for (u64 j = 0; j < MT_WHEEL; j += P[i]) w[j] = (uint8_t)(w[j] + (bl | 1));
  }
  for (u64 j = 0; j < MT_WHEEL; j += 4) w[j] |= 0x80;
  for (u64 j = 0; j < MT_WHEEL; j += 9) w[j] |= 0x80;
}

// prime-index boundaries for a segment with prime rule p*p <= y2
struct PrimeCut { uint32_t first, warp_end, small_end, large_end; };
static PrimeCut prime_cut(const std::vector<uint32_t>& p, u64 y2) {
  PrimeCut c;
  auto idx_ge = [&](u64 v) { return (uint32_t)(std::lower_bound(p.begin(), p.end(), (uint32_t)std::min<u64>(v, 0xFFFFFFFFull)) - p.begin()); };
  u64 s = isqrt_u128(y2);  // p <= floor(sqrt(y2))  <=>  p*p <= y2
  uint32_t end = (uint32_t)(std::upper_bound(p.begin(), p.end(), (uint32_t)std::min<u64>(s, 0xFFFFFFFFull)) - p.begin());
  c.first = std::min(idx_ge(5), end);
  c.warp_end = std::min(idx_ge(MT_TILE / 64), end);
  c.small_end = std::min((uint32_t)(std::upper_bound(p.begin(), p.end(), MT_TILE) - p.begin()), end);
  c.large_end = end;
  if (c.warp_end < c.first) c.warp_end = c.first;
  if (c.small_end < c.warp_end) c.small_end = c.warp_end;
  return c;
}

struct CaptureTargetH {  // mirror of CaptureTarget in mt_sieve.cu
  u64 n_lo, n_hi;
  double nd;
  int nbits;
  u64 jq0, jq1;
  int* Q;
};

// ============================================================================
// sieve-only helpers for the backend-protocol ops
// ============================================================================
struct SieveRunner {
  DevBuf d_primes, d_rp, d_lg, d_w32, d_big, d_tsum, d_tbase, d_run, d_mu, d_m, d_st;
  std::vector<uint32_t> p;
  u64 R = 0;
  int init(const uint64_t* primes, const uint8_t* logs, u64 np, const uint8_t* wheel, u64 R_) {
    R = R_;
    p.resize(np);
    std::vector<double> r(np);
    for (u64 i = 0; i < np; i++) {
      if (primes[i] > 0xFFFFFFFFull) { mt_set_error("prime beyond 2^32"); return MT_ERR_VALUE; }
      p[i] = (uint32_t)primes[i];
      r[i] = 1.0 / (double)primes[i];
    }
    std::vector<uint32_t> w32;
    build_wheel_words(wheel, w32);
    RC(dalloc(d_primes, np * 4 + 4)); RC(dalloc(d_rp, np * 8 + 8)); RC(dalloc(d_lg, np + 1));
    RC(dalloc(d_w32, w32.size() * 4));
    if (np) {
      MT_CUDA_CHECK(cudaMemcpy(d_primes.p, p.data(), np * 4, cudaMemcpyHostToDevice));
      MT_CUDA_CHECK(cudaMemcpy(d_rp.p, r.data(), np * 8, cudaMemcpyHostToDevice));
      MT_CUDA_CHECK(cudaMemcpy(d_lg.p, logs, np, cudaMemcpyHostToDevice));
    }
    MT_CUDA_CHECK(cudaMemcpy(d_w32.p, w32.data(), w32.size() * 4, cudaMemcpyHostToDevice));
    RC(dalloc(d_big, R)); RC(dalloc(d_tsum, (R / MT_TILE) * 4)); RC(dalloc(d_tbase, (R / MT_TILE) * 8));
    RC(dalloc(d_run, 8));
    MT_CUDA_CHECK(cudaMemset(d_run.p, 0, 8));
    return MT_OK;
  }
  // one segment [Y0, Y0+R) with prime rule y2; outputs as requested
  int segment(u64 Y0, u64 y2, int8_t* mu, int* m, uint8_t* states, bool scan, cudaStream_t st) {
    PrimeCut c = prime_cut(p, y2);
    SieveSegment s{};
    s.Y0 = Y0; s.R = R; s.y2 = y2;
    s.big = d_big.as<uint32_t>();
    s.primes = d_primes.as<uint32_t>(); s.rprimes = d_rp.as<double>(); s.logs = d_lg.as<uint8_t>();
    s.p_large_begin = c.small_end; s.p_large_end = c.large_end; s.do_logs_large = 1;
    s.running = scan ? d_run.as<int64_t>() : nullptr;
    s.tile_base = d_tbase.as<int64_t>();
    SieveTileArgs& a = s.tile;
    a.Y0 = Y0; a.y2 = y2; a.wheel32x = d_w32.as<uint32_t>(); a.big = s.big;
    a.primes = s.primes; a.rprimes = s.rprimes; a.logs = s.logs;
    a.p_first = c.first; a.p_warp_end = c.warp_end; a.p_small_end = c.small_end;
    a.log_min = 11; a.do_logs = 1;
    a.tile_sum = d_tsum.as<int>();
    a.mu_out = mu; a.m_out = m; a.states_out = states; a.caps = nullptr; a.n_cap = 0;
    return mt_launch_sieve_segment(s, st);
  }
};

static int sieve_range_op(u64 y1, u64 y2, const uint64_t* primes, const uint8_t* logs, u64 np,
                          const uint8_t* wheel, int8_t* mu_out, uint8_t* st_out) {
  if (y2 < y1) { mt_set_error("bad block bounds [%llu, %llu]", (unsigned long long)y1, (unsigned long long)y2); return MT_ERR_VALUE; }
  const u64 R = 1ull << 24;
  SieveRunner S;
  RC(S.init(primes, logs, np, wheel, R));
  DevBuf d_out;
  RC(dalloc(d_out, R));
  u64 Y0 = (y1 / MT_TILE) * MT_TILE;
  for (; Y0 <= y2; Y0 += R) {
    int8_t* mu = st_out ? nullptr : d_out.as<int8_t>();
    uint8_t* sts = st_out ? d_out.as<uint8_t>() : nullptr;
    RC(S.segment(Y0, y2, mu, nullptr, sts, false, 0));
    u64 a = std::max(Y0, y1), b = std::min(Y0 + R - 1, y2);
    void* dst = st_out ? (void*)(st_out + (a - y1)) : (void*)(mu_out + (a - y1));
    MT_CUDA_CHECK(cudaMemcpy(dst, d_out.as<uint8_t>() + (a - Y0), b - a + 1, cudaMemcpyDeviceToHost));
  }
  return MT_OK;
}

extern "C" int mt_sieve_logprime(uint64_t y1, uint64_t y2, const uint64_t* primes, const uint8_t* logs,
                                 uint64_t np, const uint8_t* wheel, int8_t* mu_out) {
  return sieve_range_op(y1, y2, primes, logs, np, wheel, mu_out, nullptr);
}

extern "C" int mt_logprime_states(uint64_t y1, uint64_t y2, const uint64_t* primes, const uint8_t* logs,
                                  uint64_t np, const uint8_t* wheel, uint8_t* states_out) {
  return sieve_range_op(y1, y2, primes, logs, np, wheel, nullptr, states_out);
}

extern "C" int mt_sieve_naive(uint64_t y1, uint64_t y2, const uint64_t* primes, uint64_t np, int8_t* mu_out) {
  // same mu via the log-prime sieve with the reference's log table and wheel
  std::vector<uint8_t> lg(np);
  for (u64 i = 0; i < np; i++) {
    int bl = 0;
    for (u64 x = primes[i] - 1; x; x >>= 1) bl++;
    lg[i] = (uint8_t)(bl | 1);
  }
  uint8_t w[MT_WHEEL];
  reference_wheel(w);
  return sieve_range_op(y1, y2, primes, lg.data(), np, w, mu_out, nullptr);
}

extern "C" int mt_mertens_range(uint64_t y1, uint64_t y2, int64_t* m_out) {
  if (y1 < 1 || y2 < y1) { mt_set_error("bad range"); return MT_ERR_VALUE; }
  PrimeTable pt;
  build_primes(ceil_sqrt_u128(y2 + MT_TILE * 2) + 1, pt);
  std::vector<uint64_t> p64(pt.p.begin(), pt.p.end());
  uint8_t w[MT_WHEEL];
  reference_wheel(w);
  const u64 R = 1ull << 24;
  SieveRunner S;
  RC(S.init(p64.data(), pt.lg.data(), p64.size(), w, R));
  DevBuf d_m;
  RC(dalloc(d_m, R * 4));
  std::vector<int> hm(R);
  for (u64 Y0 = 0; Y0 <= y2; Y0 += R) {
    RC(S.segment(Y0, Y0 + R - 1, nullptr, d_m.as<int>(), nullptr, true, 0));
    if (Y0 + R - 1 < y1) continue;
    MT_CUDA_CHECK(cudaMemcpy(hm.data(), d_m.p, R * 4, cudaMemcpyDeviceToHost));
    u64 a = std::max(Y0, y1), b = std::min(Y0 + R - 1, y2);
    for (u64 y = a; y <= b; y++) m_out[y - y1] = hm[y - Y0];
  }
  return MT_OK;
}

__global__ void k_gather_points(const int* __restrict__ M, u64 Y0, const uint64_t* __restrict__ pts,
                                u64 npts, int64_t* __restrict__ out) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npts) out[i] = M[pts[i] - Y0];
}

extern "C" int mt_mertens_at(const uint64_t* pts, uint64_t npts, int64_t* m_out) {
  if (npts == 0) return MT_OK;
  for (u64 i = 0; i < npts; i++) {
    if (pts[i] < 1 || (i && pts[i] < pts[i - 1])) { mt_set_error("points must be sorted and >= 1"); return MT_ERR_VALUE; }
  }
  const u64 ymax = pts[npts - 1];
  PrimeTable pt;
  build_primes(ceil_sqrt_u128(ymax + MT_TILE * 2) + 1, pt);
  std::vector<uint64_t> p64(pt.p.begin(), pt.p.end());
  uint8_t w[MT_WHEEL];
  reference_wheel(w);
  const u64 R = 1ull << 25;
  SieveRunner S;
  RC(S.init(p64.data(), pt.lg.data(), p64.size(), w, R));
  DevBuf d_m, d_pts, d_out;
  RC(dalloc(d_m, R * 4)); RC(dalloc(d_pts, npts * 8)); RC(dalloc(d_out, npts * 8));
  MT_CUDA_CHECK(cudaMemcpy(d_pts.p, pts, npts * 8, cudaMemcpyHostToDevice));
  u64 i0 = 0;
  for (u64 Y0 = 0; Y0 <= ymax; Y0 += R) {
    RC(S.segment(Y0, Y0 + R - 1, nullptr, d_m.as<int>(), nullptr, true, 0));
    u64 i1 = i0;
    while (i1 < npts && pts[i1] < Y0 + R) i1++;
    if (i1 > i0) {
      k_gather_points<<<(unsigned)((i1 - i0 + 255) / 256), 256>>>(d_m.as<int>(), Y0, d_pts.as<uint64_t>() + i0, i1 - i0, d_out.as<int64_t>() + i0);
      MT_CUDA_CHECK(cudaGetLastError());
    }
    i0 = i1;
  }
  MT_CUDA_CHECK(cudaMemcpy(m_out, d_out.p, npts * 8, cudaMemcpyDeviceToHost));
  return MT_OK;
}

// tiles per segment of the sieve parity ops (MT_TEST_TILES: smaller segments for
// compute-sanitizer runs; default 256)
static u64 test_tiles() {
  const char* e = getenv("MT_TEST_TILES");
  const u64 t = e ? strtoull(e, nullptr, 10) : 256;
  return t >= 1 && t <= 4096 ? t : 256;
}

// production sieve over [y1, y2] (parity tests of mt_sieve2.cu): mu and, when
// m_out is given, M(y) (then sieving starts at 0 so prefixes are absolute)
__global__ void k_m16_to_m(const int16_t* __restrict__ M16, const int64_t* __restrict__ bk, u64 n,
                           int64_t* __restrict__ out) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = M16[i] + bk[i / MT_BLK];
}

extern "C" int mt_sieve_fast(uint64_t y1, uint64_t y2, int8_t* mu_out, int64_t* m_out) {
  if (y2 < y1) { mt_set_error("bad range"); return MT_ERR_VALUE; }
  const u64 T = MT_S2_TILE, NT = test_tiles(), R = T * NT;
  u64 Y0 = m_out ? 0 : (y1 / T) * T;
  const u64 y_last = ((y2 / R) + 1) * R + Y0;
  Sieve2Host* h = nullptr;
  struct G { Sieve2Host*& h; ~G() { mt_sieve2_destroy(h); } } g{h};
  RC(mt_sieve2_create(&h, y_last, (uint32_t)NT, 0));
  DevBuf d_mu, d_m, d_bk, d_run, d_mm;
  RC(dalloc(d_mu, R)); RC(dalloc(d_m, R * 2)); RC(dalloc(d_bk, (R / MT_BLK) * 8)); RC(dalloc(d_run, 8));
  RC(dalloc(d_mm, R * 8));
  MT_CUDA_CHECK(cudaMemset(d_run.p, 0, 8));
  for (; Y0 <= y2; Y0 += R) {
    RC(mt_sieve2_run(h, Y0, (uint32_t)NT, d_run.as<int64_t>(), d_mu.as<int8_t>(), d_m.as<int16_t>(),
                     d_bk.as<int64_t>(), nullptr, nullptr, 0, 0, nullptr));
    if (Y0 + R - 1 < y1) continue;
    const u64 a = std::max(Y0, y1), b = std::min(Y0 + R - 1, y2);
    if (mu_out) MT_CUDA_CHECK(cudaMemcpy(mu_out + (a - y1), d_mu.as<int8_t>() + (a - Y0), b - a + 1, cudaMemcpyDeviceToHost));
    if (m_out) {
      k_m16_to_m<<<(unsigned)((R + 255) / 256), 256>>>(d_m.as<int16_t>(), d_bk.as<int64_t>(), R, d_mm.as<int64_t>());
      MT_CUDA_CHECK(cudaGetLastError());
      MT_CUDA_CHECK(cudaMemcpy(m_out + (a - y1), d_mm.as<int64_t>() + (a - Y0), (b - a + 1) * 8, cudaMemcpyDeviceToHost));
    }
  }
  MT_CUDA_CHECK(cudaDeviceSynchronize());
  if (mt_sieve2_overflows(h)) { /* recomputed exactly; reported only */ }
  return MT_OK;
}

// cells of wheel W with y - Y0 <= o (host mirror of Wheel<W>::ncell, Y0 a multiple of W)
static u64 wheel_ncell(int W, u64 o) {
  return W == 1 ? o + 1 : W == 2 ? (o + 1) >> 1 : 2 * (o / 6) + (o % 6 >= 1) + (o % 6 >= 5);
}

// the production sieve in wheel (tail) mode over the y of [y1, y2] coprime to the
// wheel (2: odd y; 6: gcd(y, 6) = 1), y1 >= one tile: mu_out[i] = mu of the i-th
// such y in ascending order
extern "C" int mt_sieve_wheel(uint64_t y1, uint64_t y2, int wheel, int8_t* mu_out) {
  if (wheel != 2 && wheel != 6) { mt_set_error("wheel must be 2 or 6"); return MT_ERR_VALUE; }
  const u64 SPAN = (u64)MT_S2_TILE * (wheel == 2 ? 2 : 3), NT = test_tiles(), RY = SPAN * NT;
  if (y2 < y1 || y1 < SPAN) { mt_set_error("bad range (the wheel sieve needs y1 >= one tile)"); return MT_ERR_VALUE; }
  u64 Y0 = (y1 / SPAN) * SPAN;
  const u64 first = wheel_ncell(wheel, y1 - 1 - Y0);  // cells of [Y0, y1)
  const u64 y_last = ((y2 - Y0) / RY + 1) * RY + Y0 - 1;
  Sieve2Host* h = nullptr;
  struct G { Sieve2Host*& h; ~G() { mt_sieve2_destroy(h); } } g{h};
  RC(mt_sieve2_create(&h, y_last, (uint32_t)NT, 0));
  DevBuf d_mu, d_run;
  RC(dalloc(d_mu, NT * MT_S2_TILE)); RC(dalloc(d_run, 8));
  MT_CUDA_CHECK(cudaMemset(d_run.p, 0, 8));
  u64 done = 0;  // cells of [Y0_first, Y0) copied or skipped
  for (u64 base = 0; Y0 <= y2; Y0 += RY, base += NT * MT_S2_TILE) {
    RC(mt_sieve2_run(h, Y0, (uint32_t)NT, d_run.as<int64_t>(), d_mu.as<int8_t>(), nullptr, nullptr, nullptr,
                     nullptr, 0, 0, nullptr, wheel));
    const u64 ca = base < first ? first - base : 0;                   // first wanted cell of this segment
    const u64 cb = wheel_ncell(wheel, std::min(y2, Y0 + RY - 1) - Y0);  // cells with y <= min(y2, end)
    if (cb > ca) MT_CUDA_CHECK(cudaMemcpy(mu_out + (base + ca - first), d_mu.as<int8_t>() + ca, cb - ca, cudaMemcpyDeviceToHost));
    done = base + cb;
  }
  (void)done;
  MT_CUDA_CHECK(cudaDeviceSynchronize());
  return MT_OK;
}

extern "C" int mt_sieve_odd(uint64_t y1, uint64_t y2, int8_t* mu_out) { return mt_sieve_wheel(y1, y2, 2, mu_out); }

// profiling entry: the production sieve in tail mode (sums only, no outputs)
// over nseg segments of the default size from Y0 (multiple of 2^17), with
// primes for y_last; per-kernel-class CUDA-event ms into ms_out[KT_NCLASS]
extern "C" int mt_sieve_bench2(uint64_t Y0, uint64_t nseg, uint64_t y_last, int wheel, double* ms_out) {
  if (wheel == 0) wheel = 1;
  const u64 span = (u64)MT_S2_TILE * (wheel == 6 ? 3 : wheel);
  if (Y0 % span || (wheel > 1 && Y0 == 0)) { mt_set_error("Y0 must be a positive multiple of the tile span"); return MT_ERR_VALUE; }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t NT = (uint32_t)nsm * 6;
  const u64 R = (u64)NT * span;
  if (y_last < Y0 + nseg * R) y_last = Y0 + nseg * R;
  Sieve2Host* h = nullptr;
  struct G { Sieve2Host*& h; ~G() { mt_sieve2_destroy(h); } } g{h};
  RC(mt_sieve2_create(&h, y_last, NT, 0));
  DevBuf d_run;
  RC(dalloc(d_run, 8));
  MT_CUDA_CHECK(cudaMemset(d_run.p, 0, 8));
  KTimer kt;
  kt.init(true);
  for (u64 s = 0; s < nseg; s++)
    RC(mt_sieve2_run(h, Y0 + s * R, NT, d_run.as<int64_t>(), nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, &kt,
                     wheel));
  MT_CUDA_CHECK(cudaDeviceSynchronize());
  kt.drain();
  for (int c = 0; c < KT_NCLASS; c++) ms_out[c] = kt.ms[c];
  return MT_OK;
}

extern "C" int mt_sieve_bench(uint64_t Y0, uint64_t nseg, uint64_t y_last, double* ms_out) {
  return mt_sieve_bench2(Y0, nseg, y_last, 0, ms_out);
}

// exact 128/64 division of the engine (udiv128, mt_common.cuh) on a batch: parity
// entry for the reciprocal-multiply + correction path the n >= 2^64 elements take
__global__ void k_udiv128(const u64* lo, const u64* hi, const u64* m, u64 n, u64* qlo, u64* qhi) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u128 q = udiv128(lo[i], hi[i], m[i]);
  qlo[i] = (u64)q;
  qhi[i] = (u64)(q >> 64);
}

extern "C" int mt_udiv128_batch(const uint64_t* v_lo, const uint64_t* v_hi, const uint64_t* m, uint64_t n,
                                uint64_t* q_lo, uint64_t* q_hi) {
  if (!n) return MT_OK;
  for (u64 i = 0; i < n; i++)
    if (!m[i] || (v_hi[i] >> 56)) { mt_set_error("udiv128: m >= 1 and v < 2^120 required"); return MT_ERR_VALUE; }
  DevBuf a, b, c, d, e;
  RC(dalloc(a, n * 8)); RC(dalloc(b, n * 8)); RC(dalloc(c, n * 8)); RC(dalloc(d, n * 8)); RC(dalloc(e, n * 8));
  MT_CUDA_CHECK(cudaMemcpy(a.p, v_lo, n * 8, cudaMemcpyHostToDevice));
  MT_CUDA_CHECK(cudaMemcpy(b.p, v_hi, n * 8, cudaMemcpyHostToDevice));
  MT_CUDA_CHECK(cudaMemcpy(c.p, m, n * 8, cudaMemcpyHostToDevice));
  k_udiv128<<<(unsigned)((n + 255) / 256), 256>>>(a.as<u64>(), b.as<u64>(), c.as<u64>(), n, d.as<u64>(), e.as<u64>());
  MT_CUDA_CHECK(cudaGetLastError());
  MT_CUDA_CHECK(cudaMemcpy(q_lo, d.p, n * 8, cudaMemcpyDeviceToHost));
  MT_CUDA_CHECK(cudaMemcpy(q_hi, e.p, n * 8, cudaMemcpyDeviceToHost));
  return MT_OK;
}

// ============================================================================
// backend-protocol: apply_block / finalize / divisor arrays
// ============================================================================
extern "C" int mt_apply_block(uint64_t K, int64_t* acc, const uint64_t* v, const uint64_t* lo,
                              const uint64_t* xcut, const uint64_t* mcut, uint64_t* dnext, uint64_t* ynext,
                              uint64_t y1, uint64_t y2, const int64_t* mprefix, uint64_t* counted_out,
                              uint64_t* dense_out) {
  if (y1 < 1 || y2 < y1) { mt_set_error("bad block bounds"); return MT_ERR_VALUE; }
  u64 L = y2 - y1 + 1;
  DevBuf a, vv, l, x, mc, dn, yn, mp, cnt;
  RC(dalloc(a, K * 8)); RC(dalloc(vv, K * 8)); RC(dalloc(l, K * 8)); RC(dalloc(x, K * 8));
  RC(dalloc(mc, K * 8)); RC(dalloc(dn, K * 8)); RC(dalloc(yn, K * 8)); RC(dalloc(mp, L * 8));
  RC(dalloc(cnt, 24));
  if (K) {
    MT_CUDA_CHECK(cudaMemcpy(a.p, acc, K * 8, cudaMemcpyHostToDevice));
    MT_CUDA_CHECK(cudaMemcpy(vv.p, v, K * 8, cudaMemcpyHostToDevice));
    MT_CUDA_CHECK(cudaMemcpy(l.p, lo, K * 8, cudaMemcpyHostToDevice));
    MT_CUDA_CHECK(cudaMemcpy(x.p, xcut, K * 8, cudaMemcpyHostToDevice));
    MT_CUDA_CHECK(cudaMemcpy(mc.p, mcut, K * 8, cudaMemcpyHostToDevice));
    MT_CUDA_CHECK(cudaMemcpy(dn.p, dnext, K * 8, cudaMemcpyHostToDevice));
    MT_CUDA_CHECK(cudaMemcpy(yn.p, ynext, K * 8, cudaMemcpyHostToDevice));
  }
  MT_CUDA_CHECK(cudaMemcpy(mp.p, mprefix, L * 8, cudaMemcpyHostToDevice));
  MT_CUDA_CHECK(cudaMemset(cnt.p, 0, 24));
  RC(mt_apply_block_dev(K, a.as<int64_t>(), vv.as<uint64_t>(), l.as<uint64_t>(), x.as<uint64_t>(),
                        mc.as<uint64_t>(), dn.as<uint64_t>(), yn.as<uint64_t>(), y1, y2, mp.as<int64_t>(),
                        cnt.as<uint64_t>(), 0));
  uint64_t c[3];
  MT_CUDA_CHECK(cudaMemcpy(c, cnt.p, 24, cudaMemcpyDeviceToHost));
  if (c[2]) { mt_set_error("harmonic accumulator exceeded the signed-64 guard range"); return MT_ERR_OVERFLOW; }
  if (K) {
    MT_CUDA_CHECK(cudaMemcpy(acc, a.p, K * 8, cudaMemcpyDeviceToHost));
    MT_CUDA_CHECK(cudaMemcpy(dnext, dn.p, K * 8, cudaMemcpyDeviceToHost));
    MT_CUDA_CHECK(cudaMemcpy(ynext, yn.p, K * 8, cudaMemcpyDeviceToHost));
  }
  *counted_out = c[0];
  *dense_out = c[1];
  return MT_OK;
}

extern "C" int mt_finalize(uint64_t K, const int64_t* tails, const uint64_t* D, int64_t* final_out) {
  DevBuf a, d, f;
  RC(dalloc(a, K * 8)); RC(dalloc(d, K * 8)); RC(dalloc(f, K * 8));
  if (!K) return MT_OK;
  MT_CUDA_CHECK(cudaMemcpy(a.p, tails, K * 8, cudaMemcpyHostToDevice));
  MT_CUDA_CHECK(cudaMemcpy(d.p, D, K * 8, cudaMemcpyHostToDevice));
  RC(mt_finalize_dev(a.as<uint64_t>(), d.as<uint64_t>(), K, f.as<int64_t>(), 0));
  MT_CUDA_CHECK(cudaMemcpy(final_out, f.p, K * 8, cudaMemcpyDeviceToHost));
  return MT_OK;
}

extern "C" int mt_build_divisor_arrays(uint64_t cap, uint64_t* magic, uint8_t* shift, uint8_t* scheme) {
  DevBuf m, s, c;
  RC(dalloc(m, (cap + 1) * 8)); RC(dalloc(s, cap + 1)); RC(dalloc(c, cap + 1));
  RC(mt_divisor_arrays_dev(cap, m.as<uint64_t>(), s.as<uint8_t>(), c.as<uint8_t>(), 0));
  MT_CUDA_CHECK(cudaMemcpy(magic, m.p, (cap + 1) * 8, cudaMemcpyDeviceToHost));
  MT_CUDA_CHECK(cudaMemcpy(shift, s.p, cap + 1, cudaMemcpyDeviceToHost));
  MT_CUDA_CHECK(cudaMemcpy(scheme, c.p, cap + 1, cudaMemcpyDeviceToHost));
  return MT_OK;
}

// ============================================================================
// the job
// ============================================================================
// element parameters (engine.py:144-158), 128-bit exact, one thread per element
struct ElemInitArgs {
  const u64* n_lo; const u64* n_hi; const u64* e0;  // per target
  int ntgt;
  u64 u;
  u64 n_elem;
  double* vd; u64* vlo; u64* vhi; uint8_t* vbits; u64* k; uint32_t* tgt;
  u64* D; u64* xcut; u64* mcut; u64* lo;
  double xalpha;                     // > 0: split at xcut = max(D, xalpha sqrt(v)) (else the reference's)
  unsigned long long* stats;         // [ntgt*4]: max working mcut, sum / max reference mcut, reference dense items
};

__device__ u64 d_isqrt128(u128 x) {
  if (x == 0) return 0;
  double d = sqrt((double)x);
  u64 s = (u64)d;
  if (s > 0xFFFFFFFFFFull) s = 0xFFFFFFFFFFull;  // x < 2^80
  while ((u128)s * s > x) s--;
  while ((u128)(s + 1) * (s + 1) <= x) s++;
  return s;
}

__global__ void k_elem_init(ElemInitArgs a) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n_elem) return;
  int t = 0;
  while (t + 1 < a.ntgt && a.e0[t + 1] <= e) t++;
  const u64 kk = e - a.e0[t] + 1;
  const u128 n = ((u128)a.n_hi[t] << 64) | a.n_lo[t];
  const u128 v = n / kk;
  const u64 D = (u64)(v / ((u128)a.u + 1));
  u64 cs = d_isqrt128(v);
  if ((u128)cs * cs < v) cs++;
  const u64 x2 = 2 * cs;
  u64 tt = 1;
  while (tt < x2) tt <<= 1;  // smallest power of two >= 2*ceil(sqrt v) (engine.py:148-149, :481)
  u64 xr = (u64)(v / tt);
  if (xr < D) xr = D;
  if (xr < 1) xr = 1;
  // the counted / dense split: any xcut >= D gives the same acc_k (summation by parts);
  // the reference's (engine.py:144-158) fixes the RunStats counters either way
  u64 xc = xr;
  if (a.xalpha > 0) {
    xc = (u64)(a.xalpha * (double)cs);
    if (xc < D) xc = D;
    if (xc < 1) xc = 1;
  }
  const u64 mc = (u64)(v / ((u128)xc + 1));
  const u64 mr = (u64)(v / ((u128)xr + 1));
  const u64 lo = D + 1 > 2 ? D + 1 : 2;
  atomicMax(&a.stats[4 * t + 0], (unsigned long long)mc);
  atomicAdd(&a.stats[4 * t + 1], (unsigned long long)mr);
  if (xr >= lo) atomicAdd(&a.stats[4 * t + 2], (unsigned long long)(xr - lo + 1));
  atomicMax(&a.stats[4 * t + 3], (unsigned long long)mr);
  a.vlo[e] = (u64)v;
  a.vhi[e] = (u64)(v >> 64);
  a.vd[e] = (v >> 64) ? fma((double)(u64)(v >> 64), 18446744073709551616.0, (double)(u64)v) : __ull2double_rn((u64)v);
  a.vbits[e] = (uint8_t)((v >> 64) ? 128 - __clzll((long long)(u64)(v >> 64)) : 64 - __clzll((long long)(u64)v));
  a.k[e] = kk;
  a.tgt[e] = (uint32_t)t;
  a.D[e] = D;
  a.xcut[e] = xc;
  a.mcut[e] = mc;
  a.lo[e] = lo;
}

// windowed / Q-gather boundary: Q-gather takes d <= J/k
__global__ void k_elem_split(u64 n_elem, const u64* __restrict__ k, const uint32_t* __restrict__ tgt,
                             const u64* __restrict__ J, const u64* __restrict__ lo,
                             const u64* __restrict__ xcut, u64* __restrict__ lo_w, u64* __restrict__ dq_hi) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_elem) return;
  const u64 jk = J[tgt[e]] / k[e];
  const u64 xc = xcut[e], l = lo[e];
  dq_hi[e] = jk < xc ? jk : xc;
  u64 lw = jk + 1;
  lo_w[e] = lw > l ? lw : l;
}

// windowed-walk split d_sp: shared-memory windows for d >= d_sp (y up to ~C sqrt(v)),
// C = min(64, cbrt(sqrt(v)/2)) so the incremental quotient walk needs <= 1
// correction per step (second difference 2y/d^2 <= 1).
__global__ void k_elem_dsp(u64 n_elem, const double* __restrict__ vd, u64* __restrict__ dsp) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_elem) return;
  double s = sqrt(vd[e]);
  double c = cbrt(0.5 * s);
  if (c > MT_WIN_SPLIT) c = MT_WIN_SPLIT;
  if (c < 1.0) c = 1.0;
  dsp[e] = (u64)ceil(s / c);
}

// per group: y-range of the window walk and the wide-walk flag
__global__ void k_group_meta(const u64* __restrict__ gstart, u64 ng, const u64* __restrict__ vlo,
                             const u64* __restrict__ vhi, const u64* __restrict__ xcut,
                             const u64* __restrict__ lo_w, const u64* __restrict__ dsp,
                             u64* __restrict__ ylo, u64* __restrict__ yhi, uint8_t* __restrict__ wide) {
  u64 g = blockIdx.x;
  if (g >= ng) return;
  u64 mn = ~0ull, mx = 0;
  int w = 0;
  for (u64 e = gstart[g] + threadIdx.x; e < gstart[g + 1]; e += blockDim.x) {
    u64 xc = xcut[e], lw = lo_w[e] > dsp[e] ? lo_w[e] : dsp[e];
    if (lw > xc) continue;
    u128 v = ((u128)vhi[e] << 64) | vlo[e];
    u128 a = v / xc, b = v / lw;
    u64 a64 = a > (u128)~0ull ? ~0ull : (u64)a, b64 = b > (u128)~0ull ? ~0ull : (u64)b;
    if (a64 < mn) mn = a64;
    if (b64 > mx) mx = b64;
    if (xc >= (1ull << 30)) w = 1;
  }
  typedef cub::BlockReduce<u64, 256> BR;
  __shared__ typename BR::TempStorage t1, t2;
  __shared__ int sw;
  if (threadIdx.x == 0) sw = 0;
  __syncthreads();
  if (w) sw = 1;
  u64 rmn = BR(t1).Reduce(mn, cub::Min());
  u64 rmx = BR(t2).Reduce(mx, cub::Max());
  __syncthreads();
  if (threadIdx.x == 0) { ylo[g] = rmn; yhi[g] = rmx; wide[g] = (uint8_t)sw; }
}

// per-target reductions: max mcut, sum mcut, sum dense items, max windowed y
__global__ void k_window_extent(u64 n_elem, const u64* __restrict__ vlo, const u64* __restrict__ vhi,
                                const u64* __restrict__ lo_w, const u64* __restrict__ xcut,
                                unsigned long long* __restrict__ out) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_elem) return;
  u64 lw = lo_w[e];
  if (lw > xcut[e]) return;
  u128 v = ((u128)vhi[e] << 64) | vlo[e];
  u128 y = v / lw;
  atomicMax(out, (unsigned long long)(y > (u128)~0ull ? ~0ull : (u64)y));
}

template <class T>
__global__ void k_copy_small(const int16_t* __restrict__ M16, const int64_t* __restrict__ bk, u64 Y0, u64 R,
                             u64 ymax, T* __restrict__ out) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 y = Y0 + i;
  if (i >= R || y > ymax) return;
  out[y] = (T)(M16[i] + bk[i / MT_BLK]);
}

__global__ void k_copy_caps(const int* __restrict__ Q, u64 jq0, u64 c_lo, u64 cnt, int64_t* __restrict__ out) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  out[i] = Q[c_lo + i - jq0];
}

// Q[j] = sum_d s_d T_d[j] + delta over one target's own tail slice, T_1 = Q:
// the wheel prefixes at floor(n/(d j)) combine to M(floor(n/j)) - M(ya - 1) up to
// a constant folded into delta
struct CombineArgs { const int* T[3]; int s[3]; int n; };
__global__ void k_q_combine(int* __restrict__ Q, CombineArgs c, u64 cnt, int delta) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  int v = Q[i] + delta;
  for (int k = 0; k < c.n; k++) v += c.s[k] * c.T[k][i];
  Q[i] = v;
}

// multi-rank output assembly: zero the capture-window entries this rank does
// not own (own tail slice [s0, s1]; the head part j >= jh belongs to rank 0)
__global__ void k_cap_mask(int* __restrict__ Q, u64 jq0, u64 c0, u64 c1, u64 s0, u64 s1, u64 jh, int head_mine) {
  const u64 j = c0 + (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > c1) return;
  const bool mine = (j >= s0 && j <= s1) || (head_mine && j >= jh);
  if (!mine) Q[j - jq0] = 0;
}

// NVTX ranges around the plan's phases (visible in nsys / ncu --nvtx; no-ops otherwise)
struct NvtxRange {
  explicit NvtxRange(const char* s) { nvtxRangePushA(s); }
  ~NvtxRange() { nvtxRangePop(); }
};

static double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// ============================================================================
// the tail split
// ============================================================================
// The tail sieves only the y coprime to the wheel W (2: odd y; 6: gcd(y, 6) = 1).
// With C_W(x) the Moebius sum over those y <= x (mu(2z) = -mu(z) for odd z,
// mu(3z) = -mu(z) for 3 not dividing z, mu = 0 on multiples of 4 and 9):
//   M(x) = sum_{d | W} mu(d) C_W(floor(x/d)),   d in {1, 2} (W = 2) or {1, 2, 3, 6} (W = 6).
// A rank owning the tail range [a, b) sieves the wheel cells of the union of
// [a/d, b/d) with one running prefix P (P(a/W - 1) = 0), cut at every a/d and
// b/d, and records P at those breakpoints.  For x in [a, b):
//   M(x) - M(a - 1) = sum_d mu(d) (P(floor(x/d)) - P(a/d - 1)).
// Boundaries are multiples of W * (tile y-span) so every a/d is a tile boundary.
struct TailWheel {
  int W = 6, nd = 4;
  u64 d[4] = {1, 2, 3, 6};
  int s[4] = {1, -1, -1, 1};
  u64 tile_y = 3ull * MT_S2_TILE;  // y per tile (2^17 cells)
  u64 align() const { return (u64)W * tile_y; }
};
static TailWheel tail_wheel(int W) {
  TailWheel t;
  if (W == 2) { t.W = 2; t.nd = 2; t.tile_y = 2ull * MT_S2_TILE; }
  return t;
}

// the y-intervals [a/d, b/d) a rank owning [a, b) sieves, merged
static std::vector<std::pair<u64, u64>> tail_union(const TailWheel& tw, u64 a, u64 b) {
  std::vector<std::pair<u64, u64>> iv, out;
  if (b <= a) return out;
  for (int k = 0; k < tw.nd; k++) iv.push_back({a / tw.d[k], b / tw.d[k]});
  std::sort(iv.begin(), iv.end());
  for (auto& x : iv) {
    if (!out.empty() && x.first <= out.back().second) out.back().second = std::max(out.back().second, x.second);
    else out.push_back(x);
  }
  return out;
}

// y-values a rank owning [a, b) covers (its cells: 1/2 or 1/3 of them)
static u64 tail_cost(const TailWheel& tw, u64 a, u64 b) {
  u64 c = 0;
  for (auto& x : tail_union(tw, a, b)) c += x.second - x.first;
  return c;
}

// boundaries H = y[0] < ... <= y[w] = E on the wheel's alignment, balancing tail_cost
static std::vector<u64> tail_partition(const TailWheel& tw, u64 H, u64 E, uint32_t w) {
  std::vector<u64> yb(w + 1, E);
  yb[0] = H;
  if (w <= 1 || E <= H) return yb;
  const u64 AL = tw.align();
  auto cover = [&](u64 c, std::vector<u64>* out) -> bool {
    u64 a = H;
    for (uint32_t r = 0; r + 1 < w; r++) {
      u64 lo = 0, hi = (E - a) / AL;  // largest step with cost <= c
      while (lo < hi) {
        const u64 mid = (lo + hi + 1) / 2;
        if (tail_cost(tw, a, a + mid * AL) <= c) lo = mid; else hi = mid - 1;
      }
      a += lo * AL;
      if (out) (*out)[r + 1] = a;
    }
    return tail_cost(tw, a, E) <= c;
  };
  u64 lo = 0, hi = tail_cost(tw, H, E);
  while (lo < hi) {
    const u64 mid = lo + (hi - lo) / 2;
    if (cover(mid, nullptr)) hi = mid; else lo = mid + 1;
  }
  cover(lo, &yb);
  yb[w] = E;
  return yb;
}

struct TailSeg { u64 Y0; uint32_t ntiles; };

// this rank's wheel segments over the union of [a/d, b/d), cut at every
// breakpoint a/d, b/d; bp[i] = the breakpoints (ascending) and snap[i] = the number
// of segments ending at or before bp[i] (P(bp[i] - 1) is the running prefix then)
static void tail_segments(const TailWheel& tw, u64 a, u64 b, u64 seg_y, std::vector<TailSeg>& out,
                          std::vector<u64>& bp, std::vector<size_t>& snap) {
  out.clear(); bp.clear(); snap.clear();
  if (b <= a) return;
  for (int k = 0; k < tw.nd; k++) { bp.push_back(a / tw.d[k]); bp.push_back(b / tw.d[k]); }
  std::sort(bp.begin(), bp.end());
  bp.erase(std::unique(bp.begin(), bp.end()), bp.end());
  for (size_t i = 0; i + 1 < bp.size(); i++) {
    const u64 x = bp[i], y = bp[i + 1];
    bool cov = false;
    for (int k = 0; k < tw.nd; k++) cov |= a / tw.d[k] <= x && y <= b / tw.d[k];
    if (!cov) continue;
    for (u64 s = x; s < y; s += seg_y)
      out.push_back({s, (uint32_t)((std::min(y, s + seg_y) - s) / tw.tile_y)});
  }
  for (u64 x : bp) {
    size_t c = 0;
    for (auto& s : out) c += s.Y0 + (u64)s.ntiles * tw.tile_y <= x;
    snap.push_back(c);
  }
}

// ============================================================================
// the plan: one exact job (N targets sharing one sieve), split at its
// exchange points so that a multi-GPU caller can run the collectives
// ============================================================================
struct mt_plan {
  int device = -1;
  int N = 0;
  u64 u = 0;
  uint32_t rank = 0, world = 1, flags = 0;
  std::vector<u128> n;
  std::vector<u64> n_lo, n_hi, K, e0;
  u64 NE = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  u64 launches = 0;  // kernels of the current execution (reset by the head step)
  u64 counted_items = 0, dense_items = 0, Ymc = 0, Ymc_ref = 0;  // Ymc: the working split's max mcut
  double xalpha = 0;  // counted / dense split: xcut = max(D, xalpha ceil(sqrt v)); 0 = the reference's
  // elements
  DevBuf d_nlo, d_nhi, d_e0, d_vd, d_vlo, d_vhi, d_vb, d_k, d_tgt, d_D, d_x, d_mc, d_lo, d_low, d_dq,
      d_acc, d_mmc, d_dsp, d_J, d_gs, d_gylo, d_gyhi, d_gw, d_fin;
  std::vector<u64> gstart;
  u64 ng = 0;
  // quotient tables Q_t[j - jq0] = M(floor(n_t/j)), j in [jq0, jq1]
  std::vector<u64> J, jq0, jq1;
  std::vector<DevBuf> d_Q;
  std::vector<TargetDev> tdev;
  std::vector<CaptureTargetH> caps_head, caps_tail;
  // own tail slice per target (j with floor(n/j) in [ya, yb); empty: sj0 > sj1)
  // and the wheel-prefix tables d_P[t * (nd - 1) + k - 1][j - sj0] = P(floor(n/(d_k j)))
  std::vector<u64> sj0, sj1;
  std::vector<DevBuf> d_P;
  // segments
  u64 Rh = 0, head_end = 0, head_segs = 0, head_lim = 0, y_last = 0;
  u64 tail_end = 0, seg_y = 0;       // tail = [head_lim, tail_end); odd segments span <= seg_y
  std::vector<u64> ybound;           // rank r owns [ybound[r], ybound[r+1])
  u64 ya = 0, yb = 0;
  std::vector<TailSeg> tsegs;
  TailWheel tw;                      // the tail's wheel (MT_TAIL_WHEEL: 6 default, or 2)
  std::vector<u64> bp;               // breakpoints a/d, b/d (ascending)
  std::vector<size_t> snap;          // P(bp[i] - 1) = the running prefix after snap[i] segments
  std::vector<int64_t> snapv;        // those prefixes (host, after the tail)
  Sieve2Host* sv = nullptr;
  DevBuf d_mu, d_m, d_bk, d_run, d_snap, d_caps_head, d_caps_tail, d_small;
  u64 cap_c_lo = 1, cap_c_hi = 0, cap_small = 0, nsmall = 0;
  bool cap32 = false;  // MT_FLAG_CAP32: int32 capture outputs (the dense full quotient map)
  UpdateCtx* uc = nullptr;
  KTimer kt;
  int64_t m_head = 0, tail_total = 0, p_end = 0;
  // P at breakpoint y (y must be one of bp)
  int64_t snap_at(u64 y) const {
    for (size_t i = 0; i < bp.size(); i++) if (bp[i] == y) return snapv[i];
    return 0;
  }
  double ms_setup = 0, ms_head = 0, ms_tail = 0, ms_gather = 0, ms_fin = 0;
  cudaEvent_t ev[6] = {};
  int phase = 0;  // 1 after sieve_update, 2 after tail_offset, 3 after gather
  bool head_done = false;
  u64 tseg_next = 0;  // next tail segment of this rank (resumable phase 1)
  ~mt_plan() {
    if (device >= 0) cudaSetDevice(device);
    mt_update_destroy(uc);
    mt_sieve2_destroy(sv);
    for (auto& e : ev) if (e) cudaEventDestroy(e);
    kt.drain();
    if (own_stream && st) cudaStreamDestroy(st);
  }
  // Q slice [j0, j1] of target t whose quotients fall in rank r's tail range (empty: j0 > j1)
  void q_slice(int t, uint32_t r, u64& j0, u64& j1) const {
    j0 = 1; j1 = 0;
    const u64 a = ybound[r], b = ybound[r + 1];
    if (a >= b || jq1[t] < jq0[t]) return;
    // floor(n/j) in [a, b)  <=>  j in [floor(n/b) + 1, floor(n/a)]
    u128 lo = n[t] / (u128)b + 1, hi = n[t] / (u128)a;
    if (lo < jq0[t]) lo = jq0[t];
    if (hi > jq1[t]) hi = jq1[t];
    if (lo > hi) return;
    j0 = (u64)lo; j1 = (u64)hi;
  }
  // first j of target t whose quotient lies in the head (y < head_lim)
  u64 head_j(int t) const { return (u64)(n[t] / (u128)head_lim) + 1; }
  u64 tail_cells() const {
    u64 c = 0;
    for (auto& s : tsegs) c += (u64)s.ntiles * MT_S2_TILE;
    return c;
  }
  int nx() const { return tw.nd - 1; }  // wheel-prefix tables per target besides Q
};

#define PLAN_DEV(p) do { if ((p)->device >= 0) MT_CUDA_CHECK(cudaSetDevice((p)->device)); } while (0)

static CaptureTargetH make_cap(u128 n, u64 j0, u64 j1, int* Q) {
  CaptureTargetH c;
  c.n_lo = (u64)n; c.n_hi = (u64)(n >> 64);
  c.nd = c.n_hi ? (double)c.n_hi * 18446744073709551616.0 + (double)c.n_lo : (double)c.n_lo;
  c.nbits = 0;
  for (u128 x = n; x; x >>= 1) c.nbits++;
  c.jq0 = j0; c.jq1 = j1; c.Q = Q;
  return c;
}

static int plan_setup(mt_plan* P, const mt_job* job) {
  auto T0 = std::chrono::steady_clock::now();
  if (!job || job->n_targets == 0) { mt_set_error("empty job"); return MT_ERR_VALUE; }
  if (job->device >= 0) MT_CUDA_CHECK(cudaSetDevice(job->device));
  MT_CUDA_CHECK(cudaGetDevice(&P->device));
  const int N = (int)job->n_targets;
  P->N = N;
  P->u = job->u;
  P->world = job->shard_world > 1 ? job->shard_world : 1;
  P->rank = job->shard_rank;
  P->flags = job->flags;
  if (P->rank >= P->world) { mt_set_error("shard_rank %u >= shard_world %u", P->rank, P->world); return MT_ERR_VALUE; }
  const u64 u = P->u;
  P->n.resize(N); P->K.resize(N); P->e0.assign(N + 1, 0);
  P->n_lo.assign(job->n_lo, job->n_lo + N);
  P->n_hi.assign(job->n_hi, job->n_hi + N);
  for (int i = 0; i < N; i++) {
    P->n[i] = ((u128)job->n_hi[i] << 64) | job->n_lo[i];
    if (P->n[i] < 4) { mt_set_error("exact job requires n >= 4"); return MT_ERR_VALUE; }
    if (job->n_hi[i] >= (1ull << 11)) { mt_set_error("n >= 2^75 is outside the engine's range"); return MT_ERR_RESOURCE; }
    if ((u128)u <= ceil_sqrt_u128(P->n[i])) { mt_set_error("u must exceed ceil(sqrt(n))"); return MT_ERR_VALUE; }
    P->K[i] = (u64)(P->n[i] / u);
    P->e0[i + 1] = P->e0[i] + P->K[i];
  }
  const u64 NE = P->NE = P->e0[N];
  if (job->stream) { P->st = (cudaStream_t)job->stream; P->own_stream = false; }
  else { MT_CUDA_CHECK(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking)); P->own_stream = true; }
  cudaStream_t st = P->st;
  P->kt.init((P->flags & MT_FLAG_TIMING) != 0);
  for (auto& e : P->ev) MT_CUDA_CHECK(cudaEventCreate(&e));

  // ---- elements (engine.py:134-159)
  RC(dalloc(P->d_nlo, N * 8)); RC(dalloc(P->d_nhi, N * 8)); RC(dalloc(P->d_e0, (N + 1) * 8));
  RC(dalloc(P->d_vd, NE * 8)); RC(dalloc(P->d_vlo, NE * 8)); RC(dalloc(P->d_vhi, NE * 8)); RC(dalloc(P->d_vb, NE));
  RC(dalloc(P->d_k, NE * 8)); RC(dalloc(P->d_tgt, NE * 4)); RC(dalloc(P->d_D, NE * 8)); RC(dalloc(P->d_x, NE * 8));
  RC(dalloc(P->d_mc, NE * 8)); RC(dalloc(P->d_lo, NE * 8)); RC(dalloc(P->d_low, NE * 8)); RC(dalloc(P->d_dq, NE * 8));
  RC(dalloc(P->d_acc, NE * 8)); RC(dalloc(P->d_mmc, NE * 4)); RC(dalloc(P->d_dsp, NE * 8)); RC(dalloc(P->d_fin, NE * 8));
  MT_CUDA_CHECK(cudaMemcpyAsync(P->d_nlo.p, job->n_lo, N * 8, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemcpyAsync(P->d_nhi.p, job->n_hi, N * 8, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemcpyAsync(P->d_e0.p, P->e0.data(), (N + 1) * 8, cudaMemcpyHostToDevice, st));
  std::vector<unsigned long long> tstat(4 * N, 0);
  {
    DevBuf d_ts;
    RC(dalloc(d_ts, 4 * N * 8));
    MT_CUDA_CHECK(cudaMemsetAsync(d_ts.p, 0, 4 * N * 8, st));
    P->xalpha = MT_XCUT_ALPHA_DEFAULT;
    if (const char* e = getenv("MT_XCUT_ALPHA")) P->xalpha = atof(e);
    const double xalpha = P->xalpha;
    ElemInitArgs a{P->d_nlo.as<u64>(), P->d_nhi.as<u64>(), P->d_e0.as<u64>(), N, u, NE,
                   P->d_vd.as<double>(), P->d_vlo.as<u64>(), P->d_vhi.as<u64>(), P->d_vb.as<uint8_t>(), P->d_k.as<u64>(),
                   P->d_tgt.as<uint32_t>(), P->d_D.as<u64>(), P->d_x.as<u64>(), P->d_mc.as<u64>(), P->d_lo.as<u64>(),
                   xalpha, d_ts.as<unsigned long long>()};
    if (NE) k_elem_init<<<(unsigned)((NE + 255) / 256), 256, 0, st>>>(a);
    MT_CUDA_CHECK(cudaGetLastError());
    MT_CUDA_CHECK(cudaMemcpyAsync(tstat.data(), d_ts.p, 4 * N * 8, cudaMemcpyDeviceToHost, st));
    MT_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  for (int i = 0; i < N; i++) {
    P->Ymc = std::max<u64>(P->Ymc, tstat[4 * i]);
    P->Ymc_ref = std::max<u64>(P->Ymc_ref, tstat[4 * i + 3]);
    P->counted_items += tstat[4 * i + 1];
    P->dense_items += tstat[4 * i + 2];
  }

  // ---- quotient tables: Q_t[j] = M(floor(n_t/j)), j in [jq0_t, jq1_t]; the tail
  // part also needs the wheel-prefix captures at floor(n/(d j)), d | W, d > 1, so a
  // table entry is budgeted at 4 bytes per divisor
  {
    int W = 6;
    if (const char* ev = getenv("MT_TAIL_WHEEL")) W = atoi(ev);
    if (W != 2 && W != 6) { mt_set_error("MT_TAIL_WHEEL must be 2 or 6"); return MT_ERR_VALUE; }
    P->tw = tail_wheel(W);
  }
  const u64 q_budget = job->q_budget_bytes ? job->q_budget_bytes : (128ull << 30);
  P->J.assign(N, 0); P->jq0.assign(N, 0); P->jq1.assign(N, 0);
  P->cap_c_lo = job->cap_c_lo; P->cap_c_hi = job->cap_c_hi;
  for (int i = 0; i < N; i++) {
    P->jq0[i] = (u64)(P->n[i] / ((u128)u + 1)) + 1;
    P->J[i] = (u64)(P->n[i] / ((u128)P->Ymc + 1));
  }
  for (int it = 0; it < 64; it++) {  // cap the tables to the budget by scaling J down uniformly
    u64 q_total = 0;
    for (int i = 0; i < N; i++) {
      u64 hi = P->J[i];
      if (i == 0 && P->cap_c_hi >= P->cap_c_lo && P->cap_c_hi > hi) hi = P->cap_c_hi;
      P->jq1[i] = hi;
      if (hi >= P->jq0[i]) q_total += (hi - P->jq0[i] + 1);
    }
    if (q_total * 4 * P->tw.nd <= q_budget) break;
    for (int i = 0; i < N; i++) P->J[i] = P->J[i] / 2;
  }
  for (int i = 0; i < N; i++)
    if (P->J[i] < P->jq0[i]) P->J[i] = 0;  // no Q-gather for this target
  P->d_Q.clear();
  P->d_Q.reserve(N);
  P->tdev.resize(N);
  for (int i = 0; i < N; i++) {
    P->d_Q.emplace_back();
    u64 cnt = P->jq1[i] >= P->jq0[i] ? P->jq1[i] - P->jq0[i] + 1 : 0;
    RC(dalloc(P->d_Q[i], cnt * 4));
    P->tdev[i].Q = P->d_Q[i].as<int>();
    P->tdev[i].jq0 = P->jq0[i];
    P->tdev[i].wlo = 0;
    P->tdev[i].whi = cnt;
    if (cnt) P->caps_head.push_back(make_cap(P->n[i], P->jq0[i], P->jq1[i], P->tdev[i].Q));
  }
  RC(dalloc(P->d_J, N * 8));
  MT_CUDA_CHECK(cudaMemcpyAsync(P->d_J.p, P->J.data(), N * 8, cudaMemcpyHostToDevice, st));
  if (NE) k_elem_split<<<(unsigned)((NE + 255) / 256), 256, 0, st>>>(NE, P->d_k.as<u64>(), P->d_tgt.as<uint32_t>(), P->d_J.as<u64>(), P->d_lo.as<u64>(), P->d_x.as<u64>(), P->d_low.as<u64>(), P->d_dq.as<u64>());
  if (NE) k_elem_dsp<<<(unsigned)((NE + 255) / 256), 256, 0, st>>>(NE, P->d_vd.as<double>(), P->d_dsp.as<u64>());
  // element groups for the window walk: consecutive k of one target, size ~clamp(k/8, 32, 1024)
  for (int i = 0; i < N; i++) {
    u64 k0 = 1;
    while (k0 <= P->K[i]) {
      P->gstart.push_back(P->e0[i] + k0 - 1);
      // power-of-two sizes: below 256 the window walk splits each element over
      // 256/size threads, above it each thread takes size/256 elements
      u64 gs = 32;
      while (gs * 2 <= std::min<u64>(1024, k0 / 8)) gs *= 2;
      k0 += gs;
    }
  }
  const u64 ng = P->ng = P->gstart.size();
  P->gstart.push_back(NE);
  RC(dalloc(P->d_gs, (ng + 1) * 8)); RC(dalloc(P->d_gylo, ng * 8)); RC(dalloc(P->d_gyhi, ng * 8)); RC(dalloc(P->d_gw, ng));
  MT_CUDA_CHECK(cudaMemcpyAsync(P->d_gs.p, P->gstart.data(), (ng + 1) * 8, cudaMemcpyHostToDevice, st));
  if (ng) k_group_meta<<<(unsigned)ng, 256, 0, st>>>(P->d_gs.as<u64>(), ng, P->d_vlo.as<u64>(), P->d_vhi.as<u64>(), P->d_x.as<u64>(), P->d_low.as<u64>(), P->d_dsp.as<u64>(), P->d_gylo.as<u64>(), P->d_gyhi.as<u64>(), P->d_gw.as<uint8_t>());
  GroupDev grp{P->d_gs.as<u64>(), P->d_gylo.as<u64>(), P->d_gyhi.as<u64>(), P->d_gw.as<uint8_t>(), ng};
  u64 head_end = P->Ymc;
  {
    DevBuf d_we;
    RC(dalloc(d_we, 8));
    MT_CUDA_CHECK(cudaMemsetAsync(d_we.p, 0, 8, st));
    if (NE) k_window_extent<<<(unsigned)((NE + 255) / 256), 256, 0, st>>>(NE, P->d_vlo.as<u64>(), P->d_vhi.as<u64>(), P->d_low.as<u64>(), P->d_x.as<u64>(), d_we.as<unsigned long long>());
    unsigned long long we = 0;
    MT_CUDA_CHECK(cudaMemcpyAsync(&we, d_we.p, 8, cudaMemcpyDeviceToHost, st));
    MT_CUDA_CHECK(cudaStreamSynchronize(st));
    head_end = std::max<u64>(head_end, we);
  }
  P->cap_small = job->cap_small;
  if (P->cap_small > head_end) head_end = P->cap_small;
  if (head_end > u) head_end = u;
  P->head_end = head_end;


  // ---- segments (production sieve tiles of 2^17 cells)
  // default tail segment = 6 tiles per SM (the persistent sieve CTAs each take 6
  // contiguous tiles; fewer per-segment fill setups and finish launches); head
  // segments default to 1 tile per SM: the head's sparse walk gathers M(y) from the
  // segment's 2-byte table, and at 39 MB it stays in the L2 half of each die (ncu:
  // 62 % L2 hits with 2 tiles per SM; measured at 1e19: head phase -1 %)
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P->device);
  u64 tiles_per_sm = 6, tiles_per_sm_head = 1;
  if (const char* e = getenv("MT_SEG_TILES_PER_SM")) tiles_per_sm = strtoull(e, nullptr, 10);
  if (const char* e = getenv("MT_SEG_TILES_PER_SM_HEAD")) tiles_per_sm_head = strtoull(e, nullptr, 10);
  P->Rh = job->seg_log2_head ? 1ull << job->seg_log2_head : (u64)nsm * tiles_per_sm_head * MT_S2_TILE;
  // tail segments: tiles of 2^17 odd cells, 2^18 y each
  const u64 tail_tiles = job->seg_log2_tail ? 1ull << (job->seg_log2_tail - 17) : (u64)nsm * tiles_per_sm;
  const u64 Rh = P->Rh;
  if (Rh < MT_S2_TILE || (Rh % MT_S2_TILE) || Rh > (1ull << 31) || (job->seg_log2_tail && job->seg_log2_tail < 17) ||
      tail_tiles == 0 || tail_tiles * MT_S2_TILE > (1ull << 31)) {
    mt_set_error("bad segment sizes");
    return MT_ERR_VALUE;
  }
  P->seg_y = tail_tiles * P->tw.tile_y;
  // the head ends on the wheel's alignment (its last segment may be shorter than Rh)
  const u64 AL = P->tw.align();
  P->head_lim = (head_end + 1 + AL - 1) / AL * AL;  // first y of the tail
  P->head_segs = (P->head_lim + Rh - 1) / Rh;
  P->tail_end = P->head_lim;
  if (u + 1 > P->head_lim) P->tail_end = (u + 1 + AL - 1) / AL * AL;
  P->ybound = tail_partition(P->tw, P->head_lim, P->tail_end, P->world);
  P->ya = P->ybound[P->rank];
  P->yb = P->ybound[P->rank + 1];
  tail_segments(P->tw, P->ya, P->yb, P->seg_y, P->tsegs, P->bp, P->snap);
  P->y_last = std::max(P->tail_end, P->head_lim) - 1;
  RC(mt_sieve2_create(&P->sv, P->y_last, (uint32_t)std::max<u64>(Rh / MT_S2_TILE, tail_tiles), st));
  RC(dalloc(P->d_mu, Rh)); RC(dalloc(P->d_m, Rh * 2)); RC(dalloc(P->d_bk, (Rh / MT_BLK) * 8 + 8));
  RC(dalloc(P->d_run, 8)); RC(dalloc(P->d_snap, 8 * 8));
  // own tail slices, their wheel-prefix tables, and the tail capture list: the
  // prefix P at floor(n/j) (into Q) and at floor(floor(n/d)/j) = floor(n/(d j)) for
  // every other divisor d of the wheel, for j in the slice
  P->sj0.assign(N, 1); P->sj1.assign(N, 0);
  P->d_P.clear();
  P->d_P.reserve((size_t)N * P->nx());
  for (int i = 0; i < N; i++) {
    u64 j0, j1;
    P->q_slice(i, P->rank, j0, j1);
    P->sj0[i] = j0; P->sj1[i] = j1;
    const u64 cnt = j1 >= j0 ? j1 - j0 + 1 : 0;
    if (cnt) P->caps_tail.push_back(make_cap(P->n[i], j0, j1, P->tdev[i].Q + (j0 - P->jq0[i])));
    for (int k = 1; k < P->tw.nd; k++) {
      P->d_P.emplace_back();
      RC(dalloc(P->d_P.back(), cnt * 4));
      if (cnt) P->caps_tail.push_back(make_cap(P->n[i] / P->tw.d[k], j0, j1, P->d_P.back().as<int>()));
    }
  }
  RC(dalloc(P->d_caps_head, P->caps_head.size() * sizeof(CaptureTargetH)));
  RC(dalloc(P->d_caps_tail, P->caps_tail.size() * sizeof(CaptureTargetH)));
  if (!P->caps_head.empty())
    MT_CUDA_CHECK(cudaMemcpyAsync(P->d_caps_head.p, P->caps_head.data(), P->caps_head.size() * sizeof(CaptureTargetH), cudaMemcpyHostToDevice, st));
  if (!P->caps_tail.empty())
    MT_CUDA_CHECK(cudaMemcpyAsync(P->d_caps_tail.p, P->caps_tail.data(), P->caps_tail.size() * sizeof(CaptureTargetH), cudaMemcpyHostToDevice, st));
  P->nsmall = P->cap_small ? P->cap_small + 1 : 0;
  P->cap32 = (P->flags & MT_FLAG_CAP32) != 0;
  RC(dalloc(P->d_small, P->nsmall * (P->cap32 ? 4 : 8)));

  ElemDev E;
  E.vd = P->d_vd.as<double>(); E.vlo = P->d_vlo.as<u64>(); E.vhi = P->d_vhi.as<u64>(); E.vbits = P->d_vb.as<uint8_t>();
  E.k = P->d_k.as<u64>(); E.tgt = P->d_tgt.as<uint32_t>(); E.mcut = P->d_mc.as<u64>(); E.xcut = P->d_x.as<u64>();
  E.lo = P->d_lo.as<u64>(); E.lo_w = P->d_low.as<u64>(); E.dq_hi = P->d_dq.as<u64>(); E.d_sp = P->d_dsp.as<u64>(); E.n = NE;
  Shard sh;
  sh.rank = P->rank; sh.world = P->world; sh.flags = P->flags;
  RC(mt_update_create(&P->uc, E, P->d_acc.as<u64>(), P->d_mmc.as<int32_t>(), P->K.data(), P->tdev.data(), N, grp, sh,
                      &P->kt, st));
  MT_CUDA_CHECK(cudaStreamSynchronize(st));
  P->ms_setup = ms_since(T0);
  return MT_OK;
}

extern "C" int mt_plan_create(const mt_job* job, mt_plan** out) {
  g_err[0] = 0;
  if (!out) { mt_set_error("null plan out"); return MT_ERR_VALUE; }
  *out = nullptr;
  mt_plan* P = new mt_plan();
  int rc = plan_setup(P, job);
  if (rc != MT_OK) { delete P; return rc; }
  *out = P;
  return MT_OK;
}

extern "C" void mt_plan_destroy(mt_plan* p) { delete p; }

// phase 1, resumable: the head (on the first step: sieve, this rank's share of
// the head update, captures) and up to max_tail_segments of this rank's odd-cell
// tail segments per call; *done = 1 once the tail is complete
extern "C" int mt_plan_sieve_step(mt_plan* P, uint64_t max_tail_segments, int* done, int64_t* m_head,
                                  int64_t* tail_total) {
  PLAN_DEV(P);
  cudaStream_t st = P->st;
  if (!P->head_done) {
    NvtxRange nv("mt.head");
    P->kt.reset();
    P->launches = 0;
    mt_update_reset_launches(P->uc);
    mt_sieve2_launches(P->sv, true);
    MT_CUDA_CHECK(cudaMemsetAsync(P->d_acc.p, 0, P->NE * 8, st));
    MT_CUDA_CHECK(cudaMemsetAsync(P->d_mmc.p, 0, P->NE * 4, st));
    MT_CUDA_CHECK(cudaMemsetAsync(P->d_run.p, 0, 8, st));
    MT_CUDA_CHECK(cudaMemsetAsync(P->d_snap.p, 0, 8 * 8, st));
    MT_CUDA_CHECK(cudaEventRecord(P->ev[0], st));
    for (u64 s = 0; s < P->head_segs; s++) {
      const u64 Y0 = s * P->Rh, R = std::min(P->Rh, P->head_lim - Y0);  // the last segment ends at head_lim
      RC(mt_sieve2_run(P->sv, Y0, (uint32_t)(R / MT_S2_TILE), P->d_run.as<int64_t>(), P->d_mu.as<int8_t>(),
                       P->d_m.as<int16_t>(), P->d_bk.as<int64_t>(), nullptr,
                       (const CaptureTarget2*)P->d_caps_head.p, (int)P->caps_head.size(), st, &P->kt));
      RC(mt_update_head_segment(P->uc, Y0, R, P->d_mu.as<int8_t>(), P->d_m.as<int16_t>(), P->d_bk.as<int64_t>(), st));
      if (P->nsmall && Y0 <= P->cap_small) {
        if (P->cap32)
          k_copy_small<int32_t><<<(unsigned)((R + 255) / 256), 256, 0, st>>>(P->d_m.as<int16_t>(), P->d_bk.as<int64_t>(), Y0, R, P->cap_small, P->d_small.as<int32_t>());
        else
          k_copy_small<int64_t><<<(unsigned)((R + 255) / 256), 256, 0, st>>>(P->d_m.as<int16_t>(), P->d_bk.as<int64_t>(), Y0, R, P->cap_small, P->d_small.as<int64_t>());
        P->launches++;
      }
    }
    int64_t mh = 0;
    MT_CUDA_CHECK(cudaMemcpyAsync(&mh, P->d_run.p, 8, cudaMemcpyDeviceToHost, st));
    MT_CUDA_CHECK(cudaMemsetAsync(P->d_run.p, 0, 8, st));  // tail prefixes are rank-local
    MT_CUDA_CHECK(cudaEventRecord(P->ev[1], st));
    MT_CUDA_CHECK(cudaStreamSynchronize(st));
    float f = 0;
    cudaEventElapsedTime(&f, P->ev[0], P->ev[1]);
    P->ms_head = f;
    P->ms_tail = 0;
    P->m_head = mh;
    P->tseg_next = 0;
    P->head_done = true;
  }
  const u64 ns = P->tsegs.size();
  const u64 room = ns > P->tseg_next ? ns - P->tseg_next : 0;
  const u64 s_end = P->tseg_next + std::min<u64>(room, max_tail_segments);
  if (P->tseg_next < s_end) {
    NvtxRange nv("mt.tail");
    MT_CUDA_CHECK(cudaEventRecord(P->ev[1], st));
    for (u64 s = P->tseg_next; s < s_end; s++) {
      RC(mt_sieve2_run(P->sv, P->tsegs[s].Y0, P->tsegs[s].ntiles, P->d_run.as<int64_t>(), nullptr, nullptr, nullptr,
                       nullptr, (const CaptureTarget2*)P->d_caps_tail.p, (int)P->caps_tail.size(), st, &P->kt,
                       P->tw.W));
      // prefix snapshots P(bp - 1) at the breakpoints a/d, b/d
      for (size_t i = 0; i < P->bp.size(); i++)
        if (P->snap[i] == s + 1)
          MT_CUDA_CHECK(cudaMemcpyAsync(P->d_snap.as<int64_t>() + i, P->d_run.p, 8, cudaMemcpyDeviceToDevice, st));
    }
    MT_CUDA_CHECK(cudaEventRecord(P->ev[2], st));
    MT_CUDA_CHECK(cudaStreamSynchronize(st));
    float f = 0;
    cudaEventElapsedTime(&f, P->ev[1], P->ev[2]);
    P->ms_tail += f;
    P->tseg_next = s_end;
  }
  MT_CUDA_CHECK(cudaGetLastError());
  *done = P->tseg_next >= ns;
  if (*done) {
    int64_t v[9] = {0};
    MT_CUDA_CHECK(cudaMemcpy(v, P->d_run.p, 8, cudaMemcpyDeviceToHost));
    MT_CUDA_CHECK(cudaMemcpy(v + 1, P->d_snap.p, 8 * 8, cudaMemcpyDeviceToHost));
    P->p_end = v[0];
    P->snapv.assign(v + 1, v + 1 + P->bp.size());
    // this rank's M-total over [ya, yb): sum_d mu(d) (P(yb/d - 1) - P(ya/d - 1))
    int64_t tt = 0;
    if (ns)
      for (int k = 0; k < P->tw.nd; k++)
        tt += P->tw.s[k] * (P->snap_at(P->yb / P->tw.d[k]) - P->snap_at(P->ya / P->tw.d[k]));
    P->tail_total = tt;
    P->phase = 1;
    if (m_head) *m_head = P->m_head;
    if (tail_total) *tail_total = P->tail_total;
  }
  return MT_OK;
}

// phase 1 in one call: head and this rank's whole tail
extern "C" int mt_plan_sieve_update(mt_plan* P, int64_t* m_head, int64_t* tail_total) {
  P->head_done = false;
  int done = 0;
  RC(mt_plan_sieve_step(P, ~0ull, &done, nullptr, nullptr));
  if (m_head) *m_head = P->m_head;
  if (tail_total) *tail_total = P->tail_total;
  return MT_OK;
}

// ---- checkpoint / resume (reference MERTCKP1 header, engine.py:646-680, with
// version 4 marking the sm100 engine state that follows it)
#pragma pack(push, 1)
struct CkptHead {
  char magic[8];
  uint32_t version, flags;
  uint64_t n_lo, n_hi, u, next_y1, K;
  int64_t m_running;
  uint64_t block_len;
};
#pragma pack(pop)
static_assert(sizeof(CkptHead) == 72, "MERTCKP1 header is <8sII QQ Q Q Q q Q>");
#define MT_CKPT_VERSION 4

static int write_all(FILE* f, const void* p, u64 bytes) {
  if (bytes && fwrite(p, 1, bytes, f) != bytes) { mt_set_error("checkpoint write failed (disk full?)"); return MT_ERR_RESOURCE; }
  return MT_OK;
}
static int write_dev(FILE* f, const void* dptr, u64 bytes) {
  const u64 CH = 256ull << 20;
  std::vector<char> h((size_t)std::min(bytes, CH));
  for (u64 o = 0; o < bytes; o += CH) {
    const u64 b = std::min(CH, bytes - o);
    MT_CUDA_CHECK(cudaMemcpy(h.data(), (const char*)dptr + o, b, cudaMemcpyDeviceToHost));
    RC(write_all(f, h.data(), b));
  }
  return MT_OK;
}
static int read_dev(FILE* f, void* dptr, u64 bytes) {
  const u64 CH = 256ull << 20;
  std::vector<char> h((size_t)std::min(bytes, CH));
  for (u64 o = 0; o < bytes; o += CH) {
    const u64 b = std::min(CH, bytes - o);
    if (fread(h.data(), 1, b, f) != b) { mt_set_error("checkpoint truncated"); return MT_ERR_CONTRACT; }
    MT_CUDA_CHECK(cudaMemcpy((char*)dptr + o, h.data(), b, cudaMemcpyHostToDevice));
  }
  return MT_OK;
}
static int read_u64(FILE* f, u64* v) {
  if (fread(v, 8, 1, f) != 1) { mt_set_error("checkpoint truncated"); return MT_ERR_CONTRACT; }
  return MT_OK;
}

// header flags: shard rank | world << 16 (one file per rank; single-target jobs)
// layout after the header: acc (K u64), M(mcut) (K i32), Q (u64 count + int32),
// P2 (u64 count + int32), small captures (u64 count + element bytes), head M,
// running prefix and the two prefix snapshots (i64 each)
static int ckpt_write(mt_plan* P, FILE* f) {
  int64_t tail[10] = {P->m_head, 0};
  MT_CUDA_CHECK(cudaMemcpy(tail + 1, P->d_run.p, 8, cudaMemcpyDeviceToHost));
  MT_CUDA_CHECK(cudaMemcpy(tail + 2, P->d_snap.p, 8 * 8, cudaMemcpyDeviceToHost));
  CkptHead h{};
  memcpy(h.magic, "MERTCKP1", 8);
  h.version = MT_CKPT_VERSION;
  h.flags = P->rank | (P->world << 16);
  h.n_lo = P->n_lo[0]; h.n_hi = P->n_hi[0]; h.u = P->u;
  h.next_y1 = P->tseg_next < P->tsegs.size() ? P->tsegs[P->tseg_next].Y0 : P->y_last + 1;
  h.K = P->K[0];
  h.m_running = P->m_head;
  h.block_len = P->seg_y;
  RC(write_all(f, &h, sizeof(h)));
  RC(write_all(f, &P->xalpha, 8));  // the counted / dense split the head state was computed with
  RC(write_dev(f, P->d_acc.p, P->NE * 8));
  RC(write_dev(f, P->d_mmc.p, P->NE * 4));
  const u64 qn = P->jq1[0] >= P->jq0[0] ? P->jq1[0] - P->jq0[0] + 1 : 0;
  RC(write_all(f, &qn, 8));
  RC(write_dev(f, P->tdev[0].Q, qn * 4));
  const u64 pn = P->sj1[0] >= P->sj0[0] ? P->sj1[0] - P->sj0[0] + 1 : 0;
  const u64 pw = pn | ((u64)P->tw.W << 56);  // the tail wheel travels with the slice size
  RC(write_all(f, &pw, 8));
  for (int k = 0; k < P->nx(); k++) RC(write_dev(f, P->d_P[k].p, pn * 4));
  const u64 sb = P->nsmall * (P->cap32 ? 4 : 8);
  RC(write_all(f, &sb, 8));
  RC(write_dev(f, P->d_small.p, sb));
  RC(write_all(f, tail, sizeof(tail)));
  return MT_OK;
}

// written to path.tmp, flushed and synced, then renamed over path: a failed
// write leaves the previous checkpoint in place
extern "C" int mt_plan_checkpoint(mt_plan* P, const char* path) {
  if (P->N != 1) { mt_set_error("checkpoints cover single-target jobs only"); return MT_ERR_CONTRACT; }
  if (!P->head_done) { mt_set_error("checkpoint before the head is sieved"); return MT_ERR_CONTRACT; }
  PLAN_DEV(P);
  MT_CUDA_CHECK(cudaStreamSynchronize(P->st));
  std::string tmp = std::string(path) + ".tmp";
  FILE* f = fopen(tmp.c_str(), "wb");
  if (!f) { mt_set_error("cannot open %s", tmp.c_str()); return MT_ERR_RESOURCE; }
  int rc = ckpt_write(P, f);
  if (rc == MT_OK && fflush(f) != 0) { mt_set_error("checkpoint flush failed"); rc = MT_ERR_RESOURCE; }
  if (rc == MT_OK && fsync(fileno(f)) != 0) { mt_set_error("checkpoint fsync failed"); rc = MT_ERR_RESOURCE; }
  if (fclose(f) != 0 && rc == MT_OK) { mt_set_error("checkpoint close failed"); rc = MT_ERR_RESOURCE; }
  if (rc != MT_OK) { remove(tmp.c_str()); return rc; }
  if (rename(tmp.c_str(), path) != 0) { remove(tmp.c_str()); mt_set_error("cannot move %s into place", tmp.c_str()); return MT_ERR_RESOURCE; }
  return MT_OK;
}

extern "C" int mt_plan_restore(mt_plan* P, const char* path) {
  if (P->N != 1) { mt_set_error("checkpoints cover single-target jobs only"); return MT_ERR_CONTRACT; }
  PLAN_DEV(P);
  FILE* f = fopen(path, "rb");
  if (!f) { mt_set_error("cannot open %s", path); return MT_ERR_VALUE; }
  struct Closer { FILE* f; ~Closer() { fclose(f); } } cl{f};
  CkptHead h{};
  if (fread(&h, sizeof(h), 1, f) != 1 || memcmp(h.magic, "MERTCKP1", 8) || h.version != MT_CKPT_VERSION) {
    mt_set_error("not an sm100 checkpoint file (version %u)", MT_CKPT_VERSION);
    return MT_ERR_CONTRACT;
  }
  if (h.n_lo != P->n_lo[0] || h.n_hi != P->n_hi[0] || h.u != P->u || h.K != P->K[0] || h.block_len != P->seg_y ||
      h.flags != (P->rank | (P->world << 16))) {
    mt_set_error("checkpoint built for another job (n, u, K, segment size or rank/world differ)");
    return MT_ERR_CONTRACT;
  }
  double xa = -1;
  if (fread(&xa, 8, 1, f) != 1 || xa != P->xalpha) {
    mt_set_error("checkpoint built with another counted / dense split (MT_XCUT_ALPHA)");
    return MT_ERR_CONTRACT;
  }
  RC(read_dev(f, P->d_acc.p, P->NE * 8));
  RC(read_dev(f, P->d_mmc.p, P->NE * 4));
  u64 qn = 0, pw = 0, sb = 0;
  RC(read_u64(f, &qn));
  const u64 qn_plan = P->jq1[0] >= P->jq0[0] ? P->jq1[0] - P->jq0[0] + 1 : 0;
  if (qn != qn_plan) { mt_set_error("checkpoint quotient table differs from this plan's"); return MT_ERR_CONTRACT; }
  RC(read_dev(f, P->tdev[0].Q, qn * 4));
  RC(read_u64(f, &pw));
  const u64 pn = pw & ((1ull << 56) - 1);
  const u64 pn_plan = P->sj1[0] >= P->sj0[0] ? P->sj1[0] - P->sj0[0] + 1 : 0;
  if (pn != pn_plan || (int)(pw >> 56) != P->tw.W) {
    mt_set_error("checkpoint tail slice or wheel differs from this plan's");
    return MT_ERR_CONTRACT;
  }
  for (int k = 0; k < P->nx(); k++) RC(read_dev(f, P->d_P[k].p, pn * 4));
  RC(read_u64(f, &sb));
  if (sb != P->nsmall * (P->cap32 ? 4 : 8)) { mt_set_error("checkpoint capture size differs"); return MT_ERR_CONTRACT; }
  RC(read_dev(f, P->d_small.p, sb));
  int64_t tail[10];
  if (fread(tail, sizeof(tail), 1, f) != 1) { mt_set_error("checkpoint truncated"); return MT_ERR_CONTRACT; }
  MT_CUDA_CHECK(cudaMemcpy(P->d_run.p, tail + 1, 8, cudaMemcpyHostToDevice));
  MT_CUDA_CHECK(cudaMemcpy(P->d_snap.p, tail + 2, 8 * 8, cudaMemcpyHostToDevice));
  P->m_head = tail[0];
  P->head_done = true;
  u64 s = 0;
  while (s < P->tsegs.size() && P->tsegs[s].Y0 != h.next_y1) s++;
  if (s == P->tsegs.size() && h.next_y1 != P->y_last + 1) {
    mt_set_error("checkpoint position is not a tail segment boundary");
    return MT_ERR_CONTRACT;
  }
  P->tseg_next = s;
  P->kt.reset();
  P->launches = 0;
  mt_update_reset_launches(P->uc);
  mt_sieve2_launches(P->sv, true);
  P->ms_head = 0;
  P->ms_tail = 0;
  return MT_OK;
}

// phase 2: absolute M on this rank's tail slices: Q[j] = sum_d mu(d) (P(floor(n/(d j)))
// - P(ya/d - 1)) + M(ya - 1), offset = M(ya - 1).  With world > 1 the capture window
// is then masked to the entries this rank owns, ready for the caller's
// sum-reduction (mt_plan_cap_window).
extern "C" int mt_plan_tail_offset(mt_plan* P, int64_t offset) {
  if (P->phase < 1) { mt_set_error("tail_offset before sieve_update"); return MT_ERR_CONTRACT; }
  PLAN_DEV(P);
  int64_t delta = offset;
  if (!P->tsegs.empty())
    for (int k = 0; k < P->tw.nd; k++) delta -= P->tw.s[k] * P->snap_at(P->ya / P->tw.d[k]);
  if (delta > INT32_MAX || delta < INT32_MIN) { mt_set_error("M offset beyond int32"); return MT_ERR_OVERFLOW; }
  for (int t = 0; t < P->N; t++) {
    if (P->sj0[t] > P->sj1[t]) continue;
    const u64 cnt = P->sj1[t] - P->sj0[t] + 1;
    CombineArgs ca{};
    ca.n = P->nx();
    for (int k = 0; k < ca.n; k++) { ca.T[k] = P->d_P[(size_t)t * P->nx() + k].as<int>(); ca.s[k] = P->tw.s[k + 1]; }
    k_q_combine<<<(unsigned)((cnt + 255) / 256), 256, 0, P->st>>>(P->tdev[t].Q + (P->sj0[t] - P->jq0[t]), ca, cnt,
                                                                  (int)delta);
    P->launches++;
    MT_CUDA_CHECK(cudaGetLastError());
  }
  if (P->world > 1 && P->cap_c_hi >= P->cap_c_lo && P->jq1[0] >= P->jq0[0]) {
    const u64 c0 = std::max(P->cap_c_lo, P->jq0[0]), c1 = std::min(P->cap_c_hi, P->jq1[0]);
    if (c1 >= c0) {
      k_cap_mask<<<(unsigned)((c1 - c0 + 1 + 255) / 256), 256, 0, P->st>>>(P->tdev[0].Q, P->jq0[0], c0, c1, P->sj0[0],
                                                                           P->sj1[0], P->head_j(0), P->rank == 0);
      P->launches++;
      MT_CUDA_CHECK(cudaGetLastError());
    }
  }
  MT_CUDA_CHECK(cudaStreamSynchronize(P->st));
  P->phase = 2;
  return MT_OK;
}

extern "C" int mt_plan_q_slice(mt_plan* P, uint32_t target, uint32_t rank, void** dptr, uint64_t* count) {
  if ((int)target >= P->N || rank >= P->world) { mt_set_error("bad target/rank"); return MT_ERR_VALUE; }
  u64 j0, j1;
  P->q_slice((int)target, rank, j0, j1);
  if (j0 > j1) { *dptr = nullptr; *count = 0; return MT_OK; }
  *dptr = (void*)(P->tdev[target].Q + (j0 - P->jq0[target]));
  *count = j1 - j0 + 1;
  return MT_OK;
}

// target 0's capture window Q[cap_c_lo .. cap_c_hi] (device int32): with world > 1,
// after tail_offset each rank holds its own entries and zeros elsewhere, so one
// sum-reduction assembles the window (the M(floor(n/c)) outputs) on every rank
extern "C" int mt_plan_cap_window(mt_plan* P, void** dptr, uint64_t* count) {
  *dptr = nullptr;
  *count = 0;
  if (P->cap_c_hi < P->cap_c_lo || P->jq1[0] < P->jq0[0]) return MT_OK;
  const u64 c0 = std::max(P->cap_c_lo, P->jq0[0]), c1 = std::min(P->cap_c_hi, P->jq1[0]);
  if (c1 < c0) return MT_OK;
  *dptr = (void*)(P->tdev[0].Q + (c0 - P->jq0[0]));
  *count = c1 - c0 + 1;
  return MT_OK;
}

extern "C" int mt_plan_acc(mt_plan* P, void** dptr, uint64_t* count) {
  *dptr = P->d_acc.p;
  *count = P->NE;
  return MT_OK;
}

// phase 3: dense items from the quotient tables -- with world > 1 rank r takes
// the items whose table entry lies in its own tail slice plus every w-th chunk
// of the items in the (replicated) head part; rank 0 also applies the
// summation-by-parts correction -M(mcut)*xcut
extern "C" int mt_plan_gather(mt_plan* P) {
  if (P->phase < 2) { mt_set_error("gather before tail_offset"); return MT_ERR_CONTRACT; }
  PLAN_DEV(P);
  NvtxRange nv("mt.gather");
  MT_CUDA_CHECK(cudaEventRecord(P->ev[3], P->st));
  const int N = P->N;
  std::vector<u64> wlo(N, 0), whi(N, 0);
  for (int t = 0; t < N; t++) whi[t] = P->jq1[t] >= P->jq0[t] ? P->jq1[t] - P->jq0[t] + 1 : 0;
  if (P->world == 1) {
    RC(mt_update_qgather(P->uc, wlo.data(), whi.data(), false, P->st));
  } else {
    std::vector<u64> slo(N, 0), shi(N, 0), hlo(N, 0);
    for (int t = 0; t < N; t++) {
      if (P->sj1[t] >= P->sj0[t]) { slo[t] = P->sj0[t] - P->jq0[t]; shi[t] = P->sj1[t] - P->jq0[t] + 1; }
      const u64 jh = P->head_j(t);
      hlo[t] = jh > P->jq0[t] ? std::min(jh - P->jq0[t], whi[t]) : 0;
    }
    RC(mt_update_qgather(P->uc, slo.data(), shi.data(), false, P->st));
    RC(mt_update_qgather(P->uc, hlo.data(), whi.data(), true, P->st));
  }
  if (P->rank == 0) RC(mt_update_finish(P->uc, P->st));
  MT_CUDA_CHECK(cudaEventRecord(P->ev[4], P->st));
  MT_CUDA_CHECK(cudaStreamSynchronize(P->st));
  float f = 0;
  cudaEventElapsedTime(&f, P->ev[3], P->ev[4]); P->ms_gather = f;
  P->phase = 3;
  return MT_OK;
}

// phase 4: level-parallel resolve of every target (engine.py:394-402) and outputs
extern "C" int mt_plan_resolve(mt_plan* P, mt_result* out) {
  if (P->phase < 3) { mt_set_error("finalize before the harmonic array is complete"); return MT_ERR_CONTRACT; }
  PLAN_DEV(P);
  NvtxRange nv("mt.resolve");
  cudaStream_t st = P->st;
  MT_CUDA_CHECK(cudaEventRecord(P->ev[4], st));
  for (int i = 0; i < P->N; i++)
    RC(mt_finalize_dev(P->d_acc.as<u64>() + P->e0[i], P->d_D.as<u64>() + P->e0[i], P->K[i], P->d_fin.as<int64_t>() + P->e0[i], st, &P->launches));
  MT_CUDA_CHECK(cudaEventRecord(P->ev[5], st));
  DevBuf d_capm;
  if (out && out->finals && P->NE)
    MT_CUDA_CHECK(cudaMemcpyAsync(out->finals, P->d_fin.p, P->NE * 8, cudaMemcpyDeviceToHost, st));
  if (out && out->acc_out && P->NE)
    MT_CUDA_CHECK(cudaMemcpyAsync(out->acc_out, P->d_acc.p, P->NE * 8, cudaMemcpyDeviceToHost, st));
  if (out && out->cap_m_out && P->cap_c_hi >= P->cap_c_lo && P->cap32) {  // int32: straight from Q
    u64 cnt = P->cap_c_hi - P->cap_c_lo + 1;
    if (P->cap_c_lo < P->jq0[0]) { mt_set_error("capture range below floor(n/(u+1))+1"); return MT_ERR_VALUE; }
    MT_CUDA_CHECK(cudaMemcpyAsync(out->cap_m_out, P->tdev[0].Q + (P->cap_c_lo - P->jq0[0]), cnt * 4, cudaMemcpyDeviceToHost, st));
  } else if (out && out->cap_m_out && P->cap_c_hi >= P->cap_c_lo) {
    u64 cnt = P->cap_c_hi - P->cap_c_lo + 1;
    if (P->cap_c_lo < P->jq0[0]) { mt_set_error("capture range below floor(n/(u+1))+1"); return MT_ERR_VALUE; }
    RC(dalloc(d_capm, cnt * 8));
    k_copy_caps<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(P->tdev[0].Q, P->jq0[0], P->cap_c_lo, cnt, d_capm.as<int64_t>());
    P->launches++;
    MT_CUDA_CHECK(cudaMemcpyAsync(out->cap_m_out, d_capm.p, cnt * 8, cudaMemcpyDeviceToHost, st));
  }
  if (out && out->small_m_out && P->nsmall)
    MT_CUDA_CHECK(cudaMemcpyAsync(out->small_m_out, P->d_small.p, P->nsmall * (P->cap32 ? 4 : 8), cudaMemcpyDeviceToHost, st));
  MT_CUDA_CHECK(cudaStreamSynchronize(st));
  MT_CUDA_CHECK(cudaGetLastError());
  P->kt.drain();
  float f = 0;
  cudaEventElapsedTime(&f, P->ev[4], P->ev[5]); P->ms_fin = f;
  if (!out) return MT_OK;
  // ---- stats (RunStats fields in closed form, engine.py:188-197)
  mt_stats& S = out->stats;
  memset(&S, 0, sizeof(S));
  S.counted_items = P->counted_items;
  S.dense_items = P->dense_items;
  S.head_end = P->head_lim;
  S.max_mcut = P->Ymc_ref;
  S.n_head_segments = P->head_segs;
  S.n_tail_segments = P->tsegs.size();
  // kernels of this execution: the plan's own, the update context's (cub scans
  // count 2 each) and the sieve's (fill + tile + finish per segment)
  S.kernel_launches = P->launches + mt_update_launches(P->uc) + mt_sieve2_launches(P->sv, false);
  u64 qe = 0;
  for (int i = 0; i < P->N; i++) qe += P->jq1[i] >= P->jq0[i] ? P->jq1[i] - P->jq0[i] + 1 : 0;
  S.q_entries = qe;
  S.ms_update_head = P->ms_head;
  S.ms_sieve_tail = P->ms_tail;
  S.ms_qgather = P->ms_gather;
  S.ms_finalize = P->ms_fin;
  S.ms_total = P->ms_head + P->ms_tail + P->ms_gather + P->ms_fin;
  S.ms_setup = P->ms_setup;
  S.m_head = P->m_head;
  S.tail_total = P->tail_total;
  S.tail_seg_begin = P->ya;
  S.tail_seg_end = P->yb;
  for (int c = 0; c < KT_NCLASS && c < 8; c++) { S.kernel_ms[c] = P->kt.ms[c]; S.kernel_count[c] = P->kt.n[c]; }
  S.ms_counted_kernel = P->kt.ms[KT_COUNTED];
  S.ms_dense_kernel = P->kt.ms[KT_DWIN] + P->kt.ms[KT_DSPARSE] + P->kt.ms[KT_QGATHER];
  S.head_cells = P->head_lim;
  S.tail_cells = P->tail_cells();
  return MT_OK;
}

extern "C" int mt_run(const mt_job* job, mt_result* out) {
  auto T0 = std::chrono::steady_clock::now();
  if (job && job->shard_world > 1) {
    mt_set_error("mt_run is single-rank; use the plan API for shard_world > 1");
    return MT_ERR_VALUE;
  }
  mt_plan* P = nullptr;
  RC(mt_plan_create(job, &P));
  struct G { mt_plan* p; ~G() { mt_plan_destroy(p); } } g{P};
  int64_t mh = 0, tt = 0;
  RC(mt_plan_sieve_update(P, &mh, &tt));
  RC(mt_plan_tail_offset(P, mh));
  RC(mt_plan_gather(P));
  RC(mt_plan_resolve(P, out));
  if (out) out->stats.ms_total = ms_since(T0);
  return MT_OK;
}
