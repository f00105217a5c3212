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
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "mt_common.cuh"
#include "mt_internal.h"

static thread_local char g_err[2048];

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
  ~DevBuf() { if (p) cudaFree(p); }
  template <class T> T* as() { return (T*)p; }
};
static int dalloc(DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(&b.p, bytes);
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
  u64 xc = (u64)(v / tt);
  if (xc < D) xc = D;
  if (xc < 1) xc = 1;
  const u64 mc = (u64)(v / ((u128)xc + 1));
  a.vlo[e] = (u64)v;
  a.vhi[e] = (u64)(v >> 64);
  a.vd[e] = (v >> 64) ? fma((double)(u64)(v >> 64), 18446744073709551616.0, (double)(u64)v) : __ull2double_rn((u64)v);
  a.vbits[e] = (uint8_t)((v >> 64) ? 128 - __clzll((long long)(u64)(v >> 64)) : 64 - __clzll((long long)(u64)v));
  a.k[e] = kk;
  a.tgt[e] = (uint32_t)t;
  a.D[e] = D;
  a.xcut[e] = xc;
  a.mcut[e] = mc;
  a.lo[e] = D + 1 > 2 ? D + 1 : 2;
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

__global__ void k_tile_meta(u64 n_elem, const u64* __restrict__ mcut, const uint8_t* __restrict__ vbits,
                            u64* __restrict__ tmax, uint8_t* __restrict__ tbits) {
  u64 t = blockIdx.x;
  u64 e = t * MT_CT + threadIdx.x;
  u64 m = 0;
  int b = 0;
  if (e < n_elem) { m = mcut[e]; b = vbits[e]; }
  typedef cub::BlockReduce<u64, MT_CT> BR;
  typedef cub::BlockReduce<int, MT_CT> BRi;
  __shared__ typename BR::TempStorage s1;
  __shared__ typename BRi::TempStorage s2;
  u64 mx = BR(s1).Reduce(m, cub::Max());
  int bx = BRi(s2).Reduce(b, cub::Max());
  if (threadIdx.x == 0) { tmax[t] = mx; tbits[t] = (uint8_t)bx; }
}

// per-target reductions: max mcut, sum mcut, sum dense items, max windowed y
__global__ void k_elem_stats(u64 n_elem, const uint32_t* __restrict__ tgt, const u64* __restrict__ mcut,
                             const u64* __restrict__ xcut, const u64* __restrict__ lo,
                             unsigned long long* __restrict__ out /*[ntgt*3]*/) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_elem) return;
  uint32_t t = tgt[e];
  atomicMax(&out[3 * t + 0], (unsigned long long)mcut[e]);
  atomicAdd(&out[3 * t + 1], (unsigned long long)mcut[e]);
  u64 xc = xcut[e], l = lo[e];
  if (xc >= l) atomicAdd(&out[3 * t + 2], (unsigned long long)(xc - l + 1));
}

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

__global__ void k_copy_small(const int16_t* __restrict__ M16, const int64_t* __restrict__ bk, u64 Y0, u64 R,
                             u64 ymax, int64_t* __restrict__ out) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 y = Y0 + i;
  if (i >= R || y > ymax) return;
  out[y] = M16[i] + bk[i / MT_BLK];
}

__global__ void k_copy_caps(const int* __restrict__ Q, u64 jq0, u64 c_lo, u64 cnt, int64_t* __restrict__ out) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  out[i] = Q[c_lo + i - jq0];
}

static double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

extern "C" int mt_run(const mt_job* job, mt_result* out) {
  auto T0 = std::chrono::steady_clock::now();
  g_err[0] = 0;
  if (!job || !out || job->n_targets == 0) { mt_set_error("empty job"); return MT_ERR_VALUE; }
  if (job->device >= 0) MT_CUDA_CHECK(cudaSetDevice(job->device));
  const int N = (int)job->n_targets;
  const u64 u = job->u;
  std::vector<u128> n(N);
  std::vector<u64> K(N), e0(N + 1);
  e0[0] = 0;
  for (int i = 0; i < N; i++) {
    n[i] = ((u128)job->n_hi[i] << 64) | job->n_lo[i];
    if (n[i] < 4) { mt_set_error("exact job requires n >= 4"); return MT_ERR_VALUE; }
    if (job->n_hi[i] >= (1ull << 11)) { mt_set_error("n >= 2^75 is outside the engine's range"); return MT_ERR_RESOURCE; }
    if ((u128)u <= ceil_sqrt_u128(n[i])) { mt_set_error("u must exceed ceil(sqrt(n))"); return MT_ERR_VALUE; }
    K[i] = (u64)(n[i] / u);
    e0[i + 1] = e0[i] + K[i];
  }
  const u64 NE = e0[N];
  cudaStream_t st;
  MT_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamDestroy(s); } } sg{st};
  u64 launches = 0;

  // ---- elements
  DevBuf d_nlo, d_nhi, d_e0, d_vd, d_vlo, d_vhi, d_vb, d_k, d_tgt, d_D, d_x, d_mc, d_lo, d_low, d_dq, d_acc, d_mmc, d_dsp;
  RC(dalloc(d_nlo, N * 8)); RC(dalloc(d_nhi, N * 8)); RC(dalloc(d_e0, (N + 1) * 8));
  RC(dalloc(d_vd, NE * 8)); RC(dalloc(d_vlo, NE * 8)); RC(dalloc(d_vhi, NE * 8)); RC(dalloc(d_vb, NE));
  RC(dalloc(d_k, NE * 8)); RC(dalloc(d_tgt, NE * 4)); RC(dalloc(d_D, NE * 8)); RC(dalloc(d_x, NE * 8));
  RC(dalloc(d_mc, NE * 8)); RC(dalloc(d_lo, NE * 8)); RC(dalloc(d_low, NE * 8)); RC(dalloc(d_dq, NE * 8));
  RC(dalloc(d_acc, NE * 8)); RC(dalloc(d_mmc, NE * 4)); RC(dalloc(d_dsp, NE * 8));
  MT_CUDA_CHECK(cudaMemcpyAsync(d_nlo.p, job->n_lo, N * 8, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemcpyAsync(d_nhi.p, job->n_hi, N * 8, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemcpyAsync(d_e0.p, e0.data(), (N + 1) * 8, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemsetAsync(d_acc.p, 0, NE * 8, st));
  MT_CUDA_CHECK(cudaMemsetAsync(d_mmc.p, 0, NE * 4, st));
  {
    ElemInitArgs a{d_nlo.as<u64>(), d_nhi.as<u64>(), d_e0.as<u64>(), N, u, NE,
                   d_vd.as<double>(), d_vlo.as<u64>(), d_vhi.as<u64>(), d_vb.as<uint8_t>(), d_k.as<u64>(),
                   d_tgt.as<uint32_t>(), d_D.as<u64>(), d_x.as<u64>(), d_mc.as<u64>(), d_lo.as<u64>()};
    if (NE) k_elem_init<<<(unsigned)((NE + 255) / 256), 256, 0, st>>>(a);
    launches++;
    MT_CUDA_CHECK(cudaGetLastError());
  }
  std::vector<unsigned long long> tstat(3 * N, 0);
  {
    DevBuf d_ts;
    RC(dalloc(d_ts, 3 * N * 8));
    MT_CUDA_CHECK(cudaMemsetAsync(d_ts.p, 0, 3 * N * 8, st));
    if (NE) k_elem_stats<<<(unsigned)((NE + 255) / 256), 256, 0, st>>>(NE, d_tgt.as<uint32_t>(), d_mc.as<u64>(), d_x.as<u64>(), d_lo.as<u64>(), d_ts.as<unsigned long long>());
    launches++;
    MT_CUDA_CHECK(cudaMemcpyAsync(tstat.data(), d_ts.p, 3 * N * 8, cudaMemcpyDeviceToHost, st));
    MT_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  u64 Ymc = 0, counted_items = 0, dense_items = 0;
  for (int i = 0; i < N; i++) {
    Ymc = std::max<u64>(Ymc, tstat[3 * i]);
    counted_items += tstat[3 * i + 1];
    dense_items += tstat[3 * i + 2];
  }

  // ---- quotient tables: Q_t[j] = M(floor(n_t/j)), j in [jq0_t, jq1_t]
  const u64 q_budget = job->q_budget_bytes ? job->q_budget_bytes : (48ull << 30);
  std::vector<u64> J(N), jq0(N), jq1(N);
  u64 q_total = 0;
  for (int i = 0; i < N; i++) {
    jq0[i] = (u64)(n[i] / ((u128)u + 1)) + 1;
    J[i] = (u64)(n[i] / ((u128)Ymc + 1));
  }
  // cap the tables to the budget by scaling J down uniformly
  for (int it = 0; it < 64; it++) {
    q_total = 0;
    for (int i = 0; i < N; i++) {
      u64 hi = J[i];
      if (i == 0 && job->cap_c_hi >= job->cap_c_lo && job->cap_c_hi > hi) hi = job->cap_c_hi;
      jq1[i] = hi;
      if (hi >= jq0[i]) q_total += (hi - jq0[i] + 1);
    }
    if (q_total * 4 <= q_budget) break;
    for (int i = 0; i < N; i++) J[i] = J[i] / 2;
  }
  u64 head_end = Ymc;
  for (int i = 0; i < N; i++) {
    if (J[i] < jq0[i]) J[i] = 0;  // no Q-gather for this target
  }
  std::vector<DevBuf> d_Q(N);
  std::vector<TargetDev> tdev(N);
  std::vector<CaptureTargetH> caps;
  for (int i = 0; i < N; i++) {
    u64 cnt = jq1[i] >= jq0[i] ? jq1[i] - jq0[i] + 1 : 0;
    RC(dalloc(d_Q[i], cnt * 4));
    tdev[i].Q = d_Q[i].as<int>();
    tdev[i].jq0 = jq0[i];
    if (cnt) {
      CaptureTargetH c;
      c.n_lo = job->n_lo[i]; c.n_hi = job->n_hi[i];
      c.nd = job->n_hi[i] ? (double)job->n_hi[i] * 18446744073709551616.0 + (double)job->n_lo[i] : (double)job->n_lo[i];
      c.nbits = 0;
      for (u128 x = n[i]; x; x >>= 1) c.nbits++;
      c.jq0 = jq0[i]; c.jq1 = jq1[i]; c.Q = tdev[i].Q;
      caps.push_back(c);
    }
  }
  DevBuf d_J;
  RC(dalloc(d_J, N * 8));
  MT_CUDA_CHECK(cudaMemcpyAsync(d_J.p, J.data(), N * 8, cudaMemcpyHostToDevice, st));
  if (NE) k_elem_split<<<(unsigned)((NE + 255) / 256), 256, 0, st>>>(NE, d_k.as<u64>(), d_tgt.as<uint32_t>(), d_J.as<u64>(), d_lo.as<u64>(), d_x.as<u64>(), d_low.as<u64>(), d_dq.as<u64>());
  if (NE) k_elem_dsp<<<(unsigned)((NE + 255) / 256), 256, 0, st>>>(NE, d_vd.as<double>(), d_dsp.as<u64>());
  launches += 2;
  // element groups for the window walk: consecutive k of one target, size clamp(k/8, 32, 1024)
  std::vector<u64> gstart;
  for (int i = 0; i < N; i++) {
    u64 k0 = 1;
    while (k0 <= K[i]) {
      gstart.push_back(e0[i] + k0 - 1);
      u64 g = std::min<u64>(1024, std::max<u64>(32, k0 / 8));
      k0 += g;
    }
  }
  const u64 ng = gstart.size();
  gstart.push_back(NE);
  DevBuf d_gs, d_gylo, d_gyhi, d_gw;
  RC(dalloc(d_gs, (ng + 1) * 8)); RC(dalloc(d_gylo, ng * 8)); RC(dalloc(d_gyhi, ng * 8)); RC(dalloc(d_gw, ng));
  MT_CUDA_CHECK(cudaMemcpyAsync(d_gs.p, gstart.data(), (ng + 1) * 8, cudaMemcpyHostToDevice, st));
  if (ng) k_group_meta<<<(unsigned)ng, 256, 0, st>>>(d_gs.as<u64>(), ng, d_vlo.as<u64>(), d_vhi.as<u64>(), d_x.as<u64>(), d_low.as<u64>(), d_dsp.as<u64>(), d_gylo.as<u64>(), d_gyhi.as<u64>(), d_gw.as<uint8_t>());
  launches++;
  GroupDev grp{d_gs.as<u64>(), d_gylo.as<u64>(), d_gyhi.as<u64>(), d_gw.as<uint8_t>(), ng};
  {
    DevBuf d_we;
    RC(dalloc(d_we, 8));
    MT_CUDA_CHECK(cudaMemsetAsync(d_we.p, 0, 8, st));
    if (NE) k_window_extent<<<(unsigned)((NE + 255) / 256), 256, 0, st>>>(NE, d_vlo.as<u64>(), d_vhi.as<u64>(), d_low.as<u64>(), d_x.as<u64>(), d_we.as<unsigned long long>());
    launches++;
    unsigned long long we = 0;
    MT_CUDA_CHECK(cudaMemcpyAsync(&we, d_we.p, 8, cudaMemcpyDeviceToHost, st));
    MT_CUDA_CHECK(cudaStreamSynchronize(st));
    head_end = std::max<u64>(head_end, we);
  }
  if (job->cap_small > head_end) head_end = job->cap_small;
  if (head_end > u) head_end = u;

  // tiles metadata for the counted walk
  const u64 ntiles = (NE + MT_CT - 1) / MT_CT;
  DevBuf d_tmax, d_tbits;
  RC(dalloc(d_tmax, ntiles * 8)); RC(dalloc(d_tbits, ntiles));
  if (ntiles) k_tile_meta<<<(unsigned)ntiles, MT_CT, 0, st>>>(NE, d_mc.as<u64>(), d_vb.as<uint8_t>(), d_tmax.as<u64>(), d_tbits.as<uint8_t>());
  launches++;

  // ---- segments
  const u64 Rh = 1ull << (job->seg_log2_head ? job->seg_log2_head : 24);
  const u64 Rt = 1ull << (job->seg_log2_tail ? job->seg_log2_tail : 27);
  if (Rh < MT_TILE || Rt < Rh || (Rt % Rh)) { mt_set_error("bad segment sizes"); return MT_ERR_VALUE; }
  const u64 head_segs = (head_end + 1 + Rh - 1) / Rh;
  const u64 head_lim = head_segs * Rh;  // first y of the tail
  u64 tail_segs = 0;
  if (u + 1 > head_lim) tail_segs = (u + 1 - head_lim + Rt - 1) / Rt;
  const u64 y_last = head_lim + tail_segs * Rt - 1;

  PrimeTable pt;
  build_primes(std::max<u64>(ceil_sqrt_u128(y_last) + 1, 2), pt);
  uint8_t wheel[MT_WHEEL];
  reference_wheel(wheel);
  std::vector<uint32_t> w32;
  build_wheel_words(wheel, w32);
  const u64 np = pt.p.size();
  DevBuf d_p, d_rp, d_lg, d_w32, d_big, d_mu, d_m, d_half, d_bk, d_tsum, d_tbase, d_run, d_caps, d_small;
  RC(dalloc(d_p, np * 4)); RC(dalloc(d_rp, np * 8)); RC(dalloc(d_lg, np));
  RC(dalloc(d_w32, w32.size() * 4));
  MT_CUDA_CHECK(cudaMemcpyAsync(d_p.p, pt.p.data(), np * 4, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemcpyAsync(d_rp.p, pt.r.data(), np * 8, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemcpyAsync(d_lg.p, pt.lg.data(), np, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemcpyAsync(d_w32.p, w32.data(), w32.size() * 4, cudaMemcpyHostToDevice, st));
  RC(dalloc(d_big, Rt)); RC(dalloc(d_mu, Rh)); RC(dalloc(d_m, Rh * 2)); RC(dalloc(d_half, (Rt / MT_TILE) * 4)); RC(dalloc(d_bk, (Rh / MT_BLK) * 8 + 8));
  RC(dalloc(d_tsum, (Rt / MT_TILE) * 4)); RC(dalloc(d_tbase, (Rt / MT_TILE) * 8)); RC(dalloc(d_run, 8));
  MT_CUDA_CHECK(cudaMemsetAsync(d_run.p, 0, 8, st));
  RC(dalloc(d_caps, caps.size() * sizeof(CaptureTargetH)));
  if (!caps.empty())
    MT_CUDA_CHECK(cudaMemcpyAsync(d_caps.p, caps.data(), caps.size() * sizeof(CaptureTargetH), cudaMemcpyHostToDevice, st));
  const u64 nsmall = out->small_m_out ? job->cap_small + 1 : 0;
  RC(dalloc(d_small, nsmall * 8));

  ElemDev E;
  E.vd = d_vd.as<double>(); E.vlo = d_vlo.as<u64>(); E.vhi = d_vhi.as<u64>(); E.vbits = d_vb.as<uint8_t>();
  E.k = d_k.as<u64>(); E.tgt = d_tgt.as<uint32_t>(); E.mcut = d_mc.as<u64>(); E.xcut = d_x.as<u64>();
  E.lo = d_lo.as<u64>(); E.lo_w = d_low.as<u64>(); E.dq_hi = d_dq.as<u64>(); E.d_sp = d_dsp.as<u64>(); E.n = NE;
  UpdateCtx* uc = nullptr;
  RC(mt_update_create(&uc, E, d_acc.as<u64>(), d_mmc.as<int32_t>(), d_tmax.as<u64>(), d_tbits.as<uint8_t>(),
                      ntiles, tdev.data(), N, grp, st));
  struct UcGuard { UpdateCtx* c; ~UcGuard() { mt_update_destroy(c); } } ug{uc};

  cudaEvent_t ev[6];
  for (int i = 0; i < 6; i++) MT_CUDA_CHECK(cudaEventCreate(&ev[i]));
  struct EvGuard { cudaEvent_t* e; ~EvGuard() { for (int i = 0; i < 6; i++) cudaEventDestroy(e[i]); } } eg{ev};
  MT_CUDA_CHECK(cudaEventRecord(ev[0], st));

  auto make_seg = [&](u64 Y0, u64 R, bool head) {
    SieveSegment s{};
    const u64 y2 = Y0 + R - 1;
    PrimeCut c = prime_cut(pt.p, y2);
    s.Y0 = Y0; s.R = R; s.y2 = y2;
    s.big = d_big.as<uint32_t>();
    s.primes = d_p.as<uint32_t>(); s.rprimes = d_rp.as<double>(); s.logs = d_lg.as<uint8_t>();
    s.p_large_begin = c.small_end; s.p_large_end = c.large_end; s.do_logs_large = 1;
    s.running = d_run.as<int64_t>(); s.tile_base = d_tbase.as<int64_t>();
    s.bk = head ? d_bk.as<int64_t>() : nullptr;
    SieveTileArgs& a = s.tile;
    a.Y0 = Y0; a.y2 = y2; a.wheel32x = d_w32.as<uint32_t>(); a.big = s.big;
    a.primes = s.primes; a.rprimes = s.rprimes; a.logs = s.logs;
    a.p_first = c.first; a.p_warp_end = c.warp_end; a.p_small_end = c.small_end;
    a.log_min = 11; a.do_logs = 1;
    a.tile_sum = d_tsum.as<int>();
    a.mu_out = head ? d_mu.as<int8_t>() : nullptr;
    a.m_out = nullptr;
    a.m16_out = head ? d_m.as<int16_t>() : nullptr;
    a.half_out = d_half.as<int>();
    a.states_out = nullptr;
    a.caps = d_caps.p; a.n_cap = (int)caps.size();
    return s;
  };

  // ---- head
  for (u64 s = 0; s < head_segs; s++) {
    const u64 Y0 = s * Rh;
    SieveSegment sg = make_seg(Y0, Rh, true);
    RC(mt_launch_sieve_segment(sg, st));
    launches += 6;
    RC(mt_update_head_segment(uc, Y0, Rh, d_mu.as<int8_t>(), d_m.as<int16_t>(), d_bk.as<int64_t>(), st));
    if (nsmall && Y0 <= job->cap_small) {
      k_copy_small<<<(unsigned)((Rh + 255) / 256), 256, 0, st>>>(d_m.as<int16_t>(), d_bk.as<int64_t>(), Y0, Rh, job->cap_small, d_small.as<int64_t>());
      launches++;
    }
  }
  MT_CUDA_CHECK(cudaEventRecord(ev[1], st));
  // ---- tail
  for (u64 s = 0; s < tail_segs; s++) {
    const u64 Y0 = head_lim + s * Rt;
    SieveSegment sg = make_seg(Y0, Rt, false);
    RC(mt_launch_sieve_segment(sg, st));
    launches += 5;
  }
  MT_CUDA_CHECK(cudaEventRecord(ev[2], st));
  // ---- Q-gather + resolve
  RC(mt_update_qgather(uc, st));
  RC(mt_update_finish(uc, st));
  MT_CUDA_CHECK(cudaEventRecord(ev[3], st));
  DevBuf d_fin;
  RC(dalloc(d_fin, NE * 8));
  for (int i = 0; i < N; i++)
    RC(mt_finalize_dev(d_acc.as<u64>() + e0[i], d_D.as<u64>() + e0[i], K[i], d_fin.as<int64_t>() + e0[i], st));
  MT_CUDA_CHECK(cudaEventRecord(ev[4], st));
  if (out->finals && NE)
    MT_CUDA_CHECK(cudaMemcpyAsync(out->finals, d_fin.p, NE * 8, cudaMemcpyDeviceToHost, st));
  if (out->acc_out && NE)
    MT_CUDA_CHECK(cudaMemcpyAsync(out->acc_out, d_acc.p, NE * 8, cudaMemcpyDeviceToHost, st));
  DevBuf d_capm;
  if (out->cap_m_out && job->cap_c_hi >= job->cap_c_lo) {
    u64 cnt = job->cap_c_hi - job->cap_c_lo + 1;
    if (job->cap_c_lo < jq0[0]) { mt_set_error("capture range below floor(n/(u+1))+1"); return MT_ERR_VALUE; }
    RC(dalloc(d_capm, cnt * 8));
    k_copy_caps<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(tdev[0].Q, jq0[0], job->cap_c_lo, cnt, d_capm.as<int64_t>());
    MT_CUDA_CHECK(cudaMemcpyAsync(out->cap_m_out, d_capm.p, cnt * 8, cudaMemcpyDeviceToHost, st));
  }
  if (nsmall) MT_CUDA_CHECK(cudaMemcpyAsync(out->small_m_out, d_small.p, nsmall * 8, cudaMemcpyDeviceToHost, st));
  MT_CUDA_CHECK(cudaEventRecord(ev[5], st));
  MT_CUDA_CHECK(cudaStreamSynchronize(st));

  // ---- stats (RunStats fields in closed form, engine.py:188-197)
  mt_stats& S = out->stats;
  memset(&S, 0, sizeof(S));
  S.counted_items = counted_items;
  S.dense_items = dense_items;
  S.head_end = head_lim;
  S.max_mcut = Ymc;
  S.n_head_segments = head_segs;
  S.n_tail_segments = tail_segs;
  S.kernel_launches = launches + mt_update_launches(uc);
  u64 qe = 0;
  for (int i = 0; i < N; i++) qe += jq1[i] >= jq0[i] ? jq1[i] - jq0[i] + 1 : 0;
  S.q_entries = qe;
  float f;
  cudaEventElapsedTime(&f, ev[0], ev[1]); S.ms_update_head = f;
  cudaEventElapsedTime(&f, ev[1], ev[2]); S.ms_sieve_tail = f;
  cudaEventElapsedTime(&f, ev[2], ev[3]); S.ms_qgather = f;
  cudaEventElapsedTime(&f, ev[3], ev[4]); S.ms_finalize = f;
  S.ms_total = ms_since(T0);
  return MT_OK;
}
