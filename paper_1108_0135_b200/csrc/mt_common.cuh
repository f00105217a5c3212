// Shared device helpers for the B200 exact-Mertens engine.
//
// Division strategy (replaces the reference's Granlund-Montgomery table,
// _native.pyx:32-68,209-224, and its hardware-divide fallback):
//   floor(v/m) = est + corr, est = round(double(v) * rcp(m)) read straight out
//   of the mantissa of fma(vd, r, 2^52) (FP64 pipe, full rate on B200), and
//   corr in {0,-1} from the sign of the remainder v - est*m computed on the low
//   32 (or 64) bits with one IMAD.  Exact whenever m >= 2^(bitlen(v)-50),
//   i.e. v/m < 2^50 (|est - v/m| <= 0.375).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;
typedef unsigned __int128 u128;
typedef __int128 i128;

#define MT_TWO52 4503599627370496.0
#define MT_EXP52 0x4330000000000000ull

// est in {f, f+1} -> f, using a 32-bit remainder (needs m < 2^31)
__device__ __forceinline__ u64 qdiv32(double vd, double r, u32 vlo, u32 m) {
  u64 b = (u64)__double_as_longlong(fma(vd, r, MT_TWO52)) - MT_EXP52;
  int t = (int)(vlo - (u32)b * m);
  return b + (u64)(i64)(t >> 31);
}

// same with a 64-bit remainder (any m < 2^63)
__device__ __forceinline__ u64 qdiv64(double vd, double r, u64 vlo, u64 m) {
  u64 b = (u64)__double_as_longlong(fma(vd, r, MT_TWO52)) - MT_EXP52;
  i64 t = (i64)(vlo - b * m);
  return b + (u64)(t >> 63);
}

__device__ __forceinline__ int bitlen128(u64 lo, u64 hi) {
  return hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
}

// true when qdiv64 is exact for this (v, m) pair
__device__ __forceinline__ bool qdiv_ok(int vbits, u64 m) {
  int need = vbits - 50;
  return m >= 1 && (need <= 0 || m >= (1ull << need));
}

__device__ __forceinline__ double u128_to_double(u64 lo, u64 hi) {
  // correctly rounded for hi < 2^53 is not required: only used as an estimate
  // whose error is covered by qdiv_ok (relative error < 2^-52).
  return hi ? fma((double)hi, 18446744073709551616.0, (double)lo) : __ull2double_rn(lo);
}

// exact floor((hi:lo)/m), m >= 1, v < 2^120 (the engine's v < 2^75): reciprocal
// multiply with exact correction instead of the compiler's software u128/u64.
//   1. q = trunc(double(v) * rcp(m)): relative error < 2^-50, so the signed
//      remainder t = v - q m (exact, 128-bit) satisfies |t/m| < 2^-50 q + 2;
//   2. q += round(double(t) * rcp(m)) -- |t/m| < 2^70 fits the estimate's range
//      and its error is < 2 -- and t -= that multiple of m (exact);
//   3. at most two +-1 steps bring t into [0, m).
__device__ __forceinline__ u128 udiv128(u64 lo, u64 hi, u64 m) {
  const u128 v = ((u128)hi << 64) | lo;
  const double r = __drcp_rn((double)m);
  const double vd = hi ? fma((double)hi, 18446744073709551616.0, (double)lo) : __ull2double_rn(lo);
  const double qd = vd * r;
  u128 q;
  if (qd < 18446744073709551616.0) {
    q = __double2ull_rz(qd);
  } else {  // split at 2^64: both parts exact (qd has <= 53 significant bits)
    const u64 qh = __double2ull_rz(qd * 5.421010862427522e-20);  // 2^-64
    const double rest = fma(-(double)qh, 18446744073709551616.0, qd);
    q = ((u128)qh << 64) | __double2ull_rz(rest > 0.0 ? rest : 0.0);
  }
  i128 t = (i128)(v - q * (u128)m);
  const long long q2 = __double2ll_rn((double)t * r);
  q += (u128)(i128)q2;
  t -= (i128)q2 * (i128)(u128)m;
  while (t < 0) { q -= 1; t += (i128)(u128)m; }
  while (t >= (i128)(u128)m) { q += 1; t -= (i128)(u128)m; }
  return q;
}

// exact floor(v/m) choosing the fast path when it is provably exact
__device__ __forceinline__ u64 udiv_any(u64 vlo, u64 vhi, double vd, int vbits, u64 m) {
  if (qdiv_ok(vbits, m)) {
    double r = __drcp_rn((double)m);
    return qdiv64(vd, r, vlo, m);
  }
  return (u64)udiv128(vlo, vhi, m);
}

#define MT_CUDA_CHECK(x)                                                   \
  do {                                                                     \
    cudaError_t _e = (x);                                                  \
    if (_e != cudaSuccess) {                                               \
      mt_set_error("CUDA error %s at %s:%d", cudaGetErrorString(_e),       \
                   __FILE__, __LINE__);                                    \
      return MT_ERR_CUDA;                                                  \
    }                                                                      \
  } while (0)

void mt_set_error(const char* fmt, ...);
