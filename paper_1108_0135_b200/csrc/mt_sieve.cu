// Segmented Moebius sieve on sm_100a (replaces the CPU log-prime sieve of
// reference sieve.py:189-213 / _native.pyx:71-160, which the paper kept on the
// host).
//
// State semantics are the reference's exactly: an 8-bit cell per y holding
//   wheel(y mod 13860) + sum_{p>=11, p|y, p*p<=y2} l_p  (l_p = ceil(log2 p)|1)
//   | 0x80 if p*p | y for some 5 <= p, p*p <= y2
// and mu(y) = 0 if bit7, else (s > floor(log2 y)-1 ? 1-2(s&1) : 2(s&1)-1)
// (_native.pyx:143-159; the ceil-log rule of sieve.py:111-121).
//
// Layout: a segment [Y0, Y0+R) is cut into tiles of MT_TILE cells (Y0, R and
// tile bases are multiples of MT_TILE).  Primes p <= MT_TILE are sieved inside
// a tile held in shared memory (word-granular smem atomics, ~12 lanes/clk/SM
// measured); primes p > MT_TILE hit a tile at most once and are scattered by
// k_sieve_large into a per-segment byte buffer `big` with L2 atomics, which
// the tile kernel folds into its initial state together with the wheel.
// After classification each tile runs a block scan of mu, writes its tile sum,
// the in-tile prefix (head mode: the whole M array; always: the quotient
// captures M(floor(n/j)) for the j whose quotient falls in the tile).
#include "mt_common.cuh"
#include "mt_internal.h"

// --------------------------------------------------------------------------
// large primes: one thread per prime, L2 atomics into `big` (segment bytes)
// --------------------------------------------------------------------------
__global__ void k_sieve_large(u32* __restrict__ big, u64 Y0, u64 R, u64 y2,
                              const u32* __restrict__ primes, const double* __restrict__ rprimes,
                              const uint8_t* __restrict__ logs, u32 p_begin, u32 p_end,
                              int do_logs) {
  u32 i = p_begin + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p_end) return;
  u64 p = primes[i];
  u32 lg = logs[i];
  if (do_logs) {
    // first multiple of p at or above Y0 (Y0 < 2^53 so the fp64 quotient is exact)
    u64 q = qdiv64(__ull2double_rn(Y0), rprimes[i], Y0, p);
    u64 r = Y0 - q * p;
    u64 j = r ? p - r : (Y0 ? 0 : p);  // y = 0 is never marked (it would overflow into y = 1)
    for (; j < R; j += p) atomicAdd(&big[j >> 2], lg << ((j & 3) * 8));
  }
  u64 p2 = p * p;
  if (p >= 5 && p2 <= y2) {
    u64 q2 = Y0 / p2;
    u64 r2 = Y0 - q2 * p2;
    u64 j = r2 ? p2 - r2 : (Y0 ? 0 : p2);
    for (; j < R; j += p2) atomicOr(&big[j >> 2], 0x80u << ((j & 3) * 8));
  }
}

// --------------------------------------------------------------------------
// tile kernel
// --------------------------------------------------------------------------
struct CaptureTarget {  // one exact target n for quotient captures
  u64 n_lo, n_hi;
  double nd;
  int nbits;
  u64 jq0, jq1;  // capture j in [jq0, jq1]
  int* Q;        // Q[j - jq0] = M(floor(n/j)) (partial until fixup)
};

__device__ __forceinline__ int mu_of_state(u32 s, int thr) {
  if (s & 0x80) return 0;
  int par = s & 1;
  return ((int)s > thr) ? 1 - 2 * par : 2 * par - 1;
}

// floor(n / y) for a capture target, y >= 1 (128-bit n)
__device__ __forceinline__ u64 cap_div(const CaptureTarget& t, u64 y) {
  return udiv_any(t.n_lo, t.n_hi, t.nd, t.nbits, y);
}

template <int NT>
__global__ void __launch_bounds__(NT) k_sieve_tile(SieveTileArgs a) {
  extern __shared__ u32 smem[];
  u32* st = smem;                              // MT_TILE/4 words of states / mu
  int* pre32 = (int*)(smem + MT_TILE / 4);     // MT_TILE/32 inclusive partials (per 32 cells)
  __shared__ int warp_tot[NT / 32];
  const int tid = threadIdx.x;
  const u64 Yt = a.Y0 + (u64)blockIdx.x * MT_TILE;
  const u64 tile_off = (u64)blockIdx.x * MT_TILE;  // offset inside the segment

  // 1. wheel + large-prime marks
  {
    const u32 phase = (u32)((Yt % 13860ull) >> 2);
    const u32* __restrict__ w = a.wheel32x + phase;
    const u32* __restrict__ bg = a.big ? a.big + (tile_off >> 2) : nullptr;
    for (int i = tid; i < MT_TILE / 4; i += NT) {
      // both the wheel and `big` may carry the 0x80 square flag: merge it with OR
      u32 b = bg ? bg[i] : 0u;
      st[i] = (w[i] + (b & 0x7F7F7F7Fu)) | (b & 0x80808080u);
    }
  }
  __syncthreads();

  // 2. small primes (p in [p_first, p_small_end), all <= MT_TILE)
  {
    const double Yd = __ull2double_rn(Yt);
    const int lane = tid & 31, warp = tid >> 5;
    // 2a. warp per prime for p < MT_TILE/64 (many multiples per tile)
    for (u32 i = a.p_first + warp; i < a.p_warp_end; i += NT / 32) {
      u32 p = a.primes[i];
      u32 lg = a.logs[i];
      u64 q = qdiv64(Yd, a.rprimes[i], Yt, p);
      u32 r = (u32)(Yt - q * p);
      u32 j0 = r ? p - r : (Yt ? 0 : p);  // skip y = 0 (wheel already flags it 0x80)
      if (a.do_logs && p >= a.log_min) {
        u32 sh = lg;
        for (u32 j = j0 + lane * p; j < MT_TILE; j += 32 * p)
          atomicAdd(&st[j >> 2], sh << ((j & 3) * 8));
      }
      u64 p2 = (u64)p * p;
      if (p >= 5 && p2 <= a.y2) {
        u64 q2 = qdiv64(Yd, __drcp_rn((double)p2), Yt, p2);
        u64 r2 = Yt - q2 * p2;
        u64 j2 = r2 ? p2 - r2 : (Yt ? 0 : p2);
        for (u64 j = j2 + (u64)lane * p2; j < MT_TILE; j += 32 * p2)
          atomicOr(&st[j >> 2], 0x80u << ((j & 3) * 8));
      }
    }
    // 2b. thread per prime for the rest of the in-tile primes
    for (u32 i = a.p_warp_end + tid; i < a.p_small_end; i += NT) {
      u32 p = a.primes[i];
      u32 lg = a.logs[i];
      u64 q = qdiv64(Yd, a.rprimes[i], Yt, p);
      u32 r = (u32)(Yt - q * p);
      u32 j = r ? p - r : (Yt ? 0 : p);
      if (a.do_logs && p >= a.log_min)
        for (; j < MT_TILE; j += p) atomicAdd(&st[j >> 2], lg << ((j & 3) * 8));
      u64 p2 = (u64)p * p;
      if (p2 <= a.y2) {
        u64 q2 = qdiv64(Yd, __drcp_rn((double)p2), Yt, p2);
        u64 r2 = Yt - q2 * p2;
        u64 j2 = r2 ? p2 - r2 : (Yt ? 0 : p2);
        for (; j2 < MT_TILE; j2 += p2) atomicOr(&st[j2 >> 2], 0x80u << ((j2 & 3) * 8));
      }
    }
  }
  __syncthreads();

  if (a.states_out) {  // instrumented export (logprime_states parity)
    uint32_t* so = (uint32_t*)(a.states_out + tile_off);
    for (int i = tid; i < MT_TILE / 4; i += NT) so[i] = st[i];
    __syncthreads();  // the export must finish before cells are classified in place
  }

  // 3. classify in place: each thread owns CH = MT_TILE/NT consecutive cells
  constexpr int CH = MT_TILE / NT;  // cells per thread (multiple of 32)
  constexpr int CW = CH / 4;        // words per thread
  int tsum = 0;
  {
    const int flog_tile = 63 - __clzll((long long)(Yt | 1));
    const bool uniform = Yt >= MT_TILE;  // tiles are power-of-two aligned: one binade
    u32* my = st + tid * CW;
#pragma unroll 4
    for (int wi = 0; wi < CW; wi++) {
      u32 w = my[wi];
      u32 out = 0;
#pragma unroll
      for (int b = 0; b < 4; b++) {
        u32 s = (w >> (8 * b)) & 0xff;
        int thr;
        if (uniform) thr = flog_tile - 1;
        else {
          u64 y = Yt + (u64)(tid * CH + wi * 4 + b);
          thr = (y ? 63 - __clzll((long long)y) : 0) - 1;
        }
        int m = mu_of_state(s, thr);
        tsum += m;
        out |= ((u32)(m & 0xff)) << (8 * b);
      }
      my[wi] = out;
    }
  }
  // block exclusive scan of per-thread sums
  int incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if ((tid & 31) >= o) incl += t;
  }
  if ((tid & 31) == 31) warp_tot[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    int v = tid < NT / 32 ? warp_tot[tid] : 0;
    int iv = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, iv, o);
      if (tid >= o) iv += t;
    }
    if (tid < NT / 32) warp_tot[tid] = iv - v;  // exclusive
    if (tid == NT / 32 - 1) a.tile_sum[blockIdx.x] = iv;
  }
  __syncthreads();
  int run = warp_tot[tid >> 5] + incl - tsum;  // exclusive prefix of this thread's chunk

  // 4. outputs: mu (int8), in-tile prefix (int32), 32K-block-relative M (int16),
  //    per-32-cell partials for the captures
  __shared__ int s_half;
  if (tid == NT / 2) s_half = run;  // exclusive prefix at the tile's 32K midpoint
  __syncthreads();
  {
    const u32* my = st + tid * CW;
    int8_t* mu_out = a.mu_out ? a.mu_out + tile_off + (u64)tid * CH : nullptr;
    int* m_out = a.m_out ? a.m_out + tile_off + (u64)tid * CH : nullptr;
    int16_t* m16 = a.m16_out ? a.m16_out + tile_off + (u64)tid * CH : nullptr;
    const int hb = (tid >= NT / 2) ? s_half : 0;
    for (int wi = 0; wi < CW; wi++) {
      u32 w = my[wi];
      if (mu_out) ((u32*)mu_out)[wi] = w;
      int c0 = run + (int)(int8_t)(w & 0xff);
      int c1 = c0 + (int)(int8_t)((w >> 8) & 0xff);
      int c2 = c1 + (int)(int8_t)((w >> 16) & 0xff);
      int c3 = c2 + (int)(int8_t)(w >> 24);
      if (m_out) ((int4*)m_out)[wi] = make_int4(c0, c1, c2, c3);
      if (m16) {
        uint2 pk;
        pk.x = (u32)(uint16_t)(c0 - hb) | ((u32)(uint16_t)(c1 - hb) << 16);
        pk.y = (u32)(uint16_t)(c2 - hb) | ((u32)(uint16_t)(c3 - hb) << 16);
        ((uint2*)m16)[wi] = pk;
      }
      run = c3;
      if ((wi & 7) == 7) pre32[(tid * CH + wi * 4) >> 5] = run;
    }
    if (a.half_out && tid == 0) a.half_out[blockIdx.x] = s_half;
  }
  __syncthreads();

  // 5. quotient captures: for every target, j with floor(n/j) in this tile
  for (int t = 0; t < a.n_cap; t++) {
    const CaptureTarget& ct = ((const CaptureTarget*)a.caps)[t];
    // j range: floor(n/j) in [Yt, Yt+T)  <=>  j in (n/(Yt+T), n/Yt]
    u64 jhi = Yt ? cap_div(ct, Yt) : ~0ull;
    u64 jlo = cap_div(ct, Yt + MT_TILE) + 1;
    if (jlo < ct.jq0) jlo = ct.jq0;
    if (jhi > ct.jq1) jhi = ct.jq1;
    for (u64 j = jlo + tid; j <= jhi; j += NT) {
      u64 y = cap_div(ct, j);
      u32 o = (u32)(y - Yt);
      int c = o >> 5;
      int base = c ? pre32[c - 1] : 0;
      // the first tile's chunk base: pre32[c-1] covers cells < 32c
      const u32* wp = st + (c << 3);
      int s = 0;
      u32 last = o & 31;
      for (u32 wi = 0; wi <= (last >> 2); wi++) {
        u32 w = wp[wi];
        if (wi == (last >> 2)) {
          u32 keep = (last & 3) + 1;
          w = keep == 4 ? w : (w & ((1u << (8 * keep)) - 1));
        }
        s = __dp4a((int)w, 0x01010101, s);
      }
      ct.Q[j - ct.jq0] = base + s;
    }
  }
}

// exclusive tile bases for one segment + running M (device scalar)
__global__ void k_seg_scan(const int* __restrict__ tile_sum, int ntiles, i64* __restrict__ running,
                           i64* __restrict__ tile_base, const int* __restrict__ half,
                           i64* __restrict__ bk) {
  // single block of 1024 threads, sequential over chunks of 1024 tiles
  __shared__ i64 wsum[32];
  __shared__ i64 carry;
  const int tid = threadIdx.x;
  if (tid == 0) carry = *running;
  __syncthreads();
  for (int base = 0; base < ntiles; base += 1024) {
    int i = base + tid;
    i64 v = i < ntiles ? tile_sum[i] : 0;
    i64 incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      i64 t = __shfl_up_sync(0xffffffffu, incl, o);
      if ((tid & 31) >= o) incl += t;
    }
    if ((tid & 31) == 31) wsum[tid >> 5] = incl;
    __syncthreads();
    if (tid < 32) {
      i64 x = wsum[tid], ix = x;
      for (int o = 1; o < 32; o <<= 1) {
        i64 t = __shfl_up_sync(0xffffffffu, ix, o);
        if (tid >= o) ix += t;
      }
      wsum[tid] = ix - x;
    }
    __syncthreads();
    i64 excl = carry + wsum[tid >> 5] + incl - v;
    if (i < ntiles) {
      tile_base[i] = excl;
      if (bk) { bk[2 * i] = excl; bk[2 * i + 1] = excl + half[i]; }
    }
    __syncthreads();
    if (tid == 1023) carry = excl + v;
    __syncthreads();
  }
  if (tid == 0) *running = carry;
}

// head: M[y] += base(tile of y) (makes the segment M array absolute)
__global__ void k_fixup_M(int* __restrict__ M, const i64* __restrict__ tile_base, u64 R) {
  u64 i4 = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i4 * 4 >= R) return;
  int b = (int)tile_base[(i4 * 4) / MT_TILE];
  int4 v = ((int4*)M)[i4];
  v.x += b; v.y += b; v.z += b; v.w += b;
  ((int4*)M)[i4] = v;
}

// Q[j] += base(tile of floor(n/j)) for the captures of this segment (one block per tile)
__global__ void k_fixup_Q(SieveTileArgs a, const i64* __restrict__ tile_base) {
  const u64 Yt = a.Y0 + (u64)blockIdx.x * MT_TILE;
  const int b = (int)tile_base[blockIdx.x];
  for (int t = 0; t < a.n_cap; t++) {
    const CaptureTarget& ct = ((const CaptureTarget*)a.caps)[t];
    u64 jhi = Yt ? cap_div(ct, Yt) : ~0ull;
    u64 jlo = cap_div(ct, Yt + MT_TILE) + 1;
    if (jlo < ct.jq0) jlo = ct.jq0;
    if (jhi > ct.jq1) jhi = ct.jq1;
    for (u64 j = jlo + threadIdx.x; j <= jhi; j += blockDim.x) ct.Q[j - ct.jq0] += b;
  }
}

// ------------------------------------------------------------------ host side
int mt_launch_sieve_segment(const SieveSegment& s, cudaStream_t st, KTimer* kt) {
  // 1. large primes into `big`
  if (s.big) {
    MT_CUDA_CHECK(cudaMemsetAsync(s.big, 0, s.R, st));
    if (s.p_large_end > s.p_large_begin) {
      u32 n = s.p_large_end - s.p_large_begin;
      if (kt) kt->begin(KT_SIEVE_LARGE, st);
      k_sieve_large<<<(n + 255) / 256, 256, 0, st>>>(s.big, s.Y0, s.R, s.y2, s.primes, s.rprimes,
                                                     s.logs, s.p_large_begin, s.p_large_end,
                                                     s.do_logs_large);
      if (kt) kt->end(st);
      MT_CUDA_CHECK(cudaGetLastError());
    }
  }
  SieveTileArgs a = s.tile;
  int ntiles = (int)(s.R / MT_TILE);
  size_t smem = MT_TILE + (MT_TILE / 32) * sizeof(int);
  static bool attr = false;
  if (!attr) {
    MT_CUDA_CHECK(cudaFuncSetAttribute(k_sieve_tile<MT_SIEVE_THREADS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  if (kt) kt->begin(KT_SIEVE_TILE, st);
  k_sieve_tile<MT_SIEVE_THREADS><<<ntiles, MT_SIEVE_THREADS, smem, st>>>(a);
  if (kt) kt->end(st);
  MT_CUDA_CHECK(cudaGetLastError());
  if (s.running) {
    k_seg_scan<<<1, 1024, 0, st>>>(a.tile_sum, ntiles, s.running, s.tile_base, a.half_out, s.bk);
    MT_CUDA_CHECK(cudaGetLastError());
    if (a.m_out) {
      u64 n4 = s.R / 4;
      k_fixup_M<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(a.m_out, s.tile_base, s.R);
      MT_CUDA_CHECK(cudaGetLastError());
    }
    if (a.n_cap) {
      k_fixup_Q<<<ntiles, 256, 0, st>>>(a, s.tile_base);
      MT_CUDA_CHECK(cudaGetLastError());
    }
  }
  return MT_OK;
}
