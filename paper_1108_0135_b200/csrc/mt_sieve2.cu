// Production segmented Moebius sieve on sm_100a (the engine's head and tail).
//
// Replaces the CPU log-prime sieve the paper kept on the host (PAPER.md:87-115,
// reference sieve.py:189-213 / _native.pyx:71-160).  mu(y) is decided by the
// reference's rule (_native.pyx:143-159): with s = sum of l_p = ceil(log2 p)|1
// over the primes p <= sqrt(y2) dividing y (0x80 if some p^2 | y),
//   mu = 0 if s & 0x80, else (s > floor(log2 y) - 1 ? 1 - 2(s&1) : 2(s&1) - 1).
// Marking more primes than the reference (the presieve patterns below include
// 11..41 for every y) only moves y into the exact "fully factored" branch, so
// mu is unchanged; raw states are NOT the reference's and the
// instrumented logprime_states op keeps the reference kernel (mt_sieve.cu).
//
// Layout:
//   tile     = 2^17 cells (one byte each, 128 KB of shared memory, 1 CTA/SM,
//              1024 threads); tiles are 2^17-aligned, so every tile but the
//              first lies in one binade and shares one classification threshold
//   presieve = two L2-resident byte patterns added word-wise on load:
//              W1 (2,3,5,7,11 logs; 0x80 at 4,9,25,49; period 485100),
//              W2 (13,17,19,23; period 96577) -- small patterns stay in L2;
//              a third pattern for 29..41 cost more than marking those primes
//   in-tile  = primes 29 <= p <= 2^16 (warp per prime below 1024, lane per
//              prime above) and squares p^2 for 11 <= p <= 362 (shared-memory
//              byte reductions, red.shared.add / .or, on the cell's 32-bit word)
//   buckets  = primes p > 2^16 and squares p^2 > 2^17: a producer kernel per
//              segment enumerates every hit (balanced in chunks of hits) and
//              appends (offset, log) to a producer-private list per tile, square
//              flags from the list's back (shared-memory cursors, no global
//              atomics); the tile kernel applies its lists.  A list that would
//              overflow its capacity is recomputed exactly by the tile (slow path)
//   classify = SIMD within a word (4 cells), warp-parallel over words; 32-cell
//              chunk sums -> block scan -> tile total
//   CTAs     = persistent: CTA c sieves 4 contiguous tiles of the segment and
//              carries every in-tile prime's next multiple from tile to tile in
//              shared memory, so a prime costs one division per CTA, not per tile
//   scan     = tile sums -> one-block scan seeded with the running M; captures
//              M(floor(n/j)) and the head's 32K block bases are written
//              tile-relative and made absolute by one finishing pass (k_s3_finish)
#include <cstdio>

#include "mt_common.cuh"
#include "mt_internal.h"

#define S2_T (1u << 17)          // cells per tile
#define S2_W (S2_T / 4)          // words per tile
#define S2_NT 1024               // threads per tile CTA
#define S2_CH (S2_T / 32)        // 32-cell chunks per tile
#define S2_MAXPROD 512           // bucket producers whose counts are staged in shared memory
#define S2_MAXCAP 128            // capture targets whose j ranges are staged per tile
#ifndef S2_A_MAX
#define S2_A_MAX 1024u           // warp-per-prime marks below this, lane-per-prime from here
#endif
#ifndef S2_B2_MIN
#define S2_B2_MIN (1u << 15)     // in-tile primes from here on hit <= 4 times per tile (measured: 2^15 > 2^14 > 2^13)
#endif
#ifndef S2_LIST_PREFETCH
#define S2_LIST_PREFETCH 0       // L2 bulk prefetch of the tile's bucket lists at the tile start
#endif
#ifndef S2_DLOADS
#define S2_DLOADS 1              // 16-byte bucket vectors in flight per lane (measured: 1 > 2)
#endif
#ifndef S2_DPAIR
#define S2_DPAIR 1               // D: two bucket lists per fetch, walked as one
#endif

__device__ __forceinline__ void red_add(u32 saddr, u32 v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or(u32 saddr, u32 v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}

// ----------------------------------------------------------------------------
// wheel modes of a segment.  Cell c of a tile starting at Yt:
//   W = 1: y = Yt + c                  every y (the head)
//   W = 2: y = Yt + 2c + 1             odd y (tail)
//   W = 6: y = Yt + 3c + 1 + (c & 1)   y coprime to 6 (tail; Yt multiple of 6)
// The hits of a prime p >= 5 (or of a square q = p^2) on the cells form NS
// arithmetic streams of cell stride STRIDE: one stream of stride p (W = 1, 2;
// W = 2: p | 2c + 1 <=> c == (p-1)/2 mod p) or two of stride 2p (W = 6: y = p*m,
// m == 1 or 5 mod 6, at cells floor(p/3) and floor(5p/3) mod 2p).
// ----------------------------------------------------------------------------
template <int W> struct Wheel {
  static constexpr int NS = W == 6 ? 2 : 1;
  static constexpr u64 SPAN = (u64)S2_T * (W == 1 ? 1 : W == 2 ? 2 : 3);  // y per tile
  __device__ static __forceinline__ u64 cell0(u64 Y) { return W == 1 ? Y : W == 2 ? Y >> 1 : Y / 3; }
  __device__ static __forceinline__ u64 y_of(u64 c) { return W == 1 ? c : W == 2 ? 2 * c + 1 : 3 * c + 1 + (c & 1); }
  // number of cells with y' - Yt <= o (the prefix length of a capture at y = Yt + o)
  __device__ static __forceinline__ u64 ncell(u64 o) {
    return W == 1 ? o + 1 : W == 2 ? (o + 1) >> 1 : 2 * (o / 6) + (o % 6 >= 1) + (o % 6 >= 5);
  }
};

// (-Y) mod m for m < 2^50, Y < 2^53, with r = 1/m rounded (host: 1.0/m)
__device__ __forceinline__ u64 neg_mod64(u64 Y, double Yd, double r, u64 m) {
  const u64 q = qdiv64(Yd, r, Y, m);
  const u64 rem = Y - q * m;
  return rem ? m - rem : 0;
}
__device__ __forceinline__ u32 neg_mod(u64 Y, double Yd, double r, u32 p) { return (u32)neg_mod64(Y, Yd, r, p); }

// first cells >= C0 hit by modulus m (a prime or a square, m >= 5, coprime to 6
// when W = 6): j[s] = the offset from C0 of stream s's first cell, j[s] < STRIDE.
// rm = 1/m rounded (1/(2m) = rm/2 exactly).
template <int W>
__device__ __forceinline__ void first_hits(u64 C0, double Cd, double rm, u64 m, u64* j) {
  if (W == 6) {
    const u64 m2 = 2 * m;
    const u64 r = neg_mod64(C0, Cd, 0.5 * rm, m2);
    const u64 a = r + m / 3, b = r + (5 * m) / 3;
    j[0] = a >= m2 ? a - m2 : a;
    j[1] = b >= m2 ? b - m2 : b;
  } else {
    u64 r = neg_mod64(C0, Cd, rm, m);
    if (W == 2) {
      r += m >> 1;
      if (r >= m) r -= m;
    } else if (C0 == 0 && r == 0) {
      r = m;  // y = 0 is never marked
    }
    j[0] = r;
  }
}

// ----------------------------------------------------------------------------
// bucket producer: every hit of a prime p > big_min (log marks) and of p^2 > S2_T
// (square flags) in the segment's R cells, appended to the producer-private
// list of its tile.  Entry = offset (17 bits) | value << 17 (value bit 7 = OR).
// ----------------------------------------------------------------------------
// Work is balanced by hits, not by primes: small primes hit the segment up
// to 16x more often than large ones.  Each batch takes FBATCH of this
// producer's hit streams (NS per prime), computes every stream's first hit and
// hit count (one stream per thread) and cuts the hit runs into items of at most
// FITEM consecutive hits (an exclusive scan of items per stream; a thread finds
// its item's stream by binary search).  Rounds of one item per thread follow.
// Slots in a tile's list come from shared-memory counters; the entries are
// write-combined in shared memory (`bin` per tile and round) and flushed as
// runs (one bulk async copy per tile and round) instead of one 4-byte L2
// write per hit (ncu: the scattered stores were 60% of the stalls).  Entries
// past a full bin, and all square flags, are stored directly.
#define FBATCH 1024  // streams per batch
#ifndef FITEM
#define FITEM 32     // hits per item (1024 items per round: ~32k hits over the tiles)
#endif
#ifndef FILL_DIRECT
#define FILL_DIRECT 1  // streams of <= FDIRECT_MAX hits are emitted in phase 1 by their own thread
#endif
#ifndef FDIRECT_MAX
#define FDIRECT_MAX FITEM
#endif
// one run of a log stream's hits [pos, end) (cell offsets in the segment, stride
// step): four slot allocations in flight; hits past `end` count into the dummy
// rcnt[nt].  Shared addresses are explicit 32-bit (the generic stage pointer made
// the compiler rebuild the window base per store); the common case is one
// predicated st.shared, a full bin falls back to a direct global store
__device__ __forceinline__ void fill_run(u32 pos, u32 end, u32 step, u32 val, u32 rcnt_s, u32 stage_s, u32 nt,
                                         u32 bin, const u32* gcnt, u32* __restrict__ out, u32 cap) {
  for (; pos < end; pos += 4 * step) {
    u32 t[4], sl[4];
#pragma unroll
    for (int h = 0; h < 4; h++) {
      const u32 ph = pos + h * step;
      t[h] = ph < end ? ph >> 17 : nt;
    }
#pragma unroll
    for (int h = 0; h < 4; h++)
      asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(sl[h]) : "r"(rcnt_s + 4 * t[h]) : "memory");
    bool spill = false;
#pragma unroll
    for (int h = 0; h < 4; h++) {
      const u32 e = ((pos + h * step) & (S2_T - 1)) | val;
      const bool in = t[h] < nt && sl[h] < bin;
      if (in) asm volatile("st.shared.u32 [%0], %1;" ::"r"(stage_s + 4 * (t[h] * bin + sl[h])), "r"(e) : "memory");
      spill |= t[h] < nt && sl[h] >= bin;
    }
    if (spill) {  // rare: a full bin
#pragma unroll
      for (int h = 0; h < 4; h++) {
        if (t[h] < nt && sl[h] >= bin) {
          const u32 g = gcnt[t[h]] + sl[h];
          if (g < cap) out[t[h] * cap + g] = ((pos + h * step) & (S2_T - 1)) | val;
        }
      }
    }
  }
}

template <int W>
__global__ void __launch_bounds__(1024, 1) k_bucket_fill(Bucket2Args a) {
  constexpr int NS = Wheel<W>::NS;
  // dynamic: rcnt[ntiles + 1] (round counts; [ntiles] = dummy), gcnt[ntiles]
  // (entries before this round), cnt2[ntiles] (square flags), stage[ntiles][bin]
  extern __shared__ __align__(16) u32 dsm[];
  u32* rcnt = dsm;
  u32* gcnt = rcnt + a.ntiles + 1;
  u32* cnt2 = gcnt + a.ntiles;
  u32* stage = dsm + ((3 * a.ntiles + 1 + 3) & ~3u);  // 16-byte aligned (bulk copies)
  const u32 rcnt_s = (u32)__cvta_generic_to_shared(rcnt);
  const u32 stage_s = (u32)__cvta_generic_to_shared(stage);
  __shared__ u32 s_q0[FBATCH];
  __shared__ u32 s_step[FBATCH];
  __shared__ u32 s_val[FBATCH];
  __shared__ u32 s_ipre[FBATCH + 1];  // exclusive prefix of items per stream
  __shared__ u32 s_wsum[32];
  __shared__ u32 s_hits;
  __shared__ u32 s_dhits;  // hits emitted directly in this batch's phase 1
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 b = blockIdx.x, NP = gridDim.x;
  const u32 nt = a.ntiles, bin = a.bin;
  if (tid == 0) { s_hits = 0; s_dhits = 0; }
  for (u32 t = tid; t < 3 * nt + 1; t += blockDim.x) dsm[t] = 0;
  const u64 C0 = Wheel<W>::cell0(a.Y0);  // first cell of the segment
  const u32 R = nt * S2_T;                // cells, <= 2^31
  const double Cd = (double)C0;
  u32* __restrict__ out = a.buf + (u64)b * nt * a.cap;
  const u32 cap = a.cap;
  // this producer's primes: log marks p_lo + b + k*NP, then squares q_lo + b + k*NP
  const u32 nlog = a.p_hi > a.p_lo + b ? (a.p_hi - a.p_lo - b + NP - 1) / NP : 0;
  const u32 nsq = a.q_hi > a.q_lo + b ? (a.q_hi - a.q_lo - b + NP - 1) / NP : 0;
  const u32 nstream = (nlog + nsq) * NS;
  // flush: each tile's run, zero-padded to a multiple of 4 entries (an entry of 0 adds 0
  // to cell 0: a no-op mark) so every run starts 16-byte aligned, goes out as one bulk
  // async copy shared -> global (block-uniform call)
  auto flush = [&]() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    for (u32 t = tid; t < nt; t += blockDim.x) {
      const u32 rc = rcnt[t], g0 = gcnt[t];
      if (!rc) continue;
      const u32 len = (rc + 3) & ~3u;
      u32* so = stage + t * bin;
      u32* go = out + t * cap + g0;
      if (rc < bin) {  // len <= bin: up to three pad words
        const u32 npad = len - rc;
        if (npad > 0) so[rc] = 0u;
        if (npad > 1) so[rc + 1] = 0u;
        if (npad > 2) so[rc + 2] = 0u;
      } else {
        for (u32 i = rc; i < len; i++) if (g0 + i < cap) go[i] = 0u;
      }
      const u32 ncp = g0 < cap ? min(min(len, bin), cap - g0) : 0u;
      if (ncp) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(go), "r"((u32)__cvta_generic_to_shared(so)), "r"(ncp * 4u) : "memory");
      }
      gcnt[t] = g0 + len;
      rcnt[t] = 0;
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
  };
  u32 pend = 0;  // direct hits staged since the last flush (block-uniform)
  for (u32 base = 0; base < nstream; base += FBATCH) {
    __syncthreads();
    // phase 1: first hit, step, value, item count of one stream per thread
    u32 c = 0;
    {
      const u32 ks = base + tid, k = ks / NS, s = ks % NS;
      u32 q0 = R, step = 1, val = 0;
      if (ks < nstream) {
        u64 j[NS];
        if (k < nlog) {
          const u32 p = a.pperm[(u64)b * a.kp + k];  // producer-major copy: coalesced; 1/p and log recomputed
          first_hits<W>(C0, Cd, __drcp_rn((double)p), p, j);
          q0 = (u32)(s ? j[NS - 1] : j[0]);
          step = NS * p;
          val = ((32u - __clz(p - 1)) | 1u) << 17;  // ceil(log2 p) | 1
        } else {
          const u64 p = a.qperm[(u64)b * a.kq + (k - nlog)];
          const u64 q = p * p;
          first_hits<W>(C0, Cd, __drcp_rn((double)q), q, j);
          const u64 js = s ? j[NS - 1] : j[0];
          q0 = js < R ? (u32)js : R;
          step = NS * q < R ? (u32)(NS * q) : R;  // one hit at most when the stride reaches R
          val = 0x80u << 17;
        }
        const u32 hits = q0 < R ? (R - 1 - q0) / step + 1 : 0;
        if (FILL_DIRECT && hits && hits <= FDIRECT_MAX && !(val & (0x80u << 17))) {
          // a stream of at most one item (the large primes at n >= 1e21) is emitted
          // right here by its own thread: no item, no search
          fill_run(q0, R, step, val, rcnt_s, stage_s, nt, bin, gcnt, out, cap);
          atomicAdd(&s_dhits, hits);
        } else {
          c = (hits + FITEM - 1) / FITEM;
          if (hits) atomicAdd(&s_hits, hits);
        }
      }
      s_q0[tid] = q0;
      s_step[tid] = step;
      s_val[tid] = val;
    }
    // block exclusive scan of item counts
    u32 incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const u32 x = s_wsum[lane];
      u32 ix = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, ix, o);
        if (lane >= o) ix += t;
      }
      s_wsum[lane] = ix - x;
      if (lane == 31) s_ipre[FBATCH] = ix;
    }
    __syncthreads();
    s_ipre[tid] = s_wsum[warp] + incl - c;
    __syncthreads();
    const u32 nit = s_ipre[FBATCH];
    pend += s_dhits;
    // items per thread and round: large primes give short items, so a round
    // takes several per thread to fill the bins (~FITEM hits per thread)
    const u32 per = nit ? max(1u, min(16u, (FITEM * nit + s_hits / 2) / max(1u, s_hits))) : 1u;
    __syncthreads();
    if (tid == 0) { s_hits = 0; s_dhits = 0; }
    for (u32 r0 = 0; r0 < nit; r0 += 1024 * per) {
      for (u32 it = r0 + tid; it < min(nit, r0 + 1024 * per); it += 1024) {
        u32 lo = 0, hi = FBATCH;  // largest k with s_ipre[k] <= it
        while (hi - lo > 1) {
          const u32 mid = (lo + hi) >> 1;
          if (s_ipre[mid] <= it) lo = mid; else hi = mid;
        }
        const u32 k = lo, ci = it - s_ipre[k];
        const u32 step = s_step[k], val = s_val[k];
        u32 pos = s_q0[k] + ci * FITEM * step;
        const u32 end = (u32)min((u64)R, (u64)pos + (u64)FITEM * step);
        if (!(val & (0x80u << 17))) {
          // four slot allocations in flight; hits past `end` count into the dummy
          // rcnt[nt].  Shared addresses are explicit 32-bit (the generic stage
          // pointer made the compiler rebuild the window base per store); the
          // common case is one predicated st.shared, a full bin falls back to a
          // direct global store
          fill_run(pos, end, step, val, rcnt_s, stage_s, nt, bin, gcnt, out, cap);
        } else {  // square flags fill each list from the back
          for (; pos < end; pos += step) {
            const u32 t = pos >> 17;
            const u32 sl = atomicAdd(&cnt2[t], 1u);
            if (sl < cap) out[t * cap + (cap - 1 - sl)] = pos & (S2_T - 1);
          }
        }
      }
      flush();
      pend = 0;
    }
    if (pend > (nt * bin) / 2) {  // direct-only batches: flush once the bins are half full
      flush();
      pend = 0;
    }
  }
  if (pend) flush();
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  for (u32 t = tid; t < nt; t += blockDim.x) {
    const u32 nl = gcnt[t], ns = cnt2[t];
    // overflow (nl + ns > cap) is flagged by an all-ones count
    a.counts[(u64)b * nt + t] = (nl + ns > cap || nl > 0xFFFF || ns > 0xFFFF) ? 0xFFFFFFFFu : (nl | (ns << 16));
  }
}

// ----------------------------------------------------------------------------
// tile kernel
// ----------------------------------------------------------------------------

// mu of the 4 cells of a state word (uniform threshold thr): packed int8 and their sum
__device__ __forceinline__ u32 mu_word(u32 w, u32 kthr, int& sum) {
  const u32 nsq = ~w & 0x80808080u;                              // not square-flagged
  const u32 g = ((w & 0x7f7f7f7fu) + kthr) & 0x80808080u;        // s > thr
  const u32 x = g ^ ((w << 7) & 0x80808080u);                    // mu = +1 iff (s > thr) xor odd
  const u32 pl = x & nsq, mi = ~x & nsq;
  const u32 out = (pl >> 7) + (mi >> 7) * 255u;                  // bytes +1 / -1 (0xff) / 0
  sum = __dp4a((int)out, 0x01010101, sum);                        // signed byte sum
  return out;
}

__device__ __forceinline__ int mu_cell(u32 s, int thr) {
  if (s & 0x80) return 0;
  int par = s & 1;
  return ((int)s > thr) ? 1 - 2 * par : 2 * par - 1;
}

// next tile's first offset of a stream whose first offset in this tile is j < stride
__device__ __forceinline__ u32 carry(u32 j, u32 tm, u32 stride) { return j >= tm ? j - tm : j + stride - tm; }

// ----------------------------------------------------------------------------
// k_sieve3: persistent tile kernel.  CTA c sieves the contiguous tiles
// [c*m, c*m + m) of the segment; the first multiple of every in-tile prime
// (and square) is computed once per CTA by division and then carried from
// tile to tile in shared memory (no per-tile division).  Captures and head
// outputs are tile-relative; k_s3_finish makes them absolute.
// ----------------------------------------------------------------------------

// an overflowed bucket list (more hits than its capacity): producer b's hits on
// the tile at cell Ct, recomputed from the primes by one warp (rare)
template <int W>
__device__ __noinline__ void d_overflow(const u32* __restrict__ primes, const double* __restrict__ rprimes,
                                       const uint8_t* __restrict__ logs, u32 p_lo, u32 p_hi, u32 q_lo, u32 q_hi,
                                       u32 nprod, unsigned long long* ovf, u32 b, u64 Ct, u32 sbase, int lane) {
  constexpr int NS = Wheel<W>::NS;
  if (lane == 0) atomicAdd(ovf, 1ull);
  const double Cd = (double)Ct;
  u64 j[NS];
  for (u64 i = (u64)p_lo + b + (u64)lane * nprod; i < p_hi; i += 32ull * nprod) {
    const u32 p = primes[i];
    first_hits<W>(Ct, Cd, rprimes[i], p, j);
    for (int s = 0; s < NS; s++)
      for (u64 jj = j[s]; jj < S2_T; jj += NS * p)
        red_add(sbase + ((u32)jj & ~3u), (u32)logs[i] << (((u32)jj & 3) * 8));
  }
  for (u64 i = (u64)q_lo + b + (u64)lane * nprod; i < q_hi; i += 32ull * nprod) {
    const u64 p = primes[i];
    first_hits<W>(Ct, Cd, __drcp_rn((double)(p * p)), p * p, j);
    for (int s = 0; s < NS; s++)
      if (j[s] < S2_T) red_or(sbase + ((u32)j[s] & ~3u), 0x80u << (((u32)j[s] & 3) * 8));
  }
}

template <int W>
__global__ void __launch_bounds__(S2_NT, 1) k_sieve3(Sieve2Args a) {
  constexpr int NS = Wheel<W>::NS;
  constexpr u64 SPAN = Wheel<W>::SPAN;
  extern __shared__ u32 st[];                   // S2_W state / mu words
  int* csum = (int*)(st + S2_W);                // S2_CH chunk sums -> exclusive chunk prefixes
  const u32 nA = a.p_warp_end - a.p_first;
  const u32 nBp = a.p_small_end - a.p_warp_end;
  const u32 nB1 = a.p_b2 - a.p_warp_end;        // B1 primes; [nB1, nBp) are B2
  const u32 nC = a.sq_end - a.sq_first;
  u32* offA = (u32*)(csum + S2_CH);             // [NS][nA] first hit of each stream (lane 0's mark), A primes
  u32* tmA = offA + NS * nA;                    // T mod stride
  u32* offB = tmA + nA;                         // [NS][nBp] first hits, B primes
  u32* offC = offB + NS * nBp;                  // [NS][nC] first hits of p^2, small squares
  u32* tmC = offC + NS * nC;                    // T mod stride
  uint16_t* pB = (uint16_t*)(tmC + nC);         // B primes as (p - 1) / 2
  __shared__ int wsum[32];
  __shared__ int s_total;
  __shared__ u32 s_dnext;
  __shared__ u32 s_cnt[S2_MAXPROD];  // this tile's bucket-list counts
  __shared__ u64 s_cj[2][S2_MAXCAP];   // capture j ranges of this tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 m = a.tiles_per_cta;
  const u32 tile0 = blockIdx.x * m;
  if (tile0 >= a.ntiles) return;
  const u32 tile_end = min(tile0 + m, a.ntiles);
  const u32 sbase = (u32)__cvta_generic_to_shared(st);
  const u32 send = sbase + S2_T;

  // ---- first multiples at the CTA's first tile
  {
    const u64 C = Wheel<W>::cell0(a.Y0 + (u64)tile0 * SPAN);
    const double Cd = (double)C;
    u64 j[NS];
    for (u32 k = tid; k < nA; k += S2_NT) {
      const u32 i = a.p_first + k, p = a.primes[i];
      first_hits<W>(C, Cd, a.rprimes[i], p, j);
      for (int s = 0; s < NS; s++) offA[s * nA + k] = (u32)j[s];
      tmA[k] = S2_T % (NS * p);
    }
    for (u32 k = tid; k < nBp; k += S2_NT) {
      const u32 i = a.p_warp_end + k, p = a.primes[i];
      first_hits<W>(C, Cd, a.rprimes[i], p, j);
      for (int s = 0; s < NS; s++) offB[s * nBp + k] = (u32)j[s];
      pB[k] = (uint16_t)((p - 1) >> 1);
    }
    for (u32 k = tid; k < nC; k += S2_NT) {
      const u32 p = a.primes[a.sq_first + k], q = p * p;
      first_hits<W>(C, Cd, __drcp_rn((double)q), q, j);
      for (int s = 0; s < NS; s++) offC[s * nC + k] = (u32)j[s];
      tmC[k] = S2_T % (NS * q);
    }
  }

  for (u32 tile = tile0; tile < tile_end; tile++) {
    const u64 Yt = a.Y0 + (u64)tile * SPAN;    // first y of the tile
    const u64 Ct = Wheel<W>::cell0(Yt);        // first cell of the tile
    __syncthreads();  // offsets ready / previous tile's outputs done
    if (tid == 0) s_dnext = 0;
    // 1. presieve patterns
    {
      const u32* __restrict__ w1 = a.w1 + (u32)((Ct % a.w1_period4) >> 2);
      const u32* __restrict__ w2 = a.w2 + (u32)((Ct % a.w2_period4) >> 2);
      for (int i = tid; i < (int)S2_W; i += S2_NT) st[i] = w1[i] + w2[i];
    }
    for (u32 b = tid; b < a.nprod && b < S2_MAXPROD; b += S2_NT) {
      const u32 cw = a.counts[(u64)b * a.ntiles + tile];
      s_cnt[b] = cw;
#if S2_LIST_PREFETCH
      // the tile's bucket lists (~140 KB, written by the fill, mostly in DRAM) start
      // moving into L2 now and are read in phase D after the presieve and marks
      if (cw != 0xFFFFFFFFu && (cw & 0xFFFF)) {
        const u32* L = a.buf + ((u64)b * a.ntiles + tile) * a.cap;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(L), "r"((cw & 0xFFFF) * 4u) : "memory");
      }
#endif
    }
    __syncthreads();
    // 2. marks
    // A: warp per prime (W = 6: half-warp per stream), snake order over the warps
    for (u32 r = 0; r * 32 < nA; r++) {
      const u32 k = r * 32 + ((r & 1) ? 31 - warp : warp);
      if (k >= nA) continue;
      const u32 i = a.p_first + k;
      const u32 p = a.primes[i];
      const u32 lg = a.logs[i];
      const u32 stride = NS * p;
      const int s = NS == 2 ? lane >> 4 : 0;
      const u32 li = NS == 2 ? lane & 15 : lane;
      const u32 j0 = offA[s * nA + k];
      const u32 j = j0 + li * stride;
      const u32 v = lg << ((j & 3) * 8);
      const u32 astep = 32 * p;  // (32 / NS) lanes x stride
#pragma unroll 4
      for (u32 ad = sbase + (j & ~3u); ad < send; ad += astep) red_add(ad, v);
      __syncwarp();
      if (li == 0) offA[s * nA + k] = carry(j0, tmA[k], stride);
    }
    // B: lane per prime, groups of 32 in snake order (single loop, predicated tail)
    //    B1 = [1024, S2_B2_MIN): four interleaved streams per prime
    {
      const u32 nG = (nB1 + 31) / 32;
      for (u32 r = 0; r * 32 < nG; r++) {
        const u32 g = r * 32 + ((r & 1) ? 31 - warp : warp);
        if (g >= nG) continue;
        const u32 k = g * 32 + lane;
        if (k < nB1) {
          const u32 p = 2u * pB[k] + 1u;
          const u32 lg = (32 - __clz(p - 1)) | 1;
          // streams in ascending order a0 < a1 < a2 < a3 < a0 + 4p, stepping 4p:
          // W = 1, 2: j, j+p, j+2p, j+3p; W = 6: lo, hi, lo+2p, hi+2p of the two streams
          u32 e0, e1, e2, e3;
          if (NS == 2) {
            const u32 x = offB[k], y = offB[nBp + k];
            e0 = min(x, y); e1 = max(x, y); e2 = e0 + 2 * p; e3 = e1 + 2 * p;
          } else {
            e0 = offB[k]; e1 = e0 + p; e2 = e1 + p; e3 = e2 + p;
          }
          const u32 p4 = 4 * p;
          const u32 v0 = lg << ((e0 & 3) * 8), v1 = lg << ((e1 & 3) * 8);
          const u32 v2 = lg << ((e2 & 3) * 8), v3 = lg << ((e3 & 3) * 8);
          u32 a0 = sbase + (e0 & ~3u), a1 = sbase + (e1 & ~3u), a2 = sbase + (e2 & ~3u), a3 = sbase + (e3 & ~3u);
          // streams past the tile end add into a per-lane scratch word (csum[lane],
          // rewritten by the classify pass) instead of branching around the reduction
          const u32 scratch = send + 4 * lane;  // csum[lane]: one word per lane, no contention
          u32 jn = e0;
          for (; a0 < send; a0 += p4, a1 += p4, a2 += p4, a3 += p4, jn += p4) {
            red_add(a0, v0);
            red_add(a1 < send ? a1 : scratch, v1);
            red_add(a2 < send ? a2 : scratch, v2);
            red_add(a3 < send ? a3 : scratch, v3);
          }
          if (NS == 2) {
            const u32 tm = S2_T % (2 * p);
            offB[k] = carry(offB[k], tm, 2 * p);
            offB[nBp + k] = carry(offB[nBp + k], tm, 2 * p);
          } else {
            // jn is stream 0's next multiple; the first multiple past the tile is
            // one of jn - 3p .. jn (three conditional steps, no division)
            jn = jn - p >= S2_T && jn >= p ? jn - p : jn;
            jn = jn - p >= S2_T && jn >= p ? jn - p : jn;
            jn = jn - p >= S2_T && jn >= p ? jn - p : jn;
            offB[k] = jn - S2_T;
          }
        }
      }
    }
    //    B2 = [S2_B2_MIN, big_min): at most T / S2_B2_MIN hits per tile and stream,
    //    plain streams (per-prime setup dominates here, so it is kept minimal)
    {
      const u32 nG = (nBp - nB1 + 31) / 32;
      for (u32 r = 0; r * 32 < nG; r++) {
        const u32 g = r * 32 + ((r & 1) ? 31 - warp : warp);
        if (g >= nG) continue;
        const u32 k = nB1 + g * 32 + lane;
        if (k < nBp) {
          const u32 p = 2u * pB[k] + 1u;
          const u32 lg = (32 - __clz(p - 1)) | 1;
          const u32 stride = NS * p;
#pragma unroll
          for (int s = 0; s < NS; s++) {
            u32 j = offB[s * nBp + k];
            for (; j < S2_T; j += stride) red_add(sbase + (j & ~3u), lg << ((j & 3) * 8));
            offB[s * nBp + k] = j - S2_T;
          }
        }
      }
    }
    // C: warp per small square (W = 6: half-warp per stream)
    for (u32 k = warp; k < nC; k += 32) {
      const u32 p = a.primes[a.sq_first + k], q = p * p;
      const u32 stride = NS * q;
      const int s = NS == 2 ? lane >> 4 : 0;
      const u32 li = NS == 2 ? lane & 15 : lane;
      const u32 j0 = offC[s * nC + k];
      for (u32 j = j0 + li * stride; j < S2_T; j += 32 * q) red_or(sbase + (j & ~3u), 0x80u << ((j & 3) * 8));
      __syncwarp();
      if (li == 0) offC[s * nC + k] = carry(j0, tmC[k], stride);
    }
    // D: bucket lists (primes > big_min, squares > 2^17), dealt to warps from a
    //    shared counter so warps that finished A-C early take more lists; with
    //    S2_DPAIR a warp takes two lists (b, b + 1) and walks them as one run
    //    (more loads in flight, fuller lanes on short lists, half the fetches)
    if (a.nprod) {
      const u32 dn_s = (u32)__cvta_generic_to_shared(&s_dnext);
      constexpr u32 DP = S2_DPAIR ? 2 : 1;
      for (;;) {
        u32 b = 0;
        if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(b) : "r"(dn_s), "n"(DP) : "memory");
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b >= a.nprod) break;
        u32 cw0 = b < S2_MAXPROD ? s_cnt[b] : a.counts[(u64)b * a.ntiles + tile];
        u32 cw1 = 0;
        if (DP == 2 && b + 1 < a.nprod) cw1 = b + 1 < S2_MAXPROD ? s_cnt[b + 1] : a.counts[(u64)(b + 1) * a.ntiles + tile];
        // overflowed list: this producer's hits on the tile, recomputed exactly
        for (u32 h = 0; h < DP; h++) {
          u32& cw = h ? cw1 : cw0;
          if (cw != 0xFFFFFFFFu) continue;
          d_overflow<W>(a.primes, a.rprimes, a.logs, a.p_lo, a.p_hi, a.q_lo, a.q_hi, a.nprod, a.overflow, b + h, Ct,
                        sbase, lane);
          cw = 0;
        }
        const u32* __restrict__ L0 = a.buf + ((u64)b * a.ntiles + tile) * a.cap;
        const u32* __restrict__ L1 = L0 + (u64)a.ntiles * a.cap;  // list b + 1 of the tile
        // log entries (front): every run is a multiple of 4 (the fill pads it with
        // no-op zero entries), so the lists are read as 16-byte vectors, S2_DLOADS
        // per lane in flight; vector k < n0 is list b's, k >= n0 list b + 1's
        const u32 n0 = (cw0 & 0xFFFF) >> 2, n4 = n0 + ((cw1 & 0xFFFF) >> 2);
        const uint4* __restrict__ A4 = (const uint4*)L0;
        const uint4* __restrict__ B4 = (const uint4*)L1 - n0;
        for (u32 k = lane; k < n4; k += 32 * S2_DLOADS) {
          uint4 e[S2_DLOADS];
#pragma unroll
          for (int h = 0; h < S2_DLOADS; h++) {
            const u32 kk = k + 32 * h;
            e[h] = kk < n4 ? (kk < n0 ? A4 : B4)[kk] : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int h = 0; h < S2_DLOADS; h++) {
            red_add(sbase + (e[h].x & 0x1FFFCu), (e[h].x >> 17) << ((e[h].x & 3) * 8));
            red_add(sbase + (e[h].y & 0x1FFFCu), (e[h].y >> 17) << ((e[h].y & 3) * 8));
            red_add(sbase + (e[h].z & 0x1FFFCu), (e[h].z >> 17) << ((e[h].z & 3) * 8));
            red_add(sbase + (e[h].w & 0x1FFFCu), (e[h].w >> 17) << ((e[h].w & 3) * 8));
          }
        }
        // square flags (back of each list)
        const u32 s0 = cw0 >> 16, ns = s0 + (cw1 >> 16);
        const u32* __restrict__ Q0 = L0 + a.cap - 1;
        const u32* __restrict__ Q1 = L1 + a.cap - 1 + s0;
        for (u32 k = lane; k < ns; k += 32) {
          const u32 e = *((k < s0 ? Q0 : Q1) - k);
          red_or(sbase + (e & 0x1FFFCu), 0x80u << ((e & 3) * 8));
        }
      }
    }
    __syncthreads();
    if (a.states_out) {  // instrumented export (debug)
      u32* so = (u32*)(a.states_out + (u64)tile * S2_T);
      for (int i = tid; i < (int)S2_W; i += S2_NT) so[i] = st[i];
      __syncthreads();
    }
    // 3. classify (warp w: words [w*1024, (w+1)*1024), lane l: 4 words per step)
    {
      // one threshold for the tile when its y lie in one binade (always for W = 1, 2
      // and y >= SPAN; W = 6 tiles are not power-of-two aligned)
      const int thr_t = 62 - __clzll((long long)(Yt | 1));
      const bool uniform = Yt >= SPAN && (63 - __clzll((long long)(Yt + SPAN - 1))) == thr_t + 1;
      const u32 kthr = uniform ? (u32)(127 - thr_t) * 0x01010101u : 0u;
      uint4* st4 = (uint4*)st;
#pragma unroll 2
      for (int it = 0; it < 8; it++) {
        const int q = warp * 256 + it * 32 + lane;
        uint4 w = st4[q];
        int s = 0;
        if (uniform) {
          w.x = mu_word(w.x, kthr, s);
          w.y = mu_word(w.y, kthr, s);
          w.z = mu_word(w.z, kthr, s);
          w.w = mu_word(w.w, kthr, s);
        } else {
          u32* wv = (u32*)&w;
          for (int k = 0; k < 4; k++) {
            u32 mw = 0;
            for (int bb = 0; bb < 4; bb++) {
              const u64 y = Yt + Wheel<W>::y_of((u64)(q * 4 + k) * 4 + bb);
              const int thr = (y ? 63 - __clzll((long long)y) : 0) - 1;
              const int mm = mu_cell((wv[k] >> (8 * bb)) & 0xff, thr);
              s += mm;
              mw |= ((u32)(mm & 0xff)) << (8 * bb);
            }
            wv[k] = mw;
          }
        }
        st4[q] = w;
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (!(lane & 1)) csum[q >> 1] = s;
      }
    }
    __syncthreads();
    // 4. exclusive scan of the 4096 chunk sums (tile-relative)
    {
      int v0 = csum[tid * 4], v1 = csum[tid * 4 + 1], v2 = csum[tid * 4 + 2], v3 = csum[tid * 4 + 3];
      int tsum = v0 + v1 + v2 + v3;
      int incl = tsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        int x = wsum[lane], ix = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int t = __shfl_up_sync(0xffffffffu, ix, o);
          if (lane >= o) ix += t;
        }
        wsum[lane] = ix - x;
        if (lane == 31) s_total = ix;
      }
      __syncthreads();
      int e = wsum[warp] + incl - tsum;
      csum[tid * 4] = e;
      csum[tid * 4 + 1] = e + v0;
      csum[tid * 4 + 2] = e + v0 + v1;
      csum[tid * 4 + 3] = e + v0 + v1 + v2;
    }
    __syncthreads();
    if (tid == 0) a.tile_sum[tile] = s_total;
    // 5. head outputs (tile-relative block starts; k_s3_finish makes bk absolute)
    if (a.mu_out) {
      u32* mo = (u32*)(a.mu_out + (u64)tile * S2_T);
      for (int i = tid; i < (int)S2_W; i += S2_NT) mo[i] = st[i];
    }
    if (W == 1 && a.m16_out) {
      if (tid < 4) a.bkrel[(u64)tile * 4 + tid] = csum[tid * 1024];
      int16_t* m16 = a.m16_out + (u64)tile * S2_T;
      for (int c = tid; c < (int)S2_CH; c += S2_NT) {
        const int bstart = csum[(c >> 10) << 10];
        int run = csum[c] - bstart;
        const u32* wp = st + c * 8;
        uint4 o[4];
        u32* ov = (u32*)o;
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const u32 w = wp[k];
          const int c0 = run + (int)(int8_t)(w & 0xff);
          const int c1 = c0 + (int)(int8_t)((w >> 8) & 0xff);
          const int c2 = c1 + (int)(int8_t)((w >> 16) & 0xff);
          const int c3 = c2 + (int)(int8_t)(w >> 24);
          ov[2 * k] = (u32)(uint16_t)c0 | ((u32)(uint16_t)c1 << 16);
          ov[2 * k + 1] = (u32)(uint16_t)c2 | ((u32)(uint16_t)c3 << 16);
          run = c3;
        }
        uint4* dst = (uint4*)(m16 + (u64)c * 32);
#pragma unroll
        for (int k = 0; k < 4; k++) dst[k] = o[k];
      }
    }
    // 6. captures, tile-relative: Q_t[j] = (prefix at floor(n_t/j)) - (prefix at Yt - 1),
    //    the prefix being M (W = 1) or the wheel's cell sum (W = 2, 6).  The j range of
    //    every target on this tile is computed once per tile by one thread each.
    for (int t0 = 0; t0 < a.n_cap; t0 += S2_MAXCAP) {
      const int nc = min(a.n_cap - t0, S2_MAXCAP);
      __syncthreads();
      if (tid < nc) {
        const CaptureTarget2& ct = a.caps[t0 + tid];
        u64 jhi = Yt ? udiv_any(ct.n_lo, ct.n_hi, ct.nd, ct.nbits, Yt) : ~0ull;
        u64 jlo = udiv_any(ct.n_lo, ct.n_hi, ct.nd, ct.nbits, Yt + SPAN) + 1;
        s_cj[0][tid] = jlo < ct.jq0 ? ct.jq0 : jlo;
        s_cj[1][tid] = jhi > ct.jq1 ? ct.jq1 : jhi;
      }
      __syncthreads();
     for (int t = 0; t < nc; t++) {
      const CaptureTarget2& ct = a.caps[t0 + t];
      const u64 jlo = s_cj[0][t], jhi = s_cj[1][t];
      for (u64 j = jlo + tid; j <= jhi; j += S2_NT) {
        const u64 y = udiv_any(ct.n_lo, ct.n_hi, ct.nd, ct.nbits, j);
        const u32 ncell = (u32)Wheel<W>::ncell(y - Yt);  // cells with y' <= y
        if (ncell == 0) { ct.Q[j - ct.jq0] = 0; continue; }
        const u32 o = ncell - 1;
        const int c = o >> 5;
        const u32* wp = st + (c << 3);
        int s = 0;
        const u32 last = o & 31;
        for (u32 k = 0; k <= (last >> 2); k++) {
          u32 w = wp[k];
          if (k == (last >> 2)) {
            const u32 keep = (last & 3) + 1;
            w = keep == 4 ? w : (w & ((1u << (8 * keep)) - 1));
          }
          s = __dp4a((int)w, 0x01010101, s);
        }
        ct.Q[j - ct.jq0] = csum[c] + s;
      }
     }
    }
  }
}

// Segment finish in one launch (one block per tile): each block sums
// the tile totals before it (<= ntiles L2-resident ints) for its own base,
// writes its head block bases and fixes its captures; the block of the last
// tile leaves M(Y0 + R - 1) in done[1] and the last block to finish moves it
// to *running (every block has read *running by then) and re-arms the counter.
__global__ void __launch_bounds__(256) k_s3_finish(const int* __restrict__ tile_sum, u32 ntiles, i64* running,
                                                   const int* __restrict__ bkrel, i64* __restrict__ bk,
                                                   const CaptureTarget2* __restrict__ caps, int n_cap, u64 Y0,
                                                   u64 span, unsigned long long* done) {
  __shared__ i64 wred[8];
  __shared__ i64 s_base;
  const u32 t = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  i64 part = 0;
  for (u32 i = tid; i < t; i += blockDim.x) part += tile_sum[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) wred[warp] = part;
  __syncthreads();
  if (tid == 0) {
    i64 b = *(volatile i64*)running;
    for (int w = 0; w < 8; w++) b += wred[w];
    s_base = b;
  }
  __syncthreads();
  const i64 base = s_base;
  if (bk && tid < 4) bk[(u64)t * 4 + tid] = base + bkrel[(u64)t * 4 + tid];
  const u64 Yt = Y0 + (u64)t * span;
  // the tile's j range of every capture target, one thread per target (two divisions each)
  __shared__ u64 s_j[2][S2_MAXCAP];
  for (int c0 = 0; c0 < n_cap; c0 += S2_MAXCAP) {
    const int nc = min(n_cap - c0, S2_MAXCAP);
    __syncthreads();
    if (tid < nc) {
      const CaptureTarget2& ct = caps[c0 + tid];
      const u64 jhi = Yt ? udiv_any(ct.n_lo, ct.n_hi, ct.nd, ct.nbits, Yt) : ~0ull;
      const u64 jlo = udiv_any(ct.n_lo, ct.n_hi, ct.nd, ct.nbits, Yt + span) + 1;
      s_j[0][tid] = jlo < ct.jq0 ? ct.jq0 : jlo;
      s_j[1][tid] = jhi > ct.jq1 ? ct.jq1 : jhi;
    }
    __syncthreads();
    for (int c = 0; c < nc; c++) {
      const CaptureTarget2& ct = caps[c0 + c];
      for (u64 j = s_j[0][c] + tid; j <= s_j[1][c]; j += blockDim.x) ct.Q[j - ct.jq0] += (int)base;
    }
  }
  if (tid == 0) {
    if (t == ntiles - 1) ((volatile i64*)done)[1] = base + tile_sum[t];
    __threadfence();
    const unsigned long long prev = atomicAdd(done, 1ull);
    if (prev == ntiles - 1) {
      __threadfence();
      *(volatile i64*)running = ((volatile i64*)done)[1];
      *(volatile unsigned long long*)done = 0ull;
    }
  }
}

// ------------------------------------------------------------------ host side
template <int W>
static void launch_segment(const Sieve2Args& a, const Bucket2Args& b, size_t bs, size_t smem, u32 grid,
                           cudaStream_t st, KTimer* kt) {
  if (a.nprod) {
    if (kt) kt->begin(KT_SIEVE_LARGE, st);
    k_bucket_fill<W><<<b.nprod_grid, 1024, bs, st>>>(b);
    if (kt) kt->end(st);
  }
  if (kt) kt->begin(KT_SIEVE_TILE, st);
  k_sieve3<W><<<grid, S2_NT, smem, st>>>(a);
  if (kt) kt->end(st);
  if (kt) kt->begin(KT_OTHER, st);
  k_s3_finish<<<a.ntiles, 256, 0, st>>>(a.tile_sum, a.ntiles, a.running, a.bkrel, a.bk, a.caps, a.n_cap, a.Y0,
                                        Wheel<W>::SPAN, a.tstate);
  if (kt) kt->end(st);
}

// shared memory of k_sieve3: the tile, chunk sums, and the in-tile primes' offsets
static size_t sieve3_smem(const Sieve2Args& a) {
  const u32 nA = a.p_warp_end - a.p_first, nBp = a.p_small_end - a.p_warp_end, nC = a.sq_end - a.sq_first;
  const u32 ns = a.wheel == 6 ? 2 : 1;
  return S2_T + S2_CH * sizeof(int) + (size_t)((ns + 1) * nA + ns * nBp + (ns + 1) * nC) * 4 + (size_t)nBp * 2 + 16;
}

int mt_sieve2_segment(const Sieve2Segment& g, cudaStream_t st, KTimer* kt) {
  const Sieve2Args& a = g.tile;
  const Bucket2Args& b = g.bucket;
  const size_t bs = (((3 * (size_t)b.ntiles + 1 + 3) & ~(size_t)3) + (size_t)b.ntiles * b.bin) * sizeof(u32);
  const size_t smem = sieve3_smem(a);
  const u32 grid = (a.ntiles + a.tiles_per_cta - 1) / a.tiles_per_cta;
  if (a.wheel == 6) launch_segment<6>(a, b, bs, smem, grid, st, kt);
  else if (a.wheel == 2) launch_segment<2>(a, b, bs, smem, grid, st, kt);
  else launch_segment<1>(a, b, bs, smem, grid, st, kt);
  MT_CUDA_CHECK(cudaGetLastError());
  return MT_OK;
}

// ============================================================================
// host context
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

namespace {
struct Buf {
  void* p = nullptr;
  ~Buf() { if (p) mt_dfree(p); }
};
int balloc(Buf& b, size_t n) {
  if (!n) n = 16;
  cudaError_t e = mt_dmalloc(&b.p, n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    mt_set_error("device allocation of %zu bytes failed: %s", n, cudaGetErrorString(e));
    return MT_ERR_RESOURCE;
  }
  return MT_OK;
}
u64 isqrt64(u64 x) {
  u64 s = (u64)std::sqrt((long double)x);
  while (s * s > x) s--;
  while ((s + 1) * (s + 1) <= x) s++;
  return s;
}
uint8_t logp(u64 p) {  // ceil(log2 p) | 1  (sieve.py:111-121)
  int bl = 0;
  for (u64 x = p - 1; x; x >>= 1) bl++;
  return (uint8_t)(bl | 1);
}
// byte pattern of period P (cells) replicated over 4P + T bytes, as words: the
// logs of `logp_primes` and the 0x80 flags of `sq` on the cells of wheel W
// (cell c <-> y = c, 2c + 1 or 3c + 1 + (c & 1); P a multiple of each period)
std::vector<uint32_t> pattern_words(u64 P, const std::vector<u32>& logp_primes, const std::vector<u32>& sq, int W) {
  std::vector<uint8_t> one(P, 0);
  for (u64 c = 0; c < P; c++) {
    const u64 y = W == 1 ? c : W == 2 ? 2 * c + 1 : 3 * c + 1 + (c & 1);
    for (u32 p : logp_primes) if (y % p == 0) one[c] = (uint8_t)(one[c] + logp(p));
    for (u32 q : sq) if (y % q == 0) one[c] |= 0x80;
  }
  const u64 nbytes = 4 * P + S2_T;
  std::vector<uint32_t> w(nbytes / 4);
  for (u64 i = 0; i < nbytes / 4; i++) {
    u32 v = 0;
    for (int b = 0; b < 4; b++) v |= (u32)one[(4 * i + b) % P] << (8 * b);
    w[i] = v;
  }
  return w;
}
}  // namespace

struct Sieve2Host {
  // presieve patterns per wheel W (index 0: W = 1, 1: W = 2, 2: W = 6), periods in cells:
  //   W = 1: 2^2 3^2 5^2 7^2 11 = 485100 (2,3,5,7,11; 4,9,25,49) and 13 17 19 23 = 96577
  //   W = 2: 3^2 5^2 7^2 11 = 121275 (3,5,7,11; 9,25,49) and 96577
  //   W = 6: 2 5^2 7^2 11 = 26950 (5,7,11; 25,49) and 2 x 96577 (two cells per 6 y)
  Buf w1[3], w2[3], prm, rp, lg, buf, counts, tstate, ovf, tsum, tbase, bkrel;
  u64 P1[3] = {485100, 121275, 26950}, P2[3] = {96577, 96577, 193154};
  int nsm = 148;
  std::vector<u32> p;
  u32 nprod = 0, cap = 0, max_tiles = 0;
  u32 fill_smem = 0;  // dynamic shared memory available to k_bucket_fill
  u32 sieve3_smem_max = 0;  // dynamic shared memory available to k_sieve3
  // bucket primes in producer-major order: pperm[b * kp + k] = p[P_lo + b + k * nprod]
  // (log marks), qperm[b * kq + k] = p[Q_lo + b + k * nprod] (square flags)
  Buf pperm, qperm;
  u32 kp = 0, kq = 0, P_lo = 0, Q_lo = 0;
  u32 big_min = S2_T / 2;  // primes above this go to the bucket lists (2^16: measured 1.2 % better than 2^17 at 1e19)
  uint64_t overflows_host = 0;
  uint64_t launches = 0;  // kernels launched by mt_sieve2_run (fill + tile + finish per segment)
};

int mt_sieve2_create(Sieve2Host** out, uint64_t y_last, uint32_t max_tiles, cudaStream_t st) {
  Sieve2Host* h = new Sieve2Host();
  *out = h;
  h->max_tiles = max_tiles;
  // primes up to ceil(sqrt(y_last)) + 1
  const u64 lim = isqrt64(y_last) + 2;
  {
    std::vector<uint8_t> f(lim + 1, 1);
    f[0] = 0;
    if (lim >= 1) f[1] = 0;
    for (u64 i = 2; i * i <= lim; i++)
      if (f[i]) for (u64 j = i * i; j <= lim; j += i) f[j] = 0;
    for (u64 i = 2; i <= lim; i++) if (f[i]) h->p.push_back((u32)i);
  }
  const size_t np = h->p.size();
  std::vector<double> r(np);
  std::vector<uint8_t> l(np);
  for (size_t i = 0; i < np; i++) { r[i] = 1.0 / (double)h->p[i]; l[i] = logp(h->p[i]); }
  if (balloc(h->prm, np * 4) || balloc(h->rp, np * 8) || balloc(h->lg, np)) return MT_ERR_RESOURCE;
  MT_CUDA_CHECK(cudaMemcpyAsync(h->prm.p, h->p.data(), np * 4, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemcpyAsync(h->rp.p, r.data(), np * 8, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaMemcpyAsync(h->lg.p, l.data(), np, cudaMemcpyHostToDevice, st));
  // presieve patterns
  auto up = [&](Buf& b, const std::vector<uint32_t>& w) -> int {
    if (balloc(b, w.size() * 4)) return MT_ERR_RESOURCE;
    MT_CUDA_CHECK(cudaMemcpyAsync(b.p, w.data(), w.size() * 4, cudaMemcpyHostToDevice, st));
    MT_CUDA_CHECK(cudaStreamSynchronize(st));  // the host vector dies at return
    return MT_OK;
  };
  if (up(h->w1[0], pattern_words(h->P1[0], {2, 3, 5, 7, 11}, {4, 9, 25, 49}, 1))) return MT_ERR_RESOURCE;
  if (up(h->w1[1], pattern_words(h->P1[1], {3, 5, 7, 11}, {9, 25, 49}, 2))) return MT_ERR_RESOURCE;
  if (up(h->w1[2], pattern_words(h->P1[2], {5, 7, 11}, {25, 49}, 6))) return MT_ERR_RESOURCE;
  for (int i = 0; i < 3; i++)
    if (up(h->w2[i], pattern_words(h->P2[i], {13, 17, 19, 23}, {}, i == 0 ? 1 : i == 1 ? 2 : 6))) return MT_ERR_RESOURCE;
  if (const char* e = getenv("MT_S2_BIG_LOG2")) h->big_min = 1u << atoi(e);
  // bucket space: producers = SMs; capacity from the expected hits per (producer, tile)
  int dev, nsm;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double e = 0;
  for (size_t i = 0; i < np; i++) {
    const double pp = h->p[i];
    if (pp > h->big_min) e += S2_T / pp + 1.0 / 64;
    if (pp > 362 && pp * pp <= (double)y_last * 1.0001) e += S2_T / (pp * pp);
  }
  const bool any = np && (h->p.back() > h->big_min || (double)h->p.back() > 362.0);
  if (any && e > 0) {
    h->nprod = (u32)nsm;
    const double m = e / h->nprod;
    // + the fill's zero padding: <= 3 entries per tile and round, a round being
    //   ~1024 * FITEM hits of one producer spread over the segment's tiles
    const double rounds = m * max_tiles / (1024.0 * FITEM) + 1.0;
    h->cap = (u32)std::ceil(m + 8.0 * std::sqrt(m) + 2.0 * rounds + 32.0);
    if (const char* ev = getenv("MT_S2_CAP")) h->cap = std::min<u32>(h->cap, (u32)std::max(32, atoi(ev)));  // test hook
    h->cap = (h->cap + 31) & ~31u;
    if (balloc(h->buf, (size_t)h->nprod * max_tiles * h->cap * 4) ||
        balloc(h->counts, (size_t)h->nprod * max_tiles * 4))
      return MT_ERR_RESOURCE;
    auto gt = [&](u64 v) { return (u32)(std::upper_bound(h->p.begin(), h->p.end(), (u32)v) - h->p.begin()); };
    h->P_lo = gt(h->big_min);
    h->Q_lo = gt(362);
    auto perm = [&](Buf& dst, u32 lo, u32& kk) -> int {
      kk = np > lo ? (u32)((np - lo + h->nprod - 1) / h->nprod) : 0;
      std::vector<u32> v((size_t)h->nprod * kk + 1, 0);
      for (u32 b = 0; b < h->nprod; b++)
        for (u32 k = 0; k < kk; k++) {
          const size_t i = (size_t)lo + b + (size_t)k * h->nprod;
          if (i < np) v[(size_t)b * kk + k] = h->p[i];
        }
      if (balloc(dst, v.size() * 4)) return MT_ERR_RESOURCE;
      MT_CUDA_CHECK(cudaMemcpyAsync(dst.p, v.data(), v.size() * 4, cudaMemcpyHostToDevice, st));
      MT_CUDA_CHECK(cudaStreamSynchronize(st));
      return MT_OK;
    };
    if (perm(h->pperm, h->P_lo, h->kp) || perm(h->qperm, h->Q_lo, h->kq)) return MT_ERR_RESOURCE;
  }
  h->nsm = nsm;
  if (balloc(h->tstate, ((size_t)max_tiles + 1) * 8) || balloc(h->ovf, 8) || balloc(h->tsum, (size_t)max_tiles * 4) ||
      balloc(h->tbase, (size_t)max_tiles * 8) || balloc(h->bkrel, (size_t)max_tiles * 16))
    return MT_ERR_RESOURCE;
  MT_CUDA_CHECK(cudaMemsetAsync(h->ovf.p, 0, 8, st));
  MT_CUDA_CHECK(cudaMemsetAsync(h->tstate.p, 0, 16, st));  // k_s3_finish: done counter, next running
  {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes f1, f2, f6;
    MT_CUDA_CHECK(cudaFuncGetAttributes(&f1, k_sieve3<1>));
    MT_CUDA_CHECK(cudaFuncGetAttributes(&f2, k_sieve3<2>));
    MT_CUDA_CHECK(cudaFuncGetAttributes(&f6, k_sieve3<6>));
    const int s3 = optin - (int)std::max({f1.sharedSizeBytes, f2.sharedSizeBytes, f6.sharedSizeBytes});
    MT_CUDA_CHECK(cudaFuncSetAttribute(k_sieve3<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3));
    MT_CUDA_CHECK(cudaFuncSetAttribute(k_sieve3<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3));
    MT_CUDA_CHECK(cudaFuncSetAttribute(k_sieve3<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3));
    h->sieve3_smem_max = (u32)s3;
    MT_CUDA_CHECK(cudaFuncGetAttributes(&f1, k_bucket_fill<1>));
    MT_CUDA_CHECK(cudaFuncGetAttributes(&f2, k_bucket_fill<2>));
    MT_CUDA_CHECK(cudaFuncGetAttributes(&f6, k_bucket_fill<6>));
    h->fill_smem = (u32)(optin - (int)std::max({f1.sharedSizeBytes, f2.sharedSizeBytes, f6.sharedSizeBytes}));
    MT_CUDA_CHECK(cudaFuncSetAttribute(k_bucket_fill<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->fill_smem));
    MT_CUDA_CHECK(cudaFuncSetAttribute(k_bucket_fill<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->fill_smem));
    MT_CUDA_CHECK(cudaFuncSetAttribute(k_bucket_fill<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->fill_smem));
  }
  if (max_tiles > 16384) { mt_set_error("too many tiles per segment (max 2^31 cells)"); return MT_ERR_VALUE; }
  MT_CUDA_CHECK(cudaStreamSynchronize(st));
  return MT_OK;
}

void mt_sieve2_destroy(Sieve2Host* h) { delete h; }

uint64_t mt_sieve2_overflows(Sieve2Host* h) {
  unsigned long long v = 0;
  cudaMemcpy(&v, h->ovf.p, 8, cudaMemcpyDeviceToHost);
  return v;
}

int mt_sieve2_run(Sieve2Host* h, uint64_t Y0, uint32_t ntiles, int64_t* running, int8_t* mu_out,
                  int16_t* m16_out, int64_t* bk, uint8_t* states_out, const CaptureTarget2* caps,
                  int n_cap, cudaStream_t st, KTimer* kt, int wheel) {
  if (ntiles == 0) return MT_OK;
  if (wheel != 1 && wheel != 2 && wheel != 6) { mt_set_error("wheel must be 1, 2 or 6"); return MT_ERR_VALUE; }
  const u64 span = (u64)S2_T * (wheel == 6 ? 3 : wheel);
  const int wi = wheel == 1 ? 0 : wheel == 2 ? 1 : 2;
  if (ntiles > h->max_tiles || (Y0 % span) || (wheel == 6 && Y0 % 6)) { mt_set_error("bad sieve segment"); return MT_ERR_VALUE; }
  if (wheel != 1 && (m16_out || bk || Y0 < span)) {
    mt_set_error("wheel segments give mu and sums only, above the first tile");
    return MT_ERR_VALUE;
  }
  const u64 y2 = Y0 + (u64)ntiles * span - 1;
  const std::vector<u32>& p = h->p;
  const u64 s = isqrt64(y2);  // p <= floor(sqrt(y2))  <=>  p*p <= y2
  auto idx_gt = [&](u64 v) { return (u32)(std::upper_bound(p.begin(), p.end(), (u32)std::min<u64>(v, 0xFFFFFFFFull)) - p.begin()); };
  const u32 end = idx_gt(s);
  Sieve2Segment g{};
  Sieve2Args& a = g.tile;
  a.Y0 = Y0;
  a.ntiles = ntiles;
  a.tstate = (unsigned long long*)h->tstate.p;
  a.ticket = (uint32_t*)((unsigned long long*)h->tstate.p + ntiles);
  a.running = running;
  a.wheel = (u32)wheel;
  a.w1 = (const u32*)h->w1[wi].p; a.w2 = (const u32*)h->w2[wi].p;
  a.w1_period4 = 4 * h->P1[wi]; a.w2_period4 = 4 * h->P2[wi];
  a.primes = (const u32*)h->prm.p; a.rprimes = (const double*)h->rp.p; a.logs = (const uint8_t*)h->lg.p;
  a.p_first = std::min(idx_gt(28), end);  // A primes start at 29 (2..23 are presieved, or those of them >= the wheel's)
  a.p_warp_end = std::max(a.p_first, std::min(idx_gt(S2_A_MAX - 1), end));
  a.p_small_end = std::max(a.p_warp_end, std::min(idx_gt(h->big_min), end));
  a.p_b2 = std::max(a.p_warp_end, std::min(idx_gt(S2_B2_MIN - 1), a.p_small_end));
  a.sq_first = std::min(idx_gt(10), end);
  a.sq_end = std::max(a.sq_first, std::min(idx_gt(362), end));
  a.p_lo = a.p_small_end; a.p_hi = end;
  a.q_lo = std::max(a.sq_end, std::min(idx_gt(362), end)); a.q_hi = end;
  a.nprod = (h->nprod && (a.p_hi > a.p_lo || a.q_hi > a.q_lo)) ? h->nprod : 0;
  a.cap = h->cap;
  a.counts = (const u32*)h->counts.p; a.buf = (const u32*)h->buf.p;
  a.overflow = (unsigned long long*)h->ovf.p;
  a.states_out = states_out; a.mu_out = mu_out; a.m16_out = m16_out; a.bk = bk;
  a.tile_sum = (int*)h->tsum.p;
  a.tile_base = (int64_t*)h->tbase.p;
  a.bkrel = (int*)h->bkrel.p;
  a.tiles_per_cta = (ntiles + h->nsm - 1) / h->nsm;
  a.caps = caps; a.n_cap = n_cap;
  Bucket2Args& b = g.bucket;
  b.Y0 = Y0; b.ntiles = ntiles; b.cap = h->cap; b.nprod_grid = a.nprod;
  {  // write-combining bin per tile: what fits next to the counters, 16..128 entries
    const u64 head = 4ull * ((3ull * ntiles + 1 + 3) & ~3ull);
    const u64 room = h->fill_smem > head ? h->fill_smem - head : 0;
    u64 bin = std::min<u64>(128, room / (4ull * ntiles)) & ~7ull;
    if (const char* e = getenv("MT_FILL_BIN")) bin = std::min<u64>(bin, (u64)atoi(e)) & ~7ull;
    b.bin = bin >= 16 ? (u32)bin : 0;
  }
  b.primes = a.primes; b.rprimes = a.rprimes; b.logs = a.logs;
  b.p_lo = a.p_lo; b.p_hi = a.p_hi; b.q_lo = a.q_lo; b.q_hi = a.q_hi;
  b.pperm = (const u32*)h->pperm.p; b.qperm = (const u32*)h->qperm.p; b.kp = h->kp; b.kq = h->kq;
  if ((b.p_hi > b.p_lo && b.p_lo != h->P_lo) || (b.q_hi > b.q_lo && b.q_lo != h->Q_lo)) {
    mt_set_error("bucket prime ranges do not match the producer-major tables");
    return MT_ERR_VALUE;
  }
  b.buf = (u32*)h->buf.p; b.counts = (u32*)h->counts.p;
  if (sieve3_smem(a) > h->sieve3_smem_max) { mt_set_error("sieve tile needs more shared memory than the device has"); return MT_ERR_RESOURCE; }
  h->launches += (a.nprod ? 1 : 0) + 2;
  return mt_sieve2_segment(g, st, kt);
}

uint64_t mt_sieve2_launches(Sieve2Host* h, bool reset) {
  const uint64_t n = h->launches;
  if (reset) h->launches = 0;
  return n;
}
