// Harmonic-array update on sm_100a — the paper's accelerator contribution
// and the reference's hot loop apply_block
// (_native.pyx:227-310, pure.py:110-148), restructured for the GPU.
//
// For element k (v = floor(n/k)) the reference accumulates, over all y-blocks,
//   acc_k = sum_{m=1}^{mcut} M(m) (q_m - q'_{m+1})     counted walk (:263-284)
//         + sum_{d=lo}^{xcut} M(floor(v/d))            dense walk   (:285-307)
// with q_m = floor(v/m) and the top term clipped at xcut.  By summation by
// parts the counted walk equals
//   sum_{m=1}^{mcut} mu(m) floor(v/m)  -  M(mcut) * xcut
// (floor(v/(mcut+1)) <= xcut always), so it needs only mu(m) != 0 (61% of m),
// one exact division per item and no prefix values.  acc_k is therefore
// computed as (all mod 2^64):
//   counted  : tiles of (256 entries x 8192 m) per head segment; the tile's
//              squarefree m coprime to 6 are staged in shared memory as (1/m, m)
//              and every thread walks them with the fp64-reciprocal exact division
//              (the other m come from entries dk: S(v,x) = sum_{d|6} mu(d) S_6(v/d, x/d)).
//   windowed : dense items whose quotient y = v/d lies in the head, gathered
//              from the segment's M array (load-balanced item ranges).
//   Q-gather : dense items with k*d <= J read M(floor(n/(kd))) straight from
//              the captured quotient table Q[j] (no division at all).
// The split (xcut, mcut) is the engine's (xcut ~ 0.39 sqrt(v), mt_engine.cu k_elem_init: any
// split gives the same acc_k); the RunStats counters are the reference's split's.
#include <cub/cub.cuh>

#include "mt_common.cuh"
#include "mt_internal.h"

#include <algorithm>
#include <vector>

#define IPT 32  // items per lane per work chunk

struct UpdateCtx {
  ElemDev E;
  uint64_t* acc;
  int32_t* Mmc;
  CountedEntries C;          // counted-walk entries (elements + virtual j = 2k, 3k, 6k > K)
  uint64_t* tile_max;        // [ntiles] max walk limit of each MT_CT-entry tile
  uint8_t* tile_vbits;       // [ntiles] max bit length of v in the tile
  uint64_t ntiles;
  TargetDev* tgts;  // device
  std::vector<TargetDev> tgts_h;  // host copy (windows are set per Q-gather pass)
  int ntgt;
  // scratch
  uint64_t* units;   // [ntiles+1]
  uint64_t* cnt;     // [n+1]
  uint64_t* dtop;    // [n]
  uint64_t* off;     // [n+1]
  uint64_t* qcnt;    // [n+1]
  uint64_t* qoff;    // [n+1]
  uint64_t* counter; // work counters [4]
  GroupDev G;
  uint64_t* gunits;  // [ng+1] windows per group, then exclusive offsets
  uint64_t* guoff;   // [ng+1]
  uint64_t* gwfirst; // [ng]
  void* cub_tmp;
  size_t cub_bytes;
  uint64_t launches;
  int nsm;
  Shard sh;
  KTimer* kt;
};

// ---------------------------------------------------------------- counted walk
// Wheel-6 form (round 2).  With S(v, x) = sum_{m<=x} mu(m) floor(v/m) and S_6 the
// same sum over the m coprime to 6, mu(d m') = mu(d) mu(m') for d | 6 and m'
// coprime to 6, and floor(v/(d m')) = floor(floor(v/d)/m') give
//   S(v, x) = S_6(v, x) - S_6(v/2, x/2) - S_6(v/3, x/3) + S_6(v/6, x/6)
// (floors throughout), and floor(v_k/d) = v_{dk}.  So the counted sum of element k,
// C_k = S(v_k, mcut_k), needs only the m coprime to 6 (a third of the m), and its
// d-parts are prefixes of the walks of entries dk.  Every "counted entry" j walks
// the squarefree m coprime to 6 up to its largest limit and, for each role
//   r = 0 (d = 1): + S_6(v_j, mcut_j)          to acc[j]      (its own part)
//   r = 1, 2, 3 (d = 2, 3, 6), d | j:
//          mu(d) S_6(v_j, floor(mcut_{j/d} / d)) to acc[j/d]
// Entries 0..NE-1 are the elements; the values floor(n/j) with j = 2k, 3k, 6k > K
// (k <= K) get virtual entries (roles r >= 1 only, k_ce_virtual).  Work per element
// drops from the odd m (4/pi^2 of the m) to 3/pi^2 of them, plus the virtual parts.
// Work units are (tile of MT_CT entries) x (MT_CU consecutive m, <= MT_CM of them
// coprime to 6).
#ifndef MT_CU
#define MT_CU 8192  // m per counted unit (measured: 8192 > 4096)
#endif
static_assert((MT_CU & (MT_CU - 1)) == 0, "counted units must be powers of two (units never straddle 2^32)");
static_assert(MT_CM >= MT_CU / 3 + 1 && MT_CM % 4 == 0, "the list holds a unit's m coprime to 6, in 4-entry blocks");

__global__ void k_counted_plan(const uint64_t* __restrict__ tile_max, uint64_t ntiles, u64 Y0,
                               u64 R, uint64_t* __restrict__ units) {
  u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  if (t == ntiles) { units[t] = 0; return; }
  u64 mx = tile_max[t];
  u64 n = 0;
  if (mx >= Y0 && mx >= 1) {
    n = (mx - Y0) / MT_CU + 1;
    u64 cap = R / MT_CU;
    if (n > cap) n = cap;
  }
  units[t] = n;
}

// counted entries from the elements (one thread per element): roles 0 (own) and
// d = 2, 3, 6 for d | k (the d-part of element k/d, at index e - (k - k/d))
__global__ void k_ce_init(ElemDev E, CountedEntries C) {
  const u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E.n) return;
  const u64 k = E.k[e];
  C.vd[e] = E.vd[e]; C.vlo[e] = E.vlo[e]; C.vhi[e] = E.vhi[e]; C.vbits[e] = E.vbits[e];
  C.lim[0][e] = E.mcut[e]; C.tg[0][e] = (u32)e;
  const u32 dd[3] = {2, 3, 6};
#pragma unroll
  for (int r = 1; r < CE_ROLES; r++) {
    const u32 d = dd[r - 1];
    if (k % d == 0) {
      const u64 ep = e - (k - k / d);
      C.lim[r][e] = E.mcut[ep] / d; C.tg[r][e] = (u32)ep;
    } else {
      C.lim[r][e] = 0; C.tg[r][e] = 0xFFFFFFFFu;
    }
  }
}

// j <= x with j mod 6 in {0, 2, 3, 4} (the j divisible by 2 or 3)
__host__ __device__ __forceinline__ u64 ce_cnt23(u64 x) { const u64 r = x % 6; return 4 * (x / 6) + (r >= 2) + (r >= 3) + (r >= 4); }

// virtual entries of one target (K, its first element index ebase): the j > K of the
// form 2k, 3k, 6k (k <= K) in increasing j: A = j in (K, 2K] divisible by 2 or 3,
// B = 3i in (2K, 3K], C = 6i in (3K, 6K]; VirtSpec holds per target the first
// entry index and the A/B/C counts
struct VirtSpec { u64 base, K, ebase, nA, nB, nC; };
__global__ void k_ce_virtual(ElemDev E, const VirtSpec* __restrict__ vs, int ntgt, u64 ntot, CountedEntries C) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntot) return;
  int t = 0;
  while (t + 1 < ntgt && vs[t + 1].base <= vs[0].base + i) t++;
  const VirtSpec S = vs[t];
  const u64 c = vs[0].base + i, s = c - S.base, K = S.K;
  u64 j;
  if (s < S.nA) {
    const u64 q = ce_cnt23(K) + s;  // 0-based rank among the j divisible by 2 or 3
    const u64 r = q % 4;
    j = 6 * (q / 4) + (r == 0 ? 2 : r == 1 ? 3 : r == 2 ? 4 : 6);
  } else if (s < S.nA + S.nB) {
    j = 3 * ((2 * K) / 3 + 1 + (s - S.nA));
  } else {
    j = 6 * (K / 2 + 1 + (s - S.nA - S.nB));
  }
  C.lim[0][c] = 0; C.tg[0][c] = 0xFFFFFFFFu;
  const u32 dd[3] = {2, 3, 6};
  bool have = false;
#pragma unroll
  for (int r = 1; r < CE_ROLES; r++) {
    const u32 d = dd[r - 1];
    if (j % d == 0 && j / d <= K) {
      const u64 ep = S.ebase + j / d - 1;
      C.lim[r][c] = E.mcut[ep] / d; C.tg[r][c] = (u32)ep;
      if (!have) {  // v_j = floor(v_{j/d} / d) (< 2^64: j > K = floor(n/u) gives v_j <= u)
        const u128 v = (((u128)E.vhi[ep] << 64) | E.vlo[ep]) / d;
        const u64 vl = (u64)v;
        C.vd[c] = __ull2double_rn(vl); C.vlo[c] = vl; C.vhi[c] = 0;
        C.vbits[c] = (uint8_t)(vl ? 64 - __clzll((long long)vl) : 0);
        have = true;
      }
    } else {
      C.lim[r][c] = 0; C.tg[r][c] = 0xFFFFFFFFu;
    }
  }
}

__global__ void k_ce_tiles(CountedEntries C, uint64_t* __restrict__ tmax, uint8_t* __restrict__ tbits) {
  const u64 t = blockIdx.x, c = t * MT_CT + threadIdx.x;
  u64 m = 0;
  int b = 0;
  if (c < C.n) {
#pragma unroll
    for (int r = 0; r < CE_ROLES; r++) m = max(m, C.lim[r][c]);
    b = C.vbits[c];
  }
  typedef cub::BlockReduce<u64, MT_CT> BR;
  typedef cub::BlockReduce<int, MT_CT> BRi;
  __shared__ typename BR::TempStorage s1;
  __shared__ typename BRi::TempStorage s2;
  const u64 mx = BR(s1).Reduce(m, cub::Max());
  const int bx = BRi(s2).Reduce(b, cub::Max());
  if (threadIdx.x == 0) { tmax[t] = mx; tbits[t] = (uint8_t)bx; }
}

__device__ __forceinline__ u64 upper_idx(const uint64_t* __restrict__ off, u64 n, u64 x) {
  // largest i in [0, n) with off[i] <= x   (off non-decreasing, off[0] = 0)
  u64 lo = 0, hi = n;
  while (hi - lo > 1) {
    u64 mid = (lo + hi) >> 1;
    if (off[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// the same search by a whole warp (x warp-uniform): 32 probes per round cut the
// range 33-fold, so ~4 dependent loads instead of ~17 for 10^5 entries
__device__ __forceinline__ u64 upper_idx_warp(const uint64_t* __restrict__ off, u64 n, u64 x) {
  const int lane = threadIdx.x & 31;
  u64 lo = 0, hi = n;
  while (hi - lo > 1) {
    const u64 step = (hi - lo + 32) / 33;
    const u64 p = lo + step * (u64)(lane + 1);
    const bool ok = p < hi && off[p] <= x;  // monotone in lane
    const u32 c = __popc(__ballot_sync(0xffffffffu, ok));
    const u64 nlo = c ? lo + step * c : lo;
    const u64 nhi = lo + step * (c + 1);
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
  }
  return lo;
}

struct CountedArgs {
  CountedEntries C;
  uint64_t* acc;
  const uint64_t* tile_max;
  const uint8_t* tile_vbits;
  const uint64_t* off;  // [ntiles+1] exclusive scan of units
  uint64_t ntiles;
  const int8_t* mu;     // segment mu
  u64 Y0;
  uint64_t* counter;
  u32 rank, world, force_wide;
};

// S_o over the first bp plus-list and bn minus-list entries for one entry (all
// paths; the caller picks it for units off the fast path).  Returns the signed sum.
__device__ __noinline__ u64 counted_one(const CountedArgs& a, u64 c, u64 tau, u64 mlo, u64 mhi, int bp_, int bn_,
                                           const double* rmL, const u32* mL) {
  const u64 mhw = mlo & 0xFFFFFFFF00000000ull;  // high word shared by the chunk
  const double vd = a.C.vd[c];
  const u64 vlo = a.C.vlo[c];
  const int vb = a.tile_vbits[tau];
  const bool ok = !(a.force_wide & MT_FLAG_FORCE_SLOWDIV) && ((vb <= 50) || (mlo >= (1ull << (vb - 50))));
  if (ok && mhi <= (1ull << 31) && !(a.force_wide & MT_FLAG_FORCE_WIDE)) {
    const u32 v32 = (u32)vlo;
    u64 ap = 0, an = 0;
    u32 cp = 0, cn = 0;
#pragma unroll 8
    for (int i = 0; i < bp_; i++) {
      u64 b = (u64)__double_as_longlong(fma(vd, rmL[i], MT_TWO52));
      int t = (int)(v32 + (u32)b * mL[i]);
      ap += b; cp += (u32)t >> 31;
    }
#pragma unroll 8
    for (int i = 0; i < bn_; i++) {
      int idx = MT_CM - 1 - i;
      u64 b = (u64)__double_as_longlong(fma(vd, rmL[idx], MT_TWO52));
      int t = (int)(v32 + (u32)b * mL[idx]);
      an += b; cn += (u32)t >> 31;
    }
    return (ap - (u64)bp_ * MT_EXP52 - cp) - (an - (u64)bn_ * MT_EXP52 - cn);
  } else if (ok) {
    // 64-bit remainder: the estimate must be stripped of the exponent
    // bits before it is multiplied by m (m >= 2^31 here)
    u64 ap = 0, an = 0, cp = 0, cn = 0;
    for (int i = 0; i < bp_; i++) {
      u64 b = (u64)__double_as_longlong(fma(vd, rmL[i], MT_TWO52)) - MT_EXP52;
      i64 t = (i64)(vlo - b * (mhw | (0u - mL[i])));
      ap += b; cp += (u64)t >> 63;
    }
    for (int i = 0; i < bn_; i++) {
      int idx = MT_CM - 1 - i;
      u64 b = (u64)__double_as_longlong(fma(vd, rmL[idx], MT_TWO52)) - MT_EXP52;
      i64 t = (i64)(vlo - b * (mhw | (0u - mL[idx])));
      an += b; cn += (u64)t >> 63;
    }
    return (ap - cp) - (an - cn);
  }
  // exact path (small m with wide v): reciprocal 128/64 division with correction
  const u64 vhi = a.C.vhi[c];
  u64 sp = 0, sn = 0;
  for (int i = 0; i < bp_; i++) sp += (u64)udiv128(vlo, vhi, mhw | (0u - mL[i]));
  for (int i = 0; i < bn_; i++) sn += (u64)udiv128(vlo, vhi, mhw | (0u - mL[MT_CM - 1 - i]));
  return sp - sn;
}

// entries of the ascending list [0, tot) (plus) or [MT_CM - tot, MT_CM) read
// backwards (minus) with m <= mc
__device__ __forceinline__ int count_le(const u32* mL, u64 mhw, int tot, u64 mc, bool minus) {
  int lo = 0, hi = tot;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const u32 w = minus ? mL[MT_CM - 1 - mid] : mL[mid];
    if ((mhw | (0u - w)) <= mc) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// fast-path walks over list entries [i0, i1): two entries jointly (every entry
// read from shared memory serves both) or one alone.  Sums of the estimates'
// double bits and counts of negative 32-bit remainders (the corrections).
#ifndef CT_VEC
#define CT_VEC 1  // list entries read as 16-byte vectors (4 entries: 2 x 16 B of 1/m, 16 B of m)
#endif
#ifndef CT_RCP_PASS
#define CT_RCP_PASS 1  // reciprocals of the unit's list in a separate uniform pass
#endif
#ifndef CT_VUNROLL
#define CT_VUNROLL 4  // 4-entry blocks per iteration of the joint walk (measured: 4 > 2; 108 registers)
#endif
#define MT_PRAGMA_(x) _Pragma(#x)
#define MT_UNROLL(n) MT_PRAGMA_(unroll n)
template <bool MINUS>
__device__ __forceinline__ void walk2(const double* rmL, const u32* mL, int i0, int i1, double vdA, u32 vA,
                                      double vdB, u32 vB, u64& pA, u32& cA, u64& pB, u32& cB) {
  auto item = [&](double r, u32 m) {
    const u64 bA = (u64)__double_as_longlong(fma(vdA, r, MT_TWO52));
    const u64 bB = (u64)__double_as_longlong(fma(vdB, r, MT_TWO52));
    pA += bA; cA += (vA + (u32)bA * m) >> 31;
    pB += bB; cB += (vB + (u32)bB * m) >> 31;
  };
  int i = i0;
#if CT_VEC
  // blocks of 4 entries at indices 4k.. (minus list: MT_CM - 4 - 4k.., read in any
  // order: only the set summed matters), scalar entries before and after
#pragma unroll 1
  for (; i < i1 && (i & 3); i++) {
    const int idx = MINUS ? MT_CM - 1 - i : i;
    item(rmL[idx], mL[idx]);
  }
  MT_UNROLL(CT_VUNROLL)
  for (; i + 4 <= i1; i += 4) {
    const int b = MINUS ? MT_CM - 4 - i : i;
    const double2 r01 = *(const double2*)(rmL + b), r23 = *(const double2*)(rmL + b + 2);
    const uint4 m4 = *(const uint4*)(mL + b);
    item(r01.x, m4.x); item(r01.y, m4.y); item(r23.x, m4.z); item(r23.y, m4.w);
  }
#else
#pragma unroll 8
#endif
  for (; i < i1; i++) {
    const int idx = MINUS ? MT_CM - 1 - i : i;
    item(rmL[idx], mL[idx]);
  }
}
template <bool MINUS>
__device__ __forceinline__ void walk1(const double* rmL, const u32* mL, int i0, int i1, double vd, u32 v, u64& p,
                                      u32& c) {
  auto item = [&](double r, u32 m) {
    const u64 b = (u64)__double_as_longlong(fma(vd, r, MT_TWO52));
    p += b; c += (v + (u32)b * m) >> 31;
  };
  int i = i0;
#if CT_VEC
#pragma unroll 1
  for (; i < i1 && (i & 3); i++) {
    const int idx = MINUS ? MT_CM - 1 - i : i;
    item(rmL[idx], mL[idx]);
  }
#pragma unroll 1
  for (; i + 4 <= i1; i += 4) {
    const int b = MINUS ? MT_CM - 4 - i : i;
    const double2 r01 = *(const double2*)(rmL + b), r23 = *(const double2*)(rmL + b + 2);
    const uint4 m4 = *(const uint4*)(mL + b);
    item(r01.x, m4.x); item(r01.y, m4.y); item(r23.x, m4.z); item(r23.y, m4.w);
  }
#else
#pragma unroll 2
#endif
  for (; i < i1; i++) {
    const int idx = MINUS ? MT_CM - 1 - i : i;
    item(rmL[idx], mL[idx]);
  }
}

// one list (plus or minus) for the thread's two entries A, B with the prefix
// lengths lA[r], lB[r] of their roles r (0 = none): the walk is cut at every
// distinct positive length in ascending order (in the common case every thread
// has one, the whole list, so the walks of a warp stay in lockstep), the two
// entries walk jointly while both still need entries, and at a role's cut its
// prefix value (sum of floor(v/m) = bits - L*2^52 - corrections), signed by the
// role and the list, goes straight to the role's accumulator
template <bool MINUS>
__device__ __forceinline__ void walk_list(const double* rmL, const u32* mL, double vdA, u32 vA, double vdB, u32 vB,
                                          const int (&lA)[CE_ROLES], const int (&lB)[CE_ROLES],
                                          const u32 (&tA)[CE_ROLES], const u32 (&tB)[CE_ROLES], uint64_t* acc) {
  int mA = 0, mB = 0;
#pragma unroll
  for (int r = 0; r < CE_ROLES; r++) { mA = max(mA, lA[r]); mB = max(mB, lB[r]); }
  u64 pA = 0, pB = 0;
  u32 cA = 0, cB = 0;
  int pos = 0;
#pragma unroll 1
  for (;;) {
    int c = 0x7FFFFFFF;
#pragma unroll
    for (int r = 0; r < CE_ROLES; r++) {
      if (lA[r] > pos) c = min(c, lA[r]);
      if (lB[r] > pos) c = min(c, lB[r]);
    }
    if (c == 0x7FFFFFFF) break;
    if (mA > pos && mB > pos) walk2<MINUS>(rmL, mL, pos, c, vdA, vA, vdB, vB, pA, cA, pB, cB);
    else if (mA > pos) walk1<MINUS>(rmL, mL, pos, c, vdA, vA, pA, cA);
    else walk1<MINUS>(rmL, mL, pos, c, vdB, vB, pB, cB);
    pos = c;
    const u64 vAv = pA - (u64)c * MT_EXP52 - cA, vBv = pB - (u64)c * MT_EXP52 - cB;
#pragma unroll
    for (int r = 0; r < CE_ROLES; r++) {
      // role sign mu(d) (d = 1, 2, 3, 6: + - - +), negated on the minus list
      const bool neg = ((r == 1 || r == 2) != MINUS);
      if (lA[r] == c) atomicAdd((unsigned long long*)(acc + tA[r]), (unsigned long long)(neg ? 0ull - vAv : vAv));
      if (lB[r] == c) atomicAdd((unsigned long long*)(acc + tB[r]), (unsigned long long)(neg ? 0ull - vBv : vBv));
    }
  }
}

// Two entries per thread (c and c + MT_CT/2 of the unit's tile): every list
// entry read from shared memory serves both walks, which cuts the loads and
// loop overhead per item (the walk is issue-bound).
#define CT_THREADS (MT_CT / 2)
#ifndef CT_MINB
#define CT_MINB 5  // 5 CTAs of 128 threads per SM (<= 102 registers; measured: 5 > 4 > 6)
#endif
__global__ void __launch_bounds__(CT_THREADS, CT_MINB) k_counted(CountedArgs a) {
  // dynamic: rmL[MT_CM] (1/m), then mL[MT_CM]: the low word of m, stored NEGATED (the
  // 32-bit remainder is one IMAD, v + q * (-m))
  extern __shared__ __align__(16) double rmL[];
  u32* mL = (u32*)(rmL + MT_CM);
  __shared__ u64 s_unit;
  __shared__ int wp[CT_THREADS / 32], wn[CT_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 total = a.off[a.ntiles];
  // thread 0 fetches the next unit while the CTA works on the current one
  u64 nxt = 0;
  if (tid == 0) nxt = atomicAdd((unsigned long long*)a.counter, 1ull) * a.world + a.rank;
  for (;;) {
    if (tid == 0) s_unit = nxt;
    __syncthreads();
    const u64 unit = s_unit;
    if (unit >= total) break;
    if (tid == 0) nxt = atomicAdd((unsigned long long*)a.counter, 1ull) * a.world + a.rank;
    const u64 tau = upper_idx_warp(a.off, a.ntiles + 1, unit);
    const u64 cu = unit - a.off[tau];
    const u64 mlo = a.Y0 + cu * MT_CU;  // even (Y0 and MT_CU are)
    u64 mhi = mlo + MT_CU;  // exclusive
    const u64 mx = a.tile_max[tau];
    if (mhi > mx + 1) mhi = mx + 1;

    // ---- the unit's squarefree m coprime to 6: plus from the front, minus from the back
    constexpr int PER = MT_CU / CT_THREADS;  // 64 m per thread
    const u64 m0 = mlo + (u64)tid * PER;
    const u32 r3 = (u32)(m0 % 3);
    u64 bits[PER / 8];
#pragma unroll
    for (int q = 0; q < PER / 8; q++) bits[q] = m0 + 8 * q < mhi ? *(const u64*)(a.mu + (m0 + 8 * q - a.Y0)) : 0;
    int np = 0, nn = 0;
#pragma unroll
    for (int b = 1; b < PER; b += 2) {  // odd m (m0 is even) not divisible by 3
      const u32 s3 = r3 + (u32)(b % 3);
      const int8_t mu = (s3 == 0 || s3 == 3) ? 0 : (int8_t)((bits[b >> 3] >> (8 * (b & 7))) & 0xff);
      const bool in = m0 + b < mhi;
      np += (in && mu > 0);
      nn += (in && mu < 0);
    }
    // block exclusive scan of (np, nn)
    int ip = np, in_ = nn;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int tp = __shfl_up_sync(0xffffffffu, ip, o), tn = __shfl_up_sync(0xffffffffu, in_, o);
      if (lane >= o) { ip += tp; in_ += tn; }
    }
    if (lane == 31) { wp[warp] = ip; wn[warp] = in_; }
    __syncthreads();
    int bp = 0, bn = 0, totp = 0, totn = 0;
#pragma unroll
    for (int w = 0; w < CT_THREADS / 32; w++) {
      if (w < warp) { bp += wp[w]; bn += wn[w]; }
      totp += wp[w]; totn += wn[w];
    }
    int op = bp + ip - np, on = bn + in_ - nn;
#pragma unroll
    for (int b = 1; b < PER; b += 2) {
      const u32 s3 = r3 + (u32)(b % 3);
      const int8_t mu = (s3 == 0 || s3 == 3) ? 0 : (int8_t)((bits[b >> 3] >> (8 * (b & 7))) & 0xff);
      const u64 m = m0 + b;
#if CT_RCP_PASS
      // compaction stores only the (negated) low word; the reciprocals follow in one
      // uniform pass over the compacted list (no divergent fp64 reciprocal here)
      if (m < mhi && mu != 0) {
        const int idx = mu > 0 ? op : MT_CM - 1 - on;
        mL[idx] = 0u - (u32)m;  // units never straddle 2^32
        op += mu > 0; on += mu < 0;
      }
#else
      if (m < mhi && mu != 0) {
        const double r = __drcp_rn((double)m);
        if (mu > 0) { rmL[op] = r; mL[op] = 0u - (u32)m; op++; }
        else { const int idx = MT_CM - 1 - on; rmL[idx] = r; mL[idx] = 0u - (u32)m; on++; }  // units never straddle 2^32
      }
#endif
    }
    __syncthreads();
    const u64 mhw = mlo & 0xFFFFFFFF00000000ull;
#if CT_RCP_PASS
    for (int i = tid; i < totp + totn; i += CT_THREADS) {
      const int idx = i < totp ? i : MT_CM - totn + (i - totp);
      rmL[idx] = __drcp_rn((double)(mhw | (0u - mL[idx])));
    }
    __syncthreads();
#endif

    // ---- the two entries' roles: prefix lengths of every role's limit in both lists
    const u64 cA = tau * MT_CT + tid, cB = cA + CT_THREADS;
    int pA[CE_ROLES], nA[CE_ROLES], pB[CE_ROLES], nB[CE_ROLES];
    u32 tA[CE_ROLES], tB[CE_ROLES];
    auto lens = [&](u64 lim, int& pl, int& nl) {
      if (lim < mlo) { pl = nl = 0; return; }
      if (lim + 1 >= mhi) { pl = totp; nl = totn; return; }
      pl = count_le(mL, mhw, totp, lim, false);
      nl = count_le(mL, mhw, totn, lim, true);
    };
#pragma unroll
    for (int r = 0; r < CE_ROLES; r++) {
      pA[r] = nA[r] = pB[r] = nB[r] = 0;
      tA[r] = cA < a.C.n ? a.C.tg[r][cA] : 0xFFFFFFFFu;
      tB[r] = cB < a.C.n ? a.C.tg[r][cB] : 0xFFFFFFFFu;
      if (tA[r] != 0xFFFFFFFFu) lens(a.C.lim[r][cA], pA[r], nA[r]);
      if (tB[r] != 0xFFFFFFFFu) lens(a.C.lim[r][cB], pB[r], nB[r]);
    }
    const int vb = a.tile_vbits[tau];
    const bool fast = !(a.force_wide & (MT_FLAG_FORCE_SLOWDIV | MT_FLAG_FORCE_WIDE)) &&
                      ((vb <= 50) || (mlo >= (1ull << (vb - 50)))) && mhi <= (1ull << 31);
    if (fast) {
      const double vdA = cA < a.C.n ? a.C.vd[cA] : 0.0, vdB = cB < a.C.n ? a.C.vd[cB] : 0.0;
      const u32 vA = cA < a.C.n ? (u32)a.C.vlo[cA] : 0u, vB = cB < a.C.n ? (u32)a.C.vlo[cB] : 0u;
      walk_list<false>(rmL, mL, vdA, vA, vdB, vB, pA, pB, tA, tB, a.acc);
      walk_list<true>(rmL, mL, vdA, vA, vdB, vB, nA, nB, tA, tB, a.acc);
    } else {
#pragma unroll 1
      for (int r = 0; r < CE_ROLES; r++) {
        const bool neg = (r == 1 || r == 2);
        if (pA[r] + nA[r]) {
          const u64 S = counted_one(a, cA, tau, mlo, mhi, pA[r], nA[r], rmL, mL);
          atomicAdd((unsigned long long*)(a.acc + tA[r]), (unsigned long long)(neg ? 0ull - S : S));
        }
        if (pB[r] + nB[r]) {
          const u64 S = counted_one(a, cB, tau, mlo, mhi, pB[r], nB[r], rmL, mL);
          atomicAdd((unsigned long long*)(a.acc + tB[r]), (unsigned long long)(neg ? 0ull - S : S));
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- dense walk machinery
// walk d = dh, dh-1, ..., dl with y = floor(v/d), calling f(y) for each;
// incremental quotients: v = y (d+1) + r  =>  y(d) = y + floor((y + r)/d)
template <bool WIDE, class F>
__device__ __forceinline__ void walk_quotients(u64 vlo, u64 vhi, double vd, int vb, u64 dh, u64 dl, F f) {
  double rd = __drcp_rn((double)dh);
  u64 y = qdiv_ok(vb, dh) ? qdiv64(vd, rd, vlo, dh) : (u64)udiv128(vlo, vhi, dh);
  u64 delta = (u64)((double)y * rd);
  u64 d = dh;
  if (!WIDE) {
    u32 r = (u32)vlo - (u32)y * (u32)d;
    for (;;) {
      f(y);
      if (d == dl) break;
      --d;
      u32 t = r + (u32)y - (u32)delta * (u32)d;
      while (t >= (u32)d) {
        if ((int)t < 0) { delta--; t += (u32)d; } else { delta++; t -= (u32)d; }
      }
      r = t;
      y += delta;
    }
  } else {
    u64 r = vlo - y * d;
    for (;;) {
      f(y);
      if (d == dl) break;
      --d;
      u64 t = r + y - delta * d;
      while (t >= d) {
        if ((i64)t < 0) { delta--; t += d; } else { delta++; t -= d; }
      }
      r = t;
      y += delta;
    }
  }
}

// The window walk for d < 2^30 in 32-bit registers: d, the offset of y = v/d
// inside the window, the remainder r and the increment delta = y(d) - y(d+1)
// all fit (y < W0 + 2^15, delta <= y/d <= 2^12 in the window-walk region).
// The split d_sp keeps y/d^2 <= 1, so one correction of delta per step is
// exact; a second is never needed (a rare-path loop guards it anyway).
__device__ __forceinline__ int walk_window32(u64 vlo, u64 vhi, double vd, int vb, u64 dh64, u64 dl64, u64 W0,
                                             u32 swbase, bool& bad) {
  const double rd = __drcp_rn((double)dh64);
  const u64 y0 = qdiv_ok(vb, dh64) ? qdiv64(vd, rd, vlo, dh64) : (u64)udiv128(vlo, vhi, dh64);
  u32 delta = (u32)((double)y0 * rd);
  // all arithmetic mod 2^32 (the true ts lies in (-d, 2d)): the walk keeps -d, the
  // low word of y (the window offset is y - W0, so the load address is
  // (swbase - 2 W0) + 2 y), the remainder r and the increment delta
  int nd = -(int)(u32)dh64;
  const int ndl = -(int)(u32)dl64;
  u32 r = (u32)vlo - (u32)y0 * (u32)dh64;
  u32 yw = (u32)y0;
  u32 base = swbase - 2u * (u32)W0;
  int s = 0;
  u32 accb = 0;
  for (;;) {
    asm volatile("" : "+r"(base));  // keep the window base live (no per-item rematerialisation)
    short m16;
    asm volatile("ld.shared.s16 %0, [%1];" : "=h"(m16) : "r"(base + 2 * yw));
    s += m16;
    if (nd == ndl) break;
    ++nd;                                              // d - 1
    const int ts = (int)(r + yw) + (int)delta * nd;    // (y + r) - delta*d in (-d, 2d)
    // c = +1 if ts >= d, -1 if ts < 0, else 0 (from the two sign bits, no predicates)
    const int c = ((ts + nd) >> 31) + (ts >> 31) + 1;
    delta += (u32)c;
    const int t = ts + c * nd;                         // ts - c*d
    // t in [0, d) always holds when y/d^2 <= 1/2 but for rare floor patterns: its two
    // sign conditions are OR-ed into one word and a violation re-walks exactly
    accb |= (u32)(t | ~(t + nd));
    r = (u32)t;
    yw += delta;
  }
  bad = (accb >> 31) != 0;
  return s;
}

// floor(v/m) clamped to `clamp` (v may exceed 2^64)
__device__ __forceinline__ u64 div_clamp(u64 vlo, u64 vhi, double vd, int vb, u64 m, u64 clamp) {
  if (vhi) {
    u128 q = udiv128(vlo, vhi, m);
    return q > (u128)clamp ? clamp : (u64)q;
  }
  u64 q = udiv_any(vlo, 0, vd, vb, m);
  return q > clamp ? clamp : q;
}

// ---- shared-memory window walk: units (element group, 32K window of the segment)
__global__ void k_win_plan(GroupDev G, u64 Y0, u64 R, uint64_t* __restrict__ units,
                           uint64_t* __restrict__ wfirst) {
  u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (g > G.ng) return;
  if (g == G.ng) { units[g] = 0; return; }
  u64 lo = G.ylo[g], hi = G.yhi[g];
  u64 a = lo > Y0 ? lo : Y0, b = hi < Y0 + R - 1 ? hi : Y0 + R - 1;
  if (lo > hi || a > b) { units[g] = 0; wfirst[g] = 0; return; }
  u64 w0 = (a - Y0) / MT_BLK, w1 = (b - Y0) / MT_BLK;
  units[g] = w1 - w0 + 1;
  wfirst[g] = w0;
}

struct WinArgs {
  ElemDev E;
  uint64_t* acc;
  GroupDev G;
  const uint64_t* uoff;
  const uint64_t* wfirst;
  const int16_t* M16;
  const int64_t* bk;
  u64 Y0;
  uint64_t* counter;
  u32 rank, world, force_wide;
};

__device__ __forceinline__ void mbar_wait(u32 bar, u32 phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}

#ifndef DW_NT
#define DW_NT 256   // threads per window-walk CTA (one 64 KB window each)
#endif
#ifndef DW_MINB
#define DW_MINB 1
#endif
#ifndef DW_CTAS
#define DW_CTAS 3   // resident window-walk CTAs per SM (64 KB of shared memory each)
#endif
__global__ void __launch_bounds__(DW_NT, DW_MINB) k_dwin(WinArgs a) {
  extern __shared__ __align__(128) int4 smem_win[];
  int16_t* sw = (int16_t*)smem_win;
  const u32 swbase = (u32)__cvta_generic_to_shared(sw);
  __shared__ u64 s_unit;
  __shared__ __align__(8) unsigned long long s_bar;
  const int tid = threadIdx.x;
  const u32 bar = (u32)__cvta_generic_to_shared(&s_bar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  u32 phase = 0;
  const u64 total = a.uoff[a.G.ng];
  u64 nxt = 0;  // next unit, fetched while the current one is walked
  if (tid == 0) nxt = atomicAdd((unsigned long long*)a.counter, 1ull) * a.world + a.rank;
  for (;;) {
    if (tid == 0) s_unit = nxt;
    __syncthreads();
    const u64 unit = s_unit;
    if (unit >= total) break;
    if (tid == 0) nxt = atomicAdd((unsigned long long*)a.counter, 1ull) * a.world + a.rank;
    const u64 g = upper_idx_warp(a.uoff, a.G.ng + 1, unit);
    const u64 w = a.wfirst[g] + (unit - a.uoff[g]);
    const u64 W0 = a.Y0 + w * MT_BLK, W1 = W0 + MT_BLK;  // [W0, W1)
    // the 64 KB window arrives by one bulk async copy (TMA) while the threads
    // compute their elements' d-ranges (two divisions each); they wait on the
    // mbarrier just before their first window read
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((u32)(MT_BLK * 2)) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(swbase), "l"(a.M16 + w * MT_BLK), "r"((u32)(MT_BLK * 2)), "r"(bar) : "memory");
    }
    bool ready = false;
    const i64 base = a.bk[w];
    const bool wide = a.G.wide[g] || a.force_wide;
    const u64 e0g = a.G.start[g], e1 = a.G.start[g + 1];
    // groups smaller than the CTA: S = DW_NT/A threads per element, each walking a
    // contiguous slice of the element's d-range in this window
    const u32 A = (u32)(e1 - e0g);
    const u32 S = A < DW_NT ? DW_NT / A : 1;
    const u32 slice = A < DW_NT ? tid / A : 0;
    const u64 efirst = A < DW_NT ? e0g + tid % A : e0g + tid;
    for (u64 e = efirst; e < e1 && slice < S; e += (A < DW_NT ? e1 : DW_NT)) {
      const u64 xc = a.E.xcut[e];
      u64 lw = a.E.lo_w[e];
      const u64 sp = a.E.d_sp[e];
      if (sp > lw) lw = sp;
      if (lw > xc) continue;
      const u64 vlo = a.E.vlo[e], vhi = a.E.vhi[e];
      const double vd = a.E.vd[e];
      const int vb = a.E.vbits[e];
      u64 dh = W0 ? div_clamp(vlo, vhi, vd, vb, W0, xc) : xc;
      u64 dl = div_clamp(vlo, vhi, vd, vb, W1, xc) + 1;
      if (dl < lw) dl = lw;
      if (dh < dl) continue;
      if (S > 1) {  // this thread's slice of [dl, dh], counted from the top
        const u64 len = dh - dl + 1, piece = (len + S - 1) / S;
        if ((u64)slice * piece >= len) continue;
        const u64 top = dh - (u64)slice * piece;
        const u64 bot = top + 1 >= piece ? top - piece + 1 : 0;
        dh = top;
        if (bot > dl) dl = bot;
      }
      if (!ready) { mbar_wait(bar, phase); ready = true; }
      int s = 0;
      if (wide) {
        auto f = [&](u64 y) { s += sw[(u32)(y - W0)]; };
        walk_quotients<true>(vlo, vhi, vd, vb, dh, dl, f);
      } else {
        bool bad = false;
        s = walk_window32(vlo, vhi, vd, vb, dh, dl, W0, swbase, bad);
        if (bad) {  // never expected (d >= d_sp); exact re-walk keeps the result right regardless
          s = 0;
          auto f = [&](u64 y) { s += sw[(u32)(y - W0)]; };
          walk_quotients<true>(vlo, vhi, vd, vb, dh, dl, f);
        }
      }
      const i64 tot = (i64)s + (i64)(dh - dl + 1) * base;
      atomicAdd((unsigned long long*)(a.acc + e), (unsigned long long)tot);
    }
    // the copy must have landed before the buffer is refilled (thread 0 re-arms)
    if (tid == 0 && !ready) mbar_wait(bar, phase);
    phase ^= 1u;
    __syncthreads();
  }
}

// ---- sparse part (d < d_sp, y far above sqrt(v)): runs of consecutive d, L2 gathers
#define SPARSE_RUN 32
__global__ void k_sparse_plan(ElemDev E, u64 Y0, u64 R, uint64_t* __restrict__ runs,
                              uint64_t* __restrict__ dtop, uint64_t* __restrict__ dbot) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e > E.n) return;
  if (e == E.n) { runs[e] = 0; return; }
  u64 xc = E.xcut[e];
  const u64 sp = E.d_sp[e];
  if (sp >= 1 && sp - 1 < xc) xc = sp - 1;
  const u64 lw = E.lo_w[e];
  u64 c = 0, top = 0, bot = 0;
  if (lw <= xc) {
    const u64 vlo = E.vlo[e], vhi = E.vhi[e];
    const double vd = E.vd[e];
    const int vb = E.vbits[e];
    const u64 dhi = Y0 ? div_clamp(vlo, vhi, vd, vb, Y0, xc) : xc;
    u64 dlo = div_clamp(vlo, vhi, vd, vb, Y0 + R, xc) + 1;
    if (dlo < lw) dlo = lw;
    if (dhi >= dlo) { c = (dhi - dlo) / SPARSE_RUN + 1; top = dhi; bot = dlo; }
  }
  runs[e] = c;
  dtop[e] = top;
  dbot[e] = bot;
}

struct SparseArgs {
  ElemDev E;
  uint64_t* acc;
  const uint64_t* roff;
  const uint64_t* dtop;
  const uint64_t* dbot;
  const int16_t* M16;
  const int64_t* bk;
  u64 Y0;
  uint64_t* counter;
  u32 rank, world;
};

__global__ void __launch_bounds__(256) k_dsparse(SparseArgs a) {
  const u64 total = a.roff[a.E.n];
  for (;;) {
    u64 base_unit = 0;
    const int lane = threadIdx.x & 31;
    if (lane == 0) base_unit = atomicAdd((unsigned long long*)a.counter, 32ull);
    base_unit = __shfl_sync(0xffffffffu, base_unit, 0);
    if (base_unit * a.world + a.rank >= total) break;
    const u64 unit = (base_unit + lane) * a.world + a.rank;
    if (unit >= total) continue;
    const u64 e = upper_idx(a.roff, a.E.n + 1, unit);
    const u64 j = unit - a.roff[e];
    const u64 dh = a.dtop[e] - j * SPARSE_RUN;
    const u64 bot = a.dbot[e];
    const u64 dl = dh >= bot + SPARSE_RUN - 1 ? dh - SPARSE_RUN + 1 : bot;
    const u64 vlo = a.E.vlo[e], vhi = a.E.vhi[e];
    const double vd = a.E.vd[e];
    const int vb = a.E.vbits[e];
    i64 s = 0;
    // four quotients, then their eight gathers in flight (the gathers are
    // independent; one at a time left the kernel latency-bound, ncu long_sb 66 %)
    u64 d = dh;
    for (; d >= dl + 3; d -= 4) {
      u64 o[4];
#pragma unroll
      for (int h = 0; h < 4; h++) {
        const u64 dd = d - h;
        o[h] = (qdiv_ok(vb, dd) ? qdiv64(vd, __drcp_rn((double)dd), vlo, dd) : (u64)udiv128(vlo, vhi, dd)) - a.Y0;
      }
      int16_t m[4];
      i64 b[4];
#pragma unroll
      for (int h = 0; h < 4; h++) { m[h] = a.M16[o[h]]; b[h] = a.bk[o[h] / MT_BLK]; }
#pragma unroll
      for (int h = 0; h < 4; h++) s += (i64)m[h] + b[h];
      if (d == dl + 3) { d = dl - 1; break; }
    }
    for (; d + 1 > dl; d--) {  // 0..3 left (d >= dl, d may reach 0 only when dl = 0)
      const u64 y = qdiv_ok(vb, d) ? qdiv64(vd, __drcp_rn((double)d), vlo, d) : (u64)udiv128(vlo, vhi, d);
      const u64 o = y - a.Y0;
      s += (i64)a.M16[o] + a.bk[o / MT_BLK];
      if (d == dl) break;
    }
    atomicAdd((unsigned long long*)(a.acc + e), (unsigned long long)s);
  }
}

// ---- Q-gather: dense items with k*d <= J straight from the quotient table
struct QArgs {
  ElemDev E;
  uint64_t* acc;
  const uint64_t* off;   // [n+1]
  const uint64_t* dtop;  // [n] first (largest) d of each element's run in this block
  uint64_t n;
  uint64_t* counter;
  const TargetDev* tgts;
  u32 rank, world;
};

__global__ void __launch_bounds__(256) k_qitems(QArgs a) {
  const int lane = threadIdx.x & 31;
  const u64 total = a.off[a.n];
  for (;;) {
    u64 w = 0;
    if (lane == 0) w = atomicAdd((unsigned long long*)a.counter, 1ull) * a.world + a.rank;
    w = __shfl_sync(0xffffffffu, w, 0);
    const u64 base = w * (32ull * IPT);
    if (base >= total) break;
    u64 i = base + lane;
    if (i >= total) continue;
    u64 e = upper_idx(a.off, a.n + 1, i);
    u64 e_lo = a.off[e], e_hi = a.off[e + 1];
    u64 top = a.dtop[e];
    u64 kk = a.E.k[e];
    TargetDev t = a.tgts[a.E.tgt[e]];
    i64 sum = 0;
    for (int s = 0; s < IPT;) {
      if (i >= total) break;
      if (i >= e_hi) {
        if (sum) atomicAdd((unsigned long long*)(a.acc + e), (unsigned long long)sum);
        sum = 0;
        e = upper_idx(a.off, a.n + 1, i);
        e_lo = a.off[e]; e_hi = a.off[e + 1];
        top = a.dtop[e];
        kk = a.E.k[e];
        t = a.tgts[a.E.tgt[e]];
      }
      const u64 d = top - (i - e_lo);
      if (s + 4 <= IPT && i + 96 < e_hi) {  // four gathers of one element in flight
        const int32_t* q = t.Q + (kk * d - t.jq0);
        const u64 st = kk * 32;
        const int32_t q0 = q[0], q1 = *(q - st), q2 = *(q - 2 * st), q3 = *(q - 3 * st);
        sum += (i64)q0 + q1 + q2 + q3;
        s += 4;
        i += 128;
      } else {
        sum += t.Q[kk * d - t.jq0];
        s++;
        i += 32;
      }
    }
    if (sum) atomicAdd((unsigned long long*)(a.acc + e), (unsigned long long)sum);
  }
}

__global__ void k_mcut_capture(ElemDev E, u64 Y0, u64 R, const int16_t* __restrict__ M16,
                               const int64_t* __restrict__ bk, int32_t* __restrict__ Mmc) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E.n) return;
  u64 mc = E.mcut[e];
  if (mc >= Y0 && mc < Y0 + R) Mmc[e] = (int32_t)(M16[mc - Y0] + bk[(mc - Y0) / MT_BLK]);
}

__global__ void k_acc_finish(ElemDev E, uint64_t* __restrict__ acc, const int32_t* __restrict__ Mmc) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E.n) return;
  acc[e] -= (u64)(i64)Mmc[e] * E.xcut[e];
}

// items of element e whose table index k*d - jq0 lies in the block [r0, r1):
// d in [ceil((jq0 + r0) / k), floor((jq0 + r1 - 1) / k)] within [lo, dq_hi]
__global__ void k_qgather_plan(ElemDev E, const TargetDev* __restrict__ tgts, u64 r0, u64 r1,
                               uint64_t* __restrict__ cnt, uint64_t* __restrict__ dtop) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e > E.n) return;
  if (e == E.n) { cnt[e] = 0; return; }
  const TargetDev& tg = tgts[E.tgt[e]];
  const u64 k = E.k[e], jq0 = tg.jq0;
  if (r0 < tg.wlo) r0 = tg.wlo;  // this pass's window of the target's table
  if (r1 > tg.whi) r1 = tg.whi;
  if (r0 >= r1) { cnt[e] = 0; dtop[e] = 0; return; }
  u64 hi = E.dq_hi[e], lo = E.lo[e];
  const u64 dl = (jq0 + r0 + k - 1) / k, dh = (jq0 + r1 - 1) / k;
  if (dl > lo) lo = dl;
  if (dh < hi) hi = dh;
  cnt[e] = hi >= lo ? hi - lo + 1 : 0;
  dtop[e] = hi;
}

static int scan_u64(UpdateCtx* c, const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t st) {
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, (int64_t)n, st);
  if (need > c->cub_bytes) {
    if (c->cub_tmp) mt_dfree(c->cub_tmp);
    MT_CUDA_CHECK(mt_dmalloc(&c->cub_tmp, need));
    c->cub_bytes = need;
  }
  MT_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(c->cub_tmp, need, in, out, (int64_t)n, st));
  c->launches += 2;  // cub: tile-state init kernel + scan kernel
  return MT_OK;
}

int mt_update_create(UpdateCtx** out, const ElemDev& E, uint64_t* acc, int32_t* Mmc, const uint64_t* Kt,
                     const TargetDev* tgts, int ntgt, const GroupDev& grp, const Shard& sh,
                     KTimer* kt, cudaStream_t st) {
  UpdateCtx* c = new UpdateCtx();
  c->sh = sh;
  c->kt = kt;
  c->G = grp;
  c->E = E; c->acc = acc; c->Mmc = Mmc;
  c->ntgt = ntgt;
  c->launches = 0;
  *out = c;
  MT_CUDA_CHECK(mt_dmalloc(&c->tgts, sizeof(TargetDev) * (ntgt ? ntgt : 1)));
  c->tgts_h.assign(tgts, tgts + ntgt);
  MT_CUDA_CHECK(cudaMemcpyAsync(c->tgts, tgts, sizeof(TargetDev) * ntgt, cudaMemcpyHostToDevice, st));
  // counted entries: the NE elements (target t's k = 1..K_t from ebase_t on), then
  // per target its virtual entries (k_ce_virtual)
  std::vector<VirtSpec> vs(ntgt ? ntgt : 1);
  u64 nce = E.n, eb = 0;
  for (int t = 0; t < ntgt; t++) {
    const u64 K = Kt[t];
    VirtSpec& v = vs[t];
    v.base = nce; v.K = K; v.ebase = eb;
    v.nA = ce_cnt23(2 * K) - ce_cnt23(K);
    v.nB = K - (2 * K) / 3;
    v.nC = K - K / 2;
    nce += v.nA + v.nB + v.nC;
    eb += K;
  }
  CountedEntries& C = c->C;
  C.n = nce;
  const u64 na = nce ? nce : 1;
  MT_CUDA_CHECK(mt_dmalloc(&C.vd, na * 8)); MT_CUDA_CHECK(mt_dmalloc(&C.vlo, na * 8)); MT_CUDA_CHECK(mt_dmalloc(&C.vhi, na * 8));
  MT_CUDA_CHECK(mt_dmalloc(&C.vbits, na));
  for (int r = 0; r < CE_ROLES; r++) {
    MT_CUDA_CHECK(mt_dmalloc(&C.lim[r], na * 8));
    MT_CUDA_CHECK(mt_dmalloc(&C.tg[r], na * 4));
  }
  c->ntiles = (nce + MT_CT - 1) / MT_CT;
  MT_CUDA_CHECK(mt_dmalloc(&c->tile_max, (c->ntiles + 1) * 8));
  MT_CUDA_CHECK(mt_dmalloc(&c->tile_vbits, c->ntiles + 1));
  {
    VirtSpec* dvs = nullptr;
    MT_CUDA_CHECK(mt_dmalloc(&dvs, sizeof(VirtSpec) * vs.size()));
    MT_CUDA_CHECK(cudaMemcpyAsync(dvs, vs.data(), sizeof(VirtSpec) * ntgt, cudaMemcpyHostToDevice, st));
    if (E.n) k_ce_init<<<(unsigned)((E.n + 255) / 256), 256, 0, st>>>(E, C);
    const u64 nv = nce - E.n;
    if (nv) k_ce_virtual<<<(unsigned)((nv + 255) / 256), 256, 0, st>>>(E, dvs, ntgt, nv, C);
    if (c->ntiles) k_ce_tiles<<<(unsigned)c->ntiles, MT_CT, 0, st>>>(C, c->tile_max, c->tile_vbits);
    MT_CUDA_CHECK(cudaGetLastError());
    MT_CUDA_CHECK(cudaStreamSynchronize(st));
    mt_dfree(dvs);
  }
  const u64 ntiles = c->ntiles;
  MT_CUDA_CHECK(mt_dmalloc(&c->units, sizeof(uint64_t) * (ntiles + 1) * 2));
  MT_CUDA_CHECK(mt_dmalloc(&c->cnt, sizeof(uint64_t) * (E.n + 1)));
  MT_CUDA_CHECK(mt_dmalloc(&c->dtop, sizeof(uint64_t) * (E.n + 1)));
  MT_CUDA_CHECK(mt_dmalloc(&c->off, sizeof(uint64_t) * (E.n + 1)));
  MT_CUDA_CHECK(mt_dmalloc(&c->qcnt, sizeof(uint64_t) * (E.n + 1)));
  MT_CUDA_CHECK(mt_dmalloc(&c->qoff, sizeof(uint64_t) * (E.n + 1)));
  MT_CUDA_CHECK(mt_dmalloc(&c->counter, sizeof(uint64_t) * 4));
  MT_CUDA_CHECK(mt_dmalloc(&c->gunits, sizeof(uint64_t) * (grp.ng + 1)));
  MT_CUDA_CHECK(mt_dmalloc(&c->guoff, sizeof(uint64_t) * (grp.ng + 1)));
  MT_CUDA_CHECK(mt_dmalloc(&c->gwfirst, sizeof(uint64_t) * (grp.ng + 1)));
  MT_CUDA_CHECK(cudaFuncSetAttribute(k_dwin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(MT_BLK * 2)));
  MT_CUDA_CHECK(cudaFuncSetAttribute(k_counted, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(MT_CM * 12)));
  c->cub_tmp = nullptr; c->cub_bytes = 0;
  int dev; cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, dev);
  return MT_OK;
}

void mt_update_destroy(UpdateCtx* c) {
  if (!c) return;
  mt_dfree(c->C.vd); mt_dfree(c->C.vlo); mt_dfree(c->C.vhi); mt_dfree(c->C.vbits);
  for (int r = 0; r < CE_ROLES; r++) { mt_dfree(c->C.lim[r]); mt_dfree(c->C.tg[r]); }
  mt_dfree(c->tile_max); mt_dfree(c->tile_vbits);
  mt_dfree(c->tgts); mt_dfree(c->units); mt_dfree(c->cnt); mt_dfree(c->dtop); mt_dfree(c->off);
  mt_dfree(c->qcnt); mt_dfree(c->qoff); mt_dfree(c->counter);
  mt_dfree(c->gunits); mt_dfree(c->guoff); mt_dfree(c->gwfirst);
  if (c->cub_tmp) mt_dfree(c->cub_tmp);
  delete c;
}

uint64_t mt_update_launches(UpdateCtx* c) { return c->launches; }
void mt_update_reset_launches(UpdateCtx* c) { c->launches = 0; }

int mt_update_head_segment(UpdateCtx* c, u64 Y0, u64 R, const int8_t* mu, const int16_t* M16,
                           const int64_t* bk, cudaStream_t st) {
  const ElemDev& E = c->E;
  // counted walk
  {
    uint64_t* units = c->units;
    uint64_t* off = c->units + (c->ntiles + 1);
    k_counted_plan<<<(unsigned)((c->ntiles + 1 + 255) / 256), 256, 0, st>>>(c->tile_max, c->ntiles, Y0, R, units);
    c->launches++;
    int rc = scan_u64(c, units, off, c->ntiles + 1, st);
    if (rc) return rc;
    MT_CUDA_CHECK(cudaMemsetAsync(c->counter, 0, sizeof(uint64_t) * 4, st));
    CountedArgs a{c->C, c->acc, c->tile_max, c->tile_vbits, off, c->ntiles, mu, Y0, c->counter,
                  c->sh.rank, c->sh.world, c->sh.flags};
    c->kt->begin(KT_COUNTED, st);
    k_counted<<<c->nsm * 12, CT_THREADS, MT_CM * 12, st>>>(a);
    c->kt->end(st);
    c->launches++;
    MT_CUDA_CHECK(cudaGetLastError());
  }
  // M(mcut) captures
  k_mcut_capture<<<(unsigned)((E.n + 255) / 256), 256, 0, st>>>(E, Y0, R, M16, bk, c->Mmc);
  c->launches++;
  // windowed dense walk, shared-memory windows
  if (c->G.ng) {
    k_win_plan<<<(unsigned)((c->G.ng + 1 + 255) / 256), 256, 0, st>>>(c->G, Y0, R, c->gunits, c->gwfirst);
    c->launches++;
    int rc = scan_u64(c, c->gunits, c->guoff, c->G.ng + 1, st);
    if (rc) return rc;
    WinArgs a{E, c->acc, c->G, c->guoff, c->gwfirst, M16, bk, Y0, c->counter + 1,
              c->sh.rank, c->sh.world, (c->sh.flags & MT_FLAG_FORCE_WIDE) ? 1u : 0u};
    c->kt->begin(KT_DWIN, st);
    k_dwin<<<c->nsm * DW_CTAS, DW_NT, MT_BLK * 2, st>>>(a);
    c->kt->end(st);
    c->launches++;
    MT_CUDA_CHECK(cudaGetLastError());
  }
  // windowed dense walk, sparse part
  {
    k_sparse_plan<<<(unsigned)((E.n + 1 + 255) / 256), 256, 0, st>>>(E, Y0, R, c->cnt, c->dtop, c->qoff);
    c->launches++;
    int rc = scan_u64(c, c->cnt, c->off, E.n + 1, st);
    if (rc) return rc;
    SparseArgs a{E, c->acc, c->off, c->dtop, c->qoff, M16, bk, Y0, c->counter + 2, c->sh.rank, c->sh.world};
    c->kt->begin(KT_DSPARSE, st);
    k_dsparse<<<c->nsm * 8, 256, 0, st>>>(a);
    c->kt->end(st);
    c->launches++;
    MT_CUDA_CHECK(cudaGetLastError());
  }
  return MT_OK;
}

// The items k*d <= J read Q[k d] with stride k: one DRAM sector (~110 B of
// DRAM traffic measured) per 4-byte item when the table is swept element by
// element.  Blocking the table index into L2-sized ranges and running every
// element's items of one block before the next keeps the block in L2, so the
// table is read from HBM about once (1e19: 1.78 TB of DRAM reads unblocked).
int mt_update_qgather(UpdateCtx* c, const uint64_t* wlo, const uint64_t* whi, bool interleave, cudaStream_t st) {
  const ElemDev& E = c->E;
  u64 B = 1ull << 24;  // 64 MB of int32 table per block
  if (const char* ev = getenv("MT_QBLOCK_LOG2")) B = 1ull << atoi(ev);
  u64 lo = ~0ull, hi = 0;
  for (int t = 0; t < c->ntgt; t++) {
    c->tgts_h[t].wlo = wlo[t];
    c->tgts_h[t].whi = whi[t];
    if (whi[t] > wlo[t]) { lo = std::min<u64>(lo, wlo[t]); hi = std::max<u64>(hi, whi[t]); }
  }
  if (hi == 0) return MT_OK;
  MT_CUDA_CHECK(cudaMemcpyAsync(c->tgts, c->tgts_h.data(), sizeof(TargetDev) * c->ntgt, cudaMemcpyHostToDevice, st));
  MT_CUDA_CHECK(cudaStreamSynchronize(st));  // tgts_h may change before the copy would run
  const u32 rank = interleave ? c->sh.rank : 0u, world = interleave ? c->sh.world : 1u;
  for (u64 b = lo / B; b * B < hi; b++) {
    k_qgather_plan<<<(unsigned)((E.n + 1 + 255) / 256), 256, 0, st>>>(E, c->tgts, b * B, (b + 1) * B, c->qcnt, c->dtop);
    c->launches++;
    int rc = scan_u64(c, c->qcnt, c->qoff, E.n + 1, st);
    if (rc) return rc;
    MT_CUDA_CHECK(cudaMemsetAsync(c->counter + 3, 0, sizeof(uint64_t), st));
    QArgs a{E, c->acc, c->qoff, c->dtop, E.n, c->counter + 3, c->tgts, rank, world};
    c->kt->begin(KT_QGATHER, st);
    k_qitems<<<c->nsm * 8, 256, 0, st>>>(a);
    c->kt->end(st);
    c->launches++;
    MT_CUDA_CHECK(cudaGetLastError());
  }
  return MT_OK;
}

int mt_update_finish(UpdateCtx* c, cudaStream_t st) {
  k_acc_finish<<<(unsigned)((c->E.n + 255) / 256), 256, 0, st>>>(c->E, c->acc, c->Mmc);
  c->launches++;
  MT_CUDA_CHECK(cudaGetLastError());
  return MT_OK;
}

// ---------------------------------------------------------------- final resolve
// final[k] = 1 - acc[k] - sum_{d=2}^{D_k} final[k d]   (_native.pyx:313-334)
// Level-parallel: k in (K/2^{L+1}, K/2^L] depends only on levels above.
__global__ void k_fin_level(const uint64_t* __restrict__ acc, const uint64_t* __restrict__ D,
                            int64_t* __restrict__ fin, u64 klo, u64 khi) {
  const u64 wid = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const u64 k = klo + 1 + wid;
  if (k > khi) return;
  const u64 dk = D[k - 1];
  u64 s = 0;
  for (u64 d = 2 + lane; d <= dk; d += 32) s += (u64)fin[k * d - 1];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) fin[k - 1] = (int64_t)(1ull - acc[k - 1] - s);
}

int mt_finalize_dev(const uint64_t* acc, const uint64_t* D, uint64_t K, int64_t* fin, cudaStream_t st,
                    uint64_t* launches) {
  if (K == 0) return MT_OK;
  u64 khi = K;
  while (khi > 0) {
    u64 klo = khi / 2;
    u64 n = khi - klo;
    u64 threads = n * 32;
    k_fin_level<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(acc, D, fin, klo, khi);
    MT_CUDA_CHECK(cudaGetLastError());
    if (launches) ++*launches;
    khi = klo;
  }
  return MT_OK;
}

// ------------------------------------------------------ plugin: apply_block
// Exact per-block semantics of _native.pyx:227-310 (thread per element).
__global__ void k_apply_block(u64 K, int64_t* __restrict__ acc, const uint64_t* __restrict__ v,
                              const uint64_t* __restrict__ lo, const uint64_t* __restrict__ xcut,
                              const uint64_t* __restrict__ mcut, uint64_t* __restrict__ dnext,
                              uint64_t* __restrict__ ynext, u64 a, u64 b,
                              const int64_t* __restrict__ mp, uint64_t* __restrict__ counters) {
  u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const u64 vk = v[k];
  const double vd = __ull2double_rn(vk);
  const int vb = vk ? 64 - __clzll((long long)vk) : 0;
  u64 counted = 0, dense = 0;
  const u64 mc = mcut[k];
  if (mc >= a) {
    u64 hi = mc < b ? mc : b;
    u64 qn = udiv_any(vk, 0, vd, vb, hi + 1);
    if (hi == mc && qn < xcut[k]) qn = xcut[k];
    i128 delta = 0;
    for (u64 m = hi; m >= a && m >= 1; m--) {
      u64 q = udiv_any(vk, 0, vd, vb, m);
      delta += (i128)(i64)(q - qn) * mp[m - a];
      qn = q;
    }
    counted = hi - a + 1;
    delta += acc[k];
    const i128 lim = (i128)1 << 62;
    if (delta > lim || delta < -lim) { atomicAdd((unsigned long long*)&counters[2], 1ull); return; }
    acc[k] = (int64_t)delta;
  }
  if (ynext[k] <= b) {
    u64 d = dnext[k];
    const u64 lok = lo[k];
    u64 d_lo = udiv_any(vk, 0, vd, vb, b + 1) + 1;
    if (d_lo < lok) d_lo = lok;
    u64 q = ynext[k];
    i64 delta = 0;
    for (;;) {
      delta += mp[q - a];
      dense++;
      if (d == d_lo) break;
      d--;
      q = udiv_any(vk, 0, vd, vb, d);
    }
    acc[k] += delta;
    dnext[k] = d_lo - 1;
    ynext[k] = (d_lo - 1 >= lok) ? udiv_any(vk, 0, vd, vb, d_lo - 1) : ~0ull;
  }
  if (counted) atomicAdd((unsigned long long*)&counters[0], (unsigned long long)counted);
  if (dense) atomicAdd((unsigned long long*)&counters[1], (unsigned long long)dense);
}

int mt_apply_block_dev(uint64_t K, int64_t* acc, const uint64_t* v, const uint64_t* lo,
                       const uint64_t* xcut, const uint64_t* mcut, uint64_t* dnext, uint64_t* ynext,
                       uint64_t y1, uint64_t y2, const int64_t* mp, uint64_t* counters, cudaStream_t st) {
  if (K == 0) return MT_OK;
  k_apply_block<<<(unsigned)((K + 127) / 128), 128, 0, st>>>(K, acc, v, lo, xcut, mcut, dnext, ynext, y1, y2, mp, counters);
  MT_CUDA_CHECK(cudaGetLastError());
  return MT_OK;
}

// ------------------------------------------------ plugin: build_divisor_arrays
// _native.pyx:32-68 (Granlund-Montgomery constants), one thread per divisor.
__global__ void k_divisor(u64 cap, uint64_t* magic, uint8_t* shift, uint8_t* scheme) {
  u64 d = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (d > cap) return;
  if (d == 0) { magic[0] = 0; shift[0] = 0; scheme[0] = 0; return; }
  int s = 63 - __clzll((long long)d);
  if ((d & (d - 1)) == 0) { magic[d] = 0; shift[d] = (uint8_t)s; scheme[d] = 2; return; }
  u128 num = (u128)1 << (64 + s);
  u64 m0 = (u64)(num / d);
  u64 rem = (u64)(num - (u128)m0 * d);
  if (d - rem < (1ull << s)) { magic[d] = m0 + 1; shift[d] = (uint8_t)s; scheme[d] = 0; }
  else {
    u128 big = (s == 63) ? (~(u128)0) / d + 1 : (((u128)1 << (64 + s + 1)) + d - 1) / d;
    magic[d] = (u64)big; shift[d] = (uint8_t)s; scheme[d] = 1;
  }
}

int mt_divisor_arrays_dev(uint64_t cap, uint64_t* magic, uint8_t* shift, uint8_t* scheme, cudaStream_t st) {
  k_divisor<<<(unsigned)((cap + 1 + 255) / 256), 256, 0, st>>>(cap, magic, shift, scheme);
  MT_CUDA_CHECK(cudaGetLastError());
  return MT_OK;
}
