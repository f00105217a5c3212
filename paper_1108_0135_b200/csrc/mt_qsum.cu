// The paper's approximate algorithm (Eq. 2):
//   q_n(x) = 2 sum_{i<=n} a_i cos(z_i * delta + b'_i),   delta = ln x - x0,
// over a zero table shifted to x0 (b'_i = (b_i + z_i x0) mod 2 pi, done on the host
// in exact arithmetic, paper_1108_0135_b200/explicit.py).  The paper's GPU workload
// besides the exact path (§8(f) rank 4).
//
// Grid form (q_batch): delta_j = delta0 + j*h.  A CTA takes QB consecutive grid points;
// each thread takes every QT-th term and walks the points by rotating
// (cos, sin)(z delta_j + b') with the fixed step (cos, sin)(z h) -- 4 FMA per point
// instead of a transcendental -- re-seeded from sincos every QB points, so the
// rotation error stays ~QB ulp.  Partial sums reduce through warp shuffles and
// shared memory in a fixed order (deterministic: ascending i within a thread,
// fixed tree across threads).  fp64 throughout (the paper: single precision is
// not enough unless both n and x are small).
#include "mt_common.cuh"
#include "mt_internal.h"

#define QT 256  // threads per CTA
#define QB 32   // grid points per CTA (one rotation run)

__global__ void __launch_bounds__(QT) k_qgrid(const double* __restrict__ z, const double* __restrict__ a,
                                              const double* __restrict__ b, u64 nt, double d0, double h, u64 count,
                                              const double* __restrict__ pts, double* __restrict__ out) {
  __shared__ double red[QT / 32][QB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 p0 = (u64)blockIdx.x * QB;
  double acc[QB];
#pragma unroll
  for (int k = 0; k < QB; k++) acc[k] = 0.0;
  if (pts) {  // arbitrary points: one sincos per term and point
    for (u64 i = tid; i < nt; i += QT) {
      const double zi = z[i], ai = a[i], bi = b[i];
#pragma unroll
      for (int k = 0; k < QB; k++) {
        const u64 p = p0 + k < count ? p0 + k : count - 1;
        acc[k] = fma(ai, cos(fma(zi, pts[p], bi)), acc[k]);
      }
    }
  } else {
    const double dstart = fma((double)p0, h, d0);
    for (u64 i = tid; i < nt; i += QT) {
      const double zi = z[i], ai = a[i];
      double s, c, sh, ch;
      sincos(fma(zi, dstart, b[i]), &s, &c);
      sincos(zi * h, &sh, &ch);
#pragma unroll
      for (int k = 0; k < QB; k++) {
        acc[k] = fma(ai, c, acc[k]);
        const double c2 = fma(c, ch, -s * sh);  // cos(t + zh)
        s = fma(s, ch, c * sh);                 // sin(t + zh)
        c = c2;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < QB; k++) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (tid < QB && p0 + tid < count) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < QT / 32; w++) v += red[w][tid];
    out[p0 + tid] = 2.0 * v;
  }
}

static int qsum(const double* z, const double* a, const double* b, uint64_t nt, double d0, double h,
                const double* pts, uint64_t count, double* out) {
  if (!count) return MT_OK;
  if (nt == 0) {
    for (u64 i = 0; i < count; i++) out[i] = 0.0;
    return MT_OK;
  }
  double *dz = nullptr, *da = nullptr, *db = nullptr, *dp = nullptr, *dout = nullptr;
  struct F { double** p[5]; ~F() { for (auto q : p) if (*q) mt_dfree(*q); } } f{{&dz, &da, &db, &dp, &dout}};
  MT_CUDA_CHECK(mt_dmalloc(&dz, nt * 8));
  MT_CUDA_CHECK(mt_dmalloc(&da, nt * 8));
  MT_CUDA_CHECK(mt_dmalloc(&db, nt * 8));
  MT_CUDA_CHECK(mt_dmalloc(&dout, count * 8));
  MT_CUDA_CHECK(cudaMemcpy(dz, z, nt * 8, cudaMemcpyHostToDevice));
  MT_CUDA_CHECK(cudaMemcpy(da, a, nt * 8, cudaMemcpyHostToDevice));
  MT_CUDA_CHECK(cudaMemcpy(db, b, nt * 8, cudaMemcpyHostToDevice));
  if (pts) {
    MT_CUDA_CHECK(mt_dmalloc(&dp, count * 8));
    MT_CUDA_CHECK(cudaMemcpy(dp, pts, count * 8, cudaMemcpyHostToDevice));
  }
  k_qgrid<<<(unsigned)((count + QB - 1) / QB), QT>>>(dz, da, db, nt, d0, h, count, dp, dout);
  MT_CUDA_CHECK(cudaGetLastError());
  MT_CUDA_CHECK(cudaMemcpy(out, dout, count * 8, cudaMemcpyDeviceToHost));
  return MT_OK;
}

extern "C" int mt_q_batch(const double* z, const double* a, const double* b, uint64_t n_terms, double delta0,
                          double step, uint64_t count, double* out) {
  return qsum(z, a, b, n_terms, delta0, step, nullptr, count, out);
}

extern "C" int mt_q_points(const double* z, const double* a, const double* b, uint64_t n_terms,
                           const double* delta, uint64_t count, double* out) {
  return qsum(z, a, b, n_terms, 0.0, 0.0, delta, count, out);
}
