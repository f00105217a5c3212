// Microbenchmarks for the sieve redesign (r01): shared-memory byte-add marks
// with sieve strides, and distributed-shared-memory reds across a cluster.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_sieve mb_sieve.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;

__global__ void k_local(const uint32_t* primes, int np, int words, int iters, uint32_t* out) {
  extern __shared__ uint32_t st[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) st[i] = 0;
  __syncthreads();
  const uint32_t T = words * 4u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int it = 0; it < iters; it++) {
    uint32_t base = (blockIdx.x * 7919u + it * 104729u);
    for (int i = warp; i < np; i += nw) {
      uint32_t p = primes[i];
      uint32_t j0 = p - (base % p);
      for (uint32_t j = j0 + lane * p; j < T; j += 32 * p) atomicAdd(&st[j >> 2], 5u << ((j & 3) * 8));
    }
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) s += st[i];
  atomicAdd(out, s);
}

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}

// each thread performs `n` reds into pseudo-random words of random cluster ranks
__global__ void k_dsmem(int words, int n, uint32_t* out, int remote_only) {
  extern __shared__ uint32_t st[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < words; i += blockDim.x) st[i] = 0;
  cl.sync();
  const uint32_t C = cl.num_blocks(), me = cl.block_rank();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(st);
  uint32_t x = blockIdx.x * 1315423911u + threadIdx.x * 2654435761u;
  for (int i = 0; i < n; i++) {
    x = x * 1664525u + 1013904223u;
    uint32_t r = (x >> 24) % C;
    if (remote_only && r == me) r = (r + 1) % C;
    uint32_t w = (x >> 3) % words;
    uint32_t a = mapa(base + 4 * w, r);
    asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(a), "r"(1u) : "memory");
  }
  cl.sync();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) s += st[i];
  atomicAdd(out, s);
}

// local random smem atomics, same shape as k_dsmem (reference point)
__global__ void k_lrand(int words, int n, uint32_t* out) {
  extern __shared__ uint32_t st[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) st[i] = 0;
  __syncthreads();
  uint32_t x = blockIdx.x * 1315423911u + threadIdx.x * 2654435761u;
  for (int i = 0; i < n; i++) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(&st[(x >> 3) % words], 1u);
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) s += st[i];
  atomicAdd(out, s);
}

// returning smem atomics vs match.any-based warp aggregation (slot allocation)
__global__ void k_atoms_ret(int n, uint32_t* out) {
  __shared__ uint32_t cnt[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint32_t x = blockIdx.x * 1315423911u + threadIdx.x * 2654435761u, acc = 0;
  for (int i = 0; i < n; i++) {
    x = x * 1664525u + 1013904223u;
    acc += atomicAdd(&cnt[(x >> 8) % 592], 1u);
  }
  if (acc == 0x12345678) out[0] = acc;
}
__global__ void k_match(int n, uint32_t* out) {
  __shared__ uint16_t cnt[32][600];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = lane; i < 600; i += 32) cnt[w][i] = 0;
  __syncwarp();
  uint32_t x = blockIdx.x * 1315423911u + threadIdx.x * 2654435761u, acc = 0;
  for (int i = 0; i < n; i++) {
    x = x * 1664525u + 1013904223u;
    const uint32_t t = (x >> 8) % 592;
    const uint32_t m = __match_any_sync(0xffffffffu, t);
    const uint32_t rank = __popc(m & ((1u << lane) - 1));
    const uint32_t base = cnt[w][t];
    __syncwarp();
    if (rank == __popc(m) - 1) cnt[w][t] = (uint16_t)(base + __popc(m));
    __syncwarp();
    acc += base + rank;
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  int dev = 0, nsm, clk;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double ghz = clk / 1e6;
  uint32_t* d_out;
  cudaMalloc(&d_out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // primes
  std::vector<uint32_t> P;
  std::vector<char> f(1 << 18, 1);
  for (int i = 2; i < (1 << 18); i++)
    if (f[i]) { P.push_back(i); for (int j = 2 * i; j < (1 << 18); j += i) f[j] = 0; }
  uint32_t* d_p;
  cudaMalloc(&d_p, P.size() * 4);
  cudaMemcpy(d_p, P.data(), P.size() * 4, cudaMemcpyHostToDevice);
  for (int cfg = 0; cfg < 4; cfg++) {
    int T = (cfg < 2) ? (1 << 17) : (1 << 16);
    int threads = (cfg % 2 == 0) ? 1024 : 512;
    int words = T / 4;
    int lo = 0, hi = 0;
    while (P[lo] < 29) lo++;
    while (hi < (int)P.size() && P[hi] <= (uint32_t)T) hi++;
    double marks = 0;
    for (int i = lo; i < hi; i++) marks += (double)T / P[i];
    cudaFuncSetAttribute(k_local, cudaFuncAttributeMaxDynamicSharedMemorySize, T);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_local, threads, T);
    int grid = nsm * per_sm, iters = 8;
    k_local<<<grid, threads, T>>>(d_p + lo, hi - lo, words, 1, d_out);
    cudaEventRecord(a);
    k_local<<<grid, threads, T>>>(d_p + lo, hi - lo, words, iters, d_out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double tot = marks * grid * iters;
    printf("local marks T=%d thr=%d ctas/sm=%d primes[29,%d] %.3f ms  %.3f marks/clk/SM  (%.3g marks/s, cells/s at 1.27 marks/cell %.3g) %s\n",
           T, threads, per_sm, T, ms, tot / (ms * 1e-3) / nsm / (ghz * 1e9), tot / (ms * 1e-3),
           tot / (ms * 1e-3) / 1.27, cudaGetErrorString(cudaGetLastError()));
  }
  // local random
  {
    int words = 1 << 15, n = 4096, threads = 1024;
    cudaFuncSetAttribute(k_lrand, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4);
    k_lrand<<<nsm, threads, words * 4>>>(words, n, d_out);
    cudaEventRecord(a);
    k_lrand<<<nsm, threads, words * 4>>>(words, n, d_out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double tot = (double)nsm * threads * n;
    printf("local random atomics: %.3f ops/clk/SM %s\n", tot / (ms * 1e-3) / nsm / (ghz * 1e9), cudaGetErrorString(cudaGetLastError()));
  }
  {
    int n = 4096, threads = 1024;
    k_atoms_ret<<<nsm, threads>>>(n, d_out);
    cudaEventRecord(a);
    k_atoms_ret<<<nsm, threads>>>(n, d_out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("returning smem atomics: %.3f lanes/clk/SM\n", (double)nsm * threads * n / (ms * 1e-3) / nsm / (ghz * 1e9));
    k_match<<<nsm, threads>>>(n, d_out);
    cudaEventRecord(a);
    k_match<<<nsm, threads>>>(n, d_out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("match.any slot allocation: %.3f lanes/clk/SM %s\n", (double)nsm * threads * n / (ms * 1e-3) / nsm / (ghz * 1e9),
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int C : {2, 4, 8, 16}) {
    for (int ro = 0; ro < 2; ro++) {
      int words = 1 << 15, n = 2048, threads = 1024;
      cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4);
      cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      int grid = (nsm / C) * C;
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = words * 4;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      cudaOccupancyMaxActiveClusters(&ncl, k_dsmem, &cfg);
      cudaLaunchKernelEx(&cfg, k_dsmem, words, n, d_out, ro);
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, k_dsmem, words, n, d_out, ro);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double tot = (double)grid * threads * n;
      printf("dsmem red cluster=%2d remote_only=%d active_clusters=%d grid=%d: %.3f ms %.3f reds/clk/SM %s\n", C, ro, ncl,
             grid, ms, tot / (ms * 1e-3) / grid / (ghz * 1e9), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
