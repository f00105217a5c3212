// Pipe-throughput microbenchmarks for the Mertens hot loops on sm_100a.
// Each kernel reports lane-ops/s; used to size the update/sieve kernels
// and to measure the INT (IMAD) peak that the roofline fraction uses.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s %s:%d\n",cudaGetErrorString(e),__FILE__,__LINE__); return 1;}}while(0)

__global__ void k_imad(uint32_t* out, int iters, uint32_t a) {
  uint32_t x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<16;j++){ x0=x0*a+x1; x1=x1*a+x2; x2=x2*a+x3; x3=x3*a+x4; x4=x4*a+x5; x5=x5*a+x6; x6=x6*a+x7; x7=x7*a+x0; }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0^x1^x2^x3^x4^x5^x6^x7;
}
__global__ void k_dfma(double* out, int iters, double a) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<16;j++){ x0=fma(x0,a,x1); x1=fma(x1,a,x2); x2=fma(x2,a,x3); x3=fma(x3,a,x4); x4=fma(x4,a,x5); x5=fma(x5,a,x6); x6=fma(x6,a,x7); x7=fma(x7,a,x0);}
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_iadd(uint32_t* out, int iters, uint32_t a) {
  uint32_t x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<16;j++){ x0=(x0^a)+x1; x1=(x1^a)+x2; x2=(x2^a)+x3; x3=(x3^a)+x4; x4=(x4^a)+x5; x5=(x5^a)+x6; x6=(x6^a)+x7; x7=(x7^a)+x0; }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0^x1^x2^x3^x4^x5^x6^x7;
}
// counted-walk prototype: per squarefree m in a smem list, est=rint(v*rm), 32-bit correction, u64 accumulate
struct Ent { double rm; uint32_t m; uint32_t pad; };
__global__ void k_counted(unsigned long long* out, int reps, uint64_t vbase) {
  __shared__ Ent L[2048];
  for (int i=threadIdx.x;i<2048;i+=blockDim.x){ uint32_t m=100000+i*3; L[i].rm=1.0/(double)m; L[i].m=m; }
  __syncthreads();
  uint64_t v = vbase + (uint64_t)(blockIdx.x*blockDim.x+threadIdx.x)*7919ull;
  double vd = __ull2double_rn(v); uint32_t vlo=(uint32_t)v;
  const double C = 4503599627370496.0; // 2^52
  unsigned long long acc=0; int corr=0;
  for (int r=0;r<reps;r++){
#pragma unroll 8
    for (int i=0;i<2048;i++){
      double e = fma(vd, L[i].rm, C);
      unsigned long long b = __double_as_longlong(e);
      int32_t t = (int32_t)(vlo - (uint32_t)b * L[i].m);
      acc += b; corr += (int)((uint32_t)t >> 31);
    }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc-corr;
}
// reference-style: hardware u64 division per item
__global__ void k_div(unsigned long long* out, int reps, uint64_t vbase) {
  __shared__ uint32_t L[2048];
  for (int i=threadIdx.x;i<2048;i+=blockDim.x){ L[i]=100000+i*3; }
  __syncthreads();
  uint64_t v = vbase + (uint64_t)(blockIdx.x*blockDim.x+threadIdx.x)*7919ull;
  unsigned long long acc=0;
  for (int r=0;r<reps;r++){
    for (int i=0;i<2048;i++){ acc += v / L[i]; }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc;
}
__global__ void k_atoms(uint32_t* out, int iters) {
  __shared__ uint32_t S[8192];
  for (int i=threadIdx.x;i<8192;i+=blockDim.x) S[i]=0;
  __syncthreads();
  uint32_t h = threadIdx.x*2654435761u + blockIdx.x;
  for (int i=0;i<iters;i++){
#pragma unroll 8
    for (int j=0;j<8;j++){ h = h*1664525u+1013904223u; atomicAdd(&S[h>>19], 1u<<((h&3)*8)); }
  }
  __syncthreads();
  out[blockIdx.x*blockDim.x+threadIdx.x]=S[threadIdx.x];
}
__global__ void k_ldsgather(uint32_t* out, int iters) {
  __shared__ uint32_t S[8192];
  for (int i=threadIdx.x;i<8192;i+=blockDim.x) S[i]=i*7;
  __syncthreads();
  uint32_t h = threadIdx.x*2654435761u + blockIdx.x; uint32_t acc=0;
  for (int i=0;i<iters;i++){
#pragma unroll 8
    for (int j=0;j<8;j++){ h = h*1664525u+1013904223u; acc += S[h>>19]; }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc;
}
// byte RMW by warp-owned subranges (non-atomic), stride-p marks
__global__ void k_bytemark(uint32_t* out, int iters) {
  __shared__ uint8_t S[32768];
  for (int i=threadIdx.x;i<32768;i+=blockDim.x) S[i]=0;
  __syncthreads();
  int w=threadIdx.x>>5, l=threadIdx.x&31;
  uint8_t* mine = S + w*1024;
  for (int it=0; it<iters; it++){
    for (int p=11; p<64; p+=2){ for (int j=l*p; j<1024; j+=32*p) mine[j]+= (uint8_t)p; }
  }
  __syncthreads();
  out[blockIdx.x*blockDim.x+threadIdx.x]=S[threadIdx.x*3];
}

int main(){
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,0));
  printf("dev %s sms %d clock %d kHz smemPerBlockOptin %zu\n", pr.name, pr.multiProcessorCount, pr.clockRate, pr.sharedMemPerBlockOptin);
  int sms=pr.multiProcessorCount;
  void* buf; CK(cudaMalloc(&buf, 64<<20));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  int th=512, bl=sms*4;
  double lanes=(double)th*bl;
  #define TIME(call, ops, name) { call; CK(cudaDeviceSynchronize()); cudaEventRecord(a); call; cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b); printf("%-12s %8.3f ms  %.3e ops/s  %.2f ops/clk/SM\n", name, ms, (ops)/(ms*1e-3), (ops)/(ms*1e-3)/sms/(pr.clockRate*1e3)); }
  int it=2000;
  TIME((k_imad<<<bl,th>>>((uint32_t*)buf,it,3u)), lanes*it*128, "imad");
  TIME((k_dfma<<<bl,th>>>((double*)buf,it,1.0000001)), lanes*it*128, "dfma");
  TIME((k_iadd<<<bl,th>>>((uint32_t*)buf,it,3u)), lanes*it*256, "xor+add");
  int reps=200;
  TIME((k_counted<<<bl,th>>>((unsigned long long*)buf,reps,4000000000000000000ull)), lanes*reps*2048.0, "counted");
  TIME((k_div<<<bl,th>>>((unsigned long long*)buf,10,4000000000000000000ull)), lanes*10*2048.0, "u64div");
  TIME((k_atoms<<<bl,1024>>>((uint32_t*)buf,500)), (double)bl*1024*500*8, "atoms");
  TIME((k_ldsgather<<<bl,1024>>>((uint32_t*)buf,500)), (double)bl*1024*500*8, "ldsgather");
  double marks=0; for(int p=11;p<64;p+=2) marks += 1024.0/p; marks*=32.0*bl*50;
  TIME((k_bytemark<<<bl,1024>>>((uint32_t*)buf,50)), marks, "bytemark");
  return 0;
}
