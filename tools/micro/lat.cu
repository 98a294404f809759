// Latency microbenchmarks (one warp, dependent chains) for the patch solver
// design: DMMA m8n8k4 f64, DFMA, rsqrt(double), __syncthreads (8 warps),
// LDS.64.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat.cu -o lat
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k(long long* out, double* sink, int n) {
  __shared__ double sm[1024];
  __shared__ long long t[8];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double a = 1.0 + lane * 1e-7, b = 0.999, c0 = 0, c1 = 0;
  long long t0, t1;
  // DMMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(c0, c1, a, b);
  t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
  // 4 independent DMMA chains
  double e0 = 0, e1 = 0, f0 = 0, f1 = 0, g0 = 0, g1 = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { dmma(c0, c1, a, b); dmma(e0, e1, a, b); dmma(f0, f1, a, b); dmma(g0, g1, a, b); }
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / n;
  // DFMA chain
  double x = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, 1e-3);
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / n;
  // rsqrt chain
  double r = 2.0 + a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) r = rsqrt(r) + 1.5;
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / n;
  // LDS chain (pointer chase on index)
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = ((int)sm[idx & 1023]) + (idx & 7);
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / n;
  // syncthreads
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / n;
  // shfl chain
  double sv = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) sv = __shfl_sync(0xffffffffu, sv, (lane + 1) & 31) + 1e-9;
  t1 = clock64();
  if (threadIdx.x == 0) out[6] = (t1 - t0) / n;
  // sqrt chain
  double q = 2.0 + a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) q = sqrt(q) + 1.5;
  t1 = clock64();
  if (threadIdx.x == 0) out[7] = (t1 - t0) / n;
  sink[threadIdx.x] = c0 + c1 + e0 + e1 + f0 + f1 + g0 + g1 + x + r + idx + sv + q;
}
int main() {
  long long* o; double* s;
  cudaMalloc(&o, 64 * 8); cudaMalloc(&s, 1024 * 8);
  k<<<1, 256>>>(o, s, 1000);
  k<<<1, 256>>>(o, s, 1000);
  long long h[8];
  cudaMemcpy(h, o, 64, cudaMemcpyDeviceToHost);
  printf("cycles: dmma_chain %lld  dmma_4chains %lld  dfma %lld  rsqrt %lld  lds %lld  syncthreads(8w) %lld  shfl %lld  sqrt %lld\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
}
