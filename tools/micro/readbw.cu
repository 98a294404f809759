// Achievable HBM read bandwidth: grid-stride double2 streaming reduction over
// a 782 MB buffer (the size of the finest-level symmetric S B S at q=10).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ a, long long n, double* out) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double2 v = __ldg(a + i);
    s += v.x + v.y;
  }
  if (s == 1.2345) out[0] = s;
}
__global__ void rd4(const double2* __restrict__ a, long long n, double* out) {
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double2 v0 = __ldg(a + i), v1 = __ldg(a + i + stride), v2 = __ldg(a + i + 2 * stride),
            v3 = __ldg(a + i + 3 * stride);
    s += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
  }
  for (; i < n; i += stride) { double2 v = __ldg(a + i); s += v.x + v.y; }
  if (s == 1.2345) out[0] = s;
}
int main() {
  const long long bytes = 782LL << 20;
  const long long n = bytes / 16;
  double2* a; double* o;
  cudaMalloc(&a, bytes); cudaMalloc(&o, 8);
  cudaMemset(a, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grids[] = {148 * 4, 148 * 8, 148 * 16, 148 * 32};
  for (int kind = 0; kind < 2; ++kind)
    for (int g : grids) {
      for (int w = 0; w < 3; ++w) kind ? rd4<<<g, 256>>>(a, n, o) : rd<<<g, 256>>>(a, n, o);
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) kind ? rd4<<<g, 256>>>(a, n, o) : rd<<<g, 256>>>(a, n, o);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%s grid %d: %.1f us, %.0f GB/s\n", kind ? "rd4" : "rd", g, ms * 100, bytes / (ms / 10 * 1e-3) / 1e9);
    }
}
