// Latency of the register 8x8 Cholesky + inverse (one warp, no contention).
#include <cstdio>
#include "../../paper_1503_03467_b200/csrc/gb_common.cuh"
#include "../../paper_1503_03467_b200/csrc/gb_tiled_chol.cuh"
using namespace gb;
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double t[64], t0[64];
  const int lane = threadIdx.x;
  for (int e = lane; e < 64; e += 32) {
    const int r = e >> 3, c = e & 7;
    t0[eidx(r, c)] = (r == c) ? 10.0 + r : 1.0 / (1 + r + c);
  }
  __syncwarp();
  long long total = 0;
  for (int i = 0; i < n; ++i) {
    for (int e = lane; e < 64; e += 32) t[e] = t0[e];
    __syncwarp();
    long long a = clock64();
    warp_chol8_inv(t);
    long long b = clock64();
    total += b - a;
  }
  if (lane == 0) cyc[0] = total / n;
  for (int e = lane; e < 64; e += 32) out[e] = t[e];
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8);
  k<<<1, 32>>>(o, c, 100);
  k<<<1, 32>>>(o, c, 100);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("warp_chol8_inv: %lld cycles\n", h);
}
