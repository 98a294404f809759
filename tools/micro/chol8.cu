// Latency of the register 8x8 Cholesky + inverse (one warp, no contention).
#include <cstdio>
#ifndef OLD
#define OLD 0
#endif
#include "../../paper_1503_03467_b200/csrc/gb_common.cuh"
#include "../../paper_1503_03467_b200/csrc/gb_tiled_chol.cuh"
namespace gb {
__device__ __forceinline__ bool warp_chol8_inv_old(double* t, double* scratch) {
  const int lane = threadIdx.x & 31;
  const int r = lane & 7;
  double v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = (c <= r) ? t[eidx(r, c)] : 0.0;
  double il_r = 0.0;  // 1 / L_rr, kept by lane r
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double d = __shfl_sync(0xffffffffu, v[j], j);
    ok = ok && (d > 0.0);
    const double il = rsqrt(d);
    if (r > j) v[j] *= il;
    if (r == j) {
      v[j] = d * il;
      il_r = il;
    }
#pragma unroll
    for (int c = j + 1; c < 8; ++c) {
      const double lcj = __shfl_sync(0xffffffffu, v[j], c);
      if (r > j && c <= r) v[c] = fma(-v[j], lcj, v[c]);
    }
  }
  if (!ok) return false;
  if (lane < 8) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c <= r) t[eidx(r, c)] = v[c];
    scratch[r] = il_r;  // diagonal of L^-1, read back below
  }
  __syncwarp();
  // L^-1, column r by lane r: x_i = -(sum_{r<=k<i} L_ik x_k) / L_ii, x_r = 1/L_rr
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) acc = fma(t[eidx(i, k)], x[k], acc);
    const double ii = scratch[i];
    x[i] = (i > r) ? -acc * ii : ((i == r) ? ii : 0.0);
  }
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) t[eidx(i, r)] = x[i];  // column r of L^-1 (upper = 0)
  }
  __syncwarp();
  return true;
}


}
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
    if (OLD) warp_chol8_inv_old(t, t0 + 0); else warp_chol8_inv(t);
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
