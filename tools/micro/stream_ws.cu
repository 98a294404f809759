// Streaming pattern of the warp-specialized symmetric SpMV without compute:
// persistent CTAs, one producer warp issuing 1-D bulk copies of CH-pair
// chunks from NW contiguous blocks per tile into an NS-stage ring, NW consumer
// warps that only wait and release.  Measures the HBM rate of the pattern.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int NS, int NW, int CH>
__global__ void k(const double2* __restrict__ U, long long ntile, int nch, long long blkpairs, double* out) {
  extern __shared__ __align__(16) unsigned char dsm[];
  unsigned long long* full = (unsigned long long*)dsm;
  unsigned long long* empty = full + NS;
  double2* ring = (double2*)(dsm + 16 * NS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(full + s)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(empty + s)), "r"(NW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc = 0;
  if (warp == NW) {
    if (lane == 0) {
      long long g = 0;
      for (long long t = blockIdx.x; t < ntile; t += gridDim.x)
        for (int kk = 0; kk < nch; ++kk, ++g) {
          int st = g % NS; long long r = g / NS;
          if (r > 0) asm volatile("{.reg .pred P; W%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W%=;}" ::"r"(su(empty + st)), "r"((unsigned)((r - 1) & 1)) : "memory");
          unsigned bytes = CH * 32 * 16;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(full + st)), "r"(bytes * NW) : "memory");
          for (int cw = 0; cw < NW; ++cw) {
            const double2* src = U + (t * NW + cw) * blkpairs * 32 + (long long)kk * CH * 32;
            double2* dst = ring + ((long long)st * NW + cw) * CH * 32;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst)), "l"(src), "r"(bytes), "r"(su(full + st)) : "memory");
          }
        }
    }
  } else {
    long long g = 0;
    for (long long t = blockIdx.x; t < ntile; t += gridDim.x)
      for (int kk = 0; kk < nch; ++kk, ++g) {
        int st = g % NS;
        asm volatile("{.reg .pred P; W%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W%=;}" ::"r"(su(full + st)), "r"((unsigned)((g / NS) & 1)) : "memory");
        acc += ring[((long long)st * NW + warp) * CH * 32 + lane].x;
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(empty + st)) : "memory");
      }
  }
  if (acc == 1.234) out[0] = acc;
}
template <int NS, int NW, int CH>
void run(const double2* U, long long total_pairs, double* o, const char* name) {
  const int nch = 20;  // chunks per block
  const long long blkpairs = (long long)nch * CH;
  const long long ntile = total_pairs / (blkpairs * 32 * NW);
  size_t sm = 16 * NS + (size_t)NS * NW * CH * 32 * 16;
  cudaFuncSetAttribute(k<NS, NW, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k<NS, NW, CH><<<148, 32 * (NW + 1), sm>>>(U, ntile, nch, blkpairs, o);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<NS, NW, CH><<<148, 32 * (NW + 1), sm>>>(U, ntile, nch, blkpairs, o);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double bytes = (double)ntile * NW * blkpairs * 32 * 16;
  printf("%s: %.1f us, %.0f GB/s (err %s)\n", name, ms * 200, bytes / (ms / 5 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const long long bytes = 782LL << 20;
  double2* U; double* o; cudaMalloc(&U, bytes); cudaMalloc(&o, 8); cudaMemset(U, 0, bytes);
  const long long tp = bytes / 16;
  run<4, 8, 9>(U, tp, o, "NS4 NW8 CH9 (current)");
  run<2, 8, 9>(U, tp, o, "NS2 NW8 CH9");
  run<3, 8, 18>(U, tp, o, "NS3 NW8 CH18");
  run<6, 8, 9>(U, tp, o, "NS6 NW8 CH9");
  run<4, 4, 18>(U, tp, o, "NS4 NW4 CH18");
  run<8, 4, 9>(U, tp, o, "NS8 NW4 CH9");
}
