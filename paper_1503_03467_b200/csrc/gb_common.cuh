// Shared device helpers for the gamblet B200 kernels.
//
// Data layout ("box stencil"): every level operator of the localized gamblet
// transform is a bounded box stencil on a 2-D index grid.
// A square box matrix on an L x L grid with `nr` components per grid point and
// half-width `w` stores, for row r = (s*L + t)*nr + c, the values of columns
// (s+ds, t+dt, c') for |ds|,|dt| <= w, c' < nc, row-major:
//
//     val[r * S + ((ds+w)*(2w+1) + (dt+w))*nc + c'],   S = (2w+1)^2 * nc.
//
// Out-of-domain, dropped and exactly-zero entries are stored as 0.0; the CSR
// export keeps exactly the entries != 0, which is the reference's as_csr
// semantics (sparse_core.py:47-67: explicit zeros eliminated).
//
// psi^(k) rows (fine-grid support that grows per level) use an
// origin-clamped square window of width `wd` per dimension:
// row i of level k has corner c = (s*h, t*h), h = 2^(q-k), window origin
// o = clamp(c + lo, 0, n - wd) per dimension, value at fine node (fs, ft) is
// val[i * wd*wd + (fs-o_s)*wd + (ft-o_t)].
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gb {

// status words (int64) in the device status block
enum : long long {
  ST_OK = 0,
  ST_NONPOS_DIAG = 1,   // detail = row
  ST_NOT_SPD = 2,       // detail = patch id
  ST_OUTSIDE_BOX = 3,   // detail = row (input CSR entry outside the box)
  ST_CG_BREAKDOWN = 4,  // detail = iteration
};

__device__ __forceinline__ void raise_status(long long* st, long long code,
                                             long long detail) {
  if (atomicCAS(reinterpret_cast<unsigned long long*>(st), 0ull,
                static_cast<unsigned long long>(code)) == 0ull) {
    st[1] = detail;
  }
}

// max of non-negative doubles through their (order-preserving) bit patterns
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

__host__ __device__ __forceinline__ int box_side(int w) { return 2 * w + 1; }
__host__ __device__ __forceinline__ int box_slots(int w, int nc) {
  return (2 * w + 1) * (2 * w + 1) * nc;
}
__host__ __device__ __forceinline__ int slot_of(int w, int nc, int ds, int dt,
                                                int c) {
  return ((ds + w) * (2 * w + 1) + (dt + w)) * nc + c;
}
__host__ __device__ __forceinline__ int clampi(int x, int lo, int hi) {
  return x < lo ? lo : (x > hi ? hi : x);
}
__host__ __device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// block-wide sum with a fixed reduction tree (deterministic); all threads get
// the result.  `sh` needs blockDim/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}
__device__ __forceinline__ double block_max(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < nw ? sh[lane] : 0.0;
    t = warp_max(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}

// orthonormal / chain null-basis templates arrive as 12 doubles (3 rows x 4
// children, hierarchy.py:31-42); passed by value in kernel parameters.
struct WTemplate {
  double w[3][4];
};

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default
// memory pool, whose release threshold is zero unless told otherwise: every
// synchronize hands the pool's memory back to the driver and the next
// allocation maps it again -- on this pool's microVM hosts that remap stalls
// for tens to hundreds of milliseconds now and then.  Keep the pool's memory.
inline void keep_default_pool() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

}  // namespace gb
