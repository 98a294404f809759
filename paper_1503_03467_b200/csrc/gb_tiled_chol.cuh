// Tiled SPD patch solver for one CTA: left-looking Cholesky on 8x8 FP64
// tiles with the DMMA tensor-core op (mma.sync.m8n8k4.f64), shared-memory
// resident, right-hand side folded in as an extra tile row so the forward
// substitution happens inside the factorization.
//
// Storage ("tile-packed lower"): tile (it, jt), jt <= it < T, lives at tile
// index it(it+1)/2 + jt; the RHS row is tile row T (tiles (T, jt), only row 0
// used).  Within a tile, element (r, c) sits at r*8 + (c ^ ((r & 2) << 1)):
// the XOR swizzle makes the DMMA fragment loads (row = lane>>2, col = k0 +
// (lane&3)) bank-conflict free per half warp.
#pragma once
#include "gb_common.cuh"

namespace gb {

__device__ __forceinline__ int tidx(int it, int jt) { return ((it * (it + 1)) >> 1) + jt; }
__device__ __forceinline__ int eidx(int r, int c) { return (r << 3) + (c ^ ((r & 2) << 1)); }

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Factor the 8x8 diagonal tile (one warp, rows in lanes 0..7, registers and
// shuffles), form L^-1 and store it OVER the tile: diagonal L tiles are never
// DMMA operands, every later use (TRSM, back substitution) needs L_kk^-1.
// `scratch` holds 8 doubles.  Returns false if a pivot is not positive.
__device__ __forceinline__ bool warp_chol8_inv(double* t, double* scratch) {
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

// Left-looking tiled Cholesky + forward substitution of the RHS row.
// tl: tile storage (diagonal tiles end up holding L_kk^-1), T: tiles per
// dimension, scratch: 8 doubles, flag: shared int.  Warp 0 owns the diagonal tile of every step;
// warps 1.. own the off-diagonal tiles (round robin), keep them in registers
// across the update and the TRSM (two DMMAs with L_kk^-T).  Returns false
// (CTA-uniform) when the matrix is not SPD.
__device__ bool tiled_chol_fwd(double* tl, int T, double* scratch, int* flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int e0 = eidx(fr, 2 * fk), e1 = eidx(fr, 2 * fk + 1);
  if (threadIdx.x == 0) *flag = 0;
  __syncthreads();
  for (int kt = 0; kt < T; ++kt) {
    const double* bk = tl + tidx(kt, 0) * 64;
    // (1) updates: C(it,kt) -= sum_{jt<kt} L(it,jt) L(kt,jt)^T
    if (warp == 0) {
      double* ct = tl + tidx(kt, kt) * 64;
      double c0 = ct[e0], c1 = ct[e1];
      for (int jt = 0; jt < kt; ++jt) {
        const double* b = bk + jt * 64;
        dmma_884(c0, c1, -b[eidx(fr, fk)], b[eidx(fr, fk)]);
        dmma_884(c0, c1, -b[eidx(fr, 4 + fk)], b[eidx(fr, 4 + fk)]);
      }
      ct[e0] = c0;
      ct[e1] = c1;
      __syncwarp();
      if (!warp_chol8_inv(ct, scratch) && lane == 0) *flag = 1;
    } else {
      for (int it = kt + warp; it <= T; it += nw - 1) {
        double* ct = tl + tidx(it, kt) * 64;
        double c0 = ct[e0], c1 = ct[e1];
        const double* ai = tl + tidx(it, 0) * 64;
        for (int jt = 0; jt < kt; ++jt) {
          const double* a = ai + jt * 64;
          const double* b = bk + jt * 64;
          dmma_884(c0, c1, -a[eidx(fr, fk)], b[eidx(fr, fk)]);
          dmma_884(c0, c1, -a[eidx(fr, 4 + fk)], b[eidx(fr, 4 + fk)]);
        }
        ct[e0] = c0;
        ct[e1] = c1;
      }
    }
    __syncthreads();
    if (*flag) return false;
    // (2) TRSM: L(it,kt) = C(it,kt) L_kk^-T as a product with Linv^T (DMMA)
    if (warp != 0) {
      const double* li = tl + tidx(kt, kt) * 64;  // L_kk^-1
      const double bl0 = li[eidx(fr, fk)], bl1 = li[eidx(fr, 4 + fk)];
      for (int it = kt + warp; it <= T; it += nw - 1) {
        double* ct = tl + tidx(it, kt) * 64;
        const double a0 = ct[eidx(fr, fk)], a1 = ct[eidx(fr, 4 + fk)];
        double d0 = 0.0, d1 = 0.0;
        dmma_884(d0, d1, a0, bl0);
        dmma_884(d0, d1, a1, bl1);
        __syncwarp();
        ct[e0] = d0;
        ct[e1] = d1;
      }
    }
    __syncthreads();
  }
  return true;
}

// Back substitution L^T z = y with the L_kk^-1 held in the diagonal tiles;
// y is row 0 of the RHS tiles, z (8T) written to `z`.  part: 8 * nwarps.
__device__ void tiled_back_subst(const double* tl, int T, double* z, double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < 8 * T; i += blockDim.x)
    z[i] = tl[tidx(T, i >> 3) * 64 + eidx(0, i & 7)];
  __syncthreads();
  const int r = lane & 7, cg = lane >> 3;
  for (int it = T - 1; it >= 0; --it) {
    double acc = 0.0;
    for (int jt = it + 1 + warp; jt < T; jt += nw) {
      const double* t = tl + tidx(jt, it) * 64;
      const double* zj = z + 8 * jt;
      acc += t[eidx(2 * cg, r)] * zj[2 * cg] + t[eidx(2 * cg + 1, r)] * zj[2 * cg + 1];
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 8);
    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
    if (lane < 8) part[warp * 8 + lane] = acc;
    __syncthreads();
    if (warp == 0) {
      double v = 0.0;
      if (lane < 8) {
        v = z[8 * it + lane];
        for (int w = 0; w < nw; ++w) v -= part[w * 8 + lane];
      }
      // z_it = L_kk^-T v: z[r] = sum_{c >= r} Linv[c][r] v[c]
      const double* li = tl + tidx(it, it) * 64;
      double zr = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double vc = __shfl_sync(0xffffffffu, v, c);
        if (c >= r) zr += li[eidx(c, r)] * vc;
      }
      if (lane < 8) z[8 * it + lane] = zr;
    }
    __syncthreads();
  }
}

}  // namespace gb
