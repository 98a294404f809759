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

// Left-looking tiled Cholesky + forward substitution of the RHS row, with a
// one-column lookahead.  Invariant at the start of step kt: every tile
// (it, kt), it >= kt, already holds the contributions of columns < kt-1.
// Step kt: warp 0 adds column kt-1 to the diagonal tile and factors it
// (L_kk^-1 over the tile); meanwhile warps 1.. finish the rest of column kt
// (one DMMA pair per tile) and pre-accumulate column kt+1 from columns
// 0..kt-1 (the bulk of the flops, two independent accumulator chains per
// tile).  Then all warps apply the TRSM L(it,kt) = C(it,kt) L_kk^-T (two
// DMMAs with L_kk^-1).  The serial chain per step is one DMMA pair, the
// 8x8 factor and the TRSM.  tl: tile storage (diagonal tiles end up
// holding L_kk^-1), T: tiles per dimension, flag: shared int.  Returns false
// (CTA-uniform) when the matrix is not SPD.
#ifdef GB_PATCH_PROF
__device__ unsigned long long g_fprof[8];
#endif
__device__ bool tiled_chol_fwd(double* tl, int T, double* scratch, int* flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int e0 = eidx(fr, 2 * fk), e1 = eidx(fr, 2 * fk + 1);
  const int ea = eidx(fr, fk), eb = eidx(fr, 4 + fk);
  if (threadIdx.x == 0) *flag = 0;
  __syncthreads();
  for (int kt = 0; kt < T; ++kt) {
#ifdef GB_PATCH_PROF
    long long q0 = clock64();
#endif
    const double* lk1 = tl + tidx(kt, 0) * 64 + (kt - 1) * 64;  // L(kt, kt-1)
    if (warp == 0) {
      double* ct = tl + tidx(kt, kt) * 64;
      if (kt > 0) {
        double c0 = ct[e0], c1 = ct[e1];
        dmma_884(c0, c1, -lk1[ea], lk1[ea]);
        dmma_884(c0, c1, -lk1[eb], lk1[eb]);
        ct[e0] = c0;
        ct[e1] = c1;
        __syncwarp();
      }
      if (!warp_chol8_inv(ct, scratch) && lane == 0) *flag = 1;
    } else {
      if (kt > 0) {  // finish column kt: C(it,kt) -= L(it,kt-1) L(kt,kt-1)^T
        const double b0 = lk1[ea], b1 = lk1[eb];
        for (int it = kt + warp; it <= T; it += nw - 1) {
          double* ct = tl + tidx(it, kt) * 64;
          const double* a = tl + tidx(it, kt - 1) * 64;
          double c0 = ct[e0], c1 = ct[e1];
          dmma_884(c0, c1, -a[ea], b0);
          dmma_884(c0, c1, -a[eb], b1);
          ct[e0] = c0;
          ct[e1] = c1;
        }
      }
      if (kt + 1 < T) {  // pre-accumulate column kt+1 from columns 0..kt-1
        const double* bk = tl + tidx(kt + 1, 0) * 64;
        for (int it = kt + warp; it <= T; it += nw - 1) {
          double* ct = tl + tidx(it, kt + 1) * 64;
          const double* ai = tl + tidx(it, 0) * 64;
          double c0 = ct[e0], c1 = ct[e1], d0 = 0.0, d1 = 0.0;
          int jt = 0;
          for (; jt + 1 < kt; jt += 2) {
            const double* a = ai + jt * 64;
            const double* b = bk + jt * 64;
            dmma_884(c0, c1, -a[ea], b[ea]);
            dmma_884(d0, d1, -a[64 + ea], b[64 + ea]);
            dmma_884(c0, c1, -a[eb], b[eb]);
            dmma_884(d0, d1, -a[64 + eb], b[64 + eb]);
          }
          if (jt < kt) {
            const double* a = ai + jt * 64;
            const double* b = bk + jt * 64;
            dmma_884(c0, c1, -a[ea], b[ea]);
            dmma_884(c0, c1, -a[eb], b[eb]);
          }
          ct[e0] = c0 + d0;
          ct[e1] = c1 + d1;
        }
      }
    }
#ifdef GB_PATCH_PROF
    if (blockIdx.x == 0 && lane == 0 && warp < 3) atomicAdd(&g_fprof[warp], clock64() - q0);
#endif
    __syncthreads();
#ifdef GB_PATCH_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_fprof[3], clock64() - q0);
    long long q1 = clock64();
#endif
    if (*flag) return false;
    // TRSM: L(it,kt) = C(it,kt) L_kk^-T as a product with Linv^T (DMMA)
    {
      const double* li = tl + tidx(kt, kt) * 64;  // L_kk^-1
      const double bl0 = li[ea], bl1 = li[eb];
      for (int it = kt + 1 + warp; it <= T; it += nw) {
        double* ct = tl + tidx(it, kt) * 64;
        const double a0 = ct[ea], a1 = ct[eb];
        double d0 = 0.0, d1 = 0.0;
        dmma_884(d0, d1, a0, bl0);
        dmma_884(d0, d1, a1, bl1);
        __syncwarp();
        ct[e0] = d0;
        ct[e1] = d1;
      }
    }
    __syncthreads();
#ifdef GB_PATCH_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_fprof[4], clock64() - q1);
#endif
  }
  return true;
}

// Back substitution L^T z = y with the L_kk^-1 held in the diagonal tiles;
// y is row 0 of the RHS tiles, z (8T) written to `z`.  One warp, no CTA
// barriers: step it, the 4 lane groups of 8 split the tiles jt > it and
// accumulate column r of L(jt,it) . z_jt, then z_it = L_kk^-T (y_it - acc).
// Called by all threads; returns after a __syncthreads with z complete.
__device__ void tiled_back_subst(const double* tl, int T, double* z, double* /*part*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    for (int i = lane; i < 8 * T; i += 32) z[i] = tl[tidx(T, i >> 3) * 64 + eidx(0, i & 7)];
    __syncwarp();
    const int r = lane & 7, cg = lane >> 3;
    for (int it = T - 1; it >= 0; --it) {
      double acc = 0.0;
      for (int jt = it + 1 + cg; jt < T; jt += 4) {
        const double* t = tl + tidx(jt, it) * 64;
        const double* zj = z + 8 * jt;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = fma(t[eidx(k, r)], zj[k], acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 8);
      acc += __shfl_xor_sync(0xffffffffu, acc, 16);
      const double v = z[8 * it + r] - acc;
      // z_it = L_kk^-T v: z[r] = sum_{c >= r} Linv[c][r] v[c]
      const double* li = tl + tidx(it, it) * 64;
      double zr = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double vc = __shfl_sync(0xffffffffu, v, c);
        if (c >= r) zr = fma(li[eidx(c, r)], vc, zr);
      }
      __syncwarp();
      if (lane < 8) z[8 * it + lane] = zr;
      __syncwarp();
    }
  }
  __syncthreads();
}

}  // namespace gb
