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

// Factor the 8x8 diagonal tile in place (one warp).  Returns false if a
// pivot is not positive.  invd[j] = 1 / L_jj.
__device__ __forceinline__ bool warp_chol8(double* t, double* invd) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
  for (int j = 0; j < 8; ++j) {
    const double d = t[eidx(j, j)];
    if (!(d > 0.0)) {
      ok = false;
      break;
    }
    const double l = sqrt(d);
    const double il = 1.0 / l;
    __syncwarp();
    if (lane > j && lane < 8) t[eidx(lane, j)] *= il;
    __syncwarp();
    for (int e = lane; e < 64; e += 32) {
      const int r = e >> 3, c = e & 7;
      if (c > j && c <= r) t[eidx(r, c)] -= t[eidx(r, j)] * t[eidx(c, j)];
    }
    __syncwarp();
    if (lane == 0) {
      t[eidx(j, j)] = l;
      invd[j] = il;
    }
    __syncwarp();
  }
  return ok;
}

// Left-looking tiled Cholesky + forward substitution of the RHS row.
// tl: tile storage, T: tiles per dimension, invd: 8*T scratch (1/L_ii),
// flag: shared int.  All threads of the CTA must call it.  Returns false
// (CTA-uniform) when the matrix is not SPD.
__device__ bool tiled_chol_fwd(double* tl, int T, double* invd, int* flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  if (threadIdx.x == 0) *flag = 0;
  __syncthreads();
  for (int kt = 0; kt < T; ++kt) {
    // (1) column kt: C(it,kt) -= sum_{jt<kt} L(it,jt) L(kt,jt)^T, it = kt..T
    for (int it = kt + warp; it <= T; it += nw) {
      double* ct = tl + tidx(it, kt) * 64;
      const int e0 = eidx(fr, 2 * fk), e1 = eidx(fr, 2 * fk + 1);
      double c0 = ct[e0], c1 = ct[e1];
      const double* ai = tl + tidx(it, 0) * 64;
      const double* bk = tl + tidx(kt, 0) * 64;
      for (int jt = 0; jt < kt; ++jt) {
        const double* a = ai + jt * 64;
        const double* b = bk + jt * 64;
        dmma_884(c0, c1, -a[eidx(fr, fk)], b[eidx(fr, fk)]);
        dmma_884(c0, c1, -a[eidx(fr, 4 + fk)], b[eidx(fr, 4 + fk)]);
      }
      ct[e0] = c0;
      ct[e1] = c1;
      if (it == kt) {
        __syncwarp();
        if (!warp_chol8(ct, invd + 8 * kt) && lane == 0) *flag = 1;
      }
    }
    __syncthreads();
    if (*flag) return false;
    // (2) TRSM: L(it,kt) = C(it,kt) L(kt,kt)^-T for it = kt+1..T; 4 tiles per
    // warp pass, one row per lane
    const double* lk = tl + tidx(kt, kt) * 64;
    const double* iv = invd + 8 * kt;
    const int ntile = T - kt;
    for (int base = warp * 4; base < ntile; base += nw * 4) {
      const int g = base + (lane >> 3);
      const int r = lane & 7;
      if (g < ntile) {
        double* ct = tl + tidx(kt + 1 + g, kt) * 64;
        double x[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          double v = ct[eidx(r, c)];
#pragma unroll
          for (int cc = 0; cc < c; ++cc) v -= x[cc] * lk[eidx(c, cc)];
          x[c] = v * iv[c];
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) ct[eidx(r, c)] = x[c];
      }
    }
    __syncthreads();
  }
  return true;
}

// Back substitution L^T z = y; y is row 0 of the RHS tiles, z (8T) written
// to `z`.  part: 8 * nwarps scratch.
__device__ void tiled_back_subst(const double* tl, int T, const double* invd, double* z,
                                 double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < 8 * T; i += blockDim.x)
    z[i] = tl[tidx(T, i >> 3) * 64 + eidx(0, i & 7)];
  __syncthreads();
  const int r = lane & 7, cg = lane >> 3;
  for (int it = T - 1; it >= 0; --it) {
    // partial sums of L(jt,it)^T z_jt over jt > it
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
      const double* t = tl + tidx(it, it) * 64;
      const double* iv = invd + 8 * it;
      // upper-triangular solve with L(it,it)^T, rows 7..0
      for (int rr = 7; rr >= 0; --rr) {
        const double xr = __shfl_sync(0xffffffffu, v, rr) * iv[rr];
        if (lane == rr) v = xr;
        if (lane < rr) v -= t[eidx(rr, lane)] * xr;
      }
      if (lane < 8) z[8 * it + lane] = v;
    }
    __syncthreads();
  }
}

}  // namespace gb
