// Correction patches, v3: left-looking tiled Cholesky with the finished L
// columns streamed through an L2-resident global scratch instead of held in
// shared memory (gamblet_fast.py:546-580; same arithmetic family as v2:
// 8x8 FP64 tiles, DMMA m8n8k4 updates, L_kk^-1 on the diagonal, the RHS
// folded in as tile row T).
//
// Why: v2 keeps the whole packed lower factor (~107 KB at m = 147) in shared
// memory, so only 2 patches fit per SM and the per-step serial chain (8x8
// diagonal factor + TRSM + barriers) leaves the SM idle most of the time
// (ncu: IPC 1.4, 13 % of the FP64 peak).  Here a CTA holds only the current
// tile column and the L row it needs (~24 KB): 6+ patches per SM overlap
// their serial chains.  Step kt gathers column kt of (S B S)[chi, chi] from
// the box, subtracts sum_jt L(it, jt) L(kt, jt)^T (A fragments streamed from
// the scratch, B fragments from the staged L row), factors the diagonal tile
// and writes L(it, kt) = C(it, kt) L_kk^-T back.  The scratch of a CTA is
// ~107 KB; all CTAs together stay inside the 126 MB L2.
//
// Scratch tile layout ("fragment order"): element (r, c) of an 8x8 tile at
// (c >> 2) * 32 + r * 4 + (c & 3), so the DMMA A / B fragment of k-chunk ch
// (row lane >> 2, column 4 ch + (lane & 3)) is the contiguous 256 B run
// ch * 32 + lane.  Diagonal tiles hold L_kk^-1.  Tile (it, jt) of the packed
// lower factor (RHS row it = T included) is at index it (it + 1) / 2 + jt.
#pragma once

namespace gb {

__device__ __forceinline__ int fpos(int r, int c) { return ((c >> 2) << 5) + (r << 2) + (c & 3); }

#ifndef GB_V3_MINB
#define GB_V3_MINB 6
#endif
constexpr int kV3Warps = 4;

struct V3Smem {
  double* col;   // 2 x (Tmax + 1) tiles, row-major 8x8: C(it, kt), it = kt..T
  double* lrow;  // Tmax tiles, fragment order: L(kt, jt), jt < kt
  double* dg;    // 64: diagonal tile, swizzled (warp_chol8_inv layout)
  double* sl;    // 8 Tmax + 8 (scale; 8 scratch doubles after it)
  double* z;     // 8 Tmax
  long long* rowb;  // 8 Tmax: (B offset of local row l minus its key) << 16 | a << 8 | b
  int* colk;     // 8 Tmax: key of local column l
  int* flag;
};

__host__ __device__ __forceinline__ size_t v3_smem_bytes(int Tmax) {
  return ((size_t)2 * (Tmax + 1) * 64 + (size_t)Tmax * 64 + 64 + (8 * Tmax + 8) + 8 * Tmax +
          8 * Tmax) * 8 + (size_t)8 * Tmax * 4 + 16;
}

__device__ __forceinline__ V3Smem v3_carve(double* sm, int Tmax) {
  V3Smem s;
  s.col = sm;  // two column buffers (ping-pong)
  s.lrow = s.col + 2 * (Tmax + 1) * 64;
  s.dg = s.lrow + Tmax * 64;
  s.sl = s.dg + 64;
  s.z = s.sl + 8 * Tmax + 8;
  s.rowb = reinterpret_cast<long long*>(s.z + 8 * Tmax);
  int* ip = reinterpret_cast<int*>(s.rowb + 8 * Tmax);
  s.colk = ip;
  s.flag = s.colk + 8 * Tmax;
  return s;
}

// gather column kt of (S B S)[chi, chi] (tiles (it, kt), it = kt..T-1, rows
// l1 = 8 kt .. 8 T - 1, row-major) and the RHS tile (T, kt) into `col`, by
// threads tl = 0..nt-1 (nt a multiple of 8): thread tl owns column c = tl & 7
// and rows l1 = 8 kt + (tl >> 3) + (nt / 8) j; entries are the reference's
// congruence (B s_i) s_j (gamblet_fast.py:136)
// 16-byte global -> shared copies (LDGSTS, L2 only); completion via v3_cp_wait
__device__ __forceinline__ void v3_cp16(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void v3_cp_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// 8-byte global -> shared copy (LDGSTS through L1); completion via v3_cp_wait
__device__ __forceinline__ void v3_cp8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}

// gather column kt of B[chi, chi] (tiles (it, kt), it = kt..T-1, rows
// l1 = 8 kt .. 8 T - 1, row-major) and the RHS tile (T, kt) into `col`, by
// threads tl = 0..nt-1 (nt a multiple of 8): thread tl owns column c = tl & 7
// and rows l1 = 8 kt + (tl >> 3) + (nt / 8) j.  Box entries are copied raw
// and asynchronously (cp.async; the caller waits before its barrier); the
// reference's congruence (B s_i) s_j (gamblet_fast.py:136) is applied when
// the update phase first reads the column (v3 step (3)); padding rows hold
// the unit diagonal and S.sl = 1 there.  One table word per row carries the
// row's box offset and its parent coordinates (the band test).
__device__ __forceinline__ void v3_gather(const V3Smem& S, double* col, int kt, int T, int m,
                                          int wB, const double* __restrict__ B, int tl, int nt) {
  const int c = tl & 7;
  const int l2 = 8 * kt + c;
  const int step = nt >> 3;
  int l1 = 8 * kt + (tl >> 3);
  double* dst = col + (tl >> 3) * 8 + c;
  if (l2 < m) {
    const int p2 = (int)S.rowb[l2];
    const int a2 = ((p2 >> 8) & 255) + wB, b2 = (p2 & 255) + wB;
    const unsigned w2 = 2 * wB;
    const double* Bc = B + S.colk[l2];
#pragma unroll 4
    for (; l1 < m; l1 += step, dst += step * 8) {
      const long long info = S.rowb[l1];
      const int lo = (int)info;
      if ((unsigned)(a2 - ((lo >> 8) & 255)) <= w2 && (unsigned)(b2 - (lo & 255)) <= w2)
        v3_cp8(dst, Bc + (info >> 16));
      else
        *dst = 0.0;
    }
    for (; l1 < 8 * T; l1 += step, dst += step * 8) *dst = 0.0;  // padding rows
  } else {  // padding column: unit diagonal
    for (; l1 < 8 * T; l1 += step, dst += step * 8) *dst = (l1 == l2) ? 1.0 : 0.0;
  }
  for (int r = tl >> 3; r < 8; r += step) col[(T - kt) * 64 + r * 8 + c] = (r == 0) ? S.z[l2] : 0.0;
}

__global__ void __launch_bounds__(32 * kV3Warps, GB_V3_MINB) k_correction_patches_v3(
    int Lp, int wB, const double* __restrict__ B, const double* __restrict__ sB, int wG,
    const double* __restrict__ G, int rho, double* __restrict__ Dt, long long* status, int Tmax,
    double* __restrict__ scratch, long long p0, long long p1) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  V3Smem S = v3_carve(sm, Tmax);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int SB = box_slots(wB, 3), SG = box_slots(wG, 1), SD = box_slots(rho, 3);
  double* L = scratch + (long long)blockIdx.x * ((Tmax * (Tmax + 1)) / 2 + Tmax) * 64;
  const int fr = lane >> 2, fk = lane & 3;
  // patches [p0, p1) (parent order; a row strip of the parent grid)
  for (long long i = p0 + blockIdx.x; i < p1; i += gridDim.x) {
    const int si = (int)(i / Lp), ti = (int)(i % Lp);
    const int s0 = imax(0, si - rho), s1 = imin(Lp - 1, si + rho);
    const int t0 = imax(0, ti - rho), t1 = imin(Lp - 1, ti + rho);
    const int nbt = t1 - t0 + 1;
    const int m = 3 * (s1 - s0 + 1) * nbt;
    const int T = (m + 7) >> 3;
    // local tables and the right-hand side s * (-G[:, i])
    double nrm = 0.0;
    for (int l = threadIdx.x; l < 8 * T; l += blockDim.x) {
      double v = 0.0;
      if (l < m) {
        const int pl = l / 3, c = l - 3 * pl;
        const int a = pl / nbt, b = pl - a * nbt;
        const long long r = ((long long)(s0 + a) * Lp + (t0 + b)) * 3 + c;
        // slot_of(wB, 3, a2 - a1, b2 - b1, c2) = key(l2) - 3 (a1 W2 + b1) + K
        const int key = (a * (2 * wB + 1) + b) * 3;
        S.rowb[l] = ((r * SB - key + (wB * (2 * wB + 1) + wB) * 3) << 16) | (a << 8) | b;
        S.colk[l] = key + c;
        S.sl[l] = sB[r];
        const int ds = si - (s0 + a), dt = ti - (t0 + b);
        double g = 0.0;
        if (ds >= -wG && ds <= wG && dt >= -wG && dt <= wG)
          g = G[r * SG + slot_of(wG, 1, ds, dt, 0)];
        v = sB[r] * (-g);
      }
      else {
        S.sl[l] = 1.0;  // padding rows: the deferred scaling leaves them as gathered
      }
      S.z[l] = v;
      nrm += v * v;
    }
    nrm = block_sum(nrm, red);  // also orders the table writes
    double* drow = Dt + i * SD;
    if (nrm == 0.0) {  // gamblet_fast.py:561-562: empty correction column
      for (int e = threadIdx.x; e < SD; e += blockDim.x) drow[e] = 0.0;
      __syncthreads();
      continue;
    }
    if (threadIdx.x == 0) *S.flag = 0;
    bool ok = true;
    const int colstride = (Tmax + 1) * 64;
    v3_gather(S, S.col, 0, T, m, wB, B, threadIdx.x, blockDim.x);
    v3_cp_wait();
    __syncthreads();
    // step kt: [update column kt] | [warp 0: factor the diagonal tile;
    // warps 1..: gather column kt + 1, stage L(kt + 1, 0..kt-1)] | [TRSM]
    for (int kt = 0; kt < T; ++kt) {
      double* cur = S.col + (kt & 1) * colstride;
      double* nxt = S.col + ((kt + 1) & 1) * colstride;
      // (3) C(it, kt) -= sum_jt L(it, jt) L(kt, jt)^T, a warp per tile row
      // (the gathered column is scaled here: C = (B s_l1) s_l2, RHS row unscaled)
      {
        const double sc0 = S.sl[8 * kt + ((2 * lane) & 7)], sc1 = S.sl[8 * kt + ((2 * lane) & 7) + 1];
        // two tile rows per warp iteration: 4 independent accumulator chains
        for (int it = kt + warp; it <= T; it += 2 * kV3Warps) {
          const int it2 = it + kV3Warps;
          const bool two = it2 <= T;
          double* ct = cur + (it - kt) * 64;
          double* ct2 = cur + ((two ? it2 : it) - kt) * 64;
          double c0 = ct[2 * lane], c1 = ct[2 * lane + 1];
          double g0 = two ? ct2[2 * lane] : 0.0, g1 = two ? ct2[2 * lane + 1] : 0.0;
          if (it < T) {
            const double sr = S.sl[8 * it + (lane >> 2)];
            c0 = c0 * sr * sc0;
            c1 = c1 * sr * sc1;
          }
          if (two && it2 < T) {
            const double sr = S.sl[8 * it2 + (lane >> 2)];
            g0 = g0 * sr * sc0;
            g1 = g1 * sr * sc1;
          }
          double d0 = 0.0, d1 = 0.0, h0 = 0.0, h1 = 0.0;
          const double* ai = L + (long long)((it * (it + 1)) >> 1) * 64;
          const double* ai2 = L + (long long)(((two ? it2 : it) * ((two ? it2 : it) + 1)) >> 1) * 64;
          int jt = 0;
          for (; jt + 1 < kt; jt += 2) {
            double a[4], q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = __ldcg(ai + jt * 64 + 32 * u + lane);
#pragma unroll
            for (int u = 0; u < 4; ++u) q[u] = two ? __ldcg(ai2 + jt * 64 + 32 * u + lane) : 0.0;
            const double* bj = S.lrow + jt * 64;
            const double b0 = bj[lane], b1 = bj[32 + lane], b2 = bj[64 + lane], b3 = bj[96 + lane];
            dmma_884(c0, c1, -a[0], b0);
            dmma_884(g0, g1, -q[0], b0);
            dmma_884(d0, d1, -a[2], b2);
            dmma_884(h0, h1, -q[2], b2);
            dmma_884(c0, c1, -a[1], b1);
            dmma_884(g0, g1, -q[1], b1);
            dmma_884(d0, d1, -a[3], b3);
            dmma_884(h0, h1, -q[3], b3);
          }
          if (jt < kt) {
            const double* bj = S.lrow + jt * 64;
            const double b0 = bj[lane], b1 = bj[32 + lane];
            const double a0 = __ldcg(ai + jt * 64 + lane), a1 = __ldcg(ai + jt * 64 + 32 + lane);
            const double q0 = two ? __ldcg(ai2 + jt * 64 + lane) : 0.0;
            const double q1 = two ? __ldcg(ai2 + jt * 64 + 32 + lane) : 0.0;
            dmma_884(c0, c1, -a0, b0);
            dmma_884(g0, g1, -q0, b0);
            dmma_884(c0, c1, -a1, b1);
            dmma_884(g0, g1, -q1, b1);
          }
          ct[2 * lane] = c0 + d0;
          ct[2 * lane + 1] = c1 + d1;
          if (two) {
            ct2[2 * lane] = g0 + h0;
            ct2[2 * lane + 1] = g1 + h1;
          }
        }
        __syncthreads();
      }
      if (warp == 0) {
        // (4) factor the diagonal tile -> L_kk^-1 (swizzled in S.dg, and the
        // scratch diagonal tile for the back substitution)
        for (int e = lane; e < 64; e += 32) S.dg[eidx(e >> 3, e & 7)] = cur[e];
        __syncwarp();
        if (!warp_chol8_inv(S.dg, S.sl + 8 * Tmax) && lane == 0) *S.flag = 1;
        __syncwarp();
        double* dt_ = L + (long long)(((kt * (kt + 1)) >> 1) + kt) * 64;
        for (int e = lane; e < 64; e += 32) dt_[fpos(e >> 3, e & 7)] = S.dg[eidx(e >> 3, e & 7)];
      } else if (kt + 1 < T) {
        // meanwhile: column kt + 1 and the finished part of L row kt + 1
        const double* src = L + (long long)(((kt + 1) * (kt + 2)) >> 1) * 64;
        for (int e = 2 * (threadIdx.x - 32); e < kt * 64; e += 2 * (blockDim.x - 32))
          v3_cp16(S.lrow + e, src + e);
        v3_gather(S, nxt, kt + 1, T, m, wB, B, threadIdx.x - 32, blockDim.x - 32);
        v3_cp_wait();
      }
      __syncthreads();
      if (*S.flag) {
        ok = false;
        break;
      }
      // (5) TRSM: L(it, kt) = C(it, kt) L_kk^-T (it = kt+1..T) -> scratch;
      // L(kt + 1, kt) also completes the staged L row
      {
        const double bl0 = S.dg[eidx(fr, fk)], bl1 = S.dg[eidx(fr, 4 + fk)];
        for (int it = kt + 1 + warp; it <= T; it += kV3Warps) {
          const double* ct = cur + (it - kt) * 64;
          const double a0 = ct[fr * 8 + fk], a1 = ct[fr * 8 + 4 + fk];
          double e0 = 0.0, e1 = 0.0;
          dmma_884(e0, e1, a0, bl0);
          dmma_884(e0, e1, a1, bl1);
          double* out = L + (long long)(((it * (it + 1)) >> 1) + kt) * 64;
          out[fpos(fr, 2 * fk)] = e0;
          out[fpos(fr, 2 * fk + 1)] = e1;
          if (it == kt + 1 && it < T) {
            S.lrow[kt * 64 + fpos(fr, 2 * fk)] = e0;
            S.lrow[kt * 64 + fpos(fr, 2 * fk + 1)] = e1;
          }
        }
      }
      __syncthreads();
    }
    if (!ok) {
      if (threadIdx.x == 0) raise_status(status, ST_NOT_SPD, i);
      __syncthreads();
      continue;
    }
    // back substitution L^T z = y (y = row 0 of the RHS tiles (T, jt)),
    // column oriented over all warps: step it finishes z_it = L_ii^-T y_it
    // (8 threads) and then subtracts L(it, jt)^T z_it from every y_jt, jt <
    // it (one thread per (jt, column)).  Row it of the packed factor (tiles
    // jt = 0..it, the diagonal one holding L_ii^-1) is staged into the idle
    // column buffers by cp.async one step ahead.
    {
      const double* yrow = L + (long long)((T * (T + 1)) >> 1) * 64;
      for (int e = threadIdx.x; e < 8 * T; e += blockDim.x)
        S.z[e] = __ldcg(yrow + (e >> 3) * 64 + fpos(0, e & 7));
      {
        const int it = T - 1;
        const double* src = L + (long long)((it * (it + 1)) >> 1) * 64;
        for (int e = 2 * threadIdx.x; e < (it + 1) * 64; e += 2 * blockDim.x)
          v3_cp16(S.col + (it & 1) * colstride + e, src + e);
      }
      for (int it = T - 1; it >= 0; --it) {
        v3_cp_wait();
        __syncthreads();  // row it staged, y_it final, buffer (it - 1) & 1 free
        if (it > 0) {
          const double* src = L + (long long)(((it - 1) * it) >> 1) * 64;
          for (int e = 2 * threadIdx.x; e < it * 64; e += 2 * blockDim.x)
            v3_cp16(S.col + ((it - 1) & 1) * colstride + e, src + e);
        }
        const double* row = S.col + (it & 1) * colstride;
        if (threadIdx.x < 8) {
          const int r = threadIdx.x;
          const double* li = row + it * 64;
          double zr = 0.0;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c >= r) zr = fma(li[fpos(c, r)], S.z[8 * it + c], zr);
          S.sl[8 * Tmax + r] = zr;
        }
        __syncthreads();
        if (threadIdx.x < 8) S.z[8 * it + threadIdx.x] = S.sl[8 * Tmax + threadIdx.x];
        for (int o = threadIdx.x; o < 8 * it; o += blockDim.x) {
          const int jt = o >> 3, c = o & 7;
          const double* t = row + jt * 64;
          // the 16 lanes of a half-warp start their sum at different k: the
          // tile words (c & 3) + 4 k of the fragment order then fall into 16
          // distinct bank pairs
          const int rot = 2 * (jt & 1) + (c >> 2);
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int kk = (k + rot) & 7;
            acc = fma(t[fpos(kk, c)], S.sl[8 * Tmax + kk], acc);
          }
          S.z[o] -= acc;
        }
      }
      __syncthreads();
    }
    // D = s z and the row-tail trim of this column of D (as v2)
    double mx = 0.0;
    for (int l = threadIdx.x; l < m; l += blockDim.x) {
      const double v = S.sl[l] * S.z[l];
      S.z[l] = v;
      mx = fmax(mx, fabs(v));
    }
    mx = block_max(mx, red);
    const double thr = 1e-11 * mx;
    for (int e = threadIdx.x; e < SD; e += blockDim.x) {
      const int c = e % 3, bs = e / 3;
      const int ps = si + bs / (2 * rho + 1) - rho, pt = ti + bs % (2 * rho + 1) - rho;
      double v = 0.0;
      if (ps >= s0 && ps <= s1 && pt >= t0 && pt <= t1) {
        v = S.z[((ps - s0) * nbt + (pt - t0)) * 3 + c];
        if (!(fabs(v) >= thr)) v = 0.0;
      }
      drow[e] = v;
    }
    __syncthreads();
  }
}

}  // namespace gb
