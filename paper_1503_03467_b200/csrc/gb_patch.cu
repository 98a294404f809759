#include <stdlib.h>
// Batched SPD patch solves (Algorithm 2 lines 2a/3 and 11).
//
// K1 mass patches  (gamblet_fast.py:464-498): per fine node i,
//     (S M S)[i^rho, i^rho] z = s_i e_i,   psi^(q)_i = s[i^rho] * z.
// K4 correction patches (gamblet_fast.py:546-591): per coarse index i,
//     (S B S)[chi_i, chi_i] z = s[chi_i] * (-G)[chi_i, i],
//     D[chi_i, i] = s[chi_i] * z, then the row-tail trim of D^T
//     (gamblet_fast.py:172-190) fused in.
//
// The reference solves every patch by CG to a relative residual that tight
// mode clamps at 1e-14; these kernels factor each patch exactly (Cholesky in
// shared memory, one CTA per patch), which matches tight mode to 1e-13
// (SURVEY.md 8(c)).  Patches that do not fit shared memory use a per-CTA
// global-memory workspace with the same code.
#include "gb_common.cuh"
#include "gb_kernels.h"
#include "gb_tiled_chol.cuh"
#ifdef GB_PATCH_PROF
#include <cstdio>
#endif

namespace gb {

// Right-looking Cholesky of the n x n row-major matrix `a` (lower triangle
// used) by the whole CTA.  `colj` is an n-vector scratch.  Returns false (CTA
// uniform) when a pivot is not positive.
__device__ bool cta_cholesky(double* a, int ld, int n, double* colj) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int j = 0; j < n; ++j) {
    const double d = a[(long long)j * ld + j];
    if (!(d > 0.0)) return false;
    const double l = sqrt(d);
    for (int i = j + 1 + tid; i < n; i += nt) {
      const double v = a[(long long)i * ld + j] / l;
      a[(long long)i * ld + j] = v;
      colj[i] = v;
    }
    __syncthreads();
    if (tid == 0) a[(long long)j * ld + j] = l;
    for (int i = j + 1 + warp; i < n; i += nw) {
      const double lij = colj[i];
      double* ai = a + (long long)i * ld;
      for (int k = j + 1 + lane; k <= i; k += 32) ai[k] -= lij * colj[k];
    }
    __syncthreads();
  }
  return true;
}

// Solves L L^T z = b in place with the factor from cta_cholesky.
__device__ void cta_chol_solve(const double* a, int ld, int n, double* b) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int j = 0; j < n; ++j) {
    __syncthreads();
    const double yj = b[j] / a[(long long)j * ld + j];
    __syncthreads();
    if (tid == 0) b[j] = yj;
    for (int i = j + 1 + tid; i < n; i += nt) b[i] -= a[(long long)i * ld + j] * yj;
  }
  for (int j = n - 1; j >= 0; --j) {
    __syncthreads();
    const double zj = b[j] / a[(long long)j * ld + j];
    __syncthreads();
    if (tid == 0) b[j] = zj;
    for (int i = tid; i < j; i += nt) b[i] -= a[(long long)j * ld + i] * zj;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// K1: mass patches.  M is a box (w = wM) on the n x n fine grid, s = diag^-1/2.
// psi window: lo = -rho, width wd (= min(2 rho + 1, n)).
// ---------------------------------------------------------------------------
__global__ void k_mass_patches(int n, int wM, const double* __restrict__ M,
                               const double* __restrict__ s, int rho, int wd,
                               double* __restrict__ psi, long long* status,
                               double* __restrict__ gws, int use_gmem) {
  extern __shared__ double sm[];
  const int side = 2 * rho + 1;
  const int nmax = side * side;
  double* a;
  if (use_gmem) a = gws + (long long)blockIdx.x * nmax * nmax;
  else a = sm;
  double* b = sm + (use_gmem ? 0 : nmax * nmax);
  double* colj = b + nmax;
  const int SM = box_slots(wM, 1);
  const long long N = (long long)n * n;
  for (long long i = blockIdx.x; i < N; i += gridDim.x) {
    const int si = (int)(i / n), ti = (int)(i % n);
    const int s0 = imax(0, si - rho), s1 = imin(n - 1, si + rho);
    const int t0 = imax(0, ti - rho), t1 = imin(n - 1, ti + rho);
    const int ns = s1 - s0 + 1, nt = t1 - t0 + 1, m = ns * nt;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int l1 = e / m, l2 = e % m;
      const int r1s = s0 + l1 / nt, r1t = t0 + l1 % nt;
      const int r2s = s0 + l2 / nt, r2t = t0 + l2 % nt;
      const int ds = r2s - r1s, dt = r2t - r1t;
      double v = 0.0;
      if (ds >= -wM && ds <= wM && dt >= -wM && dt <= wM) {
        const long long r1 = (long long)r1s * n + r1t, r2 = (long long)r2s * n + r2t;
        v = M[r1 * SM + slot_of(wM, 1, ds, dt, 0)] * s[r1] * s[r2];
      }
      a[(long long)l1 * m + l2] = v;
    }
    const int li = (si - s0) * nt + (ti - t0);
    for (int l = threadIdx.x; l < m; l += blockDim.x) b[l] = (l == li) ? s[i] : 0.0;
    __syncthreads();
    const bool ok = cta_cholesky(a, m, m, colj);
    if (!ok) {
      if (threadIdx.x == 0) raise_status(status, ST_NOT_SPD, i);
      __syncthreads();
      continue;
    }
    cta_chol_solve(a, m, m, b);
    // scatter into the origin-clamped window of row i
    const int os = clampi(si - rho, 0, n - wd), ot = clampi(ti - rho, 0, n - wd);
    double* row = psi + i * (long long)wd * wd;
    for (int e = threadIdx.x; e < wd * wd; e += blockDim.x) {
      const int fs = os + e / wd, ft = ot + e % wd;
      double v = 0.0;
      if (fs >= s0 && fs <= s1 && ft >= t0 && ft <= t1) {
        const int l = (fs - s0) * nt + (ft - t0);
        v = s[(long long)fs * n + ft] * b[l];
      }
      row[e] = v;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K4: correction patches on the parent grid (side Lp).  B: box nr=nc=3,
// half-width wB; G: box nr=3, nc=1, half-width wG; sB = diag(B)^-1/2.
// Output Dt: box on the parent grid, nr=1, nc=3, half-width rho (row i holds
// D[:, i] after the row-tail trim).
// ---------------------------------------------------------------------------
__global__ void k_correction_patches(int Lp, int wB, const double* __restrict__ B,
                                     const double* __restrict__ sB,
                                     int wG, const double* __restrict__ G,
                                     int rho, double* __restrict__ Dt,
                                     long long* status, double* __restrict__ gws,
                                     int use_gmem, int nmax) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  double* a;
  if (use_gmem) a = gws + (long long)blockIdx.x * nmax * nmax;
  else a = sm;
  double* b = sm + (use_gmem ? 0 : (long long)nmax * nmax);
  double* colj = b + nmax;
  const int SB = box_slots(wB, 3), SG = box_slots(wG, 1), SD = box_slots(rho, 3);
  const long long P = (long long)Lp * Lp;
  for (long long i = blockIdx.x; i < P; i += gridDim.x) {
    const int si = (int)(i / Lp), ti = (int)(i % Lp);
    const int s0 = imax(0, si - rho), s1 = imin(Lp - 1, si + rho);
    const int t0 = imax(0, ti - rho), t1 = imin(Lp - 1, ti + rho);
    const int nbt = t1 - t0 + 1;
    const int m = 3 * (s1 - s0 + 1) * nbt;
    // right-hand side s * (-G[:, i]) and its norm
    double nrm = 0.0;
    for (int l = threadIdx.x; l < m; l += blockDim.x) {
      const int pl = l / 3, c = l % 3;
      const int ps = s0 + pl / nbt, pt = t0 + pl % nbt;
      const long long r = ((long long)ps * Lp + pt) * 3 + c;
      const int ds = si - ps, dt = ti - pt;
      double g = 0.0;
      if (ds >= -wG && ds <= wG && dt >= -wG && dt <= wG)
        g = G[r * SG + slot_of(wG, 1, ds, dt, 0)];
      const double v = sB[r] * (-g);
      b[l] = v;
      nrm += v * v;
    }
    nrm = block_sum(nrm, red);
    double* drow = Dt + i * SD;
    if (nrm == 0.0) {  // gamblet_fast.py:561-562: empty correction column
      for (int e = threadIdx.x; e < SD; e += blockDim.x) drow[e] = 0.0;
      __syncthreads();
      continue;
    }
    for (long long e = threadIdx.x; e < (long long)m * m; e += blockDim.x) {
      const int l1 = (int)(e / m), l2 = (int)(e % m);
      const int p1 = l1 / 3, c1 = l1 % 3, p2 = l2 / 3, c2 = l2 % 3;
      const int p1s = s0 + p1 / nbt, p1t = t0 + p1 % nbt;
      const int p2s = s0 + p2 / nbt, p2t = t0 + p2 % nbt;
      const int ds = p2s - p1s, dt = p2t - p1t;
      double v = 0.0;
      if (ds >= -wB && ds <= wB && dt >= -wB && dt <= wB) {
        const long long r1 = ((long long)p1s * Lp + p1t) * 3 + c1;
        const long long r2 = ((long long)p2s * Lp + p2t) * 3 + c2;
        v = B[r1 * SB + slot_of(wB, 3, ds, dt, c2)] * sB[r1] * sB[r2];
      }
      a[(long long)l1 * m + l2] = v;
    }
    __syncthreads();
    const bool ok = cta_cholesky(a, m, m, colj);
    if (!ok) {
      if (threadIdx.x == 0) raise_status(status, ST_NOT_SPD, i);
      __syncthreads();
      continue;
    }
    cta_chol_solve(a, m, m, b);
    // D values s * z and the row-tail trim of this column of D
    double mx = 0.0;
    for (int l = threadIdx.x; l < m; l += blockDim.x) {
      const int pl = l / 3, c = l % 3;
      const int ps = s0 + pl / nbt, pt = t0 + pl % nbt;
      const long long r = ((long long)ps * Lp + pt) * 3 + c;
      const double v = sB[r] * b[l];
      b[l] = v;
      mx = fmax(mx, fabs(v));
    }
    mx = block_max(mx, red);
    const double thr = 1e-11 * mx;
    for (int e = threadIdx.x; e < SD; e += blockDim.x) {
      const int c = e % 3, bs = e / 3;
      const int ps = si + bs / (2 * rho + 1) - rho, pt = ti + bs % (2 * rho + 1) - rho;
      double v = 0.0;
      if (ps >= s0 && ps <= s1 && pt >= t0 && pt <= t1) {
        v = b[((ps - s0) * nbt + (pt - t0)) * 3 + c];
        if (!(fabs(v) >= thr)) v = 0.0;
      }
      drow[e] = v;
    }
    __syncthreads();
  }
}


// ===========================================================================
// v2: tiled DMMA Cholesky in shared memory (gb_tiled_chol.cuh), one CTA per
// patch.  The gather forms the reference's materialized congruence entry by
// entry, (x * s_i) * s_j (gamblet_fast.py:136), from the unscaled box.
// ===========================================================================
struct TileSmem {
  double* tl;
  double* sl;  // scale factor of local row l (and 8 scratch doubles after it)
  double* z;
  double* part;
  int* tij;    // packed (it << 8) | jt per lower tile
  int* rowg;   // global row of local index l
  int* ploc;   // packed (a << 8) | b local parent / node coordinates
  int* flag;
};

__host__ __device__ __forceinline__ size_t tile_smem_bytes(int Tmax, int nwarps) {
  const size_t ntile = (size_t)Tmax * (Tmax + 1) / 2 + Tmax;
  return ntile * 64 * 8 + (size_t)(16 * Tmax + 8) * 8 + (size_t)8 * nwarps * 8 +
         (size_t)(Tmax * (Tmax + 1) / 2) * 4 + (size_t)16 * Tmax * 4 + 16;
}

__device__ __forceinline__ TileSmem carve(double* sm, int Tmax, int nwarps) {
  TileSmem t;
  const int ntile = Tmax * (Tmax + 1) / 2 + Tmax;
  t.tl = sm;
  t.sl = t.tl + ntile * 64;
  t.z = t.sl + 8 * Tmax + 8;
  t.part = t.z + 8 * Tmax;
  int* ip = reinterpret_cast<int*>(t.part + 8 * nwarps);
  t.tij = ip;
  t.rowg = t.tij + Tmax * (Tmax + 1) / 2;
  t.ploc = t.rowg + 8 * Tmax;
  t.flag = t.ploc + 8 * Tmax;
  return t;
}

__global__ void __launch_bounds__(256) k_correction_patches_v2(
    int Lp, int wB, const double* __restrict__ B, const double* __restrict__ sB, int wG,
    const double* __restrict__ G, int rho, double* __restrict__ Dt, long long* status,
    int Tmax) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const int nw = blockDim.x >> 5;
  TileSmem S = carve(sm, Tmax, nw);
  const int SB = box_slots(wB, 3), SG = box_slots(wG, 1), SD = box_slots(rho, 3);
  const long long P = (long long)Lp * Lp;
#ifdef GB_PATCH_PROF
  long long tp[5] = {0, 0, 0, 0, 0}, tc = clock64(), tn;
#define GB_TICK(k) do { __syncthreads(); tn = clock64(); tp[k] += tn - tc; tc = tn; } while (0)
#else
#define GB_TICK(k) do {} while (0)
#endif
  for (long long i = blockIdx.x; i < P; i += gridDim.x) {
    const int si = (int)(i / Lp), ti = (int)(i % Lp);
    const int s0 = imax(0, si - rho), s1 = imin(Lp - 1, si + rho);
    const int t0 = imax(0, ti - rho), t1 = imin(Lp - 1, ti + rho);
    const int nbt = t1 - t0 + 1;
    const int m = 3 * (s1 - s0 + 1) * nbt;
    const int T = (m + 7) >> 3;
    const int nlt = T * (T + 1) / 2;
    // local tables and the right-hand side s * (-G[:, i])
    double nrm = 0.0;
    for (int l = threadIdx.x; l < 8 * T; l += blockDim.x) {
      double v = 0.0;
      if (l < m) {
        const int pl = l / 3, c = l - 3 * pl;
        const int a = pl / nbt, b = pl - a * nbt;
        const int ps = s0 + a, pt = t0 + b;
        const long long r = ((long long)ps * Lp + pt) * 3 + c;
        S.rowg[l] = (int)r;
        S.ploc[l] = (a << 8) | b;
        S.sl[l] = sB[r];
        const int ds = si - ps, dt = ti - pt;
        double g = 0.0;
        if (ds >= -wG && ds <= wG && dt >= -wG && dt <= wG)
          g = G[r * SG + slot_of(wG, 1, ds, dt, 0)];
        v = sB[r] * (-g);
      }
      S.z[l] = v;
      nrm += v * v;
    }
    for (int t = threadIdx.x; t < nlt; t += blockDim.x) {
      int it = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((it + 1) * (it + 2) / 2 <= t) ++it;
      while (it * (it + 1) / 2 > t) --it;
      S.tij[t] = (it << 8) | (t - it * (it + 1) / 2);
    }
    nrm = block_sum(nrm, red);  // also orders the table writes
    double* drow = Dt + i * SD;
    if (nrm == 0.0) {  // gamblet_fast.py:561-562: empty correction column
      for (int e = threadIdx.x; e < SD; e += blockDim.x) drow[e] = 0.0;
      __syncthreads();
      continue;
    }
    GB_TICK(0);
    // gather (S B S)[chi, chi] lower tiles + RHS tile row, 8 independent
    // loads in flight per thread (the B rows are L2 hits shared by the
    // neighbouring patches; the gather is latency-bound without the batching)
    {
      const int nel = nlt * 64, stride = blockDim.x;
      for (int e0 = threadIdx.x; e0 < nel; e0 += 8 * stride) {
        long long addr[8];
        double sc1[8], sc2[8], v[8];
        int dst[8], kind[8];  // kind: 0 zero, 1 load, 2 unit diagonal pad
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * stride;
          kind[u] = 0;
          dst[u] = -1;
          addr[u] = 0;
          sc1[u] = sc2[u] = 0.0;
          if (e < nel) {
            const int t = e >> 6, w = e & 63;
            const int ij = S.tij[t];
            const int r = w >> 3, c = w & 7;
            const int l1 = ((ij >> 8) << 3) + r, l2 = ((ij & 255) << 3) + c;
            dst[u] = t * 64 + eidx(r, c);
            if (l1 < m && l2 < m) {
              const int p1 = S.ploc[l1 / 3 * 3], p2 = S.ploc[l2 / 3 * 3];
              const int ds = (p2 >> 8) - (p1 >> 8), dt = (p2 & 255) - (p1 & 255);
              if (ds >= -wB && ds <= wB && dt >= -wB && dt <= wB) {
                kind[u] = 1;
                addr[u] = (long long)S.rowg[l1] * SB + slot_of(wB, 3, ds, dt, l2 % 3);
                sc1[u] = S.sl[l1];
                sc2[u] = S.sl[l2];
              }
            } else if (l1 == l2) {
              kind[u] = 2;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = kind[u] == 1 ? __ldg(B + addr[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (dst[u] >= 0)
            S.tl[dst[u]] = kind[u] == 1 ? v[u] * sc1[u] * sc2[u] : (kind[u] == 2 ? 1.0 : 0.0);
      }
    }
    for (int e = threadIdx.x; e < T * 64; e += blockDim.x) {
      const int jt = e >> 6, w = e & 63;
      const int r = w >> 3, c = w & 7;
      S.tl[(nlt + jt) * 64 + eidx(r, c)] = (r == 0) ? S.z[jt * 8 + c] : 0.0;
    }
    __syncthreads();
    GB_TICK(1);
    if (!tiled_chol_fwd(S.tl, T, S.sl + 8 * Tmax, S.flag)) {
      if (threadIdx.x == 0) raise_status(status, ST_NOT_SPD, i);
      __syncthreads();
      continue;
    }
    GB_TICK(2);
    tiled_back_subst(S.tl, T, S.z, S.part);
    GB_TICK(3);
    // D = s z and the row-tail trim of this column of D
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
    GB_TICK(4);
  }
#ifdef GB_PATCH_PROF
  if (threadIdx.x == 0 && blockIdx.x < 4)
    printf("patch prof blk %d: tables %lld gather %lld factor %lld backsubst %lld out %lld"
           " | blk0 factor: w0A %llu w1A %llu w2A %llu A+sync %llu trsm %llu\n",
           blockIdx.x, tp[0], tp[1], tp[2], tp[3], tp[4], g_fprof[0], g_fprof[1], g_fprof[2],
           g_fprof[3], g_fprof[4]);
#endif
#undef GB_TICK
}

__global__ void __launch_bounds__(128) k_mass_patches_v2(
    int n, int wM, const double* __restrict__ M, const double* __restrict__ s, int rho,
    int wd, double* __restrict__ psi, long long* status, int Tmax) {
  extern __shared__ double sm[];
  const int nw = blockDim.x >> 5;
  TileSmem S = carve(sm, Tmax, nw);
  const int SM = box_slots(wM, 1);
  const long long N = (long long)n * n;
  for (long long i = blockIdx.x; i < N; i += gridDim.x) {
    const int si = (int)(i / n), ti = (int)(i % n);
    const int s0 = imax(0, si - rho), s1 = imin(n - 1, si + rho);
    const int t0 = imax(0, ti - rho), t1 = imin(n - 1, ti + rho);
    const int nt = t1 - t0 + 1, m = (s1 - s0 + 1) * nt;
    const int T = (m + 7) >> 3;
    const int nlt = T * (T + 1) / 2;
    const int li = (si - s0) * nt + (ti - t0);
    for (int l = threadIdx.x; l < 8 * T; l += blockDim.x) {
      if (l < m) {
        const int a = l / nt, b = l - a * nt;
        S.rowg[l] = (s0 + a) * n + (t0 + b);
        S.ploc[l] = (a << 8) | b;
        S.sl[l] = s[S.rowg[l]];
      }
    }
    for (int t = threadIdx.x; t < nlt; t += blockDim.x) {
      int it = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((it + 1) * (it + 2) / 2 <= t) ++it;
      while (it * (it + 1) / 2 > t) --it;
      S.tij[t] = (it << 8) | (t - it * (it + 1) / 2);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nlt * 64; e += blockDim.x) {
      const int t = e >> 6, w = e & 63;
      const int ij = S.tij[t];
      const int r = w >> 3, c = w & 7;
      const int l1 = ((ij >> 8) << 3) + r, l2 = ((ij & 255) << 3) + c;
      double v = 0.0;
      if (l1 < m && l2 < m) {
        const int p1 = S.ploc[l1], p2 = S.ploc[l2];
        const int ds = (p2 >> 8) - (p1 >> 8), dt = (p2 & 255) - (p1 & 255);
        if (ds >= -wM && ds <= wM && dt >= -wM && dt <= wM)
          v = M[(long long)S.rowg[l1] * SM + slot_of(wM, 1, ds, dt, 0)] * S.sl[l1] * S.sl[l2];
      } else if (l1 == l2) {
        v = 1.0;
      }
      S.tl[t * 64 + eidx(r, c)] = v;
    }
    for (int e = threadIdx.x; e < T * 64; e += blockDim.x) {
      const int jt = e >> 6, w = e & 63;
      const int r = w >> 3, c = w & 7;
      S.tl[(nlt + jt) * 64 + eidx(r, c)] = (r == 0 && jt * 8 + c == li) ? s[i] : 0.0;
    }
    __syncthreads();
    if (!tiled_chol_fwd(S.tl, T, S.sl + 8 * Tmax, S.flag)) {
      if (threadIdx.x == 0) raise_status(status, ST_NOT_SPD, i);
      __syncthreads();
      continue;
    }
    tiled_back_subst(S.tl, T, S.z, S.part);
    const int os = clampi(si - rho, 0, n - wd), ot = clampi(ti - rho, 0, n - wd);
    double* row = psi + i * (long long)wd * wd;
    for (int e = threadIdx.x; e < wd * wd; e += blockDim.x) {
      const int fs = os + e / wd, ft = ot + e % wd;
      double v = 0.0;
      if (fs >= s0 && fs <= s1 && ft >= t0 && ft <= t1) {
        const int l = (fs - s0) * nt + (ft - t0);
        v = s[(long long)fs * n + ft] * S.z[l];
      }
      row[e] = v;
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// Mass patches as banded solves (gamblet_fast.py:464-498, line 2a/3).  With
// the local nodes of the clipped (2 rho + 1)^2 box numbered row-major (nt per
// row), the 9-point mass stencil couples l only to l +- {0, 1, nt - 1, nt,
// nt + 1}: (S M S)[i^rho, i^rho] is banded with half-bandwidth b = nt + 1 and
// its Cholesky factor has the same band (no fill outside it).  One warp per
// patch: the band (m x (b+1), <= 49 x 9 at rho = 3) in shared memory,
// right-looking column steps (<= 36 independent updates per step across the
// lanes), then the forward (RHS s_i e_i) and backward band substitutions
// with shuffle dot products.  ~b^2 m instead of m^3/3 flops; the serial
// chain is m short steps instead of 7 dense 8x8 tile factorizations.
// ---------------------------------------------------------------------------
constexpr int kBandMaxM = 49, kBandMaxB = 8, kBandW = kBandMaxB + 1, kBandWarps = 4;

// type representative of a fine coordinate: rows whose ball is unclipped
// share the patch of coordinate rho (at most (2 rho + 1)^2
// distinct S M S patches when M is translation invariant)
__host__ __device__ __forceinline__ int mass_type_rep(int c, int n, int rho) {
  return (c < rho || c > n - 1 - rho) ? c : rho;
}
// rep list entry l of the (2 rho + 1)^2 representatives: coordinates
// 0..rho (rho = the interior type) then n - rho .. n - 1 per axis
__device__ __forceinline__ int mass_rep_coord(int l, int n, int rho) {
  return l <= rho ? l : n - (2 * rho + 1) + l;
}

__global__ void __launch_bounds__(32 * kBandWarps) k_mass_patches_band(
    int n, const double* __restrict__ M, const double* __restrict__ s, int rho, int wd,
    double* __restrict__ psi, long long* status, long long p0, long long p1,
    const int* __restrict__ flag = nullptr, int mode = 0) {
  // mode 0: patches [p0, p1); 1: the type representatives only (index l in
  // [p0, p1) of the rep list); 2: [p0, p1) only when *flag != 0 (M is not
  // translation invariant, the representatives cannot stand in)
  if (mode == 2 && *flag == 0) return;
  __shared__ double sLb[kBandWarps][kBandMaxM * kBandW];
  __shared__ double sSl[kBandWarps][kBandMaxM];
  __shared__ double sX[kBandWarps][kBandMaxM];
  __shared__ double sId[kBandWarps][kBandMaxM];  // 1 / L[r][r]
  __shared__ int sRC[kBandWarps][kBandMaxM];     // (r / nt) << 8 | (r % nt)
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  double* Lb = sLb[wi];
  double* sl = sSl[wi];
  double* x = sX[wi];
  double* id = sId[wi];
  int* rc = sRC[wi];
  // this lane's two trailing-update pairs p = lane, lane + 32 of the full
  // b = 8 triangle, enumerated by rows: p = rr (rr + 1) / 2 + cc, cc <= rr;
  // offsets from the pivot column: ro = rr + 1, co = cc + 1 (pairs 36.. unused)
  int ro[2], co[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int p = lane + 32 * u;
    int rr = 0;
    while ((rr + 1) * (rr + 2) / 2 <= p) ++rr;
    ro[u] = rr + 1;
    co[u] = p - rr * (rr + 1) / 2 + 1;
    if (p >= kBandMaxB * (kBandMaxB + 1) / 2) ro[u] = 99;
  }
  // patches [p0, p1) (node order; a row strip of the fine grid)
  const long long nwarps = (long long)gridDim.x * kBandWarps;
  const int R = 2 * rho + 1;
  for (long long ii = p0 + (long long)blockIdx.x * kBandWarps + wi; ii < p1; ii += nwarps) {
    const long long i = mode == 1 ? (long long)mass_rep_coord((int)(ii / R), n, rho) * n +
                                        mass_rep_coord((int)(ii % R), n, rho)
                                  : ii;
    const int si = (int)(i / n), ti = (int)(i % n);
    const int s0 = imax(0, si - rho), s1 = imin(n - 1, si + rho);
    const int t0 = imax(0, ti - rho), t1 = imin(n - 1, ti + rho);
    const int nt = t1 - t0 + 1, m = (s1 - s0 + 1) * nt;
    const int b = imin(nt + 1, m - 1);  // half-bandwidth
    const int li = (si - s0) * nt + (ti - t0);
    for (int l = lane; l < m; l += 32) {
      const int a = l / nt, c = l - a * nt;
      rc[l] = (a << 8) | c;
      sl[l] = s[(long long)(s0 + a) * n + (t0 + c)];
    }
    __syncwarp();
    // band gather: Lb[r * kBandW + d] = (S M S)[r][r - d], d = 0..b
    for (int e = lane; e < m * kBandW; e += 32) {
      const int r = e / kBandW, d = e - r * kBandW;
      const int c = r - d;
      double v = 0.0;
      if (d <= b && c >= 0) {
        const int pr = rc[r], pc = rc[c];
        const int ds = (pc >> 8) - (pr >> 8), dt = (pc & 255) - (pr & 255);
        if (ds >= -1 && ds <= 1 && dt >= -1 && dt <= 1) {
          const long long gr = (long long)(s0 + (pr >> 8)) * n + (t0 + (pr & 255));
          v = M[gr * 9 + (ds + 1) * 3 + (dt + 1)] * sl[r] * sl[c];
        }
      }
      Lb[e] = v;
    }
    __syncwarp();
    // right-hand side s_i e_li, forward-substituted inside the factorization
    for (int l = lane; l < m; l += 32) x[l] = (l == li) ? sl[li] : 0.0;
    __syncwarp();
    bool ok = true;
    // right-looking band Cholesky: column j, y_j = x_j / L_jj, then the <= 36
    // trailing updates and x_{j+k} -= L[j+k][j] y_j
    for (int j = 0; j < m; ++j) {
      const double piv = Lb[j * kBandW];
      ok = ok && (piv > 0.0);
      const double il = rsqrt(piv);
      const double yj = x[j] * il;
      const int kmax = imin(b, m - 1 - j);
      double lc = 0.0;  // L[j + lane][j], lanes 1..kmax
      if (lane >= 1 && lane <= kmax) lc = Lb[(j + lane) * kBandW + lane] * il;
      __syncwarp();
      if (lane == 0) {
        Lb[j * kBandW] = piv * il;
        id[j] = il;
        x[j] = yj;
      }
      if (lane >= 1 && lane <= kmax) {
        Lb[(j + lane) * kBandW + lane] = lc;
        x[j + lane] = fma(-lc, yj, x[j + lane]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double vr = __shfl_sync(0xffffffffu, lc, ro[u] & 31);
        const double vc = __shfl_sync(0xffffffffu, lc, co[u] & 31);
        if (ro[u] <= kmax) {
          double* a = Lb + (j + ro[u]) * kBandW + (ro[u] - co[u]);
          *a = fma(-vr, vc, *a);
        }
      }
      __syncwarp();
    }
    if (!__all_sync(0xffffffffu, ok)) {
      if (lane == 0) raise_status(status, ST_NOT_SPD, i);
      continue;
    }
    // backward, column oriented: z_r = y_r / L_rr, then y_{r-k} -= L[r][r-k] z_r
    for (int r = m - 1; r >= 0; --r) {
      const double z = x[r] * id[r];
      if (lane >= 1 && lane <= b && r - lane >= 0)
        x[r - lane] = fma(-Lb[r * kBandW + lane], z, x[r - lane]);
      __syncwarp();
      if (lane == 0) x[r] = z;
      __syncwarp();
    }
    const int os = clampi(si - rho, 0, n - wd), ot = clampi(ti - rho, 0, n - wd);
    double* row = psi + i * (long long)wd * wd;
    for (int e = lane; e < wd * wd; e += 32) {
      const int fs = os + e / wd, ft = ot + e % wd;
      double v = 0.0;
      if (fs >= s0 && fs <= s1 && ft >= t0 && ft <= t1) {
        const int l = (fs - s0) * nt + (ft - t0);
        v = sl[l] * x[l];
      }
      row[e] = v;
    }
    __syncwarp();
  }
}
// M translation invariant (every in-domain box entry of every row equals the
// interior representative's, bit for bit) -> *flag stays 0
__global__ void k_mass_invariance(int n, const double* __restrict__ M, int* flag) {
  const long long N = (long long)n * n;
  const long long c = (long long)(n / 2) * n + n / 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    const int si = (int)(i / n), ti = (int)(i % n);
    bool bad = false;
#pragma unroll
    for (int d = 0; d < 9; ++d) {
      const int ds = d / 3 - 1, dt = d % 3 - 1;
      const bool in = si + ds >= 0 && si + ds < n && ti + dt >= 0 && ti + dt < n;
      if (in && __double_as_longlong(M[i * 9 + d]) != __double_as_longlong(M[c * 9 + d]))
        bad = true;
    }
    if (bad) atomicOr(flag, 1);
  }
}

// psi row i = psi row of its type representative (window content identical)
__global__ void k_mass_broadcast(int n, int rho, int wd, double* __restrict__ psi,
                                 const int* __restrict__ flag) {
  if (*flag != 0) return;
  const long long W2 = (long long)wd * wd;
  const long long total = (long long)n * n * W2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / W2;
    const int si = (int)(i / n), ti = (int)(i % n);
    const long long r = (long long)mass_type_rep(si, n, rho) * n + mass_type_rep(ti, n, rho);
    if (r != i) psi[e] = psi[r * W2 + (e - i * W2)];
  }
}
}  // namespace gb

#include "gb_patch_l2.cuh"

using namespace gb;

static const int kMaxSmem = 227 * 1024;

size_t gbk_mass_patch_workspace(int rho, int blocks) {
  const int nmax = (2 * rho + 1) * (2 * rho + 1);
  const size_t smem = ((size_t)nmax * nmax + 2 * nmax) * 8;
  if (smem <= (size_t)kMaxSmem) return 0;
  return (size_t)blocks * nmax * nmax * 8;
}

int gbk_mass_patches(int n, int wM, const double* M, const double* s, int rho,
                     int wd, double* psi, long long* status, double* gws,
                     int blocks, cudaStream_t st) {
  const int nmax = (2 * rho + 1) * (2 * rho + 1);
  size_t smem = ((size_t)nmax * nmax + 2 * nmax) * 8;
  int use_gmem = 0;
  if (smem > (size_t)kMaxSmem) {
    use_gmem = 1;
    smem = (size_t)2 * nmax * 8;
    if (gws == nullptr) return 1;
  }
  cudaFuncSetAttribute(k_mass_patches, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  const long long N = (long long)n * n;
  int g = blocks > 0 ? blocks : (int)(N < 148 * 64 ? N : 148 * 64);
  k_mass_patches<<<g, nmax <= 64 ? 64 : 256, smem, st>>>(n, wM, M, s, rho, wd, psi,
                                                         status, gws, use_gmem);
  return (int)cudaGetLastError();
}

size_t gbk_correction_workspace(int rho, int blocks) {
  const int nmax = 3 * (2 * rho + 1) * (2 * rho + 1);
  const size_t smem = ((size_t)nmax * nmax + 2 * nmax) * 8;
  if (smem <= (size_t)kMaxSmem) return 0;
  return (size_t)blocks * nmax * nmax * 8;
}

int gbk_correction_patches(int Lp, int wB, const double* B, const double* sB,
                           int wG, const double* G, int rho, double* Dt,
                           long long* status, double* gws, int blocks,
                           cudaStream_t st) {
  const int nmax = 3 * (2 * rho + 1) * (2 * rho + 1);
  size_t smem = ((size_t)nmax * nmax + 2 * nmax) * 8;
  int use_gmem = 0;
  if (smem > (size_t)kMaxSmem) {
    use_gmem = 1;
    smem = (size_t)2 * nmax * 8;
    if (gws == nullptr) return 1;
  }
  cudaFuncSetAttribute(k_correction_patches,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const long long P = (long long)Lp * Lp;
  int g = blocks > 0 ? blocks : (int)(P < 148 * 8 ? P : 148 * 8);
  k_correction_patches<<<g, 256, smem, st>>>(Lp, wB, B, sB, wG, G, rho, Dt, status,
                                             gws, use_gmem, nmax);
  return (int)cudaGetLastError();
}

// v2/v3 entry points: pre-scaled boxes, tiled DMMA Cholesky.  GB_UNSUPPORTED
// (negative, never a CUDA error code) when no kernel of this family covers the
// patch or the row range; the caller then uses the global-workspace v1.
// launch tuning (gb_tune, test/tool use only): 0 -> total CTAs of the v2
// correction-patch grid (0 = auto); 1 -> correction kernel (1 = v3 left-looking
// with L streamed through the caller's workspace, default; 0 = the
// shared-memory-resident v2); 2 -> mass patches (0 = banded warp solver,
// default; 1 = dense tiled v2)
static int g_patch_grid = 0;
static int g_patch_v3 = 1;
static int g_mass_dense = 0;
static int g_mass_types = 1;
int gbk_tune(int what, int value) {
  extern int g_sym_ws_ctas, g_sym_ws_on, g_k3_tiled;
  int* slot = what == 0   ? &g_patch_grid
              : what == 1 ? &g_patch_v3
              : what == 2 ? &g_mass_dense
              : what == 3 ? &g_sym_ws_ctas
              : what == 4 ? &g_mass_types
              : what == 5 ? &g_sym_ws_on
              : what == 6 ? &g_k3_tiled
                          : nullptr;
  if (!slot) return -1;
  const int old = *slot;
  if (value >= 0) *slot = value;
  return old;
}

static constexpr int kV3PerSm = GB_V3_MINB;  // smem (36 KB) and register limit of the v3 CTA

static long long v3_grid(int Lp, int r0, int r1) {
  const long long P = (long long)(r1 - r0) * Lp;
  const long long gmax = 148LL * kV3PerSm;
  return P < gmax ? P : gmax;
}

// bytes of the per-CTA L scratch the v3 kernel streams finished columns
// through (L2-resident); 0 when v3 does not run for this patch size
size_t gbk_correction_v3_workspace(int Lp, int rho, int r0, int r1) {
  const int nmax = 3 * (2 * rho + 1) * (2 * rho + 1);
  const int Tmax = (nmax + 7) / 8;
  if (!g_patch_v3 || Tmax > 255 || r1 <= r0) return 0;
  return (size_t)v3_grid(Lp, r0, r1) * ((size_t)Tmax * (Tmax + 1) / 2 + Tmax) * 64 *
         sizeof(double);
}

// parent grid rows [r0, r1) only (a spatial strip; the v3 kernel is required
// for a proper strip); Dt rows outside are not touched.  `ws` is the caller's
// scratch (gbk_correction_v3_workspace bytes, stream-ordered by the caller),
// so concurrent transforms on different streams never share it.
int gbk_correction_patches_rows(int Lp, int wB, const double* B, const double* sB, int wG,
                                const double* G, int rho, double* Dt, long long* status, int r0,
                                int r1, double* ws, size_t ws_bytes, cudaStream_t st) {
  if (r0 < 0 || r1 > Lp || r0 > r1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const int nmax = 3 * (2 * rho + 1) * (2 * rho + 1);
  const int Tmax = (nmax + 7) / 8;
  const size_t need = gbk_correction_v3_workspace(Lp, rho, r0, r1);
  if (need > 0) {
    if (!ws || ws_bytes < need) return GB_UNSUPPORTED;
    const size_t smem = v3_smem_bytes(Tmax);
    cudaError_t e = cudaFuncSetAttribute(k_correction_patches_v3,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    k_correction_patches_v3<<<(int)v3_grid(Lp, r0, r1), 32 * kV3Warps, smem, st>>>(
        Lp, wB, B, sB, wG, G, rho, Dt, status, Tmax, ws, (long long)r0 * Lp,
        (long long)r1 * Lp);
    return (int)cudaGetLastError();
  }
  if (r0 != 0 || r1 != Lp) return GB_UNSUPPORTED;  // v2 runs whole levels only
  const size_t smem = tile_smem_bytes(Tmax, 8);
  if (smem > (size_t)kMaxSmem || Tmax > 255) return GB_UNSUPPORTED;
  cudaError_t e = cudaFuncSetAttribute(k_correction_patches_v2,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  const long long P = (long long)Lp * Lp;
  int per_sm = (int)((228 * 1024) / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  long long gmax = g_patch_grid > 0 ? g_patch_grid : 148LL * per_sm * 4;
  int g = (int)(P < gmax ? P : gmax);
  k_correction_patches_v2<<<g, 256, smem, st>>>(Lp, wB, B, sB, wG, G, rho, Dt, status, Tmax);
  return (int)cudaGetLastError();
}

int gbk_correction_patches_v2(int Lp, int wB, const double* B, const double* sB, int wG,
                              const double* G, int rho, double* Dt, long long* status,
                              double* ws, size_t ws_bytes, cudaStream_t st) {
  return gbk_correction_patches_rows(Lp, wB, B, sB, wG, G, rho, Dt, status, 0, Lp, ws,
                                     ws_bytes, st);
}

// fine-grid rows [r0, r1) only (the banded kernel is required for a proper
// strip)
int gbk_mass_patches_rows(int n, int wM, const double* M, const double* s, int rho, int wd,
                          double* psi, long long* status, int r0, int r1, cudaStream_t st) {
  if (r0 < 0 || r1 > n || r0 > r1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const int nmax = (2 * rho + 1) * (2 * rho + 1);
  const int Tmax = (nmax + 7) / 8;
  if (wM == 1 && rho <= 3 && !g_mass_dense && r0 == 0 && r1 == n && n >= 2 * rho + 2 &&
      g_mass_types) {
    // whole level: factor the (2 rho + 1)^2 type representatives, broadcast
    // their rows; the general pass runs only if M is not translation invariant
    int* d_flag = nullptr;  // stream-ordered, so concurrent transforms never share it
    keep_default_pool();
    cudaError_t e = cudaMallocAsync((void**)&d_flag, sizeof(int), st);
    if (e != cudaSuccess) return (int)e;
    e = cudaMemsetAsync(d_flag, 0, sizeof(int), st);
    if (e != cudaSuccess) return (int)e;
    const long long N = (long long)n * n;
    k_mass_invariance<<<(int)((N + 255) / 256 < 148 * 8 ? (N + 255) / 256 : 148 * 8), 256, 0,
                        st>>>(n, M, d_flag);
    const int R = 2 * rho + 1;
    k_mass_patches_band<<<(R * R + kBandWarps - 1) / kBandWarps, 32 * kBandWarps, 0, st>>>(
        n, M, s, rho, wd, psi, status, 0, (long long)R * R, d_flag, 1);
    k_mass_broadcast<<<148 * 16, 256, 0, st>>>(n, rho, wd, psi, d_flag);
    const long long warps = 148LL * 16 * 4;
    const long long g = (N + kBandWarps - 1) / kBandWarps;
    k_mass_patches_band<<<(int)(g < warps / kBandWarps ? g : warps / kBandWarps),
                          32 * kBandWarps, 0, st>>>(n, M, s, rho, wd, psi, status, 0, N,
                                                    d_flag, 2);
    e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    return (int)cudaFreeAsync(d_flag, st);
  }
  if (wM == 1 && rho <= 3 && !g_mass_dense) {  // banded warp solver (rho = 3: b <= 8)
    const long long warps = 148LL * 16 * 4;
    const long long np = (long long)(r1 - r0) * n;
    const long long g = (np + kBandWarps - 1) / kBandWarps;
    k_mass_patches_band<<<(int)(g < warps / kBandWarps ? g : warps / kBandWarps),
                          32 * kBandWarps, 0, st>>>(n, M, s, rho, wd, psi, status,
                                                    (long long)r0 * n, (long long)r1 * n);
    return (int)cudaGetLastError();
  }
  if (r0 != 0 || r1 != n) return GB_UNSUPPORTED;  // the dense tiled kernel runs whole grids only
  const size_t smem = tile_smem_bytes(Tmax, 4);
  if (smem > (size_t)kMaxSmem || Tmax > 255) return GB_UNSUPPORTED;
  cudaError_t e = cudaFuncSetAttribute(k_mass_patches_v2,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  const long long N = (long long)n * n;
  int g = (int)(N < 148LL * 64 ? N : 148LL * 64);
  k_mass_patches_v2<<<g, 128, smem, st>>>(n, wM, M, s, rho, wd, psi, status, Tmax);
  return (int)cudaGetLastError();
}
int gbk_mass_patches_v2(int n, int wM, const double* M, const double* s, int rho, int wd,
                        double* psi, long long* status, cudaStream_t st) {
  return gbk_mass_patches_rows(n, wM, M, s, rho, wd, psi, status, 0, n, st);
}
