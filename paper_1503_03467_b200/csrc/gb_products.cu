// Structured (box-stencil) sparse products of the localized transform.
//
// Every product below reproduces the reference's scipy SpGEMM accumulation
// order (row of the left factor, its stored columns ascending, sums starting
// at 0.0), so identical inputs give bitwise identical outputs wherever the
// reference itself is order-deterministic.
//
//   K2  X = psi A, raw = X psi^T              gamblet_fast.py:658-665
//   K3  B = W A W^T (sym fused), G = W A pibar^T, PAPt = P A P^T
//                                             gamblet_fast.py:520-544, 597-601
//   K6  R = pibar + Dt W                      gamblet_fast.py:587-590
//       BD = B D, GtD = G^T D, DtBD, raw A^(k-1) gamblet_fast.py:602-611
//       psi^(k-1) = 0.25 P psi + Dt (W psi)   gamblet_fast.py:615-622
#include "gb_common.cuh"
#include "gb_boxgemm.cuh"
#include "gb_kernels.h"

namespace gb {

// psi window helpers --------------------------------------------------------
struct PsiWin {
  int n, L, lo, wd;  // fine side, level side, window offset, window width
  int hi;            // unclipped support bound: row support in [c+lo, c+hi]
  __device__ __forceinline__ int h() const { return n / L; }
  __device__ __forceinline__ int origin(int s) const {
    return clampi(s * (n / L) + lo, 0, n - wd);
  }
};

// ---------------------------------------------------------------------------
// K2a: X = psi A (fine grid), X box half-width wX = rho + wA
// ---------------------------------------------------------------------------
__global__ void k_psi_stencil(PsiWin pw, int rho, const double* __restrict__ psi,
                              int wA, const double* __restrict__ A, int wX,
                              double* __restrict__ X, long long e0, long long e1) {
  const int n = pw.n;
  const int SX = box_slots(wX, 1), SA = box_slots(wA, 1);
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / SX;
    const int sl = (int)(e - i * SX);
    const int si = (int)(i / n), ti = (int)(i % n);
    const int us = si + sl / (2 * wX + 1) - wX, ut = ti + sl % (2 * wX + 1) - wX;
    double acc = 0.0;
    if (us >= 0 && us < n && ut >= 0 && ut < n) {
      const int os = pw.origin(si), ot = pw.origin(ti);
      const double* prow = psi + i * (long long)pw.wd * pw.wd;
      // v over psi row support (true support [i-rho, i+rho] in the window)
      const int vs0 = imax(imax(os, si - rho), us - wA);
      const int vs1 = imin(imin(os + pw.wd - 1, si + rho), us + wA);
      const int vt0 = imax(imax(ot, ti - rho), ut - wA);
      const int vt1 = imin(imin(ot + pw.wd - 1, ti + rho), ut + wA);
      for (int vs = vs0; vs <= vs1; ++vs) {
        for (int vt = vt0; vt <= vt1; ++vt) {
          const double pv = prow[(vs - os) * pw.wd + (vt - ot)];
          if (pv == 0.0) continue;
          const long long v = (long long)vs * n + vt;
          acc += pv * A[v * SA + slot_of(wA, 1, us - vs, ut - vt, 0)];
        }
      }
    }
    X[e] = acc;
  }
}

// K2b: raw[i][j] = sum_m X[i][m] psi[j][m], box half-width wR = wX + rho
__global__ void k_psi_galerkin(PsiWin pw, int rho, const double* __restrict__ psi,
                               int wX, const double* __restrict__ X, int wR,
                               double* __restrict__ raw, long long e0, long long e1) {
  const int n = pw.n;
  const int SX = box_slots(wX, 1), SR = box_slots(wR, 1);
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / SR;
    const int sl = (int)(e - i * SR);
    const int si = (int)(i / n), ti = (int)(i % n);
    const int js = si + sl / (2 * wR + 1) - wR, jt = ti + sl % (2 * wR + 1) - wR;
    double acc = 0.0;
    if (js >= 0 && js < n && jt >= 0 && jt < n) {
      const int os = pw.origin(js), ot = pw.origin(jt);
      const double* prow = psi + ((long long)js * n + jt) * pw.wd * pw.wd;
      const double* xrow = X + i * SX;
      const int ms0 = imax(imax(si - wX, 0), imax(os, js - rho));
      const int ms1 = imin(imin(si + wX, n - 1), imin(os + pw.wd - 1, js + rho));
      const int mt0 = imax(imax(ti - wX, 0), imax(ot, jt - rho));
      const int mt1 = imin(imin(ti + wX, n - 1), imin(ot + pw.wd - 1, jt + rho));
      for (int ms = ms0; ms <= ms1; ++ms) {
        for (int mt = mt0; mt <= mt1; ++mt) {
          const double xv = xrow[slot_of(wX, 1, ms - si, mt - ti, 0)];
          if (xv == 0.0) continue;
          acc += xv * prow[(ms - os) * pw.wd + (mt - ot)];
        }
      }
    }
    raw[e] = acc;
  }
}

// ---------------------------------------------------------------------------
// K2b, coalesced form: the same sums over transposed operands.  psi^(q)
// (N x wd^2 windows) and X (N x SX box slots) are transposed to plane-major
// (psiT[w][i], XT[slot][i]); a CTA owns one fine row si and 32 consecutive
// nodes ti (lane = ti offset) for all SR output slots, so every operand load
// of a warp is one contiguous 256-byte run.  Each output is the gather
// kernel's FMA chain (ms, then mt ascending) without the zero-skip (adding a
// +-0 product leaves a sum unchanged up to the sign of a zero); the 32 x SR
// output block is staged in shared memory and written contiguously.
// ---------------------------------------------------------------------------
__global__ void k_transpose_f64(long long R, int C, const double* __restrict__ in,
                                double* __restrict__ out, long long ldo) {
  __shared__ double t[32][33];
  const long long r0 = (long long)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const long long r = r0 + k;
    const int c = c0 + threadIdx.x;
    if (r < R && c < C) t[k][threadIdx.x] = in[r * C + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k;
    const long long r = r0 + threadIdx.x;
    if (r < R && c < C) out[(long long)c * ldo + r] = t[threadIdx.x][k];
  }
}

constexpr int GT_THREADS = 256;

__global__ void __launch_bounds__(GT_THREADS) k_psi_galerkin_t(PsiWin pw, int rho,
                                                               const double* __restrict__ psiT,
                                                               int wX, const double* __restrict__ XT,
                                                               int wR, double* __restrict__ raw,
                                                               int s0, int s1, long long ld) {
  extern __shared__ double ob[];  // 32 x SR
  const int n = pw.n;
  const long long N = ld;  // plane stride of psiT / XT (the node count they hold)
  const int SR = box_slots(wR, 1), WR = 2 * wR + 1, WX = 2 * wX + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncb = (n + 31) / 32;
  for (long long cta = (long long)s0 * ncb + blockIdx.x; cta < (long long)s1 * ncb;
       cta += gridDim.x) {
    const int si = (int)(cta / ncb), ti0 = (int)(cta - (long long)si * ncb) * 32;
    const int ti = ti0 + lane;
    const bool live = ti < n;
    const long long i = (long long)si * n + ti;
    for (int sl = warp; sl < SR; sl += GT_THREADS / 32) {
      const int ds = sl / WR - wR, dt = sl - (sl / WR) * WR - wR;
      const int js = si + ds, jt = ti + dt;
      double acc = 0.0;
      if (live && js >= 0 && js < n && jt >= 0 && jt < n) {
        const int os = pw.origin(js), ot = pw.origin(jt);
        const long long j = (long long)js * n + jt;
        const int ms0 = imax(imax(si - wX, 0), imax(os, js - rho));
        const int ms1 = imin(imin(si + wX, n - 1), imin(os + pw.wd - 1, js + rho));
        const int mt0 = imax(imax(ti - wX, 0), imax(ot, jt - rho));
        const int mt1 = imin(imin(ti + wX, n - 1), imin(ot + pw.wd - 1, jt + rho));
        for (int ms = ms0; ms <= ms1; ++ms) {
          const double* xp = XT + ((long long)(ms - si + wX) * WX - ti + wX) * N + i;
          const double* pp = psiT + ((long long)(ms - os) * pw.wd - ot) * N + j;
          for (int mt = mt0; mt <= mt1; ++mt)
            acc = fma(__ldg(xp + (long long)mt * N), __ldg(pp + (long long)mt * N), acc);
        }
      }
      ob[lane * SR + sl] = acc;
    }
    __syncthreads();
    const int nl = imin(32, n - ti0);
    double* dst = raw + ((long long)si * n + ti0) * SR;
    for (int e = threadIdx.x; e < nl * SR; e += GT_THREADS) dst[e] = ob[e];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K3: level blocks.  A: box on Lk x Lk (wA).  Parent grid Lp = Lk/2.
// ---------------------------------------------------------------------------
struct Blk {
  double T[4][4];
};

__device__ __forceinline__ void load_T(int Lk, int wA, const double* __restrict__ A,
                                       int ps, int pt, int qs, int qt, Blk& t) {
  const int SA = box_slots(wA, 1);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int as = 2 * ps + (a >> 1), at = 2 * pt + (a & 1);
    const long long ra = (long long)as * Lk + at;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int bs = 2 * qs + (b >> 1), bt = 2 * qt + (b & 1);
      const int ds = bs - as, dt = bt - at;
      t.T[a][b] = (ds >= -wA && ds <= wA && dt >= -wA && dt <= wA)
                      ? A[ra * SA + slot_of(wA, 1, ds, dt, 0)]
                      : 0.0;
    }
  }
}

// B_ij[c][c'] = sum_b (sum_a W[c][a] T[a][b]) W[c'][b]   (X = W A, then X W^T)
// B_ji[c'][c] = sum_a (sum_b W[c'][b] T[a][b]) W[c][a]   (same from the other side)
__device__ __forceinline__ void block_products(const WTemplate& W, const Blk& t,
                                               double X[3][4], double Bij[3][3],
                                               double Bji[3][3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (W.w[c][a] != 0.0) acc += W.w[c][a] * t.T[a][b];
      X[c][b] = acc;
    }
  }
  double Xp[3][4];  // Xp[c'][a] = sum_b W[c'][b] T[a][b]
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (W.w[c][b] != 0.0) acc += W.w[c][b] * t.T[a][b];
      Xp[c][a] = acc;
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int cp = 0; cp < 3; ++cp) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (W.w[cp][b] != 0.0) acc += X[c][b] * W.w[cp][b];
      Bij[c][cp] = acc;
      double acc2 = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (W.w[c][a] != 0.0) acc2 += Xp[cp][a] * W.w[c][a];
      Bji[cp][c] = acc2;
    }
  }
}

__global__ void k_level_diag(int Lk, int wA, const double* __restrict__ A,
                             WTemplate W, double* __restrict__ bdiag,
                             double* __restrict__ dmin, long long e0, long long e1) {
  const int Lp = Lk / 2;
  double m = __longlong_as_double(0x7ff0000000000000ll);
  for (long long p = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; p < e1;
       p += (long long)gridDim.x * blockDim.x) {
    const int ps = (int)(p / Lp), pt = (int)(p % Lp);
    Blk t;
    load_T(Lk, wA, A, ps, pt, ps, pt, t);
    double X[3][4], Bij[3][3], Bji[3][3];
    block_products(W, t, X, Bij, Bji);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double d = (Bij[c][c] + Bji[c][c]) * 0.5;
      bdiag[p * 3 + c] = d;
      m = fmin(m, d);
    }
  }
  m = warp_min(m);
  if ((threadIdx.x & 31) == 0) {
    unsigned long long* a = reinterpret_cast<unsigned long long*>(dmin);
    unsigned long long old = *a, assumed;
    do {
      assumed = old;
      if (__longlong_as_double((long long)assumed) <= m) break;
      old = atomicCAS(a, assumed, (unsigned long long)__double_as_longlong(m));
    } while (assumed != old);
  }
}

// B (nr=nc=3, wB), G (nr=3, nc=1, wB), PAPt (nr=nc=1, wB).  One thread per
// (parent, offset).  stats[0..1] = B repair max|Bij-Bji|, max|Bij|.
__global__ void k_level_blocks(int Lk, int wA, const double* __restrict__ A,
                               WTemplate W, int wB,
                               const double* __restrict__ bdiag,
                               const double* __restrict__ dmin,
                               double* __restrict__ B, double* __restrict__ G,
                               double* __restrict__ PAPt,
                               double* __restrict__ stats, long long e0, long long e1) {
  const int Lp = Lk / 2;
  const int W2 = 2 * wB + 1, NB = W2 * W2;
  const bool do_drop = *dmin > 0.0;
  const int SB = NB * 9 / 3;  // slots per B row: NB * 3
  double mdiff = 0.0, mabs = 0.0;
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long p = e / NB;
    const int bs = (int)(e - p * NB);
    const int ps = (int)(p / Lp), pt = (int)(p % Lp);
    const int ds = bs / W2 - wB, dt = bs % W2 - wB;
    const int qs = ps + ds, qt = pt + dt;
    double* Bout = B + p * 3 * SB;
    if (qs < 0 || qs >= Lp || qt < 0 || qt >= Lp) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int cp = 0; cp < 3; ++cp) Bout[c * SB + bs * 3 + cp] = 0.0;
        G[(p * 3 + c) * NB + bs] = 0.0;
      }
      PAPt[p * NB + bs] = 0.0;
      continue;
    }
    Blk t;
    load_T(Lk, wA, A, ps, pt, qs, qt, t);
    double X[3][4], Bij[3][3], Bji[3][3];
    block_products(W, t, X, Bij, Bji);
    const long long q = (long long)qs * Lp + qt;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int cp = 0; cp < 3; ++cp) {
        const double a = Bij[c][cp], b = Bji[cp][c];
        mdiff = fmax(mdiff, fabs(a - b));
        mabs = fmax(mabs, fabs(a));
        double v = (a + b) * 0.5;
        const bool diag = (ds == 0 && dt == 0 && c == cp);
        if (do_drop && !diag) {
          if (!(fabs(v) >= 1e-12 * sqrt(bdiag[p * 3 + c] * bdiag[q * 3 + cp]))) v = 0.0;
        }
        Bout[c * SB + bs * 3 + cp] = v;
      }
      // G = X pibar^T: children of q ascending, each X * 0.25
      double g = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) g += X[c][b] * 0.25;
      G[(p * 3 + c) * NB + bs] = g;
    }
    // PAPt: PA[b] = sum_a T[a][b] (a ascending), then sum_b PA[b]
    double pap = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const double pa = ((t.T[0][b] + t.T[1][b]) + t.T[2][b]) + t.T[3][b];
      pap += pa;
    }
    PAPt[p * NB + bs] = pap;
  }
  mdiff = warp_max(mdiff);
  mabs = warp_max(mabs);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(&stats[0], mdiff);
    atomic_max_nonneg(&stats[1], mabs);
  }
}

// ---------------------------------------------------------------------------
// K6: R = 0.25 P + Dt W.  R box on the parent grid, nc = 4 children, w = rho.
// ---------------------------------------------------------------------------
__global__ void k_restriction(int Lp, int rho, const double* __restrict__ Dt,
                              WTemplate W, double* __restrict__ R, long long e0,
                              long long e1) {
  const int W2 = 2 * rho + 1, NB = W2 * W2;
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / NB;
    const int bs = (int)(e - i * NB);
    const int si = (int)(i / Lp), ti = (int)(i % Lp);
    const int ds = bs / W2 - rho, dt = bs % W2 - rho;
    const int qs = si + ds, qt = ti + dt;
    double* out = R + e * 4;
    if (qs < 0 || qs >= Lp || qt < 0 || qt >= Lp) {
#pragma unroll
      for (int b = 0; b < 4; ++b) out[b] = 0.0;
      continue;
    }
    const double* d = Dt + i * (NB * 3) + bs * 3;
    const double d0 = d[0], d1 = d[1], d2 = d[2];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double acc = 0.0;
      if (W.w[0][b] != 0.0 && d0 != 0.0) acc += d0 * W.w[0][b];
      if (W.w[1][b] != 0.0 && d1 != 0.0) acc += d1 * W.w[1][b];
      if (W.w[2][b] != 0.0 && d2 != 0.0) acc += d2 * W.w[2][b];
      out[b] = (ds == 0 && dt == 0) ? 0.25 + acc : acc;
    }
  }
}

// BD[(p,c)][j] = sum_{r' asc} B[(p,c)][r'] * Dt[j][(p'-j, c')],  w = wB + rho
__global__ void k_bd(int Lp, int wB, const double* __restrict__ B, int rho,
                     const double* __restrict__ Dt, int wBD, double* __restrict__ BD,
                     long long e0, long long e1) {
  const int SB = box_slots(wB, 3), SD = box_slots(rho, 3), SBD = box_slots(wBD, 1);
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / SBD;
    const int sl = (int)(e - r * SBD);
    const long long p = r / 3;
    const int ps = (int)(p / Lp), pt = (int)(p % Lp);
    const int js = ps + sl / (2 * wBD + 1) - wBD, jt = pt + sl % (2 * wBD + 1) - wBD;
    double acc = 0.0;
    if (js >= 0 && js < Lp && jt >= 0 && jt < Lp) {
      const double* brow = B + r * SB;
      const double* drow = Dt + ((long long)js * Lp + jt) * SD;
      const int a0 = imax(imax(ps - wB, js - rho), 0), a1 = imin(imin(ps + wB, js + rho), Lp - 1);
      const int b0 = imax(imax(pt - wB, jt - rho), 0), b1 = imin(imin(pt + wB, jt + rho), Lp - 1);
      for (int qs = a0; qs <= a1; ++qs) {
        for (int qt = b0; qt <= b1; ++qt) {
          const double* bb = brow + slot_of(wB, 3, qs - ps, qt - pt, 0);
          const double* dd = drow + slot_of(rho, 3, qs - js, qt - jt, 0);
#pragma unroll
          for (int cp = 0; cp < 3; ++cp) {
            const double bv = bb[cp], dv = dd[cp];
            if (bv != 0.0 && dv != 0.0) acc += bv * dv;
          }
        }
      }
    }
    BD[e] = acc;
  }
}

// GtD[i][j] = sum_{r asc} G[r][i] * Dt[j][r],  box nr=nc=1, w = wG + rho
__global__ void k_gtd(int Lp, int wG, const double* __restrict__ G, int rho,
                      const double* __restrict__ Dt, int wGD, double* __restrict__ GtD,
                      long long e0, long long e1) {
  const int SG = box_slots(wG, 1), SD = box_slots(rho, 3), SO = box_slots(wGD, 1);
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / SO;
    const int sl = (int)(e - i * SO);
    const int is = (int)(i / Lp), it = (int)(i % Lp);
    const int js = is + sl / (2 * wGD + 1) - wGD, jt = it + sl % (2 * wGD + 1) - wGD;
    double acc = 0.0;
    if (js >= 0 && js < Lp && jt >= 0 && jt < Lp) {
      const double* drow = Dt + ((long long)js * Lp + jt) * SD;
      const int a0 = imax(imax(is - wG, js - rho), 0), a1 = imin(imin(is + wG, js + rho), Lp - 1);
      const int b0 = imax(imax(it - wG, jt - rho), 0), b1 = imin(imin(it + wG, jt + rho), Lp - 1);
      for (int ps = a0; ps <= a1; ++ps) {
        for (int pt = b0; pt <= b1; ++pt) {
          const long long p = (long long)ps * Lp + pt;
          const int gsl = slot_of(wG, 1, is - ps, it - pt, 0);
          const double* dd = drow + slot_of(rho, 3, ps - js, pt - jt, 0);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double gv = G[(p * 3 + c) * SG + gsl], dv = dd[c];
            if (gv != 0.0 && dv != 0.0) acc += gv * dv;
          }
        }
      }
    }
    GtD[e] = acc;
  }
}

// raw A^(k-1)[i][j] = ((0.0625 PAPt + GtD_ij) + GtD_ji) + DtBD_ij,
// DtBD_ij = sum_{r asc} Dt[i][r] BD[r][j].  Box w = wA2 (>= 2 rho + wB).
__global__ void k_coarse_raw(int Lp, int wB, const double* __restrict__ PAPt,
                             int wGD, const double* __restrict__ GtD, int rho,
                             const double* __restrict__ Dt, int wBD,
                             const double* __restrict__ BD, int wA2,
                             double* __restrict__ raw, long long e0, long long e1) {
  const int SP = box_slots(wB, 1), SGD = box_slots(wGD, 1), SD = box_slots(rho, 3),
            SBD = box_slots(wBD, 1), SO = box_slots(wA2, 1);
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / SO;
    const int sl = (int)(e - i * SO);
    const int is = (int)(i / Lp), it = (int)(i % Lp);
    const int ds = sl / (2 * wA2 + 1) - wA2, dt = sl % (2 * wA2 + 1) - wA2;
    const int js = is + ds, jt = it + dt;
    double v = 0.0;
    if (js >= 0 && js < Lp && jt >= 0 && jt < Lp) {
      const long long j = (long long)js * Lp + jt;
      double pap = 0.0, gij = 0.0, gji = 0.0;
      if (ds >= -wB && ds <= wB && dt >= -wB && dt <= wB)
        pap = PAPt[i * SP + slot_of(wB, 1, ds, dt, 0)];
      if (ds >= -wGD && ds <= wGD && dt >= -wGD && dt <= wGD) {
        gij = GtD[i * SGD + slot_of(wGD, 1, ds, dt, 0)];
        gji = GtD[j * SGD + slot_of(wGD, 1, -ds, -dt, 0)];
      }
      double acc = 0.0;
      const double* drow = Dt + i * SD;
      const int a0 = imax(imax(is - rho, js - wBD), 0), a1 = imin(imin(is + rho, js + wBD), Lp - 1);
      const int b0 = imax(imax(it - rho, jt - wBD), 0), b1 = imin(imin(it + rho, jt + wBD), Lp - 1);
      for (int ps = a0; ps <= a1; ++ps) {
        for (int pt = b0; pt <= b1; ++pt) {
          const double* dd = drow + slot_of(rho, 3, ps - is, pt - it, 0);
          const long long p = (long long)ps * Lp + pt;
          const int bsl = slot_of(wBD, 1, js - ps, jt - pt, 0);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double dv = dd[c];
            if (dv == 0.0) continue;
            const double bv = BD[(p * 3 + c) * SBD + bsl];
            if (bv != 0.0) acc += dv * bv;
          }
        }
      }
      v = ((0.0625 * pap + gij) + gji) + acc;
    }
    raw[e] = v;
  }
}

// ---------------------------------------------------------------------------
// psi^(k-1) = drop_row(0.25 P psi + Dt (W psi))
// Wpsi rows (p, c) on the parent grid, window (lo_k, wdw = min(wd_k + h, n))
// with parent spacing 2h.
// ---------------------------------------------------------------------------
__global__ void k_wpsi(PsiWin child, WTemplate W, const double* __restrict__ psi,
                       PsiWin par, double* __restrict__ Wpsi, long long e0, long long e1,
                       int f0, int f1) {
  // par.L = child.L / 2, par.lo = child.lo, par.wd = wdw; only window points
  // whose fine row lies in [f0, f1) are computed (column strips of psi)
  const int Lp = par.L;
  const long long per = (long long)par.wd * par.wd;
  const long long cper = (long long)child.wd * child.wd;
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long p = e / per;
    const int f = (int)(e - p * per);
    const int ps = (int)(p / Lp), pt = (int)(p % Lp);
    const int fs = par.origin(ps) + f / par.wd, ft = par.origin(pt) + f % par.wd;
    if (fs < f0 || fs >= f1) continue;
    double cv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int cs = 2 * ps + (a >> 1), ct = 2 * pt + (a & 1);
      const int os = child.origin(cs), ot = child.origin(ct);
      const int ls = fs - os, lt = ft - ot;
      cv[a] = (ls >= 0 && ls < child.wd && lt >= 0 && lt < child.wd)
                  ? psi[((long long)cs * child.L + ct) * cper + ls * child.wd + lt]
                  : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (W.w[c][a] != 0.0 && cv[a] != 0.0) acc += W.w[c][a] * cv[a];
      Wpsi[(p * 3 + c) * per + f] = acc;
    }
  }
}

// raw psi^(k-1) rows; the row-tail drop runs afterwards (k_row_tail_drop)
__global__ void k_psi_next(PsiWin child, const double* __restrict__ psi,
                           PsiWin par, const double* __restrict__ Wpsi, int rho,
                           const double* __restrict__ Dt, PsiWin out,
                           double* __restrict__ psi_next) {
  const int Lp = out.L;
  const long long per = (long long)out.wd * out.wd;
  const long long total = (long long)Lp * Lp * per;  // (whole level only)
  const long long cper = (long long)child.wd * child.wd;
  const long long wper = (long long)par.wd * par.wd;
  const int SD = box_slots(rho, 3);
  const int h = child.h();  // child spacing in fine units; parent spacing 2h
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / per;
    const int f = (int)(e - i * per);
    const int is = (int)(i / Lp), it = (int)(i % Lp);
    const int fs = out.origin(is) + f / out.wd, ft = out.origin(it) + f % out.wd;
    // P psi: the 4 children of i
    double pv = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int cs = 2 * is + (a >> 1), ct = 2 * it + (a & 1);
      const int ls = fs - child.origin(cs), lt = ft - child.origin(ct);
      if (ls >= 0 && ls < child.wd && lt >= 0 && lt < child.wd)
        pv += psi[((long long)cs * child.L + ct) * cper + ls * child.wd + lt];
    }
    // Dt (W psi): parents p in ball(i, rho) whose Wpsi support covers f.
    // support of Wpsi row p: fine [2p h + lo, (2p+1) h + hi] with
    // hi = lo + wd_child - 1 (unclamped), so 2p h in [f - h - hi, f - lo]
    const int lo = child.lo, hi = child.hi;
    double acc = 0.0;
    const double* drow = Dt + i * SD;
    const int a0 = imax(imax(is - rho, 0), (fs - h - hi + 2 * h - 1) / (2 * h) - 1);
    const int a1 = imin(imin(is + rho, Lp - 1), (fs - lo) / (2 * h) + 1);
    const int b0 = imax(imax(it - rho, 0), (ft - h - hi + 2 * h - 1) / (2 * h) - 1);
    const int b1 = imin(imin(it + rho, Lp - 1), (ft - lo) / (2 * h) + 1);
    for (int ps = a0; ps <= a1; ++ps) {
      const int ls = fs - par.origin(ps);
      if (ls < 0 || ls >= par.wd) continue;
      for (int pt = b0; pt <= b1; ++pt) {
        const int lt = ft - par.origin(pt);
        if (lt < 0 || lt >= par.wd) continue;
        const double* dd = drow + slot_of(rho, 3, ps - is, pt - it, 0);
        const long long p = (long long)ps * Lp + pt;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double dv = dd[c];
          if (dv == 0.0) continue;
          const double wv = Wpsi[(p * 3 + c) * wper + ls * par.wd + lt];
          if (wv != 0.0) acc += dv * wv;
        }
      }
    }
    psi_next[e] = 0.25 * pv + acc;
  }
}


// ---------------------------------------------------------------------------
// psi^(k-1) raw rows as a block-sparse tensor-core GEMM (DMMA m8n8k4):
// for a block of TB x TB output rows i and a tile F of 8 x 4 fine points,
// Out[i][f] = sum_r Dt[i][r] Wpsi[r][f] over the parents r in the union of
// the rows' balls whose Wpsi window meets F (K chunked by 32), then
// + 0.25 P psi in the epilogue.  The accumulation order differs from the
// reference's sequential SpGEMM; at q = 6, 7 no row-tail-drop decision
// changed (measured), values agree to ~4e-16.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_acc(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

constexpr int PN_LDA = 36, PN_LDB = 36, PN_KC = 32;
// fine-point tile of one CTA: PN_FR rows x PN_FC consecutive columns (32 points)
#ifndef GB_PN_FC
#define GB_PN_FC 4
#endif
constexpr int PN_FC = GB_PN_FC, PN_FR = 32 / PN_FC;

__device__ __forceinline__ int floordiv(int a, int b) {  // b > 0
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}

__global__ void __launch_bounds__(128) k_psi_next_mma(PsiWin child, const double* __restrict__ psi,
                                                      PsiWin par, const double* __restrict__ Wpsi,
                                                      int rho, const double* __restrict__ Dt,
                                                      PsiWin out, double* __restrict__ psi_next,
                                                      double* __restrict__ rowmax, int TB, int nfs,
                                                      int nft, int r0, int r1, int f0, int f1) {
  // double-buffered: chunk c + 1 is gathered into registers while chunk c
  // is multiplied (the gathers are L2-latency bound)
  __shared__ double As[2][16 * PN_LDA];
  __shared__ double Bs[2][PN_KC * PN_LDB];
  // separable per-k tables: B address = kbB + (fs wd + ft), A slot = kakey -
  // (row offset); window / ball tests on the packed (s << 16 | t) positions
  // (-1 = padding column)
  __shared__ long long kbB[2][PN_KC];
  __shared__ int kbpos[2][PN_KC], kakey[2][PN_KC], kapos[2][PN_KC];
  const int Lp = out.L;
  const int nbs = (Lp + TB - 1) / TB;
  // output parent rows [r0, r1) only: the row blocks meeting the strip
  const int rb0 = r0 / TB, rb1 = (r1 + TB - 1) / TB;
  const long long nblk = (long long)(rb1 - rb0) * nbs;
  const int tpb = nfs * nft;
  const long long ntiles = nblk * tpb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int side = 2 * rho + 1;
  const int SD = box_slots(rho, 3);
  const long long wper = (long long)par.wd * par.wd;
  const long long cper = (long long)child.wd * child.wd;
  const long long oper = (long long)out.wd * out.wd;
  const int h = child.h();  // child spacing (fine units); parents 2h
  const int lo = child.lo, hi = child.hi;
  // h and TB are powers of two (dyadic levels; TB = min(Lp, 4)): the floor
  // divisions of the tile setup and of the epilogue are shifts
  const int sh2h = 31 - __clz(2 * h), tbs = 31 - __clz(TB);
  const unsigned ntl = (unsigned)ntiles;  // (< 2^31 tiles: checked by the launcher)
  for (unsigned t = blockIdx.x; t < ntl; t += gridDim.x) {
    const unsigned blk = t / (unsigned)tpb;
    const int tt = (int)(t - blk * (unsigned)tpb);
    const unsigned bq = blk / (unsigned)nbs;
    const int bi_s = (rb0 + (int)bq) << tbs, bi_t = (int)(blk - bq * (unsigned)nbs) << tbs;
    const int nrs = imin(TB, Lp - bi_s), nrt = imin(TB, Lp - bi_t);
    // union of the block rows' windows (origins are monotone in the row)
    const int us0 = out.origin(bi_s), us1 = out.origin(bi_s + nrs - 1) + out.wd - 1;
    const int ut0 = out.origin(bi_t), ut1 = out.origin(bi_t + nrt - 1) + out.wd - 1;
    const int F0s = us0 + (tt / nft) * PN_FR, F0t = ut0 + (tt % nft) * PN_FC;
    if (F0s > us1 || F0t > ut1) continue;  // (uniform across the CTA)
    if (F0s + PN_FR - 1 < f0 || F0s >= f1) continue;  // no fine row of the column strip [f0, f1)
    // parents in some ball whose Wpsi support [2ph+lo, 2ph+h+hi] meets F
    int ps0 = imax(bi_s - rho, 0), ps1 = imin(bi_s + nrs - 1 + rho, Lp - 1);
    int pt0 = imax(bi_t - rho, 0), pt1 = imin(bi_t + nrt - 1 + rho, Lp - 1);
    ps0 = imax(ps0, (F0s - h - hi) >> sh2h);  // floor division by 2 h
    ps1 = imin(ps1, (F0s + PN_FR - 1 - lo) >> sh2h);
    pt0 = imax(pt0, (F0t - h - hi) >> sh2h);
    pt1 = imin(pt1, (F0t + PN_FC - 1 - lo) >> sh2h);
    const int nps = ps1 - ps0 + 1, npt = pt1 - pt0 + 1;
    const int K = (nps > 0 && npt > 0) ? nps * npt * 3 : 0;
    double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    // the A rows this thread gathers: m = threadIdx.x / 8 (+ fixed), kk strided
    const int am = threadIdx.x >> 3;  // 0..15
    const int ams = am >> tbs, amt = am - (ams << tbs);
    const int ais = bi_s + ams, ait = bi_t + amt;
    const bool arow = am < TB * TB && ams < nrs && amt < nrt && ais >= r0 && ais < r1;
    const double* drow = Dt + ((long long)ais * Lp + ait) * SD;
    const int n_ = threadIdx.x & 31;
    const int bfs = F0s + n_ / PN_FC, bft = F0t + n_ % PN_FC;
    // chunk metadata (threads < PN_KC) into buffer u
    const int arowoff = ((ais - rho) * side + (ait - rho)) * 3;
    const long long bfsw = (long long)bfs * par.wd + bft;
    auto meta = [&](int k0, int u) {
      if (threadIdx.x < PN_KC) {
        const int kk = k0 + threadIdx.x;
        long long bb = 0;
        int bpos = -1, akey = 0, apos = -1;
        if (kk < K) {
          const int pl = kk / 3;
          const int cc = kk - 3 * pl;
          const int ps = ps0 + pl / npt;
          const int pt = pt0 + pl % npt;
          const int os = par.origin(ps), ot = par.origin(pt);
          bb = ((long long)(ps * Lp + pt) * 3 + cc) * wper - (long long)os * par.wd - ot;
          bpos = (os << 16) | ot;
          akey = (ps * side + pt) * 3 + cc;
          apos = (ps << 16) | pt;
        }
        kbB[u][threadIdx.x] = bb;
        kbpos[u][threadIdx.x] = bpos;
        kakey[u][threadIdx.x] = akey;
        kapos[u][threadIdx.x] = apos;
      }
    };
    double ra[4], rb[8];
    // gather A (16 rows x 32 k: Dt, 0 outside the row's ball / padding rows)
    // and B (32 k x 32 fine points: Wpsi, 0 outside the parent's window)
    auto gather = [&](int u) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int kk = (threadIdx.x & 7) + 8 * j;
        const int ap = kapos[u][kk];
        double v = 0.0;
        if (arow && ap >= 0) {
          const unsigned ds = (unsigned)((ap >> 16) - ais + rho);
          const unsigned dt = (unsigned)((ap & 0xffff) - ait + rho);
          if (ds <= (unsigned)(2 * rho) && dt <= (unsigned)(2 * rho))
            v = drow[kakey[u][kk] - arowoff];
        }
        ra[j] = v;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int kk = (threadIdx.x >> 5) + 4 * j;
        const int bp = kbpos[u][kk];
        double v = 0.0;
        if (bp >= 0) {
          const unsigned ls = (unsigned)(bfs - (bp >> 16)), lt = (unsigned)(bft - (bp & 0xffff));
          if (ls < (unsigned)par.wd && lt < (unsigned)par.wd) v = __ldg(Wpsi + kbB[u][kk] + bfsw);
        }
        rb[j] = v;
      }
    };
    if (K > 0) {
      meta(0, 0);
      __syncthreads();
      gather(0);
    }
    for (int k0 = 0, cb = 0; k0 < K; k0 += PN_KC, cb ^= 1) {
#pragma unroll
      for (int j = 0; j < 4; ++j) As[cb][am * PN_LDA + (threadIdx.x & 7) + 8 * j] = ra[j];
#pragma unroll
      for (int j = 0; j < 8; ++j) Bs[cb][((threadIdx.x >> 5) + 4 * j) * PN_LDB + n_] = rb[j];
      const bool more = k0 + PN_KC < K;
      if (more) meta(k0 + PN_KC, cb ^ 1);
      __syncthreads();
      if (more) gather(cb ^ 1);
#pragma unroll
      for (int ks = 0; ks < PN_KC / 4; ++ks) {
        const double b = Bs[cb][(ks * 4 + (lane & 3)) * PN_LDB + warp * 8 + (lane >> 2)];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const double a = As[cb][(mt * 8 + (lane >> 2)) * PN_LDA + ks * 4 + (lane & 3)];
          dmma_acc(c[mt][0], c[mt][1], a, b);
        }
      }
    }
    __syncthreads();  // buffers are reused by the next tile
    // epilogue: + 0.25 P psi, store inside each row's window, row max
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int m = mt * 8 + (lane >> 2);
      const int ms = m >> tbs, mtt = m - (ms << tbs);
      const int is = bi_s + ms, it = bi_t + mtt;
      const bool live = m < TB * TB && ms < nrs && mtt < nrt && is >= r0 && is < r1;
      double amax = 0.0;
      if (live) {
        const int os = out.origin(is), ot = out.origin(it);
        // the four children of row (is, it): window origins and row bases once
        const int cos0 = child.origin(2 * is), cos1 = child.origin(2 * is + 1);
        const int cot0 = child.origin(2 * it), cot1 = child.origin(2 * it + 1);
        const double* cb00 = psi + ((long long)(2 * is) * child.L + 2 * it) * cper;
        const double* cb10 = cb00 + (long long)child.L * cper;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int n = warp * 8 + 2 * (lane & 3) + j;
          const int fs = F0s + n / PN_FC, ft = F0t + n % PN_FC;
          const int ls = fs - os, lt = ft - ot;
          if (ls < 0 || ls >= out.wd || lt < 0 || lt >= out.wd) continue;
          if (fs < f0 || fs >= f1) continue;
          double pv = 0.0;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const unsigned ks = (unsigned)(fs - ((a >> 1) ? cos1 : cos0));
            const unsigned kt = (unsigned)(ft - ((a & 1) ? cot1 : cot0));
            if (ks < (unsigned)child.wd && kt < (unsigned)child.wd)
              pv += ((a >> 1) ? cb10 : cb00)[(a & 1) * cper + ks * child.wd + kt];
          }
          const double v = 0.25 * pv + c[mt][j];
          psi_next[((long long)is * Lp + it) * oper + ls * out.wd + lt] = v;
          amax = fmax(amax, fabs(v));
        }
      }
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
      if (live && (lane & 3) == 0 && amax > 0.0)
        atomic_max_nonneg(rowmax + (long long)is * Lp + it, amax);
    }
  }
}

// row max of each dense row (CTA per row chunk) for the row-tail drop
constexpr int RT_CHUNK = 4096;
__global__ void k_rowmax_chunks(long long rows, long long S, const double* __restrict__ v,
                                double* __restrict__ rowmax) {
  __shared__ double sh[32];
  const long long nch = (S + RT_CHUNK - 1) / RT_CHUNK;
  for (long long b = blockIdx.x; b < rows * nch; b += gridDim.x) {
    const long long r = b / nch, j0 = (b - r * nch) * RT_CHUNK;
    const long long j1 = j0 + RT_CHUNK < S ? j0 + RT_CHUNK : S;
    double m = 0.0;
    for (long long j = j0 + threadIdx.x; j < j1; j += blockDim.x) m = fmax(m, fabs(v[r * S + j]));
    m = block_max(m, sh);
    if (threadIdx.x == 0 && m > 0.0) atomic_max_nonneg(rowmax + r, m);
    __syncthreads();
  }
}

// |x| < 1e-11 * rowmax -> 0 (gamblet_fast.py:172-190)
__global__ void k_drop_by_rowmax(long long rows, long long S, double* __restrict__ v,
                                 const double* __restrict__ rowmax) {
  const long long nch = (S + RT_CHUNK - 1) / RT_CHUNK;
  for (long long b = blockIdx.x; b < rows * nch; b += gridDim.x) {
    const long long r = b / nch, j0 = (b - r * nch) * RT_CHUNK;
    const long long j1 = j0 + RT_CHUNK < S ? j0 + RT_CHUNK : S;
    const double thr = 1e-11 * rowmax[r];
    for (long long j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      const double x = v[r * S + j];
      if (!(fabs(x) >= thr)) v[r * S + j] = 0.0;
    }
  }
}

// the same drop restricted to the window rows whose fine row lies in
// [f0, f1) (column strips of psi: the other window rows belong to other ranks)
__global__ void k_drop_by_rowmax_cols(PsiWin out, long long row0, long long rows,
                                      double* __restrict__ v, const double* __restrict__ rowmax,
                                      int f0, int f1) {
  const long long S = (long long)out.wd * out.wd;
  const long long nch = (S + RT_CHUNK - 1) / RT_CHUNK;
  for (long long b = blockIdx.x; b < rows * nch; b += gridDim.x) {
    const long long r = row0 + b / nch;
    const int os = out.origin((int)(r / out.L));
    const long long ja = (long long)imax(f0 - os, 0) * out.wd;
    const long long jb = (long long)imin(f1 - os, out.wd) * out.wd;
    long long j0 = (b % nch) * RT_CHUNK, j1 = j0 + RT_CHUNK < S ? j0 + RT_CHUNK : S;
    j0 = j0 > ja ? j0 : ja;
    j1 = j1 < jb ? j1 : jb;
    const double thr = 1e-11 * rowmax[r];
    for (long long j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      const double x = v[r * S + j];
      if (!(fabs(x) >= thr)) v[r * S + j] = 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// operand / epilogue functors of the triple-product block GEMMs (gb_boxgemm.cuh)
// ---------------------------------------------------------------------------
// Every operand address is separable: addr = ipart(i) + qpart(q), valid for
// |q - i| <= hw (slot_of is linear in the offset) -- the GEMM gathers with
// two table lookups per element instead of the per-element index chain.
struct OpBrows {  // A operand: B[(i,mc)][(q,c)]
  const double* B;
  int Lp, w, S;
  __device__ const double* base() const { return B; }
  __device__ int hw() const { return w; }
  __device__ long long ipart(int is, int it, int mc) const {
    const int W2 = 2 * w + 1;
    return (((long long)is * Lp + it) * 3 + mc) * S - (long long)(is * W2 + it) * 3 +
           (w * W2 + w) * 3;
  }
  __device__ long long qpart(int qs, int qt, int kc) const {
    return (long long)(qs * (2 * w + 1) + qt) * 3 + kc;
  }
  __device__ double operator()(int is, int it, int mc, int qs, int qt, int kc) const {
    const int ds = qs - is, dt = qt - it;
    if (ds < -w || ds > w || dt < -w || dt > w) return 0.0;
    return B[(((long long)is * Lp + it) * 3 + mc) * S + slot_of(w, 3, ds, dt, kc)];
  }
};
struct OpDtRowsA {  // A operand: Dt[i][(q,c)]
  const double* Dt;
  int Lp, rho, S;
  __device__ const double* base() const { return Dt; }
  __device__ int hw() const { return rho; }
  __device__ long long ipart(int is, int it, int) const {
    const int W2 = 2 * rho + 1;
    return ((long long)is * Lp + it) * S - (long long)(is * W2 + it) * 3 + (rho * W2 + rho) * 3;
  }
  __device__ long long qpart(int qs, int qt, int kc) const {
    return (long long)(qs * (2 * rho + 1) + qt) * 3 + kc;
  }
  __device__ double operator()(int is, int it, int, int qs, int qt, int kc) const {
    const int ds = qs - is, dt = qt - it;
    if (ds < -rho || ds > rho || dt < -rho || dt > rho) return 0.0;
    return Dt[((long long)is * Lp + it) * S + slot_of(rho, 3, ds, dt, kc)];
  }
};
struct OpDtRowsB {  // B operand: Dt[j][(q,c)]  (i.e. D)
  const double* Dt;
  int Lp, rho, S;
  __device__ const double* base() const { return Dt; }
  __device__ int hw() const { return rho; }
  __device__ long long ipart(int js, int jt, int) const {
    const int W2 = 2 * rho + 1;
    return ((long long)js * Lp + jt) * S - (long long)(js * W2 + jt) * 3 + (rho * W2 + rho) * 3;
  }
  __device__ long long qpart(int qs, int qt, int kc) const {
    return (long long)(qs * (2 * rho + 1) + qt) * 3 + kc;
  }
  __device__ double operator()(int qs, int qt, int kc, int js, int jt) const {
    const int ds = qs - js, dt = qt - jt;
    if (ds < -rho || ds > rho || dt < -rho || dt > rho) return 0.0;
    return Dt[((long long)js * Lp + jt) * S + slot_of(rho, 3, ds, dt, kc)];
  }
};
struct OpGcols {  // A operand: G^T, G[(q,c)][i]
  const double* G;
  int Lp, w, S;
  __device__ const double* base() const { return G; }
  __device__ int hw() const { return w; }
  __device__ long long ipart(int is, int it, int) const {
    return (long long)is * (2 * w + 1) + it;
  }
  __device__ long long qpart(int qs, int qt, int kc) const {
    const int W2 = 2 * w + 1;
    return (((long long)qs * Lp + qt) * 3 + kc) * S - (long long)(qs * W2 + qt) + (w * W2 + w);
  }
  __device__ double operator()(int is, int it, int, int qs, int qt, int kc) const {
    const int ds = is - qs, dt = it - qt;
    if (ds < -w || ds > w || dt < -w || dt > w) return 0.0;
    return G[(((long long)qs * Lp + qt) * 3 + kc) * S + slot_of(w, 1, ds, dt, 0)];
  }
};
struct OpBDrows {  // B operand: BD[(q,c)][j]
  const double* BD;
  int Lp, w, S;
  __device__ const double* base() const { return BD; }
  __device__ int hw() const { return w; }
  __device__ long long ipart(int js, int jt, int) const {
    return (long long)js * (2 * w + 1) + jt;
  }
  __device__ long long qpart(int qs, int qt, int kc) const {
    const int W2 = 2 * w + 1;
    return (((long long)qs * Lp + qt) * 3 + kc) * S - (long long)(qs * W2 + qt) + (w * W2 + w);
  }
  __device__ double operator()(int qs, int qt, int kc, int js, int jt) const {
    const int ds = js - qs, dt = jt - qt;
    if (ds < -w || ds > w || dt < -w || dt > w) return 0.0;
    return BD[(((long long)qs * Lp + qt) * 3 + kc) * S + slot_of(w, 1, ds, dt, 0)];
  }
};
struct StoreBox {
  double* out;
  int Lp, MC, w, S;
  __device__ void store(int is, int it, int mc, int js, int jt, double v) const {
    out[(((long long)is * Lp + it) * MC + mc) * S + slot_of(w, 1, js - is, jt - it, 0)] = v;
  }
};
struct StoreRaw {  // ((0.0625 PAPt + GtD_ij) + GtD_ji) + DtBD_ij
  double* raw;
  const double *PAPt, *GtD;
  int Lp, wB, wGD, wA2;
  __device__ void store(int is, int it, int, int js, int jt, double acc) const {
    const int ds = js - is, dt = jt - it;
    const long long i = (long long)is * Lp + it, j = (long long)js * Lp + jt;
    double pap = 0.0, gij = 0.0, gji = 0.0;
    if (ds >= -wB && ds <= wB && dt >= -wB && dt <= wB)
      pap = PAPt[i * box_slots(wB, 1) + slot_of(wB, 1, ds, dt, 0)];
    if (ds >= -wGD && ds <= wGD && dt >= -wGD && dt <= wGD) {
      gij = GtD[i * box_slots(wGD, 1) + slot_of(wGD, 1, ds, dt, 0)];
      gji = GtD[j * box_slots(wGD, 1) + slot_of(wGD, 1, -ds, -dt, 0)];
    }
    raw[i * box_slots(wA2, 1) + slot_of(wA2, 1, ds, dt, 0)] = ((0.0625 * pap + gij) + gji) + acc;
  }
};

}  // namespace gb

using namespace gb;

static inline int grid_for(long long work, int block, int cap = 148 * 32) {
  long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

static int products_use_mma = 1;
int gbk_products_mode(int mma) {
  const int old = products_use_mma;
  if (mma >= 0) products_use_mma = mma;
  return old;
}

static inline WTemplate mkW(const double* w12) {
  WTemplate W;
  for (int c = 0; c < 3; ++c)
    for (int a = 0; a < 4; ++a) W.w[c][a] = w12[c * 4 + a];
  return W;
}

// Row-range launchers (multi-GPU strips, partition.py): [r0, r1) are grid rows
// of the OUTPUT's row grid; only those rows are written, inputs are read at
// global indices (the caller provides the halo rows).  The whole-level entry
// points are the [0, L) instances, so a partition's strips reproduce the whole
// level bitwise.
static inline bool bad_rows(int r0, int r1, int L) { return r0 < 0 || r1 > L || r0 > r1; }

int gbk_psi_stencil_rows(int n, int lo, int wd, int rho, const double* psi, int wA,
                         const double* A, int wX, double* X, int r0, int r1, cudaStream_t s) {
  if (bad_rows(r0, r1, n)) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  PsiWin pw{n, n, lo, wd, -lo};
  const long long per = (long long)n * box_slots(wX, 1);
  k_psi_stencil<<<grid_for((r1 - r0) * per, 256), 256, 0, s>>>(pw, rho, psi, wA, A, wX, X,
                                                              r0 * per, r1 * per);
  return (int)cudaGetLastError();
}
int gbk_psi_stencil(int n, int lo, int wd, int rho, const double* psi, int wA,
                    const double* A, int wX, double* X, cudaStream_t s) {
  return gbk_psi_stencil_rows(n, lo, wd, rho, psi, wA, A, wX, X, 0, n, s);
}

size_t gbk_psi_galerkin_workspace(int n, int wd, int wX) {
  return (size_t)n * n * ((size_t)wd * wd + (size_t)box_slots(wX, 1)) * sizeof(double);
}
// workspace of the strip [r0, r1): planes over the nodes of the strip's rows
// widened by wR (psi) -- X uses the same plane stride
size_t gbk_psi_galerkin_workspace_rows(int n, int wd, int wX, int wR, int r0, int r1) {
  const int h0 = imax(r0 - wR, 0), h1 = imin(r1 + wR, n);
  return (size_t)(h1 - h0) * n * ((size_t)wd * wd + (size_t)box_slots(wX, 1)) * sizeof(double);
}

// fine rows [r0, r1) of raw: psi rows within wR of the strip and the strip's X
// rows are transposed into their global plane-major positions of `work`
int gbk_psi_galerkin_t_rows(int n, int lo, int wd, int rho, const double* psi, int wX,
                            const double* X, int wR, double* raw, double* work, int r0, int r1,
                            cudaStream_t s) {
  if (bad_rows(r0, r1, n)) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  PsiWin pw{n, n, lo, wd, -lo};
  const long long N = (long long)n * n;
  const int SX = box_slots(wX, 1), SR = box_slots(wR, 1);
  const dim3 tb(32, 8);
  const int h0 = imax(r0 - wR, 0), h1 = imin(r1 + wR, n);
  const long long pa = (long long)h0 * n, pn = (long long)(h1 - h0) * n;
  // planes hold the nodes [pa, pa + pn) only (plane stride pn); psiT / XT are
  // the bases shifted so that a global node index addresses them (whole
  // level: pa = 0, pn = N)
  (void)N;
  double* psiT = work - pa;
  double* XT = work + pn * wd * wd - pa;
  k_transpose_f64<<<dim3((unsigned)((pn + 31) / 32), (wd * wd + 31) / 32), tb, 0, s>>>(
      pn, wd * wd, psi + pa * wd * wd, psiT + pa, pn);
  const long long xa = (long long)r0 * n, xn = (long long)(r1 - r0) * n;
  k_transpose_f64<<<dim3((unsigned)((xn + 31) / 32), (SX + 31) / 32), tb, 0, s>>>(
      xn, SX, X + xa * SX, XT + xa, pn);
  const size_t smem = (size_t)32 * SR * sizeof(double);
  if (smem > 200 * 1024) return GB_UNSUPPORTED;
  cudaError_t e = cudaFuncSetAttribute(k_psi_galerkin_t,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  const long long nct = (long long)(r1 - r0) * ((n + 31) / 32);
  const int g = (int)(nct < 148LL * 8 ? nct : 148LL * 8);
  k_psi_galerkin_t<<<g, GT_THREADS, smem, s>>>(pw, rho, psiT, wX, XT, wR, raw, r0, r1, pn);
  return (int)cudaGetLastError();
}
int gbk_psi_galerkin_t(int n, int lo, int wd, int rho, const double* psi, int wX,
                       const double* X, int wR, double* raw, double* work, cudaStream_t s) {
  return gbk_psi_galerkin_t_rows(n, lo, wd, rho, psi, wX, X, wR, raw, work, 0, n, s);
}

int gbk_psi_galerkin(int n, int lo, int wd, int rho, const double* psi, int wX,
                     const double* X, int wR, double* raw, cudaStream_t s) {
  PsiWin pw{n, n, lo, wd, -lo};
  const long long total = (long long)n * n * box_slots(wR, 1);
  k_psi_galerkin<<<grid_for(total, 256), 256, 0, s>>>(pw, rho, psi, wX, X, wR, raw, 0, total);
  return (int)cudaGetLastError();
}

int gbk_level_diag_rows(int Lk, int wA, const double* A, const double* w12, double* bdiag,
                        double* dmin, int r0, int r1, cudaStream_t s) {
  const int Lp = Lk / 2;
  if (bad_rows(r0, r1, Lp)) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  k_level_diag<<<grid_for((long long)(r1 - r0) * Lp, 128), 128, 0, s>>>(
      Lk, wA, A, mkW(w12), bdiag, dmin, (long long)r0 * Lp, (long long)r1 * Lp);
  return (int)cudaGetLastError();
}
int gbk_level_diag(int Lk, int wA, const double* A, const double* w12,
                   double* bdiag, double* dmin, cudaStream_t s) {
  return gbk_level_diag_rows(Lk, wA, A, w12, bdiag, dmin, 0, Lk / 2, s);
}

int gbk_level_blocks_rows(int Lk, int wA, const double* A, const double* w12, int wB,
                          const double* bdiag, const double* dmin, double* B, double* G,
                          double* PAPt, double* stats, int r0, int r1, cudaStream_t s) {
  const int Lp = Lk / 2;
  if (bad_rows(r0, r1, Lp)) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long per = (long long)Lp * box_slots(wB, 1);
  k_level_blocks<<<grid_for((r1 - r0) * per, 128), 128, 0, s>>>(
      Lk, wA, A, mkW(w12), wB, bdiag, dmin, B, G, PAPt, stats, r0 * per, r1 * per);
  return (int)cudaGetLastError();
}
int gbk_level_blocks(int Lk, int wA, const double* A, const double* w12, int wB,
                     const double* bdiag, const double* dmin, double* B, double* G,
                     double* PAPt, double* stats, cudaStream_t s) {
  return gbk_level_blocks_rows(Lk, wA, A, w12, wB, bdiag, dmin, B, G, PAPt, stats, 0, Lk / 2, s);
}

int gbk_restriction_rows(int Lp, int rho, const double* Dt, const double* w12, double* R,
                         int r0, int r1, cudaStream_t s) {
  if (bad_rows(r0, r1, Lp)) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long per = (long long)Lp * box_slots(rho, 1);
  k_restriction<<<grid_for((r1 - r0) * per, 256), 256, 0, s>>>(Lp, rho, Dt, mkW(w12), R,
                                                              r0 * per, r1 * per);
  return (int)cudaGetLastError();
}
int gbk_restriction(int Lp, int rho, const double* Dt, const double* w12, double* R,
                    cudaStream_t s) {
  return gbk_restriction_rows(Lp, rho, Dt, w12, R, 0, Lp, s);
}

// Tile loops are oversubscribed (48 CTAs per SM, grid-stride): the short
// CTAs free SMs continuously, so the level engine's high-priority SpMV CTAs
// (a whole SM each) are scheduled while the products run.  A one-wave
// persistent grid measured slower: it holds every SM until the kernel ends.
template <class Kern>
static int resident_grid(Kern, int, long long ntiles) {
  return (int)(ntiles < 148LL * 48 ? ntiles : 148LL * 48);
}
// tiles of the row blocks [rb0, rb1) of the TB x TB blocking
static long long box_gemm_tiles(int Lp, int TB, int wOut, int rb0, int rb1) {
  const long long nb = (Lp + TB - 1) / TB, side = 2 * ((wOut + TB - 1) / TB) + 1;
  const long long nt = (long long)(rb1 - rb0) * nb * side * side;
  // the kernel counts tiles in 32 bits; the largest level (Lp = 2048) has 2.7e7
  return nt < (1LL << 31) ? nt : 0;
}
// the tensor-core tile kernels own whole TB-row blocks: a strip must start and
// end on a block boundary (or the grid edge)
static inline bool rows_block_aligned(int r0, int r1, int Lp, int TB) {
  return r0 % TB == 0 && (r1 % TB == 0 || r1 == Lp);
}

int gbk_bd_rows(int Lp, int wB, const double* B, int rho, const double* Dt, int wBD,
                double* BD, int r0, int r1, cudaStream_t s) {
  if (bad_rows(r0, r1, Lp)) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long per = (long long)Lp * 3 * box_slots(wBD, 1);
  const int TB = Lp < 4 ? Lp : 4;
  if (products_use_mma && rows_block_aligned(r0, r1, Lp, TB)) {
    cudaError_t e = cudaMemsetAsync(BD + r0 * per, 0, (r1 - r0) * per * sizeof(double), s);
    if (e != cudaSuccess) return (int)e;
    const int rb0 = r0 / TB, rb1 = (r1 + TB - 1) / TB;
    auto kern = k_box_gemm<3, OpBrows, OpDtRowsB, StoreBox>;
    const long long nt = box_gemm_tiles(Lp, TB, wBD, rb0, rb1);
    if (nt == 0) return GB_UNSUPPORTED;
    kern<<<resident_grid(kern, 128, nt), 128, 0, s>>>(
        Lp, TB, wB, rho, wBD, OpBrows{B, Lp, wB, box_slots(wB, 3)},
        OpDtRowsB{Dt, Lp, rho, box_slots(rho, 3)}, StoreBox{BD, Lp, 3, wBD, box_slots(wBD, 1)},
        rb0, rb1);
    return (int)cudaGetLastError();
  }
  if (products_use_mma) return GB_UNSUPPORTED;  // same arithmetic as the whole level only
  k_bd<<<grid_for((r1 - r0) * per, 256), 256, 0, s>>>(Lp, wB, B, rho, Dt, wBD, BD, r0 * per,
                                                     r1 * per);
  return (int)cudaGetLastError();
}
int gbk_bd(int Lp, int wB, const double* B, int rho, const double* Dt, int wBD,
           double* BD, cudaStream_t s) {
  return gbk_bd_rows(Lp, wB, B, rho, Dt, wBD, BD, 0, Lp, s);
}

int gbk_gtd_rows(int Lp, int wG, const double* G, int rho, const double* Dt, int wGD,
                 double* GtD, int r0, int r1, cudaStream_t s) {
  if (bad_rows(r0, r1, Lp)) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long per = (long long)Lp * box_slots(wGD, 1);
  const int TB = Lp < 4 ? Lp : 4;
  if (products_use_mma && rows_block_aligned(r0, r1, Lp, TB)) {
    cudaError_t e = cudaMemsetAsync(GtD + r0 * per, 0, (r1 - r0) * per * sizeof(double), s);
    if (e != cudaSuccess) return (int)e;
    const int rb0 = r0 / TB, rb1 = (r1 + TB - 1) / TB;
    auto kern = k_box_gemm<1, OpGcols, OpDtRowsB, StoreBox>;
    const long long nt = box_gemm_tiles(Lp, TB, wGD, rb0, rb1);
    if (nt == 0) return GB_UNSUPPORTED;
    kern<<<resident_grid(kern, 128, nt), 128, 0, s>>>(
        Lp, TB, wG, rho, wGD, OpGcols{G, Lp, wG, box_slots(wG, 1)},
        OpDtRowsB{Dt, Lp, rho, box_slots(rho, 3)}, StoreBox{GtD, Lp, 1, wGD, box_slots(wGD, 1)},
        rb0, rb1);
    return (int)cudaGetLastError();
  }
  if (products_use_mma) return GB_UNSUPPORTED;
  k_gtd<<<grid_for((r1 - r0) * per, 256), 256, 0, s>>>(Lp, wG, G, rho, Dt, wGD, GtD, r0 * per,
                                                      r1 * per);
  return (int)cudaGetLastError();
}
int gbk_gtd(int Lp, int wG, const double* G, int rho, const double* Dt, int wGD,
            double* GtD, cudaStream_t s) {
  return gbk_gtd_rows(Lp, wG, G, rho, Dt, wGD, GtD, 0, Lp, s);
}

int gbk_coarse_raw_rows(int Lp, int wB, const double* PAPt, int wGD, const double* GtD,
                        int rho, const double* Dt, int wBD, const double* BD, int wA2,
                        double* raw, int r0, int r1, cudaStream_t s) {
  if (bad_rows(r0, r1, Lp)) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long per = (long long)Lp * box_slots(wA2, 1);
  const int TB = Lp < 4 ? Lp : 4;
  if (products_use_mma && rows_block_aligned(r0, r1, Lp, TB)) {
    cudaError_t e = cudaMemsetAsync(raw + r0 * per, 0, (r1 - r0) * per * sizeof(double), s);
    if (e != cudaSuccess) return (int)e;
    const int rb0 = r0 / TB, rb1 = (r1 + TB - 1) / TB;
    auto kern = k_box_gemm<1, OpDtRowsA, OpBDrows, StoreRaw>;
    const long long nt = box_gemm_tiles(Lp, TB, wA2, rb0, rb1);
    if (nt == 0) return GB_UNSUPPORTED;
    kern<<<resident_grid(kern, 128, nt), 128, 0, s>>>(
        Lp, TB, rho, wBD, wA2, OpDtRowsA{Dt, Lp, rho, box_slots(rho, 3)},
        OpBDrows{BD, Lp, wBD, box_slots(wBD, 1)}, StoreRaw{raw, PAPt, GtD, Lp, wB, wGD, wA2},
        rb0, rb1);
    return (int)cudaGetLastError();
  }
  if (products_use_mma) return GB_UNSUPPORTED;
  k_coarse_raw<<<grid_for((r1 - r0) * per, 256), 256, 0, s>>>(Lp, wB, PAPt, wGD, GtD, rho, Dt,
                                                             wBD, BD, wA2, raw, r0 * per,
                                                             r1 * per);
  return (int)cudaGetLastError();
}
int gbk_coarse_raw(int Lp, int wB, const double* PAPt, int wGD, const double* GtD,
                   int rho, const double* Dt, int wBD, const double* BD, int wA2,
                   double* raw, cudaStream_t s) {
  return gbk_coarse_raw_rows(Lp, wB, PAPt, wGD, GtD, rho, Dt, wBD, BD, wA2, raw, 0, Lp, s);
}

// Wpsi rows of the parents in grid rows [r0, r1); only window points whose
// fine row is in [f0, f1) are written (column strips of the coarse levels)
int gbk_wpsi_rows(int n, int Lk, int lo, int wd, const double* w12, const double* psi,
                  int wdw, double* Wpsi, int r0, int r1, int f0, int f1, cudaStream_t s) {
  const int Lp = Lk / 2;
  if (bad_rows(r0, r1, Lp) || f0 < 0 || f1 > n || f0 > f1) return GB_UNSUPPORTED;
  if (r0 == r1 || f0 == f1) return 0;
  PsiWin child{n, Lk, lo, wd, 0}, par{n, Lp, lo, wdw, 0};
  const long long per = (long long)Lp * wdw * wdw;
  k_wpsi<<<grid_for((r1 - r0) * per, 256), 256, 0, s>>>(child, mkW(w12), psi, par, Wpsi,
                                                       r0 * per, r1 * per, f0, f1);
  return (int)cudaGetLastError();
}
int gbk_wpsi(int n, int Lk, int lo, int wd, const double* w12, const double* psi,
             int wdw, double* Wpsi, cudaStream_t s) {
  return gbk_wpsi_rows(n, Lk, lo, wd, w12, psi, wdw, Wpsi, 0, Lk / 2, 0, n, s);
}

// output parent rows [r0, r1) only (tensor-core mode required for a proper
// strip, GB_UNSUPPORTED otherwise): rows outside are not written.  Raw rows and
// their row maxima; window points with a fine row outside [f0, f1) are
// neither computed nor written (column strips: the caller max-reduces rowmax
// over the column owners before the drop).
int gbk_psi_next_raw_rows(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw,
                          const double* Wpsi, int rho, const double* Dt, int lo2, int wd2,
                          double* psi_next, double* rowmax, int r0, int r1, int f0, int f1,
                          cudaStream_t s) {
  PsiWin child{n, Lk, lo, wd, hi}, par{n, Lk / 2, lo, wdw, 0}, out{n, Lk / 2, lo2, wd2, 0};
  const int Lp = Lk / 2;
  if (r0 < 0 || r1 > Lp || r0 > r1 || f0 < 0 || f1 > n || f0 > f1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const bool whole = r0 == 0 && r1 == Lp && f0 == 0 && f1 == n;
  if (!products_use_mma && !whole) return GB_UNSUPPORTED;
  const long long S = (long long)wd2 * wd2;
  const long long rows = (long long)(r1 - r0) * Lp, roff = (long long)r0 * Lp;
  cudaError_t e = cudaMemsetAsync(rowmax + roff, 0, rows * sizeof(double), s);
  if (e != cudaSuccess) return (int)e;
  if (f0 == f1) return 0;
  if (products_use_mma) {
    const int TB = Lp < 4 ? Lp : 4;
    const int hp = n / Lp;  // output row spacing (fine units)
    const int span = imin(wd2 + (TB - 1) * hp, n);
    const int nfs = (span + PN_FR - 1) / PN_FR, nft = (span + PN_FC - 1) / PN_FC;
    const long long nb = (Lp + TB - 1) / TB;
    const long long nrb = (r1 + TB - 1) / TB - r0 / TB;
    const long long nt = nrb * nb * nfs * nft;
    if (nt >= (1LL << 31)) return GB_UNSUPPORTED;  // the kernel counts tiles in 32 bits
    const int g = resident_grid(k_psi_next_mma, 128, nt);
    k_psi_next_mma<<<g, 128, 0, s>>>(child, psi, par, Wpsi, rho, Dt, out, psi_next, rowmax, TB,
                                     nfs, nft, r0, r1, f0, f1);
  } else {
    const long long total = rows * S;
    k_psi_next<<<grid_for(total, 256), 256, 0, s>>>(child, psi, par, Wpsi, rho, Dt, out,
                                                     psi_next);
    const long long nch = rows * ((S + RT_CHUNK - 1) / RT_CHUNK);
    k_rowmax_chunks<<<(int)(nch < 148LL * 32 ? nch : 148LL * 32), 256, 0, s>>>(rows, S, psi_next,
                                                                              rowmax);
  }
  return (int)cudaGetLastError();
}

// the row-tail drop of psi rows [r0, r1) given their maxima; window rows with
// a fine row outside [f0, f1) are left alone
int gbk_psi_drop_rows(int n, int Lp, int lo2, int wd2, double* psi_next, const double* rowmax,
                      int r0, int r1, int f0, int f1, cudaStream_t s) {
  if (r0 < 0 || r1 > Lp || r0 > r1 || f0 < 0 || f1 > n || f0 > f1) return GB_UNSUPPORTED;
  if (r0 == r1 || f0 == f1) return 0;
  const long long S = (long long)wd2 * wd2;
  const long long rows = (long long)(r1 - r0) * Lp, roff = (long long)r0 * Lp;
  const long long nch = rows * ((S + RT_CHUNK - 1) / RT_CHUNK);
  const int g = (int)(nch < 148LL * 32 ? nch : 148LL * 32);
  if (f0 == 0 && f1 == n) {
    k_drop_by_rowmax<<<g, 256, 0, s>>>(rows, S, psi_next + roff * S, rowmax + roff);
  } else {
    PsiWin out{n, Lp, lo2, wd2, 0};
    k_drop_by_rowmax_cols<<<g, 256, 0, s>>>(out, roff, rows, psi_next, rowmax, f0, f1);
  }
  return (int)cudaGetLastError();
}

int gbk_psi_next_rows(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw,
                      const double* Wpsi, int rho, const double* Dt, int lo2, int wd2,
                      double* psi_next, double* rowmax, int r0, int r1, cudaStream_t s) {
  const int rc = gbk_psi_next_raw_rows(n, Lk, lo, hi, wd, psi, wdw, Wpsi, rho, Dt, lo2, wd2,
                                       psi_next, rowmax, r0, r1, 0, n, s);
  if (rc != 0) return rc;
  return gbk_psi_drop_rows(n, Lk / 2, lo2, wd2, psi_next, rowmax, r0, r1, 0, n, s);
}
int gbk_psi_next(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw,
                 const double* Wpsi, int rho, const double* Dt, int lo2, int wd2,
                 double* psi_next, double* rowmax, cudaStream_t s) {
  return gbk_psi_next_rows(n, Lk, lo, hi, wd, psi, wdw, Wpsi, rho, Dt, lo2, wd2, psi_next, rowmax,
                           0, Lk / 2, s);
}
