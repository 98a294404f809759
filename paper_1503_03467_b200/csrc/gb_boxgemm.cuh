// Box-stencil block GEMM on the FP64 tensor cores (DMMA m8n8k4) for the
// split triple product A^(k-1) = 0.0625 P A P^T + G^T D + D^T G + D^T B D
// (gamblet_fast.py:590-612).  One CTA computes an output tile of TB x TB row
// parents (x MC components) by TB x TB column parents; K runs over the
// parents (x 3 components) both operands can touch, in ascending
// (q_s, q_t, c) order -- the CSR column order the reference's SpGEMM
// accumulates in -- so every output is the same sequential FMA chain as the
// per-entry gather (zero products are skipped or added as +0, which does not
// change a nonzero sum).  Operand/epilogue access is supplied by functors:
//   a(i_s, i_t, m_comp, q_s, q_t, k_comp)  (0 outside the operand's box)
//   b(q_s, q_t, k_comp, j_s, j_t)
//   out.store(i_s, i_t, m_comp, j_s, j_t, acc)   called for |j - i| <= wOut
#pragma once
#include "gb_common.cuh"

namespace gb {

__device__ __forceinline__ void dmma_884b(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

constexpr int BG_KC = 32, BG_LDA = 36, BG_LDB = 20;

// MC: row components (1 or 3) -> M = 16 MC rows, N = 16 columns, 4 warps;
// warp w: n-tile w & 1, m-tiles (w >> 1) + 2 j, j < MC.
template <int MC, class AOp, class BOp, class OutOp>
__global__ void __launch_bounds__(128) k_box_gemm(int Lp, int TB, int wa, int wb, int wOut,
                                                  AOp aop, BOp bop, OutOp out, int rb0,
                                                  int rb1) {
  // double-buffered: chunk c + 1 is gathered into registers while chunk c is
  // multiplied (the operand gathers are L2-latency bound)
  __shared__ double As[2][16 * MC * BG_LDA];
  __shared__ double Bs[2][BG_KC * BG_LDB];
  __shared__ long long aro[16 * MC], bco[16], akq[2][BG_KC], bkq[2][BG_KC];  // separable offsets
  __shared__ int arp[16 * MC], bcp[16], kq[2][BG_KC];  // packed (s << 16 | t), -1 = none
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (Lp + TB - 1) / TB;
  const int nbo = (wOut + TB - 1) / TB;
  const int side = 2 * nbo + 1;
  // row blocks [rb0, rb1) of the output only (row strips; whole level: [0, nb))
  const long long ntiles = (long long)(rb1 - rb0) * nb * side * side;
  const double* Ab = aop.base();
  const double* Bb = bop.base();
  const int wA = aop.hw(), wB_ = bop.hw();
  // TB = min(Lp, 4) is a power of two: the tile-local divisions are shifts;
  // tiles are counted in 32 bits (the launchers check the count)
  const int tbs = 31 - __clz(TB);
  const unsigned ss = (unsigned)(side * side), ntl = (unsigned)ntiles;
  for (unsigned t = blockIdx.x; t < ntl; t += gridDim.x) {
    const unsigned mbl = t / ss;
    const int ob = (int)(t - mbl * ss);
    const unsigned mb = mbl + (unsigned)rb0 * (unsigned)nb;
    const int mbs = (int)(mb / (unsigned)nb), mbt = (int)(mb - (unsigned)mbs * (unsigned)nb);
    const int obs = ob / side;
    const int nbs = mbs + obs - nbo, nbt = mbt + (ob - obs * side) - nbo;
    if (nbs < 0 || nbs >= nb || nbt < 0 || nbt >= nb) continue;  // CTA-uniform
    const int i0s = mbs << tbs, i0t = mbt << tbs, j0s = nbs << tbs, j0t = nbt << tbs;
    const int nis = imin(TB, Lp - i0s), nit = imin(TB, Lp - i0t);
    const int njs = imin(TB, Lp - j0s), njt = imin(TB, Lp - j0t);
    // skip tiles with no (i, j) pair inside the output box
    if (j0s - (i0s + nis - 1) > wOut || i0s - (j0s + njs - 1) > wOut ||
        j0t - (i0t + nit - 1) > wOut || i0t - (j0t + njt - 1) > wOut)
      continue;
    const int qs0 = imax(imax(i0s - wa, j0s - wb), 0);
    const int qs1 = imin(imin(i0s + nis - 1 + wa, j0s + njs - 1 + wb), Lp - 1);
    const int qt0 = imax(imax(i0t - wa, j0t - wb), 0);
    const int qt1 = imin(imin(i0t + nit - 1 + wa, j0t + njt - 1 + wb), Lp - 1);
    const int nqs = qs1 - qs0 + 1, nqt = qt1 - qt0 + 1;
    const int K = (nqs > 0 && nqt > 0) ? nqs * nqt * 3 : 0;
    // per-tile row / column tables
    if (threadIdx.x < 16 * MC) {
      const int m = threadIdx.x;
      const int lm = m / MC, mc = m - lm * MC;
      const int ls = lm >> tbs, lt = lm - (ls << tbs);
      const bool ok = lm < TB * TB && ls < nis && lt < nit;
      arp[m] = ok ? (((i0s + ls) << 16) | (i0t + lt)) : -1;
      aro[m] = ok ? aop.ipart(i0s + ls, i0t + lt, mc) : 0;
    } else if (threadIdx.x >= 64 && threadIdx.x < 80) {
      const int nn = threadIdx.x - 64;
      const int ls = nn >> tbs, lt = nn - (ls << tbs);
      const bool ok = nn < TB * TB && ls < njs && lt < njt;
      bcp[nn] = ok ? (((j0s + ls) << 16) | (j0t + lt)) : -1;
      bco[nn] = ok ? bop.ipart(j0s + ls, j0t + lt, 0) : 0;
    }
    double c[MC][2];
#pragma unroll
    for (int j = 0; j < MC; ++j) c[j][0] = c[j][1] = 0.0;
    auto meta = [&](int k0, int u) {
      if (threadIdx.x < BG_KC) {
        const int kk = k0 + threadIdx.x;
        int code = -1;
        long long ao = 0, bo = 0;
        if (kk < K) {
          const int pl = kk / 3, cc = kk - 3 * pl;
          const int qs = qs0 + pl / nqt, qt = qt0 + pl % nqt;
          code = (qs << 16) | qt;
          ao = aop.qpart(qs, qt, cc);
          bo = bop.qpart(qs, qt, cc);
        }
        kq[u][threadIdx.x] = code;
        akq[u][threadIdx.x] = ao;
        bkq[u][threadIdx.x] = bo;
      }
    };
    double ra[4 * MC], rb[4];
    // A: (16 MC) x 32; thread: fixed k column, rows warp + 4 r.
    // B: 32 x 16; thread: fixed column nn = t & 15, rows (t >> 4) + 8 r
    auto gather = [&](int u) {
      {
        const int kk = threadIdx.x & 31;
        const int code = kq[u][kk];
        const int qs = code >> 16, qt = code & 0xffff;
        const long long ko = akq[u][kk];
#pragma unroll
        for (int r = 0; r < 4 * MC; ++r) {
          const int m = warp + 4 * r;
          const int rp = arp[m];
          double v = 0.0;
          if (code >= 0 && rp >= 0) {
            const unsigned ds = (unsigned)(qs - (rp >> 16) + wA), dt = (unsigned)(qt - (rp & 0xffff) + wA);
            if (ds <= (unsigned)(2 * wA) && dt <= (unsigned)(2 * wA)) v = Ab[aro[m] + ko];
          }
          ra[r] = v;
        }
      }
      {
        const int nn = threadIdx.x & 15;
        const int cp = bcp[nn];
        const long long co = bco[nn];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int kk = (threadIdx.x >> 4) + 8 * r;
          const int code = kq[u][kk];
          double v = 0.0;
          if (code >= 0 && cp >= 0) {
            const unsigned ds = (unsigned)((code >> 16) - (cp >> 16) + wB_);
            const unsigned dt = (unsigned)((code & 0xffff) - (cp & 0xffff) + wB_);
            if (ds <= (unsigned)(2 * wB_) && dt <= (unsigned)(2 * wB_)) v = Bb[bkq[u][kk] + co];
          }
          rb[r] = v;
        }
      }
    };
    if (K > 0) {
      meta(0, 0);
      __syncthreads();  // also publishes the row / column tables
      gather(0);
    }
    for (int k0 = 0, cb = 0; k0 < K; k0 += BG_KC, cb ^= 1) {
#pragma unroll
      for (int r = 0; r < 4 * MC; ++r) As[cb][(warp + 4 * r) * BG_LDA + (threadIdx.x & 31)] = ra[r];
#pragma unroll
      for (int r = 0; r < 4; ++r) Bs[cb][((threadIdx.x >> 4) + 8 * r) * BG_LDB + (threadIdx.x & 15)] = rb[r];
      const bool more = k0 + BG_KC < K;
      if (more) meta(k0 + BG_KC, cb ^ 1);
      __syncthreads();
      if (more) gather(cb ^ 1);
      const int nt = warp & 1;
#pragma unroll
      for (int ks = 0; ks < BG_KC / 4; ++ks) {
        const double b = Bs[cb][(ks * 4 + (lane & 3)) * BG_LDB + nt * 8 + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < MC; ++j) {
          const int mt = (warp >> 1) + 2 * j;
          const double a = As[cb][(mt * 8 + (lane >> 2)) * BG_LDA + ks * 4 + (lane & 3)];
          dmma_884b(c[j][0], c[j][1], a, b);
        }
      }
    }
    __syncthreads();  // tables and buffers are rewritten by the next tile
    // epilogue
    const int nt = warp & 1;
#pragma unroll
    for (int j = 0; j < MC; ++j) {
      const int mt = (warp >> 1) + 2 * j;
      const int m = mt * 8 + (lane >> 2);
      const int lm = m / MC, mc = m - lm * MC;
      const int ls = lm >> tbs, lt = lm - (ls << tbs);
      if (lm >= TB * TB || ls >= nis || lt >= nit) continue;
      const int is = i0s + ls, it = i0t + lt;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int nn = nt * 8 + 2 * (lane & 3) + h;
        const int ns = nn >> tbs, ntt = nn - (ns << tbs);
        if (nn >= TB * TB || ns >= njs || ntt >= njt) continue;
        const int js = j0s + ns, jt = j0t + ntt;
        if (js - is > wOut || is - js > wOut || jt - it > wOut || it - jt > wOut) continue;
        out.store(is, it, mc, js, jt, c[j][h]);
      }
    }
  }
}

}  // namespace gb
