// Symmetric band SpMV (v6) for the tiled Krylov levels (nr = 3, L % 64 == 0).
//
// S B S is symmetric, so only its upper half is streamed from HBM: for every
// parent p the 3x3 blocks U_e[c][c'] = (S B S)[(p,c), (p+d_e,c')] of the
// npos = 2w^2 + 2w positive offsets d_e (lexicographic: (0,1..w), then
// ds = 1..w, dt = -w..w) plus the full 3x3 diagonal block.  Layout: 32
// consecutive parents per block, slot pairs innermost across the 32 lanes
// (double2 per lane), NS = 9 npos + 10 slots per parent (diagonal block
// padded to 10):
//
//     U[((p >> 5) * NS/2 + m/2) * 64 + (p & 31) * 2 + (m & 1)],  m = 9e + 3c + c'.
//
// One thread per parent reads its own slots once and applies them twice:
// gather  y(p,c)      += U_e[c][c'] x(p+d_e, c')      (upper half)
// scatter y(p+d_e,c') += U_e[c][c'] x(p, c)           (lower half = U^T)
// The scatter goes to per-warp private accumulators in shared memory (for a
// fixed e the targets of a warp are distinct, e advances in program order with
// a __syncwarp: deterministic); a CTA owns a tile of kSymTH grid rows x 64
// parent columns.  Phase 1 combines the warps' accumulators in a fixed order,
// writes the tile's own rows of y (partial) and the spill-over region (rows
// below, columns left/right) to an overflow area at the tail of y.  Phase 2
// adds the neighbours' spill-over in a fixed order and does the CG / power
// reductions.  DRAM moves half the matrix bytes of the full box, every run is
// bitwise reproducible.
#pragma once
#ifndef GB_SYM_L2_STREAM
#define GB_SYM_L2_STREAM 1
#endif

#ifndef GB_SYM_TH
#define GB_SYM_TH 4
#endif
constexpr int kSymTH = GB_SYM_TH;  // grid rows per tile
constexpr int kSymTW = 64;   // parent columns per tile (two warps)
constexpr int kSymThreads = 2 * kSymTH * 32;

__host__ __device__ __forceinline__ int symb_npos(int w) { return 2 * w * w + 2 * w; }
__host__ __device__ __forceinline__ int symb_ns(int w) { return 9 * symb_npos(w) + 10; }
// spill region of a tile: rows [0, TH + w) x columns [-w, 64 + w) x 3
__host__ __device__ __forceinline__ int symb_region(int w) {
  return (kSymTH + w) * (kSymTW + 2 * w) * 3;
}
__host__ __device__ __forceinline__ long long symb_ntile(int L) {
  return (long long)(L / kSymTH) * (L / kSymTW);
}
__host__ __device__ __forceinline__ void symb_offset(int w, int e, int* ds, int* dt) {
  if (e < w) {
    *ds = 0;
    *dt = e + 1;
  } else {
    const int f = e - w;
    *ds = 1 + f / (2 * w + 1);
    *dt = f % (2 * w + 1) - w;
  }
}

// (S B S) upper blocks from the unscaled box, entry by entry the reference's
// materialized congruence (x * s_i) * s_j (gamblet_fast.py:136)
__global__ void k_scale_box_symb(int L, int w, const double* __restrict__ B,
                                 const double* __restrict__ s, double* __restrict__ U,
                                 long long e0, long long e1) {
  const int S = (2 * w + 1) * (2 * w + 1) * 3, NS = symb_ns(w), npos = symb_npos(w);
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long blk = e / (32LL * NS);
    const int rem = (int)(e - blk * 32LL * NS);
    const int m = ((rem >> 6) << 1) | (rem & 1);
    const long long p = blk * 32 + ((rem >> 1) & 31);
    const int ps = (int)(p / L), pt = (int)(p % L);
    double v = 0.0;
    if (m < 9 * npos) {
      const int eo = m / 9, c = (m % 9) / 3, cp = m % 3;
      int ds, dt;
      symb_offset(w, eo, &ds, &dt);
      const int qs = ps + ds, qt = pt + dt;
      if (qs < L && qt >= 0 && qt < L) {
        const long long r = p * 3 + c;
        v = B[r * S + slot_of(w, 3, ds, dt, cp)] * s[r] * s[((long long)qs * L + qt) * 3 + cp];
      }
    } else if (m < 9 * npos + 9) {
      const int c = (m - 9 * npos) / 3, cp = (m - 9 * npos) % 3;
      const long long r = p * 3 + c;
      v = B[r * S + slot_of(w, 3, 0, 0, cp)] * s[r] * s[p * 3 + cp];
    }
    U[e] = v;
  }
}

// spill-over sum of the neighbour tiles into own row (ps, pt, c), added to
// `own` in a fixed order (tile rows above by distance, columns left, same,
// right): the value phase 2 produces and the fused CG update consumes
__device__ __forceinline__ double symb_fix_value(double own, const double* __restrict__ ov,
                                                 int L, int w, int ps, int pt, int c) {
  const int WC = kSymTW + 2 * w, RG = symb_region(w), tpr = L / kSymTW;
  const int KI = (w + kSymTH - 1) / kSymTH;
  const int I = ps / kSymTH, h = ps - I * kSymTH, J = pt / kSymTW, j = pt - J * kSymTW;
  // the left tile's spill covers j < w, the right tile's j >= kSymTW - w
  const bool left = j < w && J > 0, right = j >= kSymTW - w && J + 1 < tpr;
  double s = own;
  for (int dI = 0; dI <= KI; ++dI) {
    const int Ip = I - dI, rr = h + dI * kSymTH;
    if (Ip < 0 || rr >= kSymTH + w) break;
    // region entry (rr, cc) of tile (Ip, Jp): (rr WC + cc + w) 3 + c
    const double* base = ov + ((long long)Ip * tpr + J) * RG + (rr * WC + w) * 3 + c;
    if (left) s += base[-RG + (j + kSymTW) * 3];
    if (dI > 0) s += base[j * 3];
    if (right) s += base[RG + (j - kSymTW) * 3];
  }
  return s;
}

// Phase 1: y_own (partial) and the tiles' spill-over, for NV vectors sharing
// one pass over U.  Vectors are zero-halo padded ((L+2w)^2 x 3); the spill
// area of y_v starts at y_v + (L+2w)^2 * 3.  red_v = 1: the CG reduction
// x_v . (A x_v) is formed here by linearity (every tile's partial sums over
// its whole region against the staged x window, out-of-domain x is the zero
// halo) and finish_reduction(mode 0) sets alpha -- the fused CG update
// (k_symb_bjcg_update) then adds the spill-over itself and no phase 2 runs.
template <int NV>
__global__ void __launch_bounds__(kSymThreads, 2) k_symb_apply(
    int L, int w, const double* __restrict__ U, const double* __restrict__ x0,
    double* __restrict__ y0, KState* s0, double* part0, int red0,
    const double* __restrict__ x1, double* __restrict__ y1, KState* s1, double* part1,
    int red1, long long tile0, long long tile1) {
  extern __shared__ double dyn[];
  __shared__ double sh[32];
  const bool live0 = !(s0 && s0->done);
  const bool live1 = NV == 2 && !(s1 && s1->done);
  if (!live0 && !live1) return;
  const bool rd0 = live0 && red0, rd1 = NV == 2 && live1 && red1;
  const int npos = symb_npos(w), NS2 = symb_ns(w) >> 1;
  const int WC = kSymTW + 2 * w, Lpad = L + 2 * w;
  const int XW = (kSymTH + w) * WC * 3;                 // x window doubles
  const int AC = 32 + 2 * w, AREG = (w + 1) * AC * 3;  // per-warp accumulator
  const int RW = WC * 3, RG = symb_region(w);
  const long long npad = (long long)Lpad * Lpad * 3;
  int* xoff = reinterpret_cast<int*>(dyn);
  int* aoff = xoff + npos;
  double* xs = dyn + ((2 * npos + 1) >> 1) + 1;
  double* acc = xs + NV * XW;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tpr = L / kSymTW;
  for (int e = tid; e < npos; e += blockDim.x) {
    int ds, dt;
    symb_offset(w, e, &ds, &dt);
    xoff[e] = (ds * WC + dt) * 3;
    aoff[e] = (ds * AC + dt) * 3;
  }
  double dot[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) dot[v] = 0.0;
  for (long long t = tile0 + blockIdx.x; t < tile1; t += gridDim.x) {
    const int I = (int)(t / tpr), J = (int)(t % tpr);
    const int ps0 = I * kSymTH, pt0 = J * kSymTW;
    // stage x windows: the tile's own rows and the w rows below (padded rows
    // ps0 + w .. ps0 + TH + 2w - 1), padded columns pt0 .. pt0 + 64 + 2w - 1
    for (int e = tid; e < XW; e += blockDim.x) {
      const int wr = e / (WC * 3), rem = e - wr * (WC * 3);
      const long long gi = ((long long)(ps0 + w + wr) * Lpad + pt0) * 3 + rem;
      xs[e] = x0[gi];
      if (NV == 2) xs[XW + e] = x1[gi];
    }
    for (int e = tid; e < NV * 2 * kSymTH * AREG; e += blockDim.x) acc[e] = 0.0;
    __syncthreads();
    const int h = warp >> 1, j = (warp & 1) * 32 + lane;
    const long long p = (long long)(ps0 + h) * L + pt0 + j;
    const double2* up = reinterpret_cast<const double2*>(U) + (p >> 5) * (32LL * NS2) + lane;
    const int xo = (h * WC + (j + w)) * 3;  // own position in the window
    const int ao = (lane + w) * 3;          // own position in the warp accumulator
    double xa[NV][3], g[NV][3];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xa[v][c] = xs[v * XW + xo + c];
        g[v][c] = 0.0;
      }
    double* aw = acc + warp * AREG;
    // software pipeline: the slots of offset pair e + 2 are in flight while
    // pair e is applied; the diagonal block is loaded up front
    double2 cur[9], nxt[9], dg[5];
  #pragma unroll
    for (int k = 0; k < 5; ++k) dg[k] = __ldg(up + (long long)(9 * npos / 2 + k) * 32);
  #pragma unroll
    for (int k = 0; k < 9; ++k) cur[k] = __ldg(up + 32 * k);
    for (int e = 0; e < npos; e += 2) {
      if (e + 2 < npos) {
        const double2* q = up + (long long)(9 * (e + 2) / 2) * 32;
  #pragma unroll
        for (int k = 0; k < 9; ++k) nxt[k] = __ldg(q + 32 * k);
      }
  #pragma unroll
      for (int ee = 0; ee < 2; ++ee) {
        double ub[9];
  #pragma unroll
        for (int i = 0; i < 9; ++i) {
          const int m = 9 * ee + i;
          ub[i] = (m & 1) ? cur[m >> 1].y : cur[m >> 1].x;
        }
        const int xe = xo + xoff[e + ee], ae = ao + aoff[e + ee];
  #pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double* xw = xs + v * XW + xe;
          const double n0 = xw[0], n1 = xw[1], n2 = xw[2];
          g[v][0] = fma(ub[0], n0, fma(ub[1], n1, fma(ub[2], n2, g[v][0])));
          g[v][1] = fma(ub[3], n0, fma(ub[4], n1, fma(ub[5], n2, g[v][1])));
          g[v][2] = fma(ub[6], n0, fma(ub[7], n1, fma(ub[8], n2, g[v][2])));
          double* a = aw + v * 2 * kSymTH * AREG + ae;
          a[0] += fma(ub[0], xa[v][0], fma(ub[3], xa[v][1], ub[6] * xa[v][2]));
          a[1] += fma(ub[1], xa[v][0], fma(ub[4], xa[v][1], ub[7] * xa[v][2]));
          a[2] += fma(ub[2], xa[v][0], fma(ub[5], xa[v][1], ub[8] * xa[v][2]));
        }
        __syncwarp();
      }
  #pragma unroll
      for (int k = 0; k < 9; ++k) cur[k] = nxt[k];
    }
    {  // diagonal block
  #pragma unroll
      for (int v = 0; v < NV; ++v) {
        double* a = aw + v * 2 * kSymTH * AREG + ao;
  #pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int m0 = 3 * c;
          const double d0 = (m0 & 1) ? dg[m0 >> 1].y : dg[m0 >> 1].x;
          const double d1 = ((m0 + 1) & 1) ? dg[(m0 + 1) >> 1].y : dg[(m0 + 1) >> 1].x;
          const double d2 = ((m0 + 2) & 1) ? dg[(m0 + 2) >> 1].y : dg[(m0 + 2) >> 1].x;
          a[c] += fma(d0, xa[v][0], fma(d1, xa[v][1], fma(d2, xa[v][2], g[v][c])));
        }
      }
    }
    __syncthreads();
    // combine the warps' accumulators over the tile region in a fixed order
    for (int idx = tid; idx < RG; idx += blockDim.x) {
      const int rr = idx / RW, rem = idx - rr * RW;
      const int cc = rem / 3 - w, c = rem % 3;
      const int h0 = rr - w > 0 ? rr - w : 0, h1 = rr < kSymTH - 1 ? rr : kSymTH - 1;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (v == 0 ? !live0 : !live1) continue;
        const double* av = acc + v * 2 * kSymTH * AREG;
        double sm = 0.0;
        for (int hh = h0; hh <= h1; ++hh) {
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const int lc = cc - half * 32 + w;
            if (lc >= 0 && lc < AC)
              sm += av[(2 * hh + half) * AREG + ((rr - hh) * AC + lc) * 3 + c];
          }
        }
        double* y = v == 0 ? y0 : y1;
        if (rr < kSymTH && cc >= 0 && cc < kSymTW)
          y[((long long)(ps0 + rr + w) * Lpad + pt0 + cc + w) * 3 + c] = sm;
        else
          y[npad + t * RG + idx] = sm;
        if (v == 0 ? rd0 : rd1) dot[v] = fma(xs[v * XW + idx], sm, dot[v]);
      }
    }
    __syncthreads();
  }
  if (!rd0 && !rd1) return;
  KState* cs = rd0 ? s0 : s1;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (!(v == 0 ? rd0 : rd1)) continue;
    const double a = block_sum(dot[v], sh);
    if (threadIdx.x == 0) (v == 0 ? part0 : part1)[2 * blockIdx.x] = a;
  }
  if (last_block(&cs->counter)) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!(v == 0 ? rd0 : rd1)) continue;
      const double* part = v == 0 ? part0 : part1;
      double a = 0.0;
      for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) a += part[2 * k];
      a = block_sum(a, sh);
      if (threadIdx.x == 0)
        finish_reduction(v == 0 ? s0 : s1, (v == 0 ? red0 : red1) == 2 ? 3 : 0, a, 0.0);
    }
    if (threadIdx.x == 0) cs->counter = 0;
  }
}

// ---------------------------------------------------------------------------
// Phase 1, warp-specialized (default): a persistent CTA per SM, 8 consumer
// warps as above plus one producer warp that streams the consumers' U blocks
// into a kSymWsStages-deep shared-memory ring with 1-D bulk copies
// (cp.async.bulk, TMA engine; full/empty mbarriers per stage).  The producer
// runs ahead across tile boundaries, so the x staging and the combine of a
// tile overlap the HBM stream of the next; bytes in flight cost no registers.
// Same arithmetic and summation order as k_symb_apply.
// ---------------------------------------------------------------------------
constexpr int kSymWsPairs = 9;  // slot pairs of one chunk (two offsets)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
// the same copy with an L2 evict-first policy: a band larger than L2 is read
// once per pass, and without the hint its 0.8 GB stream evicts the Krylov
// vectors the update kernels between two passes re-read
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, unsigned bytes,
                                                unsigned long long* b, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void consumer_sync() {  // the 8 consumer warps only
  asm volatile("bar.sync 1, %0;" ::"r"(kSymThreads) : "memory");
}

// preferred ring depth; wide stencils (w >= 5 with two vectors) fall back to
// 2 stages so that the kernel still fits in shared memory
template <int NV>
__host__ __device__ constexpr int symb_ws_stages() { return NV == 1 ? 4 : 3; }

static inline size_t symb_ws_smem(int w, int nv, int st) {
  const int npos = symb_npos(w), WC = kSymTW + 2 * w, nwarp = 2 * kSymTH;
  return (size_t)2 * st * 8 +                                        // full/empty barriers
         (size_t)st * nwarp * kSymWsPairs * 32 * 16 +                 // U ring
         (size_t)nv * (kSymTH + w) * WC * 3 * 8 +                     // x windows
         (size_t)nv * nwarp * (w + 1) * (32 + 2 * w) * 3 * 8 +        // accumulators
         (size_t)2 * npos * 4;                                        // offset tables
}

// the consumer warps of one vector only (named barrier 1 + vec)
__device__ __forceinline__ void group_sync(int vec) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + vec), "r"(kSymThreads) : "memory");
}

// NV vectors = NV groups of 8 consumer warps: group v applies the tile's U
// blocks (read from the shared ring by every group) to vector v, so a second
// vector adds warps -- latency hiding -- instead of lengthening every warp's
// dependent shared-memory chains.  Each group runs exactly the single-vector
// arithmetic (same order), the groups are independent between ring stages.
template <int NV, int NS>
__global__ void __launch_bounds__(NV * kSymThreads + 32, 1) k_symb_apply_ws(
    int L, int w, const double* __restrict__ U, const double* __restrict__ x0,
    double* __restrict__ y0, KState* s0, double* part0, int red0,
    const double* __restrict__ x1, double* __restrict__ y1, KState* s1, double* part1,
    int red1, long long tile0, long long tile1) {
  constexpr int NW = 2 * kSymTH;  // consumer warps per vector
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ double sh[32];
  const bool live0 = !(s0 && s0->done);
  const bool live1 = NV == 2 && !(s1 && s1->done);
  if (!live0 && !live1) return;
  const bool rd0 = live0 && red0, rd1 = NV == 2 && live1 && red1;
  const int npos = symb_npos(w), NS2 = symb_ns(w) >> 1, nch = npos / 2 + 1;
  const int WC = kSymTW + 2 * w, Lpad = L + 2 * w;
  const int XW = (kSymTH + w) * WC * 3;
  const int AC = 32 + 2 * w, AREG = (w + 1) * AC * 3;
  const int RW = WC * 3, RG = symb_region(w);
  const long long npad = (long long)Lpad * Lpad * 3;
  const int tpr = L / kSymTW;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(dsm);
  unsigned long long* empty = full + NS;
  double2* ring = reinterpret_cast<double2*>(dsm + 2 * NS * 8);
  double* xs_all = reinterpret_cast<double*>(ring + NS * NW * kSymWsPairs * 32);
  double* acc_all = xs_all + NV * XW;
  int* xoff = reinterpret_cast<int*>(acc_all + NV * NW * AREG);
  int* aoff = xoff + npos;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int st = 0; st < NS; ++st) {
      mbar_init(full + st, 1);
      mbar_init(empty + st, NV * NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < npos; e += blockDim.x) {
    int ds, dt;
    symb_offset(w, e, &ds, &dt);
    xoff[e] = (ds * WC + dt) * 3;
    aoff[e] = (ds * AC + dt) * 3;
  }
  __syncthreads();
  double dot = 0.0;
  const int vec = warp / NW;  // NV for the producer warp
  if (warp == NV * NW) {
    // ---- producer: chunk g = (tile iteration, k) -> stage g % NS ----
    if (lane == 0) {
      long long g = 0;
      // bands beyond the L2 capacity (levels with >= 256^2 parents) stream
      const bool streamed = GB_SYM_L2_STREAM && L >= 256;
      const unsigned long long pol = l2_evict_first_policy();
      for (long long t = tile0 + blockIdx.x; t < tile1; t += gridDim.x) {
        const int I = (int)(t / tpr), J = (int)(t % tpr);
        for (int k = 0; k < nch; ++k, ++g) {
          const int st = (int)(g % NS);
          const long long r = g / NS;
          if (r > 0) mbar_wait(empty + st, (unsigned)((r - 1) & 1));
          const int pairs = k < nch - 1 ? kSymWsPairs : 5;
          const unsigned bytes = (unsigned)pairs * 32 * 16;
          mbar_expect_tx(full + st, bytes * NW);
          double2* dst = ring + (long long)st * NW * kSymWsPairs * 32;
          for (int cw = 0; cw < NW; ++cw) {
            const long long p =
                (long long)(I * kSymTH + (cw >> 1)) * L + J * kSymTW + (cw & 1) * 32;
            const double2* src = reinterpret_cast<const double2*>(U) + (p >> 5) * (32LL * NS2) +
                                  (long long)k * kSymWsPairs * 32;
            if (streamed)
              bulk_g2s_stream(dst + cw * kSymWsPairs * 32, src, bytes, full + st, pol);
            else
              bulk_g2s(dst + cw * kSymWsPairs * 32, src, bytes, full + st);
          }
        }
      }
    }
  } else {
    // ---- consumers: group `vec`, warp cw of the tile, thread gt of the group ----
    const int cw = warp - vec * NW, gt = tid - vec * kSymThreads;
    const bool live = vec == 0 ? live0 : live1;
    const bool rd = vec == 0 ? rd0 : rd1;
    const double* __restrict__ x = vec == 0 ? x0 : x1;
    double* __restrict__ y = vec == 0 ? y0 : y1;
    double* xs = xs_all + vec * XW;
    double* acc = acc_all + vec * NW * AREG;
    int st = 0;          // ring stage of the next chunk and its phase parity
    unsigned ph = 0;
    for (long long t = tile0 + blockIdx.x; t < tile1; t += gridDim.x) {
      const int I = (int)(t / tpr), J = (int)(t % tpr);
      const int ps0 = I * kSymTH, pt0 = J * kSymTW;
      if (!live) {  // a finished vector: keep the ring moving, no arithmetic
        for (int k = 0; k < nch; ++k) {
          mbar_wait(full + st, ph);
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + st);
          if (++st == NS) st = 0, ph ^= 1;
        }
        continue;
      }
      // x window, 8 independent loads in flight per thread (L2 latency)
      for (int e0 = gt; e0 < XW; e0 += 8 * kSymThreads) {
        double va[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * kSymThreads;
          va[u] = 0.0;
          if (e < XW) {
            const int wr = e / (WC * 3), rem = e - wr * (WC * 3);
            va[u] = x[((long long)(ps0 + w + wr) * Lpad + pt0) * 3 + rem];
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * kSymThreads;
          if (e < XW) xs[e] = va[u];
        }
      }
      for (int e = gt; e < NW * AREG; e += kSymThreads) acc[e] = 0.0;
      group_sync(vec);
      const int h = cw >> 1, j = (cw & 1) * 32 + lane;
      const int xo = (h * WC + (j + w)) * 3;
      const int ao = (lane + w) * 3;
      double xa[3], gg[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xa[c] = xs[xo + c];
        gg[c] = 0.0;
      }
      double* aw = acc + cw * AREG;
      for (int k = 0; k < nch; ++k) {
        mbar_wait(full + st, ph);
        const double2* sb = ring + (st * NW + cw) * (kSymWsPairs * 32) + lane;
        if (k < nch - 1) {
#pragma unroll
          for (int ee = 0; ee < 2; ++ee) {
            double ub[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) {
              const int m = 9 * ee + i;
              const double2 d = sb[(m >> 1) * 32];
              ub[i] = (m & 1) ? d.y : d.x;
            }
            const int e = 2 * k + ee;
            const double* xw = xs + xo + xoff[e];
            const double n0 = xw[0], n1 = xw[1], n2 = xw[2];
            gg[0] = fma(ub[0], n0, fma(ub[1], n1, fma(ub[2], n2, gg[0])));
            gg[1] = fma(ub[3], n0, fma(ub[4], n1, fma(ub[5], n2, gg[1])));
            gg[2] = fma(ub[6], n0, fma(ub[7], n1, fma(ub[8], n2, gg[2])));
            double* a = aw + ao + aoff[e];
            a[0] += fma(ub[0], xa[0], fma(ub[3], xa[1], ub[6] * xa[2]));
            a[1] += fma(ub[1], xa[0], fma(ub[4], xa[1], ub[7] * xa[2]));
            a[2] += fma(ub[2], xa[0], fma(ub[5], xa[1], ub[8] * xa[2]));
            __syncwarp();
          }
        } else {  // diagonal block
          double u[10];
#pragma unroll
          for (int i = 0; i < 5; ++i) {
            const double2 d = sb[i * 32];
            u[2 * i] = d.x;
            u[2 * i + 1] = d.y;
          }
          double* a = aw + ao;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            a[c] += fma(u[3 * c], xa[0], fma(u[3 * c + 1], xa[1], fma(u[3 * c + 2], xa[2], gg[c])));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        if (++st == NS) st = 0, ph ^= 1;
      }
      group_sync(vec);
      // combine: region row rr outer (uniform warp-row range), the thread's
      // column/component fixed, so no index division in the loop
      if (gt < RW) {
        const int cc = gt / 3 - w, c = gt - 3 * (gt / 3);
        const int lc0 = cc + w, lc1 = cc - 32 + w;
        const bool in0 = lc0 < AC, in1 = lc1 >= 0;
        const bool own_col = cc >= 0 && cc < kSymTW;
        for (int rr = 0; rr < kSymTH + w; ++rr) {
          const int h0 = rr - w > 0 ? rr - w : 0, h1 = rr < kSymTH - 1 ? rr : kSymTH - 1;
          const int idx = rr * RW + gt;
          double sm = 0.0;
          for (int hh = h0; hh <= h1; ++hh) {
            const int ro = ((rr - hh) * AC) * 3 + c;
            if (in0) sm += acc[(2 * hh) * AREG + ro + lc0 * 3];
            if (in1) sm += acc[(2 * hh + 1) * AREG + ro + lc1 * 3];
          }
          if (rr < kSymTH && own_col)
            y[((long long)(ps0 + rr + w) * Lpad + pt0 + cc + w) * 3 + c] = sm;
          else
            y[npad + t * RG + idx] = sm;
          if (rd) dot = fma(xs[idx], sm, dot);
        }
      }
      group_sync(vec);
    }
  }
  __syncthreads();
  if (!rd0 && !rd1) return;
  KState* cs = rd0 ? s0 : s1;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (!(v == 0 ? rd0 : rd1)) continue;
    const double a = block_sum(vec == v ? dot : 0.0, sh);
    if (threadIdx.x == 0) (v == 0 ? part0 : part1)[2 * blockIdx.x] = a;
  }
  if (last_block(&cs->counter)) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!(v == 0 ? rd0 : rd1)) continue;
      const double* part = v == 0 ? part0 : part1;
      double a = 0.0;
      for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) a += part[2 * k];
      a = block_sum(a, sh);
      if (threadIdx.x == 0)
        finish_reduction(v == 0 ? s0 : s1, (v == 0 ? red0 : red1) == 2 ? 3 : 0, a, 0.0);
    }
    if (threadIdx.x == 0) cs->counter = 0;
  }
}

// Phase 2: y_own += the neighbours' spill-over, then the reductions of
// finish_reduction (mode 0: x.y -> alpha, 1: x.y, y.y -> lam, ynorm, 2: none).
template <int NV>
__global__ void __launch_bounds__(256) k_symb_fix(int L, int w, const double* __restrict__ x0,
                                                  double* __restrict__ y0, KState* s0,
                                                  double* part0, int mode0,
                                                  const double* __restrict__ x1,
                                                  double* __restrict__ y1, KState* s1,
                                                  double* part1, int mode1) {
  __shared__ double sh[32];
  const bool live0 = !(s0 && s0->done);
  const bool live1 = NV == 2 && !(s1 && s1->done);
  if (!live0 && !live1) return;
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * 3, R = (long long)L * L * 3;
  double d[NV][2];
#pragma unroll
  for (int v = 0; v < NV; ++v) d[v][0] = d[v][1] = 0.0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < R;
       r += (long long)gridDim.x * blockDim.x) {
    const long long pp = r / 3;
    const int c = (int)(r - pp * 3);
    const int ps = (int)(pp / L), pt = (int)(pp % L);
    const long long yi = ((long long)(ps + w) * Lpad + pt + w) * 3 + c;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (v == 0 ? !live0 : !live1) continue;
      double* y = v == 0 ? y0 : y1;
      const double s = symb_fix_value(y[yi], y + npad, L, w, ps, pt, c);
      y[yi] = s;
      const double* x = v == 0 ? x0 : x1;
      d[v][0] = fma(x[yi], s, d[v][0]);
      d[v][1] = fma(s, s, d[v][1]);
    }
  }
  const bool red0 = live0 && mode0 != 2, red1 = NV == 2 && live1 && mode1 != 2;
  if (!red0 && !red1) return;
  KState* cs = red0 ? s0 : s1;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const bool rv = v == 0 ? red0 : red1;
    if (!rv) continue;
    const double a = block_sum(d[v][0], sh);
    const double b = block_sum(d[v][1], sh);
    double* part = v == 0 ? part0 : part1;
    if (threadIdx.x == 0) {
      part[2 * blockIdx.x] = a;
      part[2 * blockIdx.x + 1] = b;
    }
  }
  if (last_block(&cs->counter)) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const bool rv = v == 0 ? red0 : red1;
      if (!rv) continue;
      double a, b;
      final_sum2(v == 0 ? part0 : part1, gridDim.x, &a, &b, sh);
      if (threadIdx.x == 0) finish_reduction(v == 0 ? s0 : s1, v == 0 ? mode0 : mode1, a, b);
    }
    if (threadIdx.x == 0) cs->counter = 0;
  }
}

static inline size_t symb_smem(int w, int nv) {
  const int npos = symb_npos(w), WC = kSymTW + 2 * w;
  return (size_t)(((2 * npos + 1) >> 1) + 1) * 8 +
         (size_t)nv * (kSymTH + w) * WC * 3 * 8 +
         (size_t)nv * 2 * kSymTH * (w + 1) * (32 + 2 * w) * 3 * 8;
}
