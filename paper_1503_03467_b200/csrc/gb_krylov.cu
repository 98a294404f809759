// Solve-phase kernels: subband / coarse CG (K8), the spectral-estimate
// building blocks (K7) and the load-dependent transfers (K9).
//
// CG follows sparse_core.py:126-165 step for step (zero start or warm start,
// stop when ||r|| <= tol ||b||, breakdown on p^T A p <= 0, max_iter reported
// not fatal).  The iteration state lives in device memory; the kernels read it
// at entry and return immediately once `done` is set, so the host can enqueue
// chunks of iterations without a round trip per step.  Reductions are two
// level with a fixed order (per-block partials summed by the last block), so
// every run is bitwise reproducible.
#include <vector>

#include "gb_common.cuh"
#include "gb_kernels.h"

namespace gb {

struct KState {
  double rs, pAp, alpha, beta, bnorm, tol_abs, rnorm, lam;
  double ynorm, res, aux0, aux1;
  int it, done, converged, max_iter, breakdown, pad0, pad1, pad2;
  unsigned int counter, pad3;
};

__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(counter, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  return am_last;
}

// deterministic sum of gridDim.x partials (pairs) by the last block
__device__ __forceinline__ void final_sum2(const double* part, int nb, double* o0,
                                          double* o1, double* sh) {
  double a = 0.0, b = 0.0;
  for (int j = threadIdx.x; j < nb; j += blockDim.x) {
    a += part[2 * j];
    b += part[2 * j + 1];
  }
  a = block_sum(a, sh);
  b = block_sum(b, sh);
  *o0 = a;
  *o1 = b;
}

// y_r = Op(x)_r for a square box (nr = nc), one warp per row.
// mode 0: sum ((B s_r) s_c) x_c        (materialized congruence S B S)
// mode 1: s_r * sum B (s_c x_c)        (_RescaledOperator, gamblet_fast.py:142-151)
__device__ __forceinline__ double box_row_apply(int L, int nr, int w,
                                                const double* __restrict__ B,
                                                const double* __restrict__ s, int mode,
                                                const double* __restrict__ x,
                                                long long r, int lane) {
  const int W2 = 2 * w + 1;
  const int S = W2 * W2 * nr;
  const long long p = r / nr;
  const int ps = (int)(p / L), pt = (int)(p % L);
  const int s0 = imax(ps - w, 0) - ps, s1 = imin(ps + w, L - 1) - ps;
  const int t0 = imax(pt - w, 0) - pt, t1 = imin(pt + w, L - 1) - pt;
  const int nt = (t1 - t0 + 1) * nr;
  const int cnt = (s1 - s0 + 1) * nt;
  const double* row = B + r * S;
  const double sr = s[r];
  double acc = 0.0;
  for (int j = lane; j < cnt; j += 32) {
    const int a = j / nt, rem = j - a * nt;
    const int ds = s0 + a;
    const int dt = t0 + rem / nr, c = rem % nr;
    const double bv = row[((ds + w) * W2 + (dt + w)) * nr + c];
    const long long col = ((long long)(ps + ds) * L + (pt + dt)) * nr + c;
    if (mode == 0) acc += (bv * sr) * s[col] * x[col];
    else acc += bv * (s[col] * x[col]);
  }
  acc = warp_sum(acc);
  return mode == 0 ? acc : sr * acc;
}

// Ap = Op(p); partial (p.Ap, 0); last block: pAp, alpha, breakdown
__global__ void k_cg_spmv(int L, int nr, int w, const double* __restrict__ B,
                          const double* __restrict__ s, int mode,
                          const double* __restrict__ p, double* __restrict__ Ap,
                          KState* st, double* part) {
  __shared__ double sh[32];
  if (st->done) return;
  const long long rows = (long long)L * L * nr;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  double dot = 0.0;
  for (long long r = wid; r < rows; r += nwarps) {
    const double y = box_row_apply(L, nr, w, B, s, mode, p, r, lane);
    if (lane == 0) {
      Ap[r] = y;
      dot += p[r] * y;
    }
  }
  dot = block_sum(dot, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = dot;
    part[2 * blockIdx.x + 1] = 0.0;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->pAp = a;
      if (!(a > 0.0)) {
        st->breakdown = st->it + 1;
        st->done = 1;
      } else {
        st->alpha = st->rs / a;
      }
    }
  }
}

// x += alpha p; r -= alpha Ap; rs_new; convergence; beta
__global__ void k_cg_update(long long n, double* __restrict__ x, double* __restrict__ r,
                            const double* __restrict__ p, const double* __restrict__ Ap,
                            KState* st, double* part) {
  __shared__ double sh[32];
  if (st->done) return;
  const double alpha = st->alpha;
  double rr = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    rr += ri * ri;
  }
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = rr;
    part[2 * blockIdx.x + 1] = 0.0;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->it += 1;
      const double rn = sqrt(a);
      st->rnorm = rn;
      if (rn <= st->tol_abs) {
        st->done = 1;
        st->converged = 1;
      } else if (st->it >= st->max_iter) {
        st->done = 1;
        st->converged = 0;
      } else {
        st->beta = a / st->rs;
        st->rs = a;
      }
    }
  }
}

__global__ void k_cg_dir(long long n, const double* __restrict__ r, double* __restrict__ p,
                         const KState* st) {
  if (st->done) return;
  const double beta = st->beta;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = r[i] + beta * p[i];
}

// init: r = b - Ax0 (Ax0 may be null => x0 = 0), x = x0 or 0, p = r;
// bnorm, rnorm, early exits of sparse_core.py:138-148
__global__ void k_cg_init(long long n, const double* __restrict__ b,
                          const double* __restrict__ x0, const double* __restrict__ Ax0,
                          double* __restrict__ x, double* __restrict__ r,
                          double* __restrict__ p, double rel_tol, int max_iter,
                          KState* st, double* part) {
  __shared__ double sh[32];
  double bb = 0.0, rr = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double bi = b[i];
    const double ri = Ax0 ? bi - Ax0[i] : bi;
    x[i] = x0 ? x0[i] : 0.0;
    r[i] = ri;
    p[i] = ri;
    bb += bi * bi;
    rr += ri * ri;
  }
  bb = block_sum(bb, sh);
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = bb;
    part[2 * blockIdx.x + 1] = rr;
  }
  if (last_block(&st->counter)) {
    double a, c;
    final_sum2(part, gridDim.x, &a, &c, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->it = 0;
      st->breakdown = 0;
      st->max_iter = max_iter;
      const double bn = sqrt(a);
      st->bnorm = bn;
      st->tol_abs = rel_tol * bn;
      const double rn = sqrt(c);
      st->rnorm = rn;
      st->rs = rn * rn;
      st->done = 0;
      st->converged = 0;
      if (bn == 0.0) {
        st->done = 1;
        st->converged = 1;
        st->rnorm = 0.0;
        st->aux0 = 1.0;  // x must be zeroed (zero rhs)
      } else if (rn <= rel_tol * bn) {
        st->done = 1;
        st->converged = 1;
        st->aux0 = 0.0;
      } else {
        st->aux0 = 0.0;
      }
    }
  }
}

// zero rhs => x = 0 (sparse_core.py:140-141)
__global__ void k_cg_zero_if(long long n, double* __restrict__ x, const KState* st) {
  if (st->aux0 == 0.0) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = 0.0;
}

// ---------------------------------------------------------------------------
// spectral building blocks (sparse_core.py:232-278)
// ---------------------------------------------------------------------------
// y = Op(x); (x.y, y.y) -> st->lam, st->ynorm
__global__ void k_pow_apply(int L, int nr, int w, const double* __restrict__ B,
                            const double* __restrict__ s, int mode,
                            const double* __restrict__ x, double* __restrict__ y,
                            KState* st, double* part) {
  __shared__ double sh[32];
  if (st->done) return;
  const long long rows = (long long)L * L * nr;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  double xy = 0.0, yy = 0.0;
  for (long long r = wid; r < rows; r += nwarps) {
    const double v = box_row_apply(L, nr, w, B, s, mode, x, r, lane);
    if (lane == 0) {
      y[r] = v;
      xy += x[r] * v;
      yy += v * v;
    }
  }
  xy = block_sum(xy, sh);
  yy = block_sum(yy, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = xy;
    part[2 * blockIdx.x + 1] = yy;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->lam = a;
      st->ynorm = sqrt(b);
      if (st->ynorm == 0.0) {
        st->lam = 0.0;
        st->done = 1;
      }
    }
  }
}

// res = ||y - lam x||; x = y / ynorm; stop test res <= 0.5 tol |lam|
__global__ void k_pow_step(long long n, double* __restrict__ x, const double* __restrict__ y,
                           double tol, KState* st, double* part) {
  __shared__ double sh[32];
  if (st->done) return;
  const double lam = st->lam, yn = st->ynorm;
  double rr = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double d = y[i] - lam * x[i];
    rr += d * d;
  }
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = rr;
    part[2 * blockIdx.x + 1] = 0.0;
  }
  // every block must finish reading x before anyone rescales it: the rescale
  // happens in k_pow_scale after this kernel completes
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->res = sqrt(a);
      st->it += 1;
      st->aux1 = (st->res <= 0.5 * tol * fabs(lam) || st->it >= st->max_iter) ? 1.0 : 0.0;
    }
  }
}

__global__ void k_pow_scale(long long n, double* __restrict__ x, const double* __restrict__ y,
                            KState* st) {
  if (st->done) return;
  const double yn = st->ynorm;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = y[i] / yn;
  // the stop flag is committed by the last thread to leave (any thread may
  // set it: the kernel boundary orders it before the next launch)
  if (blockIdx.x == 0 && threadIdx.x == 0 && st->aux1 != 0.0) st->done = 1;
}

// Lanczos step on an unnormalized iterate (one launch per step): x = u_j
// with |u_j| = beta_{j-1} = st->aux0 (x = v_1, aux0 = 1 on the first step),
// y = A x from a power-mode apply (st->lam = x.y).  With v_j = x / beta_{j-1}:
// alpha_j = x.y / beta_{j-1}^2, u_{j+1} = (y - alpha_j x) / beta_{j-1} -
// beta_{j-1} v_{j-1}; vp <- v_j, y <- u_{j+1} (the next operator input),
// beta_j = |u_{j+1}|; (alpha_j, beta_j) appended to ab.  beta_j == 0
// (invariant subspace) or it == max_iter ends the sequence.
__global__ void k_lz_step(long long n, const double* __restrict__ x, double* __restrict__ vp,
                          double* __restrict__ y, KState* st, double* part, double* ab) {
  __shared__ double sh[32];
  if (st->done) return;
  const double bp = st->aux0, ibp = 1.0 / bp;
  const double alpha = st->lam * ibp * ibp;
  double uu = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = x[i] * ibp;
    const double u = (y[i] - alpha * x[i]) * ibp - bp * vp[i];
    vp[i] = v;
    y[i] = u;
    uu += u * u;
  }
  uu = block_sum(uu, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = uu;
    part[2 * blockIdx.x + 1] = 0.0;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      const double beta = sqrt(a);
      ab[2 * st->it] = alpha;
      ab[2 * st->it + 1] = beta;
      st->it += 1;
      st->aux0 = beta;
      if (!(beta > 0.0) || st->it >= st->max_iter) st->done = 1;
    }
  }
}

__global__ void k_lz_init(KState* st) { st->aux0 = 1.0; }

// generic dot products: out[0] = a.b, out[1] = c.c  (c may be null)
__global__ void k_dot2(long long n, const double* __restrict__ a, const double* __restrict__ b,
                       const double* __restrict__ c, double* out, KState* st,
                       double* part) {
  __shared__ double sh[32];
  double s0 = 0.0, s1 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    s0 += a[i] * b[i];
    if (c) s1 += c[i] * c[i];
  }
  s0 = block_sum(s0, sh);
  s1 = block_sum(s1, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0;
    part[2 * blockIdx.x + 1] = s1;
  }
  if (last_block(&st->counter)) {
    double x0, x1;
    final_sum2(part, gridDim.x, &x0, &x1, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      out[0] = x0;
      out[1] = x1;
    }
  }
}

// y = a / sqrt(norm2[0]) ; also copies into y2 when given
__global__ void k_scale_by_norm(long long n, const double* __restrict__ a,
                                const double* __restrict__ norm2, int which,
                                double* __restrict__ y, double* __restrict__ y2) {
  const double nv = sqrt(norm2[which]);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = a[i] / nv;
    y[i] = v;
    if (y2) y2[i] = v;
  }
}

// plain y = Op(x)
__global__ void k_box_apply(int L, int nr, int w, const double* __restrict__ B,
                            const double* __restrict__ s, int mode,
                            const double* __restrict__ x, double* __restrict__ y) {
  const long long rows = (long long)L * L * nr;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nwarps) {
    const double v = box_row_apply(L, nr, w, B, s, mode, x, r, lane);
    if (lane == 0) y[r] = v;
  }
}


// ---------------------------------------------------------------------------
// v2 Krylov operator: pre-scaled box Bs = S B S (the reference materializes
// exactly this for its spectral estimates, gamblet_fast.py:123-139) applied
// to vectors in a zero-halo padded layout, so the gather needs no bounds
// checks: grid point (s,t) with components c lives at
// ((s + w) * Lpad + (t + w)) * nr + c, Lpad = L + 2w.  One warp per grid
// point computes its nr rows together, loading each x value once; the slot ->
// relative x offset table sits in shared memory.
// ---------------------------------------------------------------------------
__global__ void k_scale_box(int L, int nr, int w, const double* __restrict__ B,
                            const double* __restrict__ s, double* __restrict__ Bs) {
  const int W2 = 2 * w + 1, S = W2 * W2 * nr;
  const long long total = (long long)L * L * nr * S;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / S;
    const int sl = (int)(e - r * S);
    const int cp = sl % nr, bs = sl / nr;
    const long long p = r / nr;
    const int qs = (int)(p / L) + bs / W2 - w, qt = (int)(p % L) + bs % W2 - w;
    double v = 0.0;
    if (qs >= 0 && qs < L && qt >= 0 && qt < L)
      v = B[e] * s[r] * s[((long long)qs * L + qt) * nr + cp];
    Bs[e] = v;
  }
}

__global__ void k_pad(int L, int nr, int w, const double* __restrict__ src,
                      const double* __restrict__ scale, double* __restrict__ dst, long long e0,
                      long long e1) {
  const int Lpad = L + 2 * w;
  for (long long r = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < e1;
       r += (long long)gridDim.x * blockDim.x) {
    const long long p = r / nr;
    const int c = (int)(r - p * nr);
    const long long pr = (((long long)(p / L) + w) * Lpad + (p % L) + w) * nr + c;
    dst[pr] = scale ? scale[r] * src[r] : src[r];
  }
}

__global__ void k_unpad(int L, int nr, int w, const double* __restrict__ src,
                        const double* __restrict__ scale, double* __restrict__ dst,
                        long long e0, long long e1) {
  const int Lpad = L + 2 * w;
  for (long long r = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < e1;
       r += (long long)gridDim.x * blockDim.x) {
    const long long p = r / nr;
    const int c = (int)(r - p * nr);
    const long long pr = (((long long)(p / L) + w) * Lpad + (p % L) + w) * nr + c;
    dst[r] = scale ? scale[r] * src[pr] : src[pr];
  }
}

__device__ __forceinline__ void build_offsets(int nr, int w, int Lpad, int* off) {
  const int W2 = 2 * w + 1, S = W2 * W2 * nr;
  for (int j = threadIdx.x; j < S + 1; j += blockDim.x) {
    const int jj = j < S ? j : 0;  // pad slot (value 0) points at a valid entry
    const int c = jj % nr, bs = jj / nr;
    off[j] = ((bs / W2) * Lpad + (bs % W2)) * nr + c;
  }
  __syncthreads();
}

template <int NR>
__device__ __forceinline__ void point_apply(const double* __restrict__ blk, int S,
                                            const int* __restrict__ off,
                                            const double* __restrict__ x, long long xb,
                                            int lane, double* y) {
  double a[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) a[c] = 0.0;
#pragma unroll 4
  for (int j = lane; j < S; j += 32) {
    const double xv = x[xb + off[j]];
#pragma unroll
    for (int c = 0; c < NR; ++c) a[c] = fma(__ldg(blk + c * S + j), xv, a[c]);
  }
#pragma unroll
  for (int c = 0; c < NR; ++c) y[c] = warp_sum(a[c]);
}

// y = Bs x over padded vectors; optional fused dot x.y into the state
template <int NR>
__device__ __forceinline__ double pbox_pass(int L, int w, const double* __restrict__ Bs,
                                            const double* __restrict__ x,
                                            double* __restrict__ y, const int* off,
                                            double* yy_out) {
  const int W2 = 2 * w + 1, S = W2 * W2 * NR, Lpad = L + 2 * w;
  const long long P = (long long)L * L;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  double dot = 0.0, yy = 0.0;
  for (long long p = wid; p < P; p += nwarps) {
    const int ps = (int)(p / L), pt = (int)(p % L);
    const long long xb = ((long long)ps * Lpad + pt) * NR;
    double v[NR];
    point_apply<NR>(Bs + p * NR * S, S, off, x, xb, lane, v);
    if (lane == 0) {
      const long long yr = ((long long)(ps + w) * Lpad + pt + w) * NR;
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        y[yr + c] = v[c];
        dot += x[yr + c] * v[c];
        yy += v[c] * v[c];
      }
    }
  }
  *yy_out = yy;
  return dot;
}

template <int NR>
__global__ void __launch_bounds__(256) k_pcg_spmv(int L, int w, const double* __restrict__ Bs,
                                                  const double* __restrict__ p,
                                                  double* __restrict__ Ap, KState* st,
                                                  double* part) {
  extern __shared__ int off[];
  __shared__ double sh[32];
  if (st->done) return;
  build_offsets(NR, w, L + 2 * w, off);
  double yy;
  double dot = pbox_pass<NR>(L, w, Bs, p, Ap, off, &yy);
  dot = block_sum(dot, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = dot;
    part[2 * blockIdx.x + 1] = 0.0;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->pAp = a;
      if (!(a > 0.0)) {
        st->breakdown = st->it + 1;
        st->done = 1;
      } else {
        st->alpha = st->rs / a;
      }
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(256) k_ppow_apply(int L, int w, const double* __restrict__ Bs,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y, KState* st,
                                                    double* part) {
  extern __shared__ int off[];
  __shared__ double sh[32];
  if (st->done) return;
  build_offsets(NR, w, L + 2 * w, off);
  double yy;
  double xy = pbox_pass<NR>(L, w, Bs, x, y, off, &yy);
  xy = block_sum(xy, sh);
  yy = block_sum(yy, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = xy;
    part[2 * blockIdx.x + 1] = yy;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->lam = a;
      st->ynorm = sqrt(b);
      if (st->ynorm == 0.0) {
        st->lam = 0.0;
        st->done = 1;
      }
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(256) k_pbox_apply(int L, int w, const double* __restrict__ Bs,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y) {
  extern __shared__ int off[];
  build_offsets(NR, w, L + 2 * w, off);
  double yy;
  pbox_pass<NR>(L, w, Bs, x, y, off, &yy);
}


// ---------------------------------------------------------------------------
// v3 Krylov operator: slot-major ("transposed box") copy of S B S,
// BsT[j * R + r] for slot j, row r (R rows).  One thread per row streams its
// slots: at every slot a warp reads 32 consecutive rows (256 B, coalesced)
// and gathers x from 32 consecutive padded positions; no shuffles, long
// unrollable loops.  The slot -> relative x offset table is in shared memory
// (every thread reads the same entry: broadcast).
// ---------------------------------------------------------------------------
// strided fallback (boxes too wide for the shared-memory transpose)
__global__ void k_scale_box_T_strided(int L, int nr, int w, const double* __restrict__ B,
                                      const double* __restrict__ s, double* __restrict__ BsT) {
  const int W2 = 2 * w + 1, S = W2 * W2 * nr;
  const long long R = (long long)L * L * nr;
  const int Sp = S + (S & 1);
  const long long total = (R + 31) / 32 * 32LL * Sp;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long blk = e / (32LL * Sp);
    const int rem = (int)(e - blk * 32LL * Sp);
    const int j = ((rem >> 6) << 1) | (rem & 1);
    const long long r = blk * 32 + ((rem >> 1) & 31);
    double v = 0.0;
    if (r < R && j < S) {
      const int cp = j % nr, bs = j / nr;
      const long long p = r / nr;
      const int qs = (int)(p / L) + bs / W2 - w, qt = (int)(p % L) + bs % W2 - w;
      if (qs >= 0 && qs < L && qt >= 0 && qt < L)
        v = B[r * S + j] * s[r] * s[((long long)qs * L + qt) * nr + cp];
    }
    BsT[e] = v;
  }
}

// blocked slot-major transpose, one CTA per 32-row block: the 32 rows are
// contiguous in B (32*S doubles), staged in shared memory, written slot-pair
// major: BsT[blk*32*Sp + (j/2)*64 + (r%32)*2 + j%2], Sp = S rounded up to even
// (the pad slot is 0), so a warp reads 512 contiguous bytes per slot pair.
__global__ void k_scale_box_T(int L, int nr, int w, const double* __restrict__ B,
                              const double* __restrict__ s, double* __restrict__ BsT) {
  extern __shared__ double tile[];  // 32 * (S + 1)
  const int W2 = 2 * w + 1, S = W2 * W2 * nr;
  const long long R = (long long)L * L * nr;
  const long long nblk = (R + 31) / 32;
  for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const long long r0 = blk * 32;
    const int nrow = (int)(R - r0 < 32 ? R - r0 : 32);
    for (int e = threadIdx.x; e < 32 * S; e += blockDim.x) {
      const int rl = e / S, j = e - rl * S;
      tile[rl * (S + 1) + j] = rl < nrow ? B[(r0 + rl) * S + j] : 0.0;
    }
    __syncthreads();
    const int Sp = S + (S & 1);
    double* out = BsT + blk * 32LL * Sp;
    for (int e = threadIdx.x; e < 32 * Sp; e += blockDim.x) {
      // pair layout: e = (j >> 1) * 64 + rl * 2 + (j & 1)
      const int j = ((e >> 6) << 1) | (e & 1), rl = (e >> 1) & 31;
      double v = 0.0;
      if (rl < nrow && j < S) {
        const long long r = r0 + rl;
        const int cp = j % nr, bs = j / nr;
        const long long p = r / nr;
        const int qs = (int)(p / L) + bs / W2 - w, qt = (int)(p % L) + bs % W2 - w;
        if (qs >= 0 && qs < L && qt >= 0 && qt < L)
          v = tile[rl * (S + 1) + j] * s[r] * s[((long long)qs * L + qt) * nr + cp];
      }
      out[e] = v;
    }
    __syncthreads();
  }
}

template <int NR>
__device__ __forceinline__ double trow_apply(const double* __restrict__ BsT, long long R, int S,
                                             const int* __restrict__ off,
                                             const double* __restrict__ x, long long xb,
                                             long long r) {
  const int Sp = S + (S & 1);
  const double2* a = reinterpret_cast<const double2*>(BsT + (r >> 5) * (32LL * Sp)) + (r & 31);
  double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 4
  for (int m = 0; m < (Sp >> 1); ++m) {
    const double2 v = __ldg(a + 32 * m);
    acc0 = fma(v.x, __ldg(x + xb + off[2 * m]), acc0);
    acc1 = fma(v.y, __ldg(x + xb + off[2 * m + 1]), acc1);
  }
  return acc0 + acc1;
}

// Operators with fewer rows than this run the split form of tbox_pass (a CTA
// per 32-row block, its 8 warps each a slice of the slots): with a thread per
// row a 3 072-row level keeps 12 CTAs busy for 49 us per pass
constexpr long long kSplitMaxRows = 148LL * 256;

// y = BsT x over padded vectors for rows [0, R); returns partial dots x.y, y.y
template <int NR>
__device__ __forceinline__ void tbox_pass(int L, int w, const double* __restrict__ BsT,
                                          const double* __restrict__ x, double* __restrict__ y,
                                          const int* off, double* xy, double* yy) {
  const int W2 = 2 * w + 1, S = W2 * W2 * NR, Lpad = L + 2 * w;
  const long long R = (long long)L * L * NR;
  double d0 = 0.0, d1 = 0.0;
  if (R < kSplitMaxRows) {  // (uniform; the launchers size the grid to match)
    __shared__ double red[256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int Sp = S + (S & 1), M = Sp >> 1;
    const int per = (M + nw - 1) / nw;
    const int m0 = imin(warp * per, M), m1 = imin(m0 + per, M);
    const long long nblk = (R + 31) >> 5;
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
      const long long r = blk * 32 + lane;
      double acc0 = 0.0, acc1 = 0.0;
      long long yr = 0;
      if (r < R) {
        const long long p = r / NR;
        const int c = (int)(r - p * NR);
        const int ps = (int)(p / L), pt = (int)(p % L);
        const long long xb = ((long long)ps * Lpad + pt) * NR;
        yr = ((long long)(ps + w) * Lpad + pt + w) * NR + c;
        const double2* a = reinterpret_cast<const double2*>(BsT + blk * (32LL * Sp)) + lane;
#pragma unroll 4
        for (int m = m0; m < m1; ++m) {
          const double2 v = __ldg(a + 32 * m);
          acc0 = fma(v.x, __ldg(x + xb + off[2 * m]), acc0);
          acc1 = fma(v.y, __ldg(x + xb + off[2 * m + 1]), acc1);
        }
      }
      red[threadIdx.x] = acc0 + acc1;
      __syncthreads();
      if (warp == 0 && r < R) {
        double v = red[lane];
        for (int j = 1; j < nw; ++j) v += red[j * 32 + lane];  // slices in order
        y[yr] = v;
        d0 += x[yr] * v;
        d1 += v * v;
      }
      __syncthreads();
    }
    *xy = d0;
    *yy = d1;
    return;
  }
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < R;
       r += (long long)gridDim.x * blockDim.x) {
    const long long p = r / NR;
    const int c = (int)(r - p * NR);
    const int ps = (int)(p / L), pt = (int)(p % L);
    const long long xb = ((long long)ps * Lpad + pt) * NR;
    const double v = trow_apply<NR>(BsT, R, S, off, x, xb, r);
    const long long yr = ((long long)(ps + w) * Lpad + pt + w) * NR + c;
    y[yr] = v;
    d0 += x[yr] * v;
    d1 += v * v;
  }
  *xy = d0;
  *yy = d1;
}


// Tiled v4 SpMV for nr = 3 and L % 64 == 0: a CTA owns the 64 parents
// (ps, pt0..pt0+63) = 192 consecutive rows and stages their x window,
// (2w+1) padded grid rows x (64 + 2w) columns x 3, in shared memory.
constexpr int kTileP = 64;

__device__ __forceinline__ void tile_pass(int L, int w, const double* __restrict__ BsT,
                                          const double* __restrict__ x, double* __restrict__ y,
                                          const int* offw, double* xs, double* xy, double* yy) {
  const int W2 = 2 * w + 1, S = W2 * W2 * 3, Sp = S + (S & 1), Lpad = L + 2 * w;
  const int WC = kTileP + 2 * w;  // window columns (parents)
  const int tiles_per_row = L / kTileP;
  const long long ntile = (long long)L * tiles_per_row;
  double d0 = 0.0, d1 = 0.0;
  const int tid = threadIdx.x;  // 0..191: local row
  const int lp = tid / 3, c = tid - 3 * lp;
  for (long long t = blockIdx.x; t < ntile; t += gridDim.x) {
    const int ps = (int)(t / tiles_per_row), pt0 = (int)(t % tiles_per_row) * kTileP;
    // stage the window: padded rows ps..ps+2w, padded columns pt0..pt0+WC-1
    for (int e = tid; e < W2 * WC * 3; e += blockDim.x) {
      const int wr = e / (WC * 3), rem = e - wr * (WC * 3);
      xs[e] = x[((long long)(ps + wr) * Lpad + pt0) * 3 + rem];
    }
    __syncthreads();
    const long long r = ((long long)ps * L + pt0) * 3 + tid;
    const double2* a = reinterpret_cast<const double2*>(BsT + (r >> 5) * (32LL * Sp)) + (r & 31);
    const double* xb = xs + lp * 3;
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 4
    for (int m = 0; m < (Sp >> 1); ++m) {
      const double2 v = __ldg(a + 32 * m);
      acc0 = fma(v.x, xb[offw[2 * m]], acc0);
      acc1 = fma(v.y, xb[offw[2 * m + 1]], acc1);
    }
    const double val = acc0 + acc1;
    const long long yr = ((long long)(ps + w) * Lpad + pt0 + lp + w) * 3 + c;
    y[yr] = val;
    d0 += xs[(w * WC + lp + w) * 3 + c] * val;
    d1 += val * val;
    __syncthreads();
  }
  *xy = d0;
  *yy = d1;
}

__device__ __forceinline__ void build_offsets_window(int w, int* off) {
  const int W2 = 2 * w + 1, S = W2 * W2 * 3, WC = kTileP + 2 * w;
  for (int j = threadIdx.x; j < S + 1; j += blockDim.x) {
    const int jj = j < S ? j : 0;
    const int cc = jj % 3, bs = jj / 3;
    off[j] = ((bs / W2) * WC + (bs % W2)) * 3 + cc;
  }
}

__global__ void __launch_bounds__(192) k_tcg_spmv_tiled(int L, int w,
                                                        const double* __restrict__ BsT,
                                                        const double* __restrict__ p,
                                                        double* __restrict__ Ap, KState* st,
                                                        double* part) {
  extern __shared__ double dyn[];
  __shared__ double sh[32];
  if (st->done) return;
  const int S = (2 * w + 1) * (2 * w + 1) * 3;
  int* offw = reinterpret_cast<int*>(dyn);
  double* xs = dyn + ((S + 2) / 2 + 1);
  build_offsets_window(w, offw);
  __syncthreads();
  double dot, yy;
  tile_pass(L, w, BsT, p, Ap, offw, xs, &dot, &yy);
  dot = block_sum(dot, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = dot;
    part[2 * blockIdx.x + 1] = 0.0;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->pAp = a;
      if (!(a > 0.0)) {
        st->breakdown = st->it + 1;
        st->done = 1;
      } else {
        st->alpha = st->rs / a;
      }
    }
  }
}

__global__ void __launch_bounds__(192) k_tpow_apply_tiled(int L, int w,
                                                          const double* __restrict__ BsT,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y, KState* st,
                                                          double* part) {
  extern __shared__ double dyn[];
  __shared__ double sh[32];
  if (st->done) return;
  const int S = (2 * w + 1) * (2 * w + 1) * 3;
  int* offw = reinterpret_cast<int*>(dyn);
  double* xs = dyn + ((S + 2) / 2 + 1);
  build_offsets_window(w, offw);
  __syncthreads();
  double xy, yy;
  tile_pass(L, w, BsT, x, y, offw, xs, &xy, &yy);
  xy = block_sum(xy, sh);
  yy = block_sum(yy, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = xy;
    part[2 * blockIdx.x + 1] = yy;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->lam = a;
      st->ynorm = sqrt(b);
      if (st->ynorm == 0.0) {
        st->lam = 0.0;
        st->done = 1;
      }
    }
  }
}

__global__ void __launch_bounds__(192) k_tbox_apply_tiled(int L, int w,
                                                          const double* __restrict__ BsT,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y) {
  extern __shared__ double dyn[];
  const int S = (2 * w + 1) * (2 * w + 1) * 3;
  int* offw = reinterpret_cast<int*>(dyn);
  double* xs = dyn + ((S + 2) / 2 + 1);
  build_offsets_window(w, offw);
  __syncthreads();
  double xy, yy;
  tile_pass(L, w, BsT, x, y, offw, xs, &xy, &yy);
}


// ---------------------------------------------------------------------------
// Dual tiled SpMV: one pass over S B S serves two independent iterations
// (the subband PCG "A" and the lambda-estimate iteration "B" of the same
// level).  Each half has its own state, partials and reduction mode
// (0 = CG p.Ap -> alpha, 1 = power x.y, y.y -> lam, ynorm); a half whose
// state is done is skipped.  Block arrival is counted on A's state.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void finish_reduction(KState* st, int mode, double a, double b) {
  if (mode == 3) {  // raw partial sum of a row strip (gb_dist.cuh all-reduces it)
    st->pAp = a;
  } else if (mode == 0) {
    st->pAp = a;
    if (!(a > 0.0)) {
      st->breakdown = st->it + 1;
      st->done = 1;
    } else {
      st->alpha = st->rs / a;
    }
  } else {
    st->lam = a;
    st->ynorm = sqrt(b);
    if (st->ynorm == 0.0) {
      st->lam = 0.0;
      st->done = 1;
    }
  }
}

#include "gb_symspmv.cuh"

__global__ void __launch_bounds__(192) k_dual_apply(int L, int w, const double* __restrict__ BsT,
                                                    const double* __restrict__ xa,
                                                    double* __restrict__ ya, KState* sa,
                                                    double* pa, int ma,
                                                    const double* __restrict__ xb,
                                                    double* __restrict__ yb, KState* sb,
                                                    double* pb, int mb) {
  extern __shared__ double dyn[];
  __shared__ double sh[32];
  const bool act_a = !sa->done, act_b = !sb->done;
  if (!act_a && !act_b) return;
  if (!act_a || !act_b) {
    // one live half: plain single pass
    const double* x = act_a ? xa : xb;
    double* y = act_a ? ya : yb;
    KState* st = act_a ? sa : sb;
    double* part = act_a ? pa : pb;
    const int mode = act_a ? ma : mb;
    const int S = (2 * w + 1) * (2 * w + 1) * 3;
    int* offw = reinterpret_cast<int*>(dyn);
    double* xs = dyn + ((S + 2) / 2 + 1);
    build_offsets_window(w, offw);
    __syncthreads();
    double xy, yy;
    tile_pass(L, w, BsT, x, y, offw, xs, &xy, &yy);
    xy = block_sum(xy, sh);
    yy = block_sum(yy, sh);
    if (threadIdx.x == 0) {
      part[2 * blockIdx.x] = xy;
      part[2 * blockIdx.x + 1] = yy;
    }
    if (last_block(&st->counter)) {
      double a, b;
      final_sum2(part, gridDim.x, &a, &b, sh);
      if (threadIdx.x == 0) {
        st->counter = 0;
        finish_reduction(st, mode, a, b);
      }
    }
    return;
  }
  const int W2 = 2 * w + 1, S = W2 * W2 * 3, Sp = S + (S & 1), Lpad = L + 2 * w;
  const int WC = kTileP + 2 * w;
  int* offw = reinterpret_cast<int*>(dyn);
  double* xsa = dyn + ((S + 2) / 2 + 1);
  double* xsb = xsa + W2 * WC * 3;
  build_offsets_window(w, offw);
  __syncthreads();
  const int tiles_per_row = L / kTileP;
  const long long ntile = (long long)L * tiles_per_row;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  const int tid = threadIdx.x;
  const int lp = tid / 3, c = tid - 3 * lp;
  for (long long t = blockIdx.x; t < ntile; t += gridDim.x) {
    const int ps = (int)(t / tiles_per_row), pt0 = (int)(t % tiles_per_row) * kTileP;
    for (int e = tid; e < W2 * WC * 3; e += blockDim.x) {
      const int wr = e / (WC * 3), rem = e - wr * (WC * 3);
      const long long gi = ((long long)(ps + wr) * Lpad + pt0) * 3 + rem;
      xsa[e] = xa[gi];
      xsb[e] = xb[gi];
    }
    __syncthreads();
    const long long r = ((long long)ps * L + pt0) * 3 + tid;
    const double2* m = reinterpret_cast<const double2*>(BsT + (r >> 5) * (32LL * Sp)) + (r & 31);
    const double* xpa = xsa + lp * 3;
    const double* xpb = xsb + lp * 3;
    double u0 = 0.0, u1 = 0.0, v0 = 0.0, v1 = 0.0;
#pragma unroll 4
    for (int k = 0; k < (Sp >> 1); ++k) {
      const double2 v = __ldg(m + 32 * k);
      const int o0 = offw[2 * k], o1 = offw[2 * k + 1];
      u0 = fma(v.x, xpa[o0], u0);
      u1 = fma(v.y, xpa[o1], u1);
      v0 = fma(v.x, xpb[o0], v0);
      v1 = fma(v.y, xpb[o1], v1);
    }
    const double ua = u0 + u1, vb = v0 + v1;
    const long long yr = ((long long)(ps + w) * Lpad + pt0 + lp + w) * 3 + c;
    ya[yr] = ua;
    yb[yr] = vb;
    const int own = (w * WC + lp + w) * 3 + c;
    a0 += xsa[own] * ua;
    a1 += ua * ua;
    b0 += xsb[own] * vb;
    b1 += vb * vb;
    __syncthreads();
  }
  a0 = block_sum(a0, sh);
  a1 = block_sum(a1, sh);
  b0 = block_sum(b0, sh);
  b1 = block_sum(b1, sh);
  if (threadIdx.x == 0) {
    pa[2 * blockIdx.x] = a0;
    pa[2 * blockIdx.x + 1] = a1;
    pb[2 * blockIdx.x] = b0;
    pb[2 * blockIdx.x + 1] = b1;
  }
  if (last_block(&sa->counter)) {
    double a, b;
    final_sum2(pa, gridDim.x, &a, &b, sh);
    double cc, d;
    final_sum2(pb, gridDim.x, &cc, &d, sh);
    if (threadIdx.x == 0) {
      sa->counter = 0;
      finish_reduction(sa, ma, a, b);
      finish_reduction(sb, mb, cc, d);
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(256) k_tcg_spmv(int L, int w, const double* __restrict__ BsT,
                                                  const double* __restrict__ p,
                                                  double* __restrict__ Ap, KState* st,
                                                  double* part) {
  extern __shared__ int off[];
  __shared__ double sh[32];
  if (st->done) return;
  build_offsets(NR, w, L + 2 * w, off);
  double dot, yy;
  tbox_pass<NR>(L, w, BsT, p, Ap, off, &dot, &yy);
  dot = block_sum(dot, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = dot;
    part[2 * blockIdx.x + 1] = 0.0;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->pAp = a;
      if (!(a > 0.0)) {
        st->breakdown = st->it + 1;
        st->done = 1;
      } else {
        st->alpha = st->rs / a;
      }
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(256) k_tpow_apply(int L, int w, const double* __restrict__ BsT,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y, KState* st,
                                                    double* part) {
  extern __shared__ int off[];
  __shared__ double sh[32];
  if (st->done) return;
  build_offsets(NR, w, L + 2 * w, off);
  double xy, yy;
  tbox_pass<NR>(L, w, BsT, x, y, off, &xy, &yy);
  xy = block_sum(xy, sh);
  yy = block_sum(yy, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = xy;
    part[2 * blockIdx.x + 1] = yy;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->lam = a;
      st->ynorm = sqrt(b);
      if (st->ynorm == 0.0) {
        st->lam = 0.0;
        st->done = 1;
      }
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(256) k_tbox_apply(int L, int w, const double* __restrict__ BsT,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y) {
  extern __shared__ int off[];
  build_offsets(NR, w, L + 2 * w, off);
  double xy, yy;
  tbox_pass<NR>(L, w, BsT, x, y, off, &xy, &yy);
}


// ---------------------------------------------------------------------------
// Block-Jacobi preconditioned CG for the subband systems (S B S) z = rhs.
// Blocks: the 12 unknowns of each 2x2 group of parents (3 per parent).  The
// stopping rule is the reference's, ||r||_2 <= tol ||b||_2 on the true
// residual (sparse_core.py:161); only the iteration path differs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long bj_row_pad(int L, int w, int b, int l) {
  // block b of the (L/2)^2 block grid, local row l = (i*2 + j)*3 + c
  const int Lb = L >> 1;
  const int bs = b / Lb, bt = b - bs * Lb;
  const int pi = l / 3, c = l - 3 * pi;
  const int ps = 2 * bs + (pi >> 1), pt = 2 * bt + (pi & 1);
  const int Lpad = L + 2 * w;
  return ((long long)(ps + w) * Lpad + (pt + w)) * 3 + c;
}

// inverse of each 12x12 diagonal block of S B S (Gauss-Jordan, one warp per block)
__global__ void k_bj_setup(int L, int w, const double* __restrict__ B,
                           const double* __restrict__ s, float* __restrict__ inv, int blk0,
                           int blk1) {
  __shared__ double M[8][12][25];
  __shared__ double colk[8][12];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int Lb = L >> 1;
  const int S = box_slots(w, 3);
  for (int b = blk0 + blockIdx.x * 8 + wl; b < blk1; b += gridDim.x * 8) {
    const int bs = b / Lb, bt = b - bs * Lb;
    double (*m)[25] = M[wl];
    for (int e = lane; e < 144; e += 32) {
      const int l1 = e / 12, l2 = e % 12;
      const int p1 = l1 / 3, c1 = l1 % 3, p2 = l2 / 3, c2 = l2 % 3;
      const int ps1 = 2 * bs + (p1 >> 1), pt1 = 2 * bt + (p1 & 1);
      const int ps2 = 2 * bs + (p2 >> 1), pt2 = 2 * bt + (p2 & 1);
      const int ds = ps2 - ps1, dt = pt2 - pt1;
      const long long r1 = ((long long)ps1 * L + pt1) * 3 + c1;
      const long long r2 = ((long long)ps2 * L + pt2) * 3 + c2;
      double v = 0.0;
      if (ds >= -w && ds <= w && dt >= -w && dt <= w)
        v = B[r1 * S + slot_of(w, 3, ds, dt, c2)] * s[r1] * s[r2];
      m[l1][l2] = v;
      m[l1][12 + l2] = (l1 == l2) ? 1.0 : 0.0;
    }
    __syncwarp();
    for (int k = 0; k < 12; ++k) {
      const double piv = 1.0 / m[k][k];
      __syncwarp();
      if (lane < 24) m[k][lane] *= piv;
      if (lane < 12) colk[wl][lane] = m[lane][k];
      __syncwarp();
      for (int e = lane; e < 12 * 24; e += 32) {
        const int i = e / 24, c = e % 24;
        if (i != k) m[i][c] -= colk[wl][i] * m[k][c];
      }
      __syncwarp();
    }
    // symmetrized and rounded to fp32: the preconditioner only has to be a
    // fixed SPD operator (the residual stays fp64), half the bytes per step
    for (int e = lane; e < 144; e += 32) {
      const int i = e / 12, j = e % 12;
      inv[(long long)b * 144 + e] = (float)(0.5 * (m[i][12 + j] + m[j][12 + i]));
    }
    __syncwarp();
  }
}

// x += alpha p; r -= alpha Ap; z = Minv r; (r.r, r.z) -> convergence, beta
__global__ void __launch_bounds__(192) k_bjcg_update(int L, int w, double* __restrict__ x,
                                                     double* __restrict__ r,
                                                     const double* __restrict__ p,
                                                     const double* __restrict__ Ap,
                                                     double* __restrict__ z,
                                                     const float* __restrict__ inv,
                                                     KState* st, double* part) {
  __shared__ double rs[192];
  __shared__ double sh[32];
  if (st->done) return;
  const double alpha = st->alpha;
  const int nb = (L >> 1) * (L >> 1);
  const int lb = threadIdx.x / 12, l = threadIdx.x % 12;
  double rr = 0.0, rz = 0.0;
  for (int b0 = blockIdx.x * 16; b0 < nb; b0 += gridDim.x * 16) {
    const int b = b0 + lb;
    long long pr = -1;
    double rv = 0.0;
    if (b < nb) {
      pr = bj_row_pad(L, w, b, l);
      x[pr] += alpha * p[pr];
      rv = r[pr] - alpha * Ap[pr];
      r[pr] = rv;
      rr += rv * rv;
    }
    rs[threadIdx.x] = rv;
    __syncthreads();
    if (b < nb) {
      const float* iv = inv + (long long)b * 144 + l * 12;
      const double* rb = rs + lb * 12;
      double zv = 0.0;
      float iw[12];  // 48-byte rows of a 576-byte block: three 16-byte loads
#pragma unroll
      for (int q4 = 0; q4 < 3; ++q4) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(iv) + q4);
        iw[4 * q4] = f.x;
        iw[4 * q4 + 1] = f.y;
        iw[4 * q4 + 2] = f.z;
        iw[4 * q4 + 3] = f.w;
      }
#pragma unroll
      for (int k = 0; k < 12; ++k) zv = fma((double)iw[k], rb[k], zv);
      z[pr] = zv;
      rz += rv * zv;
    }
    __syncthreads();
  }
  rr = block_sum(rr, sh);
  rz = block_sum(rz, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = rr;
    part[2 * blockIdx.x + 1] = rz;
  }
  if (last_block(&st->counter)) {
    double a, c;
    final_sum2(part, gridDim.x, &a, &c, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->it += 1;
      const double rn = sqrt(a);
      st->rnorm = rn;
      if (rn <= st->tol_abs) {
        st->done = 1;
        st->converged = 1;
      } else if (st->it >= st->max_iter) {
        st->done = 1;
        st->converged = 0;
      } else {
        st->beta = c / st->rs;
        st->rs = c;
      }
    }
  }
}

// k_bjcg_update for the symmetric band layout: Ap of each row is the phase-1
// partial plus the neighbour tiles' spill-over (symb_fix_value, the value
// k_symb_fix would store), alpha was set by k_symb_apply (red = 1).
__global__ void __launch_bounds__(192) k_symb_bjcg_update(int L, int w, double* __restrict__ x,
                                                          double* __restrict__ r,
                                                          const double* __restrict__ p,
                                                          const double* __restrict__ Ap,
                                                          double* __restrict__ z,
                                                          const float* __restrict__ inv,
                                                          KState* st, double* part) {
  __shared__ double rs[192];
  __shared__ double sh[32];
  if (st->done) return;
  const double alpha = st->alpha;
  const int nb = (L >> 1) * (L >> 1), Lb = L >> 1, Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const int lb = threadIdx.x / 12, l = threadIdx.x % 12;
  const int pi = l / 3, c = l - 3 * pi;
  double rr = 0.0, rz = 0.0;
  for (int b0 = blockIdx.x * 16; b0 < nb; b0 += gridDim.x * 16) {
    const int b = b0 + lb;
    long long pr = -1;
    double rv = 0.0;
    if (b < nb) {
      const int bs = b / Lb, bt = b - bs * Lb;
      const int ps = 2 * bs + (pi >> 1), pt = 2 * bt + (pi & 1);
      pr = ((long long)(ps + w) * Lpad + (pt + w)) * 3 + c;
      const double ap = symb_fix_value(Ap[pr], Ap + npad, L, w, ps, pt, c);
      x[pr] += alpha * p[pr];
      rv = r[pr] - alpha * ap;
      r[pr] = rv;
      rr += rv * rv;
    }
    rs[threadIdx.x] = rv;
    __syncthreads();
    if (b < nb) {
      const float* iv = inv + (long long)b * 144 + l * 12;
      const double* rb = rs + lb * 12;
      double zv = 0.0;
      float iw[12];  // 48-byte rows of a 576-byte block: three 16-byte loads
#pragma unroll
      for (int q4 = 0; q4 < 3; ++q4) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(iv) + q4);
        iw[4 * q4] = f.x;
        iw[4 * q4 + 1] = f.y;
        iw[4 * q4 + 2] = f.z;
        iw[4 * q4 + 3] = f.w;
      }
#pragma unroll
      for (int k = 0; k < 12; ++k) zv = fma((double)iw[k], rb[k], zv);
      z[pr] = zv;
      rz += rv * zv;
    }
    __syncthreads();
  }
  rr = block_sum(rr, sh);
  rz = block_sum(rz, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = rr;
    part[2 * blockIdx.x + 1] = rz;
  }
  if (last_block(&st->counter)) {
    double a, cc;
    final_sum2(part, gridDim.x, &a, &cc, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->it += 1;
      const double rn = sqrt(a);
      st->rnorm = rn;
      if (rn <= st->tol_abs) {
        st->done = 1;
        st->converged = 1;
      } else if (st->it >= st->max_iter) {
        st->done = 1;
        st->converged = 0;
      } else {
        st->beta = cc / st->rs;
        st->rs = cc;
      }
    }
  }
}

// Lanczos step fused with phase 2 of the symmetric SpMV (layout 1): y's own
// partial plus the neighbours' spill-over is completed in registers, alpha
// comes from the phase-1 reduction by linearity (st->pAp = x.y, run with
// red = 1), then the recurrence of k_lz_step.  Interior rows only: the
// zero halo of every vector is never written.  Tile-aligned: a CTA walks
// whole tiles (kSymTH grid rows x 64 parents), so the neighbour spill
// regions are CTA-uniform and added in symb_fix_value's order without any
// per-element division.
constexpr int kLzThreads = 256;
__global__ void __launch_bounds__(kLzThreads) k_symb_lz_update(int L, int w,
                                                               const double* __restrict__ x,
                                                               double* __restrict__ y,
                                                               double* __restrict__ vp,
                                                               KState* st, double* part,
                                                               double* ab) {
  __shared__ double sh[32];
  if (st->done) return;
  const double bp = st->aux0, ibp = 1.0 / bp;
  const double alpha = st->pAp * ibp * ibp;
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const double* ov = y + npad;
  const int WC = kSymTW + 2 * w, RG = symb_region(w), tpr = L / kSymTW;
  const int KI = (w + kSymTH - 1) / kSymTH;
  const long long ntile = symb_ntile(L);
  constexpr int TE = kSymTH * kSymTW * 3;  // elements per tile
  double uu = 0.0;
  for (long long tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int I = (int)(tile / tpr), J = (int)(tile - (long long)I * tpr);
    // all loads of the thread's NE elements first (stores to y / vp would
    // otherwise order them), then the recurrence in element order
    constexpr int NE = TE / kLzThreads;
    static_assert(TE % kLzThreads == 0, "tile must split evenly over the CTA");
    double yv[NE], xv[NE], vv[NE];
    long long yis[NE];
#pragma unroll
    for (int q = 0; q < NE; ++q) {
      const int e = threadIdx.x + q * kLzThreads;
      const int h = e / (kSymTW * 3), rem = e - h * (kSymTW * 3);
      const int j = rem / 3, c = rem - 3 * j;
      const int ps = I * kSymTH + h, pt = J * kSymTW + j;
      const long long yi = ((long long)(ps + w) * Lpad + pt + w) * 3 + c;
      yis[q] = yi;
      double v = y[yi];
      // neighbour spill-over in symb_fix_value's order
      const bool left = j < w && J > 0, right = j >= kSymTW - w && J + 1 < tpr;
      for (int dI = 0; dI <= KI; ++dI) {
        const int Ip = I - dI, rr = h + dI * kSymTH;
        if (Ip < 0 || rr >= kSymTH + w) break;
        const double* base = ov + ((long long)Ip * tpr + J) * RG + (rr * WC + w) * 3 + c;
        if (left) v += base[-RG + (j + kSymTW) * 3];
        if (dI > 0) v += base[j * 3];
        if (right) v += base[RG + (j - kSymTW) * 3];
      }
      yv[q] = v;
      xv[q] = x[yis[q]];
      vv[q] = vp[yis[q]];
    }
#pragma unroll
    for (int q = 0; q < NE; ++q) {
      const double u = (yv[q] - alpha * xv[q]) * ibp - bp * vv[q];
      vp[yis[q]] = xv[q] * ibp;
      y[yis[q]] = u;
      uu += u * u;
    }
  }
  uu = block_sum(uu, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = uu;
    part[2 * blockIdx.x + 1] = 0.0;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      const double beta = sqrt(a);
      ab[2 * st->it] = alpha;
      ab[2 * st->it + 1] = beta;
      st->it += 1;
      st->aux0 = beta;
      if (!(beta > 0.0) || st->it >= st->max_iter) st->done = 1;
    }
  }
}

// start: x = s x0 (or 0), r = b - s A x0 (Ax0 null => x0 = 0), z = Minv r, p = z;
// ||b||, ||r||, r.z and the early exits of sparse_core.py:138-148.  Partials
// are (||r||^2, r.z) pairs in part[0, 2G) and ||b||^2 in part[2G, 3G), so the
// grid is capped at 2/3 of the caller's 2 * kRedBlocks partial slots.
__global__ void __launch_bounds__(192) k_bjcg_init(int L, int w, const double* __restrict__ b,
                                                   const double* __restrict__ x0,
                                                   const double* __restrict__ Ax0,
                                                   double x0_scale,
                                                   double* __restrict__ x, double* __restrict__ r,
                                                   double* __restrict__ p,
                                                   double* __restrict__ z,
                                                   const float* __restrict__ inv,
                                                   double rel_tol, int max_iter, KState* st,
                                                   double* part) {
  __shared__ double rs[192];
  __shared__ double sh[32];
  const int nb = (L >> 1) * (L >> 1);
  const int lb = threadIdx.x / 12, l = threadIdx.x % 12;
  double bb = 0.0, rr = 0.0, rz = 0.0;
  for (int b0 = blockIdx.x * 16; b0 < nb; b0 += gridDim.x * 16) {
    const int bk = b0 + lb;
    long long pr = -1;
    double rv = 0.0;
    if (bk < nb) {
      pr = bj_row_pad(L, w, bk, l);
      const double bv = b[pr];
      rv = Ax0 ? bv - x0_scale * Ax0[pr] : bv;
      x[pr] = x0 ? x0_scale * x0[pr] : 0.0;
      r[pr] = rv;
      bb += bv * bv;
      rr += rv * rv;
    }
    rs[threadIdx.x] = rv;
    __syncthreads();
    if (bk < nb) {
      const float* iv = inv + (long long)bk * 144 + l * 12;
      const double* rb = rs + lb * 12;
      double zv = 0.0;
      float iw[12];  // 48-byte rows of a 576-byte block: three 16-byte loads
#pragma unroll
      for (int q4 = 0; q4 < 3; ++q4) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(iv) + q4);
        iw[4 * q4] = f.x;
        iw[4 * q4 + 1] = f.y;
        iw[4 * q4 + 2] = f.z;
        iw[4 * q4 + 3] = f.w;
      }
#pragma unroll
      for (int k = 0; k < 12; ++k) zv = fma((double)iw[k], rb[k], zv);
      z[pr] = zv;
      p[pr] = zv;
      rz += rv * zv;
    }
    __syncthreads();
  }
  rr = block_sum(rr, sh);
  rz = block_sum(rz, sh);
  bb = block_sum(bb, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = rr;
    part[2 * blockIdx.x + 1] = rz;
    part[2 * gridDim.x + blockIdx.x] = bb;
  }
  if (last_block(&st->counter)) {
    double a, c;
    final_sum2(part, gridDim.x, &a, &c, sh);
    double bsum = 0.0;
    for (int j = threadIdx.x; j < (int)gridDim.x; j += blockDim.x) bsum += part[2 * gridDim.x + j];
    bsum = block_sum(bsum, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      st->it = 0;
      st->breakdown = 0;
      st->max_iter = max_iter;
      const double bn = sqrt(bsum);
      st->bnorm = bn;
      st->tol_abs = rel_tol * bn;
      const double rn = sqrt(a);
      st->rnorm = rn;
      st->rs = c;
      st->done = 0;
      st->converged = 0;
      st->aux0 = 0.0;
      if (bn == 0.0) {
        st->done = 1;
        st->converged = 1;
        st->rnorm = 0.0;
        st->aux0 = 1.0;  // x must be zeroed (zero rhs)
      } else if (rn <= rel_tol * bn) {
        st->done = 1;
        st->converged = 1;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K9 transfers
// ---------------------------------------------------------------------------
// out[(p,c)] = s[(p,c)] * sum_a W[c][a] g[child_a(p)]   (s may be null)
__global__ void k_apply_w(int Lp, WTemplate W, const double* __restrict__ g,
                          const double* __restrict__ s, double* __restrict__ out,
                          long long e0, long long e1) {
  const int Lk = 2 * Lp;
  for (long long p = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; p < e1;
       p += (long long)gridDim.x * blockDim.x) {
    const int ps = (int)(p / Lp), pt = (int)(p % Lp);
    double gv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
      gv[a] = g[(long long)(2 * ps + (a >> 1)) * Lk + 2 * pt + (a & 1)];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (W.w[c][a] != 0.0) acc += W.w[c][a] * gv[a];
      out[p * 3 + c] = s ? s[p * 3 + c] * acc : acc;
    }
  }
}

// v[child_a(p)] = sum_c W[c][a] w[(p,c)]   (W^T w, csc scatter order)
__global__ void k_apply_wt(int Lp, WTemplate W, const double* __restrict__ w,
                           double* __restrict__ v, long long e0, long long e1) {
  const int Lk = 2 * Lp;
  for (long long p = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; p < e1;
       p += (long long)gridDim.x * blockDim.x) {
    const int ps = (int)(p / Lp), pt = (int)(p % Lp);
    const double w0 = w[p * 3], w1 = w[p * 3 + 1], w2 = w[p * 3 + 2];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double acc = 0.0;
      if (W.w[0][a] != 0.0) acc += W.w[0][a] * w0;
      if (W.w[1][a] != 0.0) acc += W.w[1][a] * w1;
      if (W.w[2][a] != 0.0) acc += W.w[2][a] * w2;
      v[(long long)(2 * ps + (a >> 1)) * Lk + 2 * pt + (a & 1)] = acc;
    }
  }
}

// g'[i] = sum over R row i in ascending column order (ds, alpha, dt, beta)
__global__ void k_apply_r(int Lp, int rho, const double* __restrict__ R,
                          const double* __restrict__ g, double* __restrict__ out,
                          long long e0, long long e1) {
  const int W2 = 2 * rho + 1, Lk = 2 * Lp;
  const int S = W2 * W2 * 4;
  for (long long i = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e1;
       i += (long long)gridDim.x * blockDim.x) {
    const int is = (int)(i / Lp), it = (int)(i % Lp);
    const double* row = R + i * S;
    double acc = 0.0;
    for (int dsi = 0; dsi < W2; ++dsi) {
      const int qs = is + dsi - rho;
      if (qs < 0 || qs >= Lp) continue;
      for (int alpha = 0; alpha < 2; ++alpha) {
        for (int dti = 0; dti < W2; ++dti) {
          const int qt = it + dti - rho;
          if (qt < 0 || qt >= Lp) continue;
          for (int beta = 0; beta < 2; ++beta) {
            const double rv = row[(dsi * W2 + dti) * 4 + 2 * alpha + beta];
            if (rv != 0.0)
              acc += rv * g[(long long)(2 * qs + alpha) * Lk + 2 * qt + beta];
          }
        }
      }
    }
    out[i] = acc;
  }
}

// inc[f] = sum_{j asc} psi[j][f] v[j]   (psi^T v, csc scatter order)
__global__ void k_psi_t_apply(int n, int L, int lo, int wd, const double* __restrict__ psi,
                              const double* __restrict__ v, double* __restrict__ inc,
                              int F0, int F1, int j_lo, int j_hi) {
  const int h = n / L;
  const int hi = lo + wd - 1;  // only meaningful when the window is unclipped
  const long long per = (long long)wd * wd;
  for (long long f = (long long)F0 * n + blockIdx.x * (long long)blockDim.x + threadIdx.x;
       f < (long long)F1 * n; f += (long long)gridDim.x * blockDim.x) {
    const int fs = (int)(f / n), ft = (int)(f % n);
    // rows j whose window covers f; windows are monotone in j, use a safe range
    int j0s, j1s, j0t, j1t;
    if (wd >= n) {
      j0s = 0; j1s = L - 1; j0t = 0; j1t = L - 1;
    } else {
      j0s = imax(0, (fs - hi) / h - 1); j1s = imin(L - 1, (fs - lo) / h + 1);
      j0t = imax(0, (ft - hi) / h - 1); j1t = imin(L - 1, (ft - lo) / h + 1);
    }
    j0s = imax(j0s, j_lo);
    j1s = imin(j1s, j_hi - 1);
    double acc = 0.0;
    for (int js = j0s; js <= j1s; ++js) {
      const int ls = fs - clampi(js * h + lo, 0, n - wd);
      if (ls < 0 || ls >= wd) continue;
      for (int jt = j0t; jt <= j1t; ++jt) {
        const int lt = ft - clampi(jt * h + lo, 0, n - wd);
        if (lt < 0 || lt >= wd) continue;
        const long long j = (long long)js * L + jt;
        const double pv = psi[j * per + ls * wd + lt];
        if (pv != 0.0) acc += pv * v[j];
      }
    }
    inc[f] = acc;
  }
}

// out[i] = sum over row i's window (ascending) psi[i][f] b[f]   (psi @ b)
__global__ void k_psi_apply(int n, int L, int lo, int wd, const double* __restrict__ psi,
                            const double* __restrict__ b, double* __restrict__ out) {
  const long long rows = (long long)L * L;
  const int h = n / L;
  const long long per = (long long)wd * wd;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = wid; i < rows; i += nwarps) {
    const int os = clampi((int)(i / L) * h + lo, 0, n - wd);
    const int ot = clampi((int)(i % L) * h + lo, 0, n - wd);
    const double* row = psi + i * per;
    double acc = 0.0;
    for (long long e = lane; e < per; e += 32) {
      const double v = row[e];
      if (v != 0.0) acc += v * b[(long long)(os + e / wd) * n + ot + e % wd];
    }
    acc = warp_sum(acc);
    if (lane == 0) out[i] = acc;
  }
}

__global__ void k_axpby(long long n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (y ? a * x[i] + b * y[i] : a * x[i]);
}

__global__ void k_vmul(long long n, const double* __restrict__ a, const double* __restrict__ b,
                       double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}

__global__ void k_vadd(long long n, const double* __restrict__ a, const double* __restrict__ b,
                       double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}

#include "gb_dist.cuh"

}  // namespace gb

using namespace gb;

#ifndef GB_RED_BLOCKS
#define GB_RED_BLOCKS (148 * 8)
#endif
static const int kRedBlocks = GB_RED_BLOCKS;  // 8 per SM on 148 SMs; partials sized by the caller

static inline int grid_for(long long work, int block, int cap) {
  long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

static inline WTemplate mkW(const double* w12) {
  WTemplate W;
  for (int c = 0; c < 3; ++c)
    for (int a = 0; a < 4; ++a) W.w[c][a] = w12[c * 4 + a];
  return W;
}

size_t gbk_kstate_bytes() { return sizeof(KState); }
int gbk_red_blocks() { return kRedBlocks; }

namespace gb {
__global__ void k_state_reset(KState* st, int max_iter) {
  KState z = {};
  z.max_iter = max_iter;
  *st = z;
}
}  // namespace gb

int gbk_state_reset(void* st, int max_iter, cudaStream_t s) {
  k_state_reset<<<1, 1, 0, s>>>((KState*)st, max_iter);
  return (int)cudaGetLastError();
}

int gbk_cg_init(long long n, const double* b, const double* x0, const double* Ax0,
                double* x, double* r, double* p, double rel_tol, int max_iter,
                void* st, double* part, cudaStream_t s) {
  const int g = grid_for(n, 256, kRedBlocks);
  k_cg_init<<<g, 256, 0, s>>>(n, b, x0, Ax0, x, r, p, rel_tol, max_iter, (KState*)st,
                              part);
  k_cg_zero_if<<<grid_for(n, 256, kRedBlocks), 256, 0, s>>>(n, x, (KState*)st);
  return (int)cudaGetLastError();
}

int gbk_cg_iterations(int L, int nr, int w, const double* B, const double* sv,
                      int mode, double* x, double* r, double* p, double* Ap,
                      int iters, void* st, double* part, cudaStream_t s) {
  const long long n = (long long)L * L * nr;
  const int gs = grid_for(n * 32, 256, kRedBlocks);
  const int gv = grid_for(n, 256, kRedBlocks);
  KState* k = (KState*)st;
  for (int i = 0; i < iters; ++i) {
    k_cg_spmv<<<gs, 256, 0, s>>>(L, nr, w, B, sv, mode, p, Ap, k, part);
    k_cg_update<<<gv, 256, 0, s>>>(n, x, r, p, Ap, k, part);
    k_cg_dir<<<gv, 256, 0, s>>>(n, r, p, k);
  }
  return (int)cudaGetLastError();
}

int gbk_pow_iterations(int L, int nr, int w, const double* B, const double* sv,
                       int mode, double* x, double* y, double tol, int iters,
                       void* st, double* part, cudaStream_t s) {
  const long long n = (long long)L * L * nr;
  const int gs = grid_for(n * 32, 256, kRedBlocks);
  const int gv = grid_for(n, 256, kRedBlocks);
  KState* k = (KState*)st;
  for (int i = 0; i < iters; ++i) {
    k_pow_apply<<<gs, 256, 0, s>>>(L, nr, w, B, sv, mode, x, y, k, part);
    k_pow_step<<<gv, 256, 0, s>>>(n, x, y, tol, k, part);
    k_pow_scale<<<gv, 256, 0, s>>>(n, x, y, k);
  }
  return (int)cudaGetLastError();
}


// ---- v2 (pre-scaled, padded) launchers ----
int gbk_scale_box(int L, int nr, int w, const double* B, const double* sv, double* Bs,
                  cudaStream_t s) {
  const long long total = (long long)L * L * nr * (2 * w + 1) * (2 * w + 1) * nr;
  k_scale_box<<<grid_for(total, 256, 148 * 16), 256, 0, s>>>(L, nr, w, B, sv, Bs);
  return (int)cudaGetLastError();
}
int gbk_pad(int L, int nr, int w, const double* src, const double* scale, double* dst,
            cudaStream_t s) {
  return gbk_pad_rows(L, nr, w, src, scale, dst, 0, L, s);
}
int gbk_pad_rows(int L, int nr, int w, const double* src, const double* scale, double* dst,
                 int r0, int r1, cudaStream_t s) {
  if (r0 < 0 || r1 > L || r0 > r1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long per = (long long)L * nr;
  k_pad<<<grid_for((r1 - r0) * per, 256, 148 * 16), 256, 0, s>>>(L, nr, w, src, scale, dst,
                                                                 r0 * per, r1 * per);
  return (int)cudaGetLastError();
}
int gbk_unpad(int L, int nr, int w, const double* src, const double* scale, double* dst,
              cudaStream_t s) {
  return gbk_unpad_rows(L, nr, w, src, scale, dst, 0, L, s);
}
int gbk_unpad_rows(int L, int nr, int w, const double* src, const double* scale, double* dst,
                   int r0, int r1, cudaStream_t s) {
  if (r0 < 0 || r1 > L || r0 > r1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long per = (long long)L * nr;
  k_unpad<<<grid_for((r1 - r0) * per, 256, 148 * 16), 256, 0, s>>>(L, nr, w, src, scale, dst,
                                                                   r0 * per, r1 * per);
  return (int)cudaGetLastError();
}
static inline size_t off_smem(int nr, int w) {
  return ((size_t)(2 * w + 1) * (2 * w + 1) * nr + 2) * sizeof(int);
}
static inline int point_grid(int L) {
  return grid_for((long long)L * L * 32, 256, kRedBlocks);
}
int gbk_pcg_iterations(int L, int nr, int w, const double* Bs, double* x, double* r,
                       double* p, double* Ap, int iters, void* st, double* part,
                       cudaStream_t s) {
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * nr;
  const int gs = point_grid(L);
  const int gv = grid_for(npad, 256, kRedBlocks);
  const size_t sm = off_smem(nr, w);
  KState* k = (KState*)st;
  for (int i = 0; i < iters; ++i) {
    if (nr == 3) k_pcg_spmv<3><<<gs, 256, sm, s>>>(L, w, Bs, p, Ap, k, part);
    else k_pcg_spmv<1><<<gs, 256, sm, s>>>(L, w, Bs, p, Ap, k, part);
    k_cg_update<<<gv, 256, 0, s>>>(npad, x, r, p, Ap, k, part);
    k_cg_dir<<<gv, 256, 0, s>>>(npad, r, p, k);
  }
  return (int)cudaGetLastError();
}
int gbk_ppow_iterations(int L, int nr, int w, const double* Bs, double* x, double* y,
                        double tol, int iters, void* st, double* part, cudaStream_t s) {
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * nr;
  const int gs = point_grid(L);
  const int gv = grid_for(npad, 256, kRedBlocks);
  const size_t sm = off_smem(nr, w);
  KState* k = (KState*)st;
  for (int i = 0; i < iters; ++i) {
    if (nr == 3) k_ppow_apply<3><<<gs, 256, sm, s>>>(L, w, Bs, x, y, k, part);
    else k_ppow_apply<1><<<gs, 256, sm, s>>>(L, w, Bs, x, y, k, part);
    k_pow_step<<<gv, 256, 0, s>>>(npad, x, y, tol, k, part);
    k_pow_scale<<<gv, 256, 0, s>>>(npad, x, y, k);
  }
  return (int)cudaGetLastError();
}
int gbk_pbox_apply(int L, int nr, int w, const double* Bs, const double* x, double* y,
                   cudaStream_t s) {
  const int gs = point_grid(L);
  const size_t sm = off_smem(nr, w);
  if (nr == 3) k_pbox_apply<3><<<gs, 256, sm, s>>>(L, w, Bs, x, y);
  else k_pbox_apply<1><<<gs, 256, sm, s>>>(L, w, Bs, x, y);
  return (int)cudaGetLastError();
}


// ---- v3 (slot-major) launchers ----
static inline int row_grid(long long R) {
  // small operators: a CTA per 32-row block (tbox_pass, split form)
  if (R < kSplitMaxRows) return grid_for((R + 31) / 32 * 256, 256, kRedBlocks);
  return grid_for(R, 256, kRedBlocks);
}
static inline bool use_tiled(int L, int nr, int w) {
  return nr == 3 && L % kTileP == 0 && w <= 8;
}
static inline size_t tiled_smem(int w) {
  const int S = (2 * w + 1) * (2 * w + 1) * 3;
  return ((S + 2) / 2 + 1) * sizeof(double) +
         (size_t)(2 * w + 1) * (kTileP + 2 * w) * 3 * sizeof(double);
}
static inline int tiled_grid(int L) {
  const long long nt = (long long)L * (L / kTileP);
  return (int)(nt < kRedBlocks ? nt : kRedBlocks);
}
size_t gbk_boxT_elems(int L, int nr, int w) {
  const long long R = (long long)L * L * nr;
  const long long S = (long long)(2 * w + 1) * (2 * w + 1) * nr;
  return (size_t)((R + 31) / 32) * 32 * (S + (S & 1));
}
int gbk_scale_box_T(int L, int nr, int w, const double* B, const double* sv, double* BsT,
                    cudaStream_t s) {
  const int S = (2 * w + 1) * (2 * w + 1) * nr;
  const size_t smem = (size_t)32 * (S + 1) * sizeof(double);
  if (smem > 200 * 1024) {
    const long long total = (long long)gbk_boxT_elems(L, nr, w);
    k_scale_box_T_strided<<<grid_for(total, 256, 148 * 16), 256, 0, s>>>(L, nr, w, B, sv, BsT);
    return (int)cudaGetLastError();
  }
  cudaFuncSetAttribute(k_scale_box_T, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const long long nblk = ((long long)L * L * nr + 31) / 32;
  k_scale_box_T<<<(int)(nblk < 148 * 8 ? nblk : 148 * 8), 256, smem, s>>>(L, nr, w, B, sv, BsT);
  return (int)cudaGetLastError();
}
static inline bool use_sym(int layout, int L, int nr, int w) {
  return layout == 1 && use_tiled(L, nr, w) && L % kSymTH == 0 &&
         symb_smem(w, 2) <= 226 * 1024;
}
// phase 1 of the symmetric band SpMV for nv = 1 or 2 vectors; red_v = 1 forms
// the CG reduction x_v.(A x_v) -> alpha in the same pass (the consumer is then
// k_symb_bjcg_update, which adds the spill-over itself)
#ifndef GB_SYM_WS
#define GB_SYM_WS 1  // warp-specialized bulk-copy phase 1 (0: register-pipelined)
#endif
int g_sym_ws_ctas = 0;  // gb_tune(3): CTA cap of the warp-specialized phase 1 (0: 148)
int g_sym_ws_on = 1;    // gb_tune(5): 0 = register-pipelined phase 1 (smaller CTAs)
static void sym_phase1(int L, int w, const double* U, int nv, const double* x0, double* y0,
                       KState* s0, double* p0, int r0, const double* x1, double* y1,
                       KState* s1, double* p1, int r1, cudaStream_t s, long long t0 = 0,
                       long long t1 = -1) {
  if (t1 < 0) t1 = symb_ntile(L);
  const int nt = (int)(t1 - t0);
  // dynamic shared memory attribute raised to what a launch needs (the
  // kernels also have static shared memory, so the 227 KB cap is not usable)
  static size_t attr[2][3] = {{0, 0, 0}, {0, 0, 0}};
  static size_t attr2[3] = {0, 0, 0};  // the 2-stage instances
  const int st_pref = nv == 1 ? symb_ws_stages<1>() : symb_ws_stages<2>();
#ifndef GB_SYM_MIN_STAGES
#define GB_SYM_MIN_STAGES 2
#endif
  const int st = symb_ws_smem(w, nv, st_pref) <= 226 * 1024 ? st_pref : GB_SYM_MIN_STAGES;
  const bool ws = GB_SYM_WS && g_sym_ws_on && symb_ws_smem(w, nv, st) <= 226 * 1024;
  if (ws) {
    // persistent: one CTA per SM, at most g_sym_ws_ctas (the HBM stream
    // saturates on fewer SMs; the rest stay free for the concurrent setup)
    const int cap = g_sym_ws_ctas > 0 && g_sym_ws_ctas < 148 ? g_sym_ws_ctas : 148;
    const int gp = nt < cap ? nt : cap;
    const size_t sm = symb_ws_smem(w, nv, st);
    size_t& have = st == st_pref ? attr[1][nv] : attr2[nv];
    if (sm > have) {
      if (nv == 2 && st == 3)
        cudaFuncSetAttribute(k_symb_apply_ws<2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
      else if (nv == 2)
        cudaFuncSetAttribute(k_symb_apply_ws<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
      else if (st == 4)
        cudaFuncSetAttribute(k_symb_apply_ws<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
      else
        cudaFuncSetAttribute(k_symb_apply_ws<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
      have = sm;
    }
    if (nv == 2 && st == 3)
      k_symb_apply_ws<2, 3><<<gp, 2 * kSymThreads + 32, sm, s>>>(L, w, U, x0, y0, s0, p0, r0, x1,
                                                                 y1, s1, p1, r1, t0, t1);
    else if (nv == 2)
      k_symb_apply_ws<2, 2><<<gp, 2 * kSymThreads + 32, sm, s>>>(L, w, U, x0, y0, s0, p0, r0, x1,
                                                                 y1, s1, p1, r1, t0, t1);
    else if (st == 4)
      k_symb_apply_ws<1, 4><<<gp, kSymThreads + 32, sm, s>>>(L, w, U, x0, y0, s0, p0, r0, nullptr,
                                                             nullptr, nullptr, nullptr, 0, t0, t1);
    else
      k_symb_apply_ws<1, 2><<<gp, kSymThreads + 32, sm, s>>>(L, w, U, x0, y0, s0, p0, r0, nullptr,
                                                             nullptr, nullptr, nullptr, 0, t0, t1);
    return;
  }
  const int gp = nt < kRedBlocks ? nt : kRedBlocks;
  const size_t sm = symb_smem(w, nv);
  if (sm > attr[0][nv]) {
    if (nv == 2)
      cudaFuncSetAttribute(k_symb_apply<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    else
      cudaFuncSetAttribute(k_symb_apply<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr[0][nv] = sm;
  }
  if (nv == 2)
    k_symb_apply<2><<<gp, kSymThreads, sm, s>>>(L, w, U, x0, y0, s0, p0, r0, x1, y1, s1, p1, r1,
                                                 t0, t1);
  else
    k_symb_apply<1><<<gp, kSymThreads, sm, s>>>(L, w, U, x0, y0, s0, p0, r0, nullptr, nullptr,
                                                 nullptr, nullptr, 0, t0, t1);
}
// phase 2 alone (spill-over + reductions of mode m_v) for nv vectors
static void sym_phase2(int L, int w, int nv, const double* x0, double* y0, KState* s0,
                       double* p0, int m0, const double* x1, double* y1, KState* s1, double* p1,
                       int m1, cudaStream_t s) {
  const int gf = grid_for((long long)L * L * 3, 256, kRedBlocks);
  if (nv == 2)
    k_symb_fix<2><<<gf, 256, 0, s>>>(L, w, x0, y0, s0, p0, m0, x1, y1, s1, p1, m1);
  else
    k_symb_fix<1><<<gf, 256, 0, s>>>(L, w, x0, y0, s0, p0, m0, nullptr, nullptr, nullptr,
                                     nullptr, 2);
}
// one complete symmetric-band application y_v = (S B S) x_v (phase 1 + 2)
static int sym_apply(int L, int w, const double* U, int nv, const double* x0, double* y0,
                     KState* s0, double* p0, int m0, const double* x1, double* y1, KState* s1,
                     double* p1, int m1, cudaStream_t s) {
  sym_phase1(L, w, U, nv, x0, y0, s0, p0, 0, x1, y1, s1, p1, 0, s);
  sym_phase2(L, w, nv, x0, y0, s0, p0, m0, x1, y1, s1, p1, m1, s);
  return (int)cudaGetLastError();
}
int gbk_tcg_iterations(int L, int nr, int w, const double* BsT, double* x, double* r,
                       double* p, double* Ap, int iters, void* st, double* part,
                       cudaStream_t s, int layout) {
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * nr;
  const int gs = row_grid((long long)L * L * nr);
  const int gv = grid_for(npad, 256, kRedBlocks);
  const size_t sm = off_smem(nr, w);
  KState* k = (KState*)st;
  const bool tl = use_tiled(L, nr, w);
  const bool sy = use_sym(layout, L, nr, w);
  for (int i = 0; i < iters; ++i) {
    if (sy) sym_apply(L, w, BsT, 1, p, Ap, k, part, 0, nullptr, nullptr, nullptr, nullptr, 2, s);
    else if (tl) k_tcg_spmv_tiled<<<tiled_grid(L), 192, tiled_smem(w), s>>>(L, w, BsT, p, Ap, k, part);
    else if (nr == 3) k_tcg_spmv<3><<<gs, 256, sm, s>>>(L, w, BsT, p, Ap, k, part);
    else k_tcg_spmv<1><<<gs, 256, sm, s>>>(L, w, BsT, p, Ap, k, part);
    k_cg_update<<<gv, 256, 0, s>>>(npad, x, r, p, Ap, k, part);
    k_cg_dir<<<gv, 256, 0, s>>>(npad, r, p, k);
  }
  return (int)cudaGetLastError();
}
int gbk_tpow_iterations(int L, int nr, int w, const double* BsT, double* x, double* y,
                        double tol, int iters, void* st, double* part, cudaStream_t s,
                        int layout) {
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * nr;
  const int gs = row_grid((long long)L * L * nr);
  const int gv = grid_for(npad, 256, kRedBlocks);
  const size_t sm = off_smem(nr, w);
  KState* k = (KState*)st;
  const bool tl = use_tiled(L, nr, w);
  const bool sy = use_sym(layout, L, nr, w);
  for (int i = 0; i < iters; ++i) {
    if (sy) sym_apply(L, w, BsT, 1, x, y, k, part, 1, nullptr, nullptr, nullptr, nullptr, 2, s);
    else if (tl) k_tpow_apply_tiled<<<tiled_grid(L), 192, tiled_smem(w), s>>>(L, w, BsT, x, y, k, part);
    else if (nr == 3) k_tpow_apply<3><<<gs, 256, sm, s>>>(L, w, BsT, x, y, k, part);
    else k_tpow_apply<1><<<gs, 256, sm, s>>>(L, w, BsT, x, y, k, part);
    k_pow_step<<<gv, 256, 0, s>>>(npad, x, y, tol, k, part);
    k_pow_scale<<<gv, 256, 0, s>>>(npad, x, y, k);
  }
  return (int)cudaGetLastError();
}
int gbk_tbox_apply(int L, int nr, int w, const double* BsT, const double* x, double* y,
                   cudaStream_t s, int layout) {
  const int gs = row_grid((long long)L * L * nr);
  const size_t sm = off_smem(nr, w);
  if (use_sym(layout, L, nr, w))
    sym_apply(L, w, BsT, 1, x, y, nullptr, nullptr, 2, nullptr, nullptr, nullptr, nullptr, 2, s);
  else if (use_tiled(L, nr, w)) k_tbox_apply_tiled<<<tiled_grid(L), 192, tiled_smem(w), s>>>(L, w, BsT, x, y);
  else if (nr == 3) k_tbox_apply<3><<<gs, 256, sm, s>>>(L, w, BsT, x, y);
  else k_tbox_apply<1><<<gs, 256, sm, s>>>(L, w, BsT, x, y);
  return (int)cudaGetLastError();
}


// ---- block-Jacobi PCG launchers ----
int gbk_bj_setup(int L, int w, const double* B, const double* sv, float* inv,
                 cudaStream_t s) {
  return gbk_bj_setup_rows(L, w, B, sv, inv, 0, L, s);
}
// the 2x2-parent blocks of grid rows [r0, r1) (both even)
int gbk_bj_setup_rows(int L, int w, const double* B, const double* sv, float* inv, int r0,
                      int r1, cudaStream_t s) {
  if (r0 < 0 || r1 > L || r0 > r1 || (r0 & 1) || (r1 & 1)) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const int Lb = L / 2, b0 = (r0 / 2) * Lb, b1 = (r1 / 2) * Lb;
  k_bj_setup<<<grid_for(b1 - b0, 8, 148 * 16), 256, 0, s>>>(L, w, B, sv, inv, b0, b1);
  return (int)cudaGetLastError();
}
static inline int bj_grid(int L) {
  const int nb = (L / 2) * (L / 2);
  return grid_for(nb, 16, kRedBlocks);
}
static inline int bj_init_grid(int L) {
  const int nb = (L / 2) * (L / 2);
  return grid_for(nb, 16, (2 * kRedBlocks) / 3);
}
int gbk_bjcg_init(int L, int w, const double* b, const double* x0, const double* Ax0,
                  double x0_scale, double* x, double* r, double* p, double* z, const float* inv,
                  double rel_tol, int max_iter, void* st, double* part, cudaStream_t s) {
  k_bjcg_init<<<bj_init_grid(L), 192, 0, s>>>(L, w, b, x0, Ax0, x0_scale, x, r, p, z, inv,
                                              rel_tol, max_iter, (KState*)st, part);
  if (x0) {
    const long long npad = (long long)(L + 2 * w) * (L + 2 * w) * 3;
    k_cg_zero_if<<<grid_for(npad, 256, kRedBlocks), 256, 0, s>>>(npad, x, (KState*)st);
  }
  return (int)cudaGetLastError();
}
int gbk_bjcg_iterations(int L, int w, const double* BsT, const float* inv, double* x,
                        double* r, double* p, double* Ap, double* z, int iters, void* st,
                        double* part, cudaStream_t s, int layout) {
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const int gs = row_grid((long long)L * L * 3);
  const int gv = grid_for(npad, 256, kRedBlocks);
  const size_t sm = off_smem(3, w);
  KState* k = (KState*)st;
  const bool sy = use_sym(layout, L, 3, w);
  for (int i = 0; i < iters; ++i) {
    if (sy) {  // alpha from phase 1, spill-over added by the fused update
      sym_phase1(L, w, BsT, 1, p, Ap, k, part, 1, nullptr, nullptr, nullptr, nullptr, 0, s);
      k_symb_bjcg_update<<<bj_grid(L), 192, 0, s>>>(L, w, x, r, p, Ap, z, inv, k, part);
    } else {
      if (use_tiled(L, 3, w))
        k_tcg_spmv_tiled<<<tiled_grid(L), 192, tiled_smem(w), s>>>(L, w, BsT, p, Ap, k, part);
      else
        k_tcg_spmv<3><<<gs, 256, sm, s>>>(L, w, BsT, p, Ap, k, part);
      k_bjcg_update<<<bj_grid(L), 192, 0, s>>>(L, w, x, r, p, Ap, z, inv, k, part);
    }
    k_cg_dir<<<gv, 256, 0, s>>>(npad, z, p, k);
  }
  return (int)cudaGetLastError();
}

int gbk_dot2(long long n, const double* a, const double* b, const double* c,
             double* out, void* st, double* part, cudaStream_t s) {
  k_dot2<<<grid_for(n, 256, kRedBlocks), 256, 0, s>>>(n, a, b, c, out, (KState*)st, part);
  return (int)cudaGetLastError();
}

int gbk_scale_by_norm(long long n, const double* a, const double* norm2, int which,
                      double* y, double* y2, cudaStream_t s) {
  k_scale_by_norm<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, a, norm2, which, y, y2);
  return (int)cudaGetLastError();
}

int gbk_box_apply(int L, int nr, int w, const double* B, const double* sv, int mode,
                  const double* x, double* y, cudaStream_t s) {
  const long long n = (long long)L * L * nr;
  k_box_apply<<<grid_for(n * 32, 256, 148 * 16), 256, 0, s>>>(L, nr, w, B, sv, mode, x, y);
  return (int)cudaGetLastError();
}

int gbk_apply_w(int Lp, const double* w12, const double* g, const double* sv, double* out,
                cudaStream_t s) {
  return gbk_apply_w_rows(Lp, w12, g, sv, out, 0, Lp, s);
}
int gbk_apply_w_rows(int Lp, const double* w12, const double* g, const double* sv, double* out,
                     int r0, int r1, cudaStream_t s) {
  if (r0 < 0 || r1 > Lp || r0 > r1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  k_apply_w<<<grid_for((long long)(r1 - r0) * Lp, 256, 148 * 16), 256, 0, s>>>(
      Lp, mkW(w12), g, sv, out, (long long)r0 * Lp, (long long)r1 * Lp);
  return (int)cudaGetLastError();
}

int gbk_apply_wt(int Lp, const double* w12, const double* w, double* v, cudaStream_t s) {
  return gbk_apply_wt_rows(Lp, w12, w, v, 0, Lp, s);
}
int gbk_apply_wt_rows(int Lp, const double* w12, const double* w, double* v, int r0, int r1,
                      cudaStream_t s) {
  if (r0 < 0 || r1 > Lp || r0 > r1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  k_apply_wt<<<grid_for((long long)(r1 - r0) * Lp, 256, 148 * 16), 256, 0, s>>>(
      Lp, mkW(w12), w, v, (long long)r0 * Lp, (long long)r1 * Lp);
  return (int)cudaGetLastError();
}

int gbk_apply_r(int Lp, int rho, const double* R, const double* g, double* out,
                cudaStream_t s) {
  return gbk_apply_r_rows(Lp, rho, R, g, out, 0, Lp, s);
}
int gbk_apply_r_rows(int Lp, int rho, const double* R, const double* g, double* out, int r0,
                     int r1, cudaStream_t s) {
  if (r0 < 0 || r1 > Lp || r0 > r1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  k_apply_r<<<grid_for((long long)(r1 - r0) * Lp, 128, 148 * 16), 128, 0, s>>>(
      Lp, rho, R, g, out, (long long)r0 * Lp, (long long)r1 * Lp);
  return (int)cudaGetLastError();
}

int gbk_psi_t_apply(int n, int L, int lo, int wd, const double* psi, const double* v,
                    double* inc, cudaStream_t s) {
  return gbk_psi_t_apply_rows(n, L, lo, wd, psi, v, inc, 0, n, 0, L, s);
}
// fine rows [F0, F1) of inc from the psi rows in grid rows [j_lo, j_hi) only
// (a rank's partial increment; the whole level is (0, n, 0, L))
int gbk_psi_t_apply_rows(int n, int L, int lo, int wd, const double* psi, const double* v,
                         double* inc, int F0, int F1, int j_lo, int j_hi, cudaStream_t s) {
  if (F0 < 0 || F1 > n || F0 > F1 || j_lo < 0 || j_hi > L || j_lo > j_hi) return GB_UNSUPPORTED;
  if (F0 == F1) return 0;
  k_psi_t_apply<<<grid_for((long long)(F1 - F0) * n, 128, 148 * 32), 128, 0, s>>>(
      n, L, lo, wd, psi, v, inc, F0, F1, j_lo, j_hi);
  return (int)cudaGetLastError();
}

int gbk_psi_apply(int n, int L, int lo, int wd, const double* psi, const double* b,
                  double* out, cudaStream_t s) {
  const long long rows = (long long)L * L;
  k_psi_apply<<<grid_for(rows * 32, 256, 148 * 16), 256, 0, s>>>(n, L, lo, wd, psi, b, out);
  return (int)cudaGetLastError();
}

int gbk_axpby(long long n, double a, const double* x, double b, const double* y,
              double* out, cudaStream_t s) {
  k_axpby<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, a, x, b, y, out);
  return (int)cudaGetLastError();
}

int gbk_vmul(long long n, const double* a, const double* b, double* out, cudaStream_t s) {
  k_vmul<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, a, b, out);
  return (int)cudaGetLastError();
}

int gbk_vadd(long long n, const double* a, const double* b, double* out, cudaStream_t s) {
  k_vadd<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, a, b, out);
  return (int)cudaGetLastError();
}


// ---------------------------------------------------------------------------
// General CSR operator (sparse_core.cg_solve / eig_extremes on any SPD CSR):
// one warp per row, the row's stored entries in column order; mode 0 = CG
// (p.Ap -> alpha), 1 = power (x.y, y.y -> lam, ynorm), 2 = plain y = A x.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_csr_apply(long long n, const int32_t* __restrict__ indptr,
                                                   const int32_t* __restrict__ indices,
                                                   const double* __restrict__ data,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y, KState* st,
                                                   double* part, int mode) {
  __shared__ double sh[32];
  if (mode != 2 && st->done) return;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  double xy = 0.0, yy = 0.0;
  for (long long r = wid; r < n; r += nwarps) {
    double acc = 0.0;
    for (int e = indptr[r] + lane; e < indptr[r + 1]; e += 32) acc += data[e] * x[indices[e]];
    acc = warp_sum(acc);
    if (lane == 0) {
      y[r] = acc;
      xy += x[r] * acc;
      yy += acc * acc;
    }
  }
  if (mode == 2) return;
  xy = block_sum(xy, sh);
  yy = block_sum(yy, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = xy;
    part[2 * blockIdx.x + 1] = yy;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      if (mode == 0) {
        st->pAp = a;
        if (!(a > 0.0)) {
          st->breakdown = st->it + 1;
          st->done = 1;
        } else {
          st->alpha = st->rs / a;
        }
      } else {
        st->lam = a;
        st->ynorm = sqrt(b);
        if (st->ynorm == 0.0) {
          st->lam = 0.0;
          st->done = 1;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Host-side drivers: the whole iteration loop in C (one ctypes call, GIL
// released): launch a chunk of iterations, copy the state to pinned host
// memory, synchronize the stream, stop when the device says done.
// ---------------------------------------------------------------------------
static int read_state(const void* st, KState* host, cudaStream_t s) {
  cudaError_t e = cudaMemcpyAsync(host, st, sizeof(KState), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaStreamSynchronize(s);
}

int gbk_sync_read(const void* dev, void* host, size_t bytes, cudaStream_t s) {
  cudaError_t e = cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaStreamSynchronize(s);
}

int gbk_tcg_solve(int L, int nr, int w, const double* BsT, double* x, double* r, double* p,
                  double* Ap, void* st, double* part, void* host_state, int max_chunk,
                  cudaStream_t s, long long* launches, int layout) {
  KState* h = (KState*)host_state;
  int chunk = 8;
  for (;;) {
    int e = gbk_tcg_iterations(L, nr, w, BsT, x, r, p, Ap, chunk, st, part, s, layout);
    *launches += (use_sym(layout, L, nr, w) ? 4LL : 3LL) * chunk;
    if (e) return e;
    e = read_state(st, h, s);
    if (e) return e;
    if (h->done) return 0;
    chunk = chunk * 2 < max_chunk ? chunk * 2 : max_chunk;
  }
}

int gbk_bjcg_solve(int L, int w, const double* BsT, const float* inv, double* x, double* r,
                   double* p, double* Ap, double* z, void* st, double* part, void* host_state,
                   int max_chunk, cudaStream_t s, long long* launches, int layout) {
  KState* h = (KState*)host_state;
  int chunk = 8;
  for (;;) {
    int e = gbk_bjcg_iterations(L, w, BsT, inv, x, r, p, Ap, z, chunk, st, part, s, layout);
    *launches += 3LL * chunk;
    if (e) return e;
    e = read_state(st, h, s);
    if (e) return e;
    if (h->done) return 0;
    chunk = chunk * 2 < max_chunk ? chunk * 2 : max_chunk;
  }
}

// Two independent block-Jacobi PCG solves on the same operator in lockstep
// (batched repeat solves): one dual-vector phase-1 pass streams S B S once for
// both search directions, then each vector's fused update and direction.
// Every kernel computes a vector exactly as the single-vector solve does
// (same per-vector summation order, same persistent grid), so each result is
// bitwise the single solve's; a converged vector's kernels are no-ops
// (KState.done) while the other one runs on.  Symmetric band layout only.
int gbk_bjcg_solve2(int L, int w, const double* BsT, const float* inv, double* const* x,
                    double* const* r, double* const* p, double* const* Ap, double* const* z,
                    void* const* st, double* const* part, void* const* host_state,
                    int max_chunk, cudaStream_t s, long long* launches) {
  // bitwise equality with the single solve needs the same phase-1 kernel
  // family for one and two vectors (the warp-specialized one; the dot
  // partials of the register-pipelined fallback are formed in another order)
  if (!use_sym(1, L, 3, w) || !GB_SYM_WS || !g_sym_ws_on ||
      symb_ws_smem(w, 1, 2) > 226 * 1024 || symb_ws_smem(w, 2, 2) > 226 * 1024)
    return GB_UNSUPPORTED;
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const int gv = grid_for(npad, 256, kRedBlocks);
  KState* k0 = (KState*)st[0];
  KState* k1 = (KState*)st[1];
  KState* h0 = (KState*)host_state[0];
  KState* h1 = (KState*)host_state[1];
  int chunk = 8;
  for (;;) {
    for (int i = 0; i < chunk; ++i) {
      sym_phase1(L, w, BsT, 2, p[0], Ap[0], k0, part[0], 1, p[1], Ap[1], k1, part[1], 1, s);
      k_symb_bjcg_update<<<bj_grid(L), 192, 0, s>>>(L, w, x[0], r[0], p[0], Ap[0], z[0], inv,
                                                     k0, part[0]);
      k_cg_dir<<<gv, 256, 0, s>>>(npad, z[0], p[0], k0);
      k_symb_bjcg_update<<<bj_grid(L), 192, 0, s>>>(L, w, x[1], r[1], p[1], Ap[1], z[1], inv,
                                                     k1, part[1]);
      k_cg_dir<<<gv, 256, 0, s>>>(npad, z[1], p[1], k1);
    }
    *launches += 5LL * chunk;
    int e = (int)cudaGetLastError();
    if (e) return e;
    if ((e = read_state(st[0], h0, s))) return e;
    if ((e = read_state(st[1], h1, s))) return e;
    if (h0->done && h1->done) return 0;
    chunk = chunk * 2 < max_chunk ? chunk * 2 : max_chunk;
  }
}

int gbk_tpow_solve(int L, int nr, int w, const double* BsT, double* x, double* y, double tol,
                   void* st, double* part, void* host_state, int max_chunk, cudaStream_t s,
                   long long* launches, int layout) {
  KState* h = (KState*)host_state;
  int chunk = 8;
  for (;;) {
    int e = gbk_tpow_iterations(L, nr, w, BsT, x, y, tol, chunk, st, part, s, layout);
    *launches += (use_sym(layout, L, nr, w) ? 4LL : 3LL) * chunk;
    if (e) return e;
    e = read_state(st, h, s);
    if (e) return e;
    if (h->done) return 0;
    chunk = chunk * 2 < max_chunk ? chunk * 2 : max_chunk;
  }
}

size_t gbk_boxsym_elems(int L, int w) { return (size_t)L * L * symb_ns(w); }
size_t gbk_sym_overflow_elems(int L, int w) {
  return L % kSymTW == 0 && L % kSymTH == 0 ? (size_t)symb_ntile(L) * symb_region(w) : 0;
}
int gbk_sym_supported(int L, int nr, int w) { return use_sym(1, L, nr, w) ? 1 : 0; }
int gbk_scale_box_symT(int L, int w, const double* B, const double* sv, double* UsT,
                       cudaStream_t s) {
  return gbk_scale_box_symT_rows(L, w, B, sv, UsT, 0, L, s);
}
// grid rows [r0, r1) of the symmetric band copy (rows are whole 32-parent
// blocks: L % 64 == 0); reads s within w rows below the strip
int gbk_scale_box_symT_rows(int L, int w, const double* B, const double* sv, double* UsT,
                            int r0, int r1, cudaStream_t s) {
  if (r0 < 0 || r1 > L || r0 > r1 || L % 32) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long per = (long long)L * symb_ns(w);
  k_scale_box_symb<<<grid_for((r1 - r0) * per, 256, 148 * 16), 256, 0, s>>>(
      L, w, B, sv, UsT, r0 * per, r1 * per);
  return (int)cudaGetLastError();
}

static inline int csr_grid(long long n) { return grid_for(n * 32, 256, kRedBlocks); }

int gbk_csr_apply(long long n, const int32_t* indptr, const int32_t* indices,
                  const double* data, const double* x, double* y, cudaStream_t s) {
  k_csr_apply<<<csr_grid(n), 256, 0, s>>>(n, indptr, indices, data, x, y, nullptr, nullptr, 2);
  return (int)cudaGetLastError();
}

int gbk_csr_cg_solve(long long n, const int32_t* indptr, const int32_t* indices,
                     const double* data, double* x, double* r, double* p, double* Ap,
                     void* st, double* part, void* host_state, int max_chunk, cudaStream_t s,
                     long long* launches) {
  KState* h = (KState*)host_state;
  KState* k = (KState*)st;
  const int gv = grid_for(n, 256, kRedBlocks);
  int chunk = 8;
  for (;;) {
    for (int i = 0; i < chunk; ++i) {
      k_csr_apply<<<csr_grid(n), 256, 0, s>>>(n, indptr, indices, data, p, Ap, k, part, 0);
      k_cg_update<<<gv, 256, 0, s>>>(n, x, r, p, Ap, k, part);
      k_cg_dir<<<gv, 256, 0, s>>>(n, r, p, k);
    }
    *launches += 3LL * chunk;
    int e = (int)cudaGetLastError();
    if (e) return e;
    e = read_state(st, h, s);
    if (e) return e;
    if (h->done) return 0;
    chunk = chunk * 2 < max_chunk ? chunk * 2 : max_chunk;
  }
}

int gbk_csr_pow_solve(long long n, const int32_t* indptr, const int32_t* indices,
                      const double* data, double* x, double* y, double tol, void* st,
                      double* part, void* host_state, int max_chunk, cudaStream_t s,
                      long long* launches) {
  KState* h = (KState*)host_state;
  KState* k = (KState*)st;
  const int gv = grid_for(n, 256, kRedBlocks);
  int chunk = 8;
  for (;;) {
    for (int i = 0; i < chunk; ++i) {
      k_csr_apply<<<csr_grid(n), 256, 0, s>>>(n, indptr, indices, data, x, y, k, part, 1);
      k_pow_step<<<gv, 256, 0, s>>>(n, x, y, tol, k, part);
      k_pow_scale<<<gv, 256, 0, s>>>(n, x, y, k);
    }
    *launches += 3LL * chunk;
    int e = (int)cudaGetLastError();
    if (e) return e;
    e = read_state(st, h, s);
    if (e) return e;
    if (h->done) return 0;
    chunk = chunk * 2 < max_chunk ? chunk * 2 : max_chunk;
  }
}

// ---------------------------------------------------------------------------
// 3-D box operator (config 4): y = (S B S) x with the materialized
// congruence's entry ((B_rc s_r) s_c) (gamblet_fast.py:123-139) on an L^3 grid
// with nr components, half-width w; one warp per row, reductions as
// k_csr_apply (mode 0: CG pAp/alpha, 1: power x.y, |y|, 2: none)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k3_box_apply(int L, int nr, int w,
                                                   const double* __restrict__ B,
                                                   const double* __restrict__ sv,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y, KState* st,
                                                   double* part, int mode) {
  // slot tables (shared): column offset of slot e relative to the row's
  // point, and its packed (dx, dy, dz) + w for the domain test
  extern __shared__ int k3tab[];
  __shared__ double sh[32];
  if (mode != 2 && st->done) return;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long rows = (long long)L * L * L * nr;
  const int W3 = 2 * w + 1;
  const int S = W3 * W3 * W3 * nr;
  int* toff = k3tab;
  int* tpk = k3tab + S;
  for (int e = threadIdx.x; e < S; e += blockDim.x) {
    const int c = e % nr;
    int t = e / nr;
    const int dz = t % W3;
    t /= W3;
    const int dy = t % W3, dx = t / W3;
    toff[e] = (((dx - w) * L + (dy - w)) * L + (dz - w)) * nr + c;
    tpk[e] = (dx << 16) | (dy << 8) | dz;
  }
  __syncthreads();
  double xy = 0.0, yy = 0.0;
  for (long long r = wid; r < rows; r += nwarps) {
    const long long p = r / nr;
    const int pz = (int)(p % L), py = (int)((p / L) % L), px = (int)(p / ((long long)L * L));
    // in-domain offset ranges (+ w): [lo, hi] per axis
    const int xlo = imax(w - px, 0), xhi = imin(w + L - 1 - px, 2 * w);
    const int ylo = imax(w - py, 0), yhi = imin(w + L - 1 - py, 2 * w);
    const int zlo = imax(w - pz, 0), zhi = imin(w + L - 1 - pz, 2 * w);
    const double sr = sv[r];
    const double* row = B + r * S;
    const long long base = p * nr;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int e = lane;
    // rows whose whole stencil is inside the domain (warp-uniform): the same
    // sums without the per-slot domain tests
    if (xlo == 0 && xhi == 2 * w && ylo == 0 && yhi == 2 * w && zlo == 0 && zhi == 2 * w) {
      for (; e + 96 < S; e += 128) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int eu = e + 32 * u;
          const long long col = base + toff[eu];
          v[u] = (row[eu] * sr) * sv[col] * x[col];
        }
        a0 += v[0];
        a1 += v[1];
        a2 += v[2];
        a3 += v[3];
      }
      for (; e < S; e += 32) {
        const long long col = base + toff[e];
        a0 += (row[e] * sr) * sv[col] * x[col];
      }
    }
    for (; e + 96 < S; e += 128) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int eu = e + 32 * u;
        const int pk = tpk[eu];
        const int dx = pk >> 16, dy = (pk >> 8) & 255, dz = pk & 255;
        const bool in = dx >= xlo && dx <= xhi && dy >= ylo && dy <= yhi && dz >= zlo && dz <= zhi;
        const long long col = base + toff[eu];
        v[u] = in ? (row[eu] * sr) * sv[col] * x[col] : 0.0;
      }
      a0 += v[0];
      a1 += v[1];
      a2 += v[2];
      a3 += v[3];
    }
    for (; e < S; e += 32) {
      const int pk = tpk[e];
      const int dx = pk >> 16, dy = (pk >> 8) & 255, dz = pk & 255;
      if (dx >= xlo && dx <= xhi && dy >= ylo && dy <= yhi && dz >= zlo && dz <= zhi) {
        const long long col = base + toff[e];
        a0 += (row[e] * sr) * sv[col] * x[col];
      }
    }
    double acc = (a0 + a1) + (a2 + a3);
    acc = warp_sum(acc);
    if (lane == 0) {
      y[r] = acc;
      xy += x[r] * acc;
      yy += acc * acc;
    }
  }
  if (mode == 2) return;
  xy = block_sum(xy, sh);
  yy = block_sum(yy, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = xy;
    part[2 * blockIdx.x + 1] = yy;
  }
  if (last_block(&st->counter)) {
    double a, b;
    final_sum2(part, gridDim.x, &a, &b, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      if (mode == 0) {
        st->pAp = a;
        if (!(a > 0.0)) {
          st->breakdown = st->it + 1;
          st->done = 1;
        } else {
          st->alpha = st->rs / a;
        }
      } else {
        st->lam = a;
        st->ynorm = sqrt(b);
        if (st->ynorm == 0.0) {
          st->lam = 0.0;
          st->done = 1;
        }
      }
    }
  }
}

static inline size_t box3_smem(int w, int nr) {
  const size_t b = (size_t)2 * (2 * w + 1) * (2 * w + 1) * (2 * w + 1) * nr * sizeof(int);
  static size_t attr = 48 * 1024;  // raised once to what a launch needs
  if (b > attr && b <= 200 * 1024) {
    cudaFuncSetAttribute(k3_box_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
    attr = b;
  }
  return b;
}

static inline int box3_grid(long long rows) { return grid_for(rows * 32, 256, kRedBlocks); }

int gbk3_apply(int L, int nr, int w, const double* B, const double* sv, const double* x,
               double* y, cudaStream_t s) {
  const long long rows = (long long)L * L * L * nr;
  k3_box_apply<<<box3_grid(rows), 256, box3_smem(w, nr), s>>>(L, nr, w, B, sv, x, y, nullptr,
                                                               nullptr, 2);
  return (int)cudaGetLastError();
}

int gbk3_cg_solve(int L, int nr, int w, const double* B, const double* sv, double* x, double* r,
                  double* p, double* Ap, void* st, double* part, void* host_state, int max_chunk,
                  cudaStream_t s, long long* launches) {
  KState* h = (KState*)host_state;
  KState* k = (KState*)st;
  const long long n = (long long)L * L * L * nr;
  const int gv = grid_for(n, 256, kRedBlocks);
  int chunk = 8;
  for (;;) {
    for (int i = 0; i < chunk; ++i) {
      k3_box_apply<<<box3_grid(n), 256, box3_smem(w, nr), s>>>(L, nr, w, B, sv, p, Ap, k, part,
                                                               0);
      k_cg_update<<<gv, 256, 0, s>>>(n, x, r, p, Ap, k, part);
      k_cg_dir<<<gv, 256, 0, s>>>(n, r, p, k);
    }
    *launches += 3LL * chunk;
    int e = (int)cudaGetLastError();
    if (e) return e;
    e = read_state(st, h, s);
    if (e) return e;
    if (h->done) return 0;
    chunk = chunk * 2 < max_chunk ? chunk * 2 : max_chunk;
  }
}

int gbk3_pow_solve(int L, int nr, int w, const double* B, const double* sv, double* x,
                   double* y, double tol, void* st, double* part, void* host_state,
                   int max_chunk, cudaStream_t s, long long* launches) {
  KState* h = (KState*)host_state;
  KState* k = (KState*)st;
  const long long n = (long long)L * L * L * nr;
  const int gv = grid_for(n, 256, kRedBlocks);
  int chunk = 8;
  for (;;) {
    for (int i = 0; i < chunk; ++i) {
      k3_box_apply<<<box3_grid(n), 256, box3_smem(w, nr), s>>>(L, nr, w, B, sv, x, y, k, part,
                                                               1);
      k_pow_step<<<gv, 256, 0, s>>>(n, x, y, tol, k, part);
      k_pow_scale<<<gv, 256, 0, s>>>(n, x, y, k);
    }
    *launches += 3LL * chunk;
    int e = (int)cudaGetLastError();
    if (e) return e;
    e = read_state(st, h, s);
    if (e) return e;
    if (h->done) return 0;
    chunk = chunk * 2 < max_chunk ? chunk * 2 : max_chunk;
  }
}

// ---------------------------------------------------------------------------
// Level engine: the lambda estimates of S B S (sparse_core.eig_extremes,
// power iteration then inverse iteration with warm-started inner CG) paired
// with the subband PCG of the same level, every operator pass shared by both
// through k_dual_apply.  Host control flow mirrors sparse_core.py:232-278.
// ---------------------------------------------------------------------------
#include "gb_engine.h"
#include "gb_lanczos.h"
#ifndef GB_LZ_CHECK
#define GB_LZ_CHECK 32
#endif

// ---- engine building blocks (count their launches into *nl) ----
// dual pass: A (subband PCG, mode 0) and B (mode mb) on one sweep of S B S;
// b_fused: B is a block-Jacobi PCG step whose update adds the spill-over
static int launch_dual(const gb_level_engine_args* ec, double* xb, double* yb, int mb,
                       int b_fused, cudaStream_t s, long long* nl) {
  gb_level_engine_args* e = const_cast<gb_level_engine_args*>(ec);
  e->n_dual += 1;
  if (e->layout == 1) {
    cudaEvent_t* ev = (cudaEvent_t*)e->ev_events;
    const bool timed = ev && e->ev_n < e->ev_cap;
    if (timed) cudaEventRecord(ev[2 * e->ev_n], s);
    sym_phase1(e->L, e->w, e->BsT, 2, e->pa, e->apa, (KState*)e->sta, e->parta, 1, xb, yb,
               (KState*)e->stb, e->partb, b_fused, s);
    if (timed) cudaEventRecord(ev[2 * e->ev_n++ + 1], s);
    *nl += 1;
    if (!b_fused) {
      sym_phase2(e->L, e->w, 1, xb, yb, (KState*)e->stb, e->partb, mb, nullptr, nullptr,
                 nullptr, nullptr, 2, s);
      *nl += 1;
    }
    return (int)cudaGetLastError();
  }
  if (!use_tiled(e->L, 3, e->w)) {
    // levels below the tile width (L < 64): the row-per-thread kernels, one
    // launch per half
    const int gs = row_grid((long long)e->L * e->L * 3);
    const size_t sm = off_smem(3, e->w);
    k_tcg_spmv<3><<<gs, 256, sm, s>>>(e->L, e->w, e->BsT, e->pa, e->apa, (KState*)e->sta,
                                      e->parta);
    if (mb == 0)
      k_tcg_spmv<3><<<gs, 256, sm, s>>>(e->L, e->w, e->BsT, xb, yb, (KState*)e->stb, e->partb);
    else
      k_tpow_apply<3><<<gs, 256, sm, s>>>(e->L, e->w, e->BsT, xb, yb, (KState*)e->stb,
                                          e->partb);
    *nl += 2;
    return (int)cudaGetLastError();
  }
  const int W2 = 2 * e->w + 1;
  const size_t smem = ((size_t)(W2 * W2 * 3 + 2) / 2 + 1) * sizeof(double) +
                      2 * (size_t)W2 * (kTileP + 2 * e->w) * 3 * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_dual_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  k_dual_apply<<<tiled_grid(e->L), 192, smem, s>>>(
      e->L, e->w, e->BsT, e->pa, e->apa, (KState*)e->sta, e->parta, 0, xb, yb,
      (KState*)e->stb, e->partb, mb);
  *nl += 1;
  return (int)cudaGetLastError();
}

// one live Krylov half; fused: a block-Jacobi PCG step (see launch_dual)
static int launch_single(const gb_level_engine_args* e, const double* x, double* y, void* st,
                         double* part, int mode, int fused, cudaStream_t s, long long* nl) {
  const_cast<gb_level_engine_args*>(e)->n_single += 1;
  if (e->layout == 1) {
    sym_phase1(e->L, e->w, e->BsT, 1, x, y, (KState*)st, part, fused, nullptr, nullptr,
               nullptr, nullptr, 0, s);
    *nl += 1;
    if (!fused) {
      sym_phase2(e->L, e->w, 1, x, y, (KState*)st, part, mode, nullptr, nullptr, nullptr,
                 nullptr, 2, s);
      *nl += 1;
    }
    return (int)cudaGetLastError();
  }
  if (!use_tiled(e->L, 3, e->w)) {
    const int gs = row_grid((long long)e->L * e->L * 3);
    const size_t sm = off_smem(3, e->w);
    if (mode == 0)
      k_tcg_spmv<3><<<gs, 256, sm, s>>>(e->L, e->w, e->BsT, x, y, (KState*)st, part);
    else
      k_tpow_apply<3><<<gs, 256, sm, s>>>(e->L, e->w, e->BsT, x, y, (KState*)st, part);
    *nl += 1;
    return (int)cudaGetLastError();
  }
  if (mode == 0)
    k_tcg_spmv_tiled<<<tiled_grid(e->L), 192, tiled_smem(e->w), s>>>(e->L, e->w, e->BsT, x, y,
                                                                      (KState*)st, part);
  else
    k_tpow_apply_tiled<<<tiled_grid(e->L), 192, tiled_smem(e->w), s>>>(e->L, e->w, e->BsT, x,
                                                                        y, (KState*)st, part);
  *nl += 1;
  return (int)cudaGetLastError();
}

static int launch_plain(const gb_level_engine_args* e, const double* x, double* y,
                        cudaStream_t s, long long* nl) {
  if (e->layout == 1) {
    *nl += 2;
    return sym_apply(e->L, e->w, e->BsT, 1, x, y, nullptr, nullptr, 2, nullptr, nullptr, nullptr,
                     nullptr, 2, s);
  }
  if (!use_tiled(e->L, 3, e->w))
    k_tbox_apply<3><<<row_grid((long long)e->L * e->L * 3), 256, off_smem(3, e->w), s>>>(
        e->L, e->w, e->BsT, x, y);
  else
    k_tbox_apply_tiled<<<tiled_grid(e->L), 192, tiled_smem(e->w), s>>>(e->L, e->w, e->BsT, x, y);
  *nl += 1;
  return (int)cudaGetLastError();
}

// block-Jacobi PCG update + direction of one half
static void pcg_post(const gb_level_engine_args* e, double* x, double* r, double* p, double* Ap,
                     double* z, KState* k, double* part, cudaStream_t s, long long* nl) {
  const int Lpad = e->L + 2 * e->w;
  const long long npad = (long long)Lpad * Lpad * 3;
  if (e->layout == 1)
    k_symb_bjcg_update<<<bj_grid(e->L), 192, 0, s>>>(e->L, e->w, x, r, p, Ap, z, e->inv, k, part);
  else
    k_bjcg_update<<<bj_grid(e->L), 192, 0, s>>>(e->L, e->w, x, r, p, Ap, z, e->inv, k, part);
  k_cg_dir<<<grid_for(npad, 256, kRedBlocks), 256, 0, s>>>(npad, z, p, k);
  *nl += 2;
}

static void post_a(const gb_level_engine_args* e, cudaStream_t s, long long* nl) {
  pcg_post(e, e->xa, e->ra, e->pa, e->apa, e->za, (KState*)e->sta, e->parta, s, nl);
}

// lambda_min of the 3-D operator by the Lanczos moments of the unit start
// vector x (gb_lanczos.h; the 2-D engine's spectral mode 1): Lanczos steps
// on k3_box_apply (power-mode reduction) + k_lz_step, the reference's
// inverse-iteration sequence evaluated on the host every 32-64 steps, stop
// when the estimate and its stopping index are stable to lz_tol.  x, vp, w:
// n-vectors (x is overwritten); ab / hab: 2 cap doubles (device / pinned).
int gbk3_lanczos_min(int L, int nr, int w, const double* B, const double* sv, double* x,
                     double* vp, double* wv, void* st, double* part, void* host_state,
                     double* ab, double* hab, int cap, double tol, int max_outer,
                     double lz_tol, double* lam_out, int* outer_out, int* its_out,
                     cudaStream_t s, long long* launches) {
  const long long n = (long long)L * L * L * nr;
  const int gv = grid_for(n, 256, kRedBlocks);
  KState* k = (KState*)st;
  KState* h = (KState*)host_state;
  cudaError_t ce = cudaMemsetAsync(vp, 0, sizeof(double) * n, s);
  if (ce != cudaSuccess) return (int)ce;
  k_state_reset<<<1, 1, 0, s>>>(k, cap);
  k_lz_init<<<1, 1, 0, s>>>(k);
  *launches += 2;
  double* v = x;
  double* wn = wv;
  int chunk = 64;
  *its_out = 0;
  for (;;) {
    for (int i = 0; i < chunk; ++i) {
      k3_box_apply<<<box3_grid(n), 256, box3_smem(w, nr), s>>>(L, nr, w, B, sv, v, wn, k, part,
                                                               1);
      k_lz_step<<<gv, 256, 0, s>>>(n, v, vp, wn, k, part, ab);
      double* t = v;
      v = wn;
      wn = t;
    }
    *launches += 2LL * chunk;
    int err = (int)cudaGetLastError();
    if (err) return err;
    if ((err = read_state(st, h, s))) return err;
    const int m = h->it;
    if (m > 0) {
      if ((err = gbk_sync_read(ab, hab, sizeof(double) * 2 * (size_t)m, s))) return err;
      double lam;
      int outer, stable;
      const int rc = gb_lz::lanczos_check(hab, m, tol, max_outer, lz_tol, &lam, &outer, &stable);
      if (rc) return GB_UNSUPPORTED - rc;  // -2 / -3: non-SPD or a failed evaluation
      *lam_out = lam;
      *outer_out = outer;
      *its_out = m;
      if (h->done || stable) return 0;
    } else if (h->done) {
      return GB_UNSUPPORTED - 9;  // A v_1 = 0
    }
    chunk = 32;
  }
}

static int level_engine(gb_level_engine_args* e, cudaStream_t s, long long& nl);
static int lanczos_min(gb_level_engine_args* e, cudaStream_t s, long long& nl);
static int inverse_iteration(gb_level_engine_args* e, cudaStream_t s, long long& nl);
int gbk_level_engine(gb_level_engine_args* e, cudaStream_t s, long long* launches) {
  long long nl = 0;
  e->n_dual = e->n_single = 0;
  e->ev_n = 0;
  // timing events come from a per-thread pool that only grows (an engine
  // runs on one worker thread): no event is created or destroyed in a
  // steady-state step
  static thread_local std::vector<cudaEvent_t> ev;
  const bool timing = e->ev_cap > 0 && e->ev_ms;
  if (timing) {
    const size_t need = 2 * (size_t)e->ev_cap;
    while (ev.size() < need) {
      cudaEvent_t x;
      if (cudaEventCreate(&x) != cudaSuccess) break;
      ev.push_back(x);
    }
    if (ev.size() < need) e->ev_cap = (int)(ev.size() / 2);
    e->ev_events = ev.data();
  } else {
    e->ev_events = nullptr;
  }
  int rc = level_engine(e, s, nl);
  if (timing) {
    const cudaError_t se = e->ev_n > 0 ? cudaEventSynchronize(ev[2 * e->ev_n - 1]) : cudaSuccess;
    for (int i = 0; i < e->ev_n && se == cudaSuccess; ++i)
      cudaEventElapsedTime(&e->ev_ms[i], ev[2 * i], ev[2 * i + 1]);
    e->ev_events = nullptr;
    if (!rc && se != cudaSuccess) rc = (int)se;
  }
  *launches += nl;
  return rc;
}
static int level_engine(gb_level_engine_args* e, cudaStream_t s, long long& nl) {
  const int Lpad = e->L + 2 * e->w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const int gv = grid_for(npad, 256, kRedBlocks);
  KState* ka = (KState*)e->sta;
  KState* kb = (KState*)e->stb;
  KState* ha = (KState*)e->hsta;
  KState* hb = (KState*)e->hstb;
  int err;
  int chunk = 8;
  // --- power iteration (B) paired with the PCG (A) -----------------------
  for (;;) {
    const bool a_live = !ha->done;
    for (int i = 0; i < chunk; ++i) {
      if (a_live) {
        if ((err = launch_dual(e, e->xb, e->yb, 1, 0, s, &nl))) return err;
        post_a(e, s, &nl);
      } else if ((err = launch_single(e, e->xb, e->yb, e->stb, e->partb, 1, 0, s, &nl))) {
        return err;
      }
      k_pow_step<<<gv, 256, 0, s>>>(npad, e->xb, e->yb, e->tol, kb, e->partb);
      k_pow_scale<<<gv, 256, 0, s>>>(npad, e->xb, e->yb, kb);
      nl += 2;
    }
    if ((err = (int)cudaGetLastError())) return err;
    if ((err = read_state(e->sta, ha, s))) return err;
    if ((err = read_state(e->stb, hb, s))) return err;
    if (hb->done) break;
    chunk = chunk * 2 < e->max_chunk ? chunk * 2 : e->max_chunk;
  }
  e->lam_max = hb->lam;
  e->power_its = hb->it;
  e->calls = hb->it + (hb->ynorm != 0.0 ? 0 : 1);
  if (e->spectral_mode == 1) {
    if ((err = lanczos_min(e, s, nl))) return err;
  } else if ((err = inverse_iteration(e, s, nl))) {
    return err;
  }
  if (e->breakdown) return 0;
  // --- the PCG alone until it converges ---------------------------------
  chunk = 8;
  while (!ha->done) {
    for (int i = 0; i < chunk; ++i) {
      if ((err = launch_single(e, e->pa, e->apa, e->sta, e->parta, 0, 1, s, &nl))) return err;
      post_a(e, s, &nl);
    }
    if ((err = (int)cudaGetLastError())) return err;
    if ((err = read_state(e->sta, ha, s))) return err;
    chunk = chunk * 2 < e->max_chunk ? chunk * 2 : e->max_chunk;
  }
  return 0;
}

// lambda_min by the Lanczos moments of the inverse-iteration start vector x2
// (gb_lanczos.h): v_1 = x2 (unit), each step one operator pass -- paired with
// the subband PCG while it runs -- then k_lz_step.  At every
// chunk boundary the host evaluates the reference's inverse-iteration
// sequence from T_m and stops once the estimate and its stopping index are
// stable (or T_m is exact: beta = 0).
static int lanczos_min(gb_level_engine_args* e, cudaStream_t s, long long& nl) {
  const int Lpad = e->L + 2 * e->w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const int gv = grid_for(npad, 256, kRedBlocks);
  KState* ka = (KState*)e->sta;
  KState* kb = (KState*)e->stb;
  KState* ha = (KState*)e->hsta;
  KState* hb = (KState*)e->hstb;
  (void)ka;
  int err;
  // x: operator input u_j (unnormalized), w: operator output, vp: v_{j-1}.
  // x starts as the unit start vector; after each step the new u_{j+1} sits
  // in w and the two swap.  Both carry the symmetric layout's output tail.
  if ((err = (int)cudaMemcpyAsync(e->cx, e->x2, sizeof(double) * npad,
                                  cudaMemcpyDeviceToDevice, s)))
    return err;
  double* v = e->cx;
  double* vp = e->xn;  // zero before step 1
  double* w = e->yb;
  if ((err = (int)cudaMemsetAsync(vp, 0, sizeof(double) * npad, s))) return err;
  k_state_reset<<<1, 1, 0, s>>>(kb, e->lz_cap);
  k_lz_init<<<1, 1, 0, s>>>(kb);
  nl += 2;
  int chunk = 64;
  e->lz_its = 0;
  e->lz_rc = 0;
  for (;;) {
    const bool a_live = !ha->done;
    for (int i = 0; i < chunk; ++i) {
      // symmetric layout: the B-half's reduction x.y by linearity in phase 1
      // and phase 2 fused into the Lanczos update (no k_symb_fix launch)
      const int fused = e->layout == 1;
      if (a_live) {
        if ((err = launch_dual(e, v, w, fused ? 0 : 1, fused, s, &nl))) return err;
        post_a(e, s, &nl);
      } else if ((err = launch_single(e, v, w, e->stb, e->partb, fused ? 0 : 1, fused, s,
                                      &nl))) {
        return err;
      }
      if (fused)
        k_symb_lz_update<<<(int)(symb_ntile(e->L) < kRedBlocks ? symb_ntile(e->L) : kRedBlocks),
                           kLzThreads, 0, s>>>(e->L, e->w, v, w, vp, kb, e->partb, e->lz);
      else
        k_lz_step<<<gv, 256, 0, s>>>(npad, v, vp, w, kb, e->partb, e->lz);
      nl += 1;
      double* t = v;
      v = w;
      w = t;
    }
    if ((err = (int)cudaGetLastError())) return err;
    if ((err = read_state(e->sta, ha, s))) return err;
    if ((err = read_state(e->stb, hb, s))) return err;
    const int m = hb->it;
    if (m > 0) {
      if ((err = gbk_sync_read(e->lz, e->hlz, sizeof(double) * 2 * (size_t)m, s))) return err;
      double lam;
      int outer, stable;
      const int rc = gb_lz::lanczos_check(e->hlz, m, e->tol, e->max_outer, e->lz_tol, &lam,
                                          &outer, &stable);
      if (rc) {
        e->lz_rc = rc;
        e->breakdown = -2;
        return 0;
      }
      e->lam_min = lam;
      e->n_outer = outer;
      e->lz_its = m;
      if (hb->done || stable) break;
    } else if (hb->done) {  // A v_1 = 0
      e->breakdown = -1;
      return 0;
    }
    // checks 32 steps apart (the host side of a check is O(m))
    chunk = GB_LZ_CHECK;
  }
  e->calls += e->lz_its;
  return 0;
}

// lambda_min by the reference's inverse iteration (sparse_core.py:258-277),
// inner solves warm-started CG or block-Jacobi PCG, paired with the PCG
static int inverse_iteration(gb_level_engine_args* e, cudaStream_t s, long long& nl) {
  const int Lpad = e->L + 2 * e->w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const int gv = grid_for(npad, 256, kRedBlocks);
  KState* kb = (KState*)e->stb;
  KState* ha = (KState*)e->hsta;
  KState* hb = (KState*)e->hstb;
  int err;
  int chunk;
  // --- inverse iteration -------------------------------------------------
  double* cur = e->x2;     // right-hand side of the inner solve (unit vector)
  double* nxt = e->xn;     // next iterate
  double lam_prev = 1.0 / 0.0;
  int have_prev = 0;       // warm start x0 = previous normalized iterate (= cur)
  e->lam_min = e->lam_max;
  e->n_outer = 0;
  for (int outer = 0; outer < e->max_outer; ++outer) {
    // inner CG: A_op y = cur, x0 = cur when warm (its A x0 is e->ax from the
    // previous Rayleigh quotient)
    k_state_reset<<<1, 1, 0, s>>>(kb, (int)e->inner_max_iter);
    // PCG mode warm-starts from cur / lambda (the current Rayleigh quotient),
    // the reference's CG mode from cur itself (sparse_core.py:266)
    if (e->inner_pcg)
      k_bjcg_init<<<bj_init_grid(e->L), 192, 0, s>>>(
          e->L, e->w, cur, have_prev ? cur : nullptr, have_prev ? e->ax : nullptr,
          have_prev ? 1.0 / e->lam_min : 1.0, e->cx, e->cr, e->cp, e->cz, e->inv, e->inner_tol,
          (int)e->inner_max_iter, kb, e->partb);
    else
      k_cg_init<<<gv, 256, 0, s>>>(npad, cur, have_prev ? cur : nullptr,
                                   have_prev ? e->ax : nullptr, e->cx, e->cr, e->cp,
                                   e->inner_tol, (int)e->inner_max_iter, kb, e->partb);
    k_cg_zero_if<<<gv, 256, 0, s>>>(npad, e->cx, kb);
    nl += 3;
    chunk = 8;
    for (;;) {
      const bool a_live = !ha->done;
      for (int i = 0; i < chunk; ++i) {
        if (a_live) {
          if ((err = launch_dual(e, e->cp, e->cap, 0, e->inner_pcg, s, &nl))) return err;
          post_a(e, s, &nl);
        } else if ((err = launch_single(e, e->cp, e->cap, e->stb, e->partb, 0, e->inner_pcg, s,
                                        &nl))) {
          return err;
        }
        if (e->inner_pcg) {
          pcg_post(e, e->cx, e->cr, e->cp, e->cap, e->cz, kb, e->partb, s, &nl);
        } else {
          k_cg_update<<<gv, 256, 0, s>>>(npad, e->cx, e->cr, e->cp, e->cap, kb, e->partb);
          k_cg_dir<<<gv, 256, 0, s>>>(npad, e->cr, e->cp, kb);
          nl += 2;
        }
      }
      if ((err = (int)cudaGetLastError())) return err;
      if ((err = read_state(e->sta, ha, s))) return err;
      if ((err = read_state(e->stb, hb, s))) return err;
      if (hb->done) break;
      chunk = chunk * 2 < e->max_chunk ? chunk * 2 : e->max_chunk;
    }
    if (hb->breakdown) {
      e->breakdown = hb->breakdown;
      return 0;
    }
    if (outer < 64) e->inner_its[outer] = hb->it;
    e->calls += hb->it + (have_prev ? 1 : 0);
    // y -> unit vector, Rayleigh quotient x.(A x)
    k_dot2<<<gv, 256, 0, s>>>(npad, e->cx, e->cx, nullptr, e->dots, kb, e->partb);
    k_scale_by_norm<<<grid_for(npad, 256, 148 * 16), 256, 0, s>>>(npad, e->cx, e->dots, 0, nxt,
                                                                  nullptr);
    if ((err = launch_plain(e, nxt, e->ax, s, &nl))) return err;
    k_dot2<<<gv, 256, 0, s>>>(npad, nxt, e->ax, nullptr, e->dots + 2, kb, e->partb);
    nl += 3;
    e->calls += 1;
    if ((err = gbk_sync_read(e->dots, e->hdots, 4 * sizeof(double), s))) return err;
    e->n_outer = outer + 1;
    if (e->hdots[0] == 0.0) {
      e->breakdown = -1;  // A^-1 x = 0
      return 0;
    }
    const double lam = e->hdots[2];
    e->lam_min = lam;
    double* t = cur;
    cur = nxt;
    nxt = t;
    have_prev = 1;
    if (fabs(lam - lam_prev) <= 0.5 * e->tol * fabs(lam)) break;
    lam_prev = lam;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Row-strip Krylov launchers (gb_dist.cuh): rank-local pieces of the
// distributed block-Jacobi PCG / power iteration / Lanczos recurrence on the
// grid rows [r0, r1) of a tiled level.  The caller (gamblet_dist.py) exchanges
// halos and all-reduces the partial sums between them.
// ---------------------------------------------------------------------------
static inline bool dist_rows_ok(int L, int r0, int r1) {
  return r0 >= 0 && r1 <= L && r0 < r1 && r0 % kSymTH == 0 && r1 % kSymTH == 0 &&
         L % kSymTW == 0;
}
static inline int dist_bj_grid(int nblk) { return grid_for(nblk, 16, kRedBlocks); }

// phase 1 of y_v = (S B S) x_v on the strip's tiles for nv = 1, 2 vectors with
// the strip partials of x_v . (A x_v) formed by linearity -> red[0], red[1]
int gbk_dist_apply(int L, int w, const double* U, int nv, const double* x0, double* y0,
                   void* st0, double* part0, const double* x1, double* y1, void* st1,
                   double* part1, double* red, int r0, int r1, cudaStream_t s) {
  if (!dist_rows_ok(L, r0, r1) || (nv != 1 && nv != 2)) return GB_UNSUPPORTED;
  const long long tpr = L / kSymTW;
  sym_phase1(L, w, U, nv, x0, y0, (KState*)st0, part0, 2, x1, y1, (KState*)st1, part1, 2, s,
             (r0 / kSymTH) * tpr, (r1 / kSymTH) * tpr);
  k_dist_pack<<<1, 1, 0, s>>>((KState*)st0, nv == 2 ? (KState*)st1 : nullptr, red);
  return (int)cudaGetLastError();
}

int gbk_dist_pcg_init(int L, int w, const double* b, double* x, double* r, double* p, double* z,
                      const float* inv, void* st, double* part, double* out, int r0, int r1,
                      cudaStream_t s) {
  if (!dist_rows_ok(L, r0, r1)) return GB_UNSUPPORTED;
  const int Lb = L / 2, b0 = (r0 / 2) * Lb, b1 = (r1 / 2) * Lb;
  k_dist_pcg_init<<<dist_bj_grid(b1 - b0), 192, 0, s>>>(L, w, b, x, r, p, z, inv, (KState*)st,
                                                        part, out, b0, b1);
  return (int)cudaGetLastError();
}
int gbk_dist_pcg_init_commit(void* st, const double* out, double rel_tol, int max_iter,
                             cudaStream_t s) {
  k_dist_pcg_init_commit<<<1, 1, 0, s>>>((KState*)st, out, rel_tol, max_iter);
  return (int)cudaGetLastError();
}
int gbk_dist_pcg_update(int L, int w, double* x, double* r, const double* p, const double* Ap,
                        double* z, const float* inv, void* st, const double* red, double* part,
                        double* out, int r0, int r1, cudaStream_t s) {
  if (!dist_rows_ok(L, r0, r1)) return GB_UNSUPPORTED;
  const int Lb = L / 2, b0 = (r0 / 2) * Lb, b1 = (r1 / 2) * Lb;
  k_dist_pcg_update<<<dist_bj_grid(b1 - b0), 192, 0, s>>>(L, w, x, r, p, Ap, z, inv, (KState*)st,
                                                          red, part, out, b0, b1);
  return (int)cudaGetLastError();
}
// all-reduced sums -> state, then p = z + beta p on the strip
int gbk_dist_pcg_commit_dir(int L, int w, void* st, const double* red, const double* out,
                            const double* z, double* p, int r0, int r1, cudaStream_t s) {
  if (!dist_rows_ok(L, r0, r1)) return GB_UNSUPPORTED;
  const long long Lpad = L + 2 * w, off = (long long)(r0 + w) * Lpad * 3,
                  n = (long long)(r1 - r0) * Lpad * 3;
  k_dist_pcg_commit<<<1, 1, 0, s>>>((KState*)st, red, out);
  k_cg_dir<<<grid_for(n, 256, kRedBlocks), 256, 0, s>>>(n, z + off, p + off, (KState*)st);
  return (int)cudaGetLastError();
}
int gbk_dist_fix_yy(int L, int w, double* y, void* st, double* part, double* out, int r0, int r1,
                    cudaStream_t s) {
  if (!dist_rows_ok(L, r0, r1)) return GB_UNSUPPORTED;
  const long long n = (long long)(r1 - r0) * L * 3;
  k_dist_fix_yy<<<grid_for(n, 256, kRedBlocks), 256, 0, s>>>(L, w, y, (KState*)st, part, out, r0,
                                                            r1);
  return (int)cudaGetLastError();
}
// power iteration between the reductions: stage 0 (x.y and y.y all-reduced)
// sets lam, ynorm and forms the residual partial; stage 1 (residual
// all-reduced) tests convergence and rescales x = y / ynorm on the strip
int gbk_dist_pow_step(int L, int w, double* x, const double* y, void* st, const double* red,
                      const double* out_yy, double* out_res, double* part, double tol, int r0,
                      int r1, int stage, cudaStream_t s) {
  if (!dist_rows_ok(L, r0, r1)) return GB_UNSUPPORTED;
  const long long Lpad = L + 2 * w, off = (long long)(r0 + w) * Lpad * 3,
                  n = (long long)(r1 - r0) * Lpad * 3;
  const int g = grid_for(n, 256, kRedBlocks);
  if (stage == 0) {
    k_dist_pow_commit1<<<1, 1, 0, s>>>((KState*)st, red, out_yy);
    k_dist_pow_res<<<g, 256, 0, s>>>(n, x + off, y + off, (KState*)st, part, out_res);
  } else {
    k_dist_pow_commit2<<<1, 1, 0, s>>>((KState*)st, out_res, tol);
    k_pow_scale<<<g, 256, 0, s>>>(n, x + off, y + off, (KState*)st);
  }
  return (int)cudaGetLastError();
}
int gbk_dist_lz_update(int L, int w, const double* x, double* y, double* vp, void* st,
                       const double* red, double* part, double* out, int r0, int r1,
                       cudaStream_t s) {
  if (!dist_rows_ok(L, r0, r1)) return GB_UNSUPPORTED;
  const long long n = (long long)(r1 - r0) * L * 3;
  k_dist_lz_update<<<grid_for(n, 256, kRedBlocks), 256, 0, s>>>(L, w, x, y, vp, (KState*)st, red,
                                                               part, out, r0, r1);
  return (int)cudaGetLastError();
}
int gbk_dist_lz_commit(void* st, const double* red, const double* out, double* ab,
                       cudaStream_t s) {
  k_dist_lz_commit<<<1, 1, 0, s>>>((KState*)st, red, out, ab);
  return (int)cudaGetLastError();
}
int gbk_dist_lz_begin(void* st, int cap, cudaStream_t s) {
  k_state_reset<<<1, 1, 0, s>>>((KState*)st, cap);
  k_lz_init<<<1, 1, 0, s>>>((KState*)st);
  return (int)cudaGetLastError();
}
int gbk_dist_dot(long long n, const double* a, const double* b, void* st, double* part,
                 double* out, cudaStream_t s) {
  k_dist_dot<<<grid_for(n, 256, kRedBlocks), 256, 0, s>>>(n, a, b, (KState*)st, part, out);
  return (int)cudaGetLastError();
}
