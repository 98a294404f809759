// Row-strip Krylov kernels of the spatially partitioned solve (multi-GPU,
// paper_1503_03467_b200/gamblet_dist.py).  A rank owns the grid rows [r0, r1)
// of a tiled level (multiples of kSymTH): its rows of the symmetric band copy
// of S B S, of the block-Jacobi inverses and of every Krylov vector.  Vectors
// keep the global zero-halo padded layout (and the global spill-over tail), so
// the single-GPU kernels run on a tile / row range; what crosses ranks is
//   * the w rows of the operator input below the strip      (halo, neighbour)
//   * the spill-over tiles of the KI tile rows above it     (halo, neighbour)
//   * the partial sums of every reduction                   (all-reduce)
// so every kernel that forms a reduction stops at the rank's partial sum
// (deterministic two-level order) and a one-thread commit kernel applies the
// all-reduced value to the iteration state -- the same state machine as the
// single-GPU engine (sparse_core.py:126-165 for CG, :232-257 for the power
// iteration), split at the reduction points.
#pragma once

// red[0] = sa->pAp, red[1] = sb->pAp: the raw strip partials phase 1 formed
// by linearity (red mode 2); a null state contributes 0
__global__ void k_dist_pack(const KState* sa, const KState* sb, double* red) {
  red[0] = (sa && !sa->done) ? sa->pAp : 0.0;
  red[1] = (sb && !sb->done) ? sb->pAp : 0.0;
}

__device__ __forceinline__ void dist_emit(KState* st, double* part, double* out, int nout,
                                          double a, double b, double c, double* sh) {
  a = block_sum(a, sh);
  b = block_sum(b, sh);
  c = block_sum(c, sh);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = a;
    part[3 * blockIdx.x + 1] = b;
    part[3 * blockIdx.x + 2] = c;
  }
  if (last_block(&st->counter)) {
    double x = 0.0, y = 0.0, z = 0.0;
    for (int j = threadIdx.x; j < (int)gridDim.x; j += blockDim.x) {
      x += part[3 * j];
      y += part[3 * j + 1];
      z += part[3 * j + 2];
    }
    x = block_sum(x, sh);
    y = block_sum(y, sh);
    z = block_sum(z, sh);
    if (threadIdx.x == 0) {
      st->counter = 0;
      out[0] = x;
      if (nout > 1) out[1] = y;
      if (nout > 2) out[2] = z;
    }
  }
}

// block-Jacobi apply of one 12-row block: z = Minv r (fp32 inverse, fp64 sums)
__device__ __forceinline__ double dist_bj_row(const float* __restrict__ inv, long long b, int l,
                                              const double* rb) {
  const float* iv = inv + b * 144 + l * 12;
  float iw[12];
#pragma unroll
  for (int q4 = 0; q4 < 3; ++q4) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(iv) + q4);
    iw[4 * q4] = f.x;
    iw[4 * q4 + 1] = f.y;
    iw[4 * q4 + 2] = f.z;
    iw[4 * q4 + 3] = f.w;
  }
  double zv = 0.0;
#pragma unroll
  for (int k = 0; k < 12; ++k) zv = fma((double)iw[k], rb[k], zv);
  return zv;
}

// x = 0, r = b, z = Minv r, p = z on the blocks [b_lo, b_hi);
// out = (r.r, r.z, b.b) partials of the strip
__global__ void __launch_bounds__(192) k_dist_pcg_init(int L, int w, const double* __restrict__ b,
                                                       double* __restrict__ x,
                                                       double* __restrict__ r,
                                                       double* __restrict__ p,
                                                       double* __restrict__ z,
                                                       const float* __restrict__ inv, KState* st,
                                                       double* part, double* out, int b_lo,
                                                       int b_hi) {
  __shared__ double rs[192];
  __shared__ double sh[32];
  const int lb = threadIdx.x / 12, l = threadIdx.x % 12;
  double bb = 0.0, rz = 0.0;
  for (int b0 = b_lo + blockIdx.x * 16; b0 < b_hi; b0 += gridDim.x * 16) {
    const int bk = b0 + lb;
    long long pr = -1;
    double rv = 0.0;
    if (bk < b_hi) {
      pr = bj_row_pad(L, w, bk, l);
      rv = b[pr];
      x[pr] = 0.0;
      r[pr] = rv;
      bb += rv * rv;
    }
    rs[threadIdx.x] = rv;
    __syncthreads();
    if (bk < b_hi) {
      const double zv = dist_bj_row(inv, bk, l, rs + lb * 12);
      z[pr] = zv;
      p[pr] = zv;
      rz += rv * zv;
    }
    __syncthreads();
  }
  dist_emit(st, part, out, 3, bb, rz, bb, sh);
}

// the all-reduced (r.r, r.z, b.b) -> iteration state (k_bjcg_init's tail)
__global__ void k_dist_pcg_init_commit(KState* st, const double* out, double rel_tol,
                                       int max_iter) {
  st->counter = 0;
  st->it = 0;
  st->breakdown = 0;
  st->max_iter = max_iter;
  const double bn = sqrt(out[2]);
  st->bnorm = bn;
  st->tol_abs = rel_tol * bn;
  const double rn = sqrt(out[0]);
  st->rnorm = rn;
  st->rs = out[1];
  st->done = 0;
  st->converged = 0;
  st->aux0 = 0.0;
  if (bn == 0.0) {
    st->done = 1;
    st->converged = 1;
    st->rnorm = 0.0;
    st->aux0 = 1.0;
  } else if (rn <= rel_tol * bn) {
    st->done = 1;
    st->converged = 1;
  }
}

// x += alpha p; r -= alpha (A p completed by the neighbours' spill-over);
// z = Minv r on the blocks [b_lo, b_hi); alpha = rs / red[0] with red[0] the
// all-reduced p.Ap; out = (r.r, r.z) partials
__global__ void __launch_bounds__(192) k_dist_pcg_update(
    int L, int w, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
    const double* __restrict__ Ap, double* __restrict__ z, const float* __restrict__ inv,
    KState* st, const double* red, double* part, double* out, int b_lo, int b_hi) {
  __shared__ double rs[192];
  __shared__ double sh[32];
  if (st->done) return;
  const double pAp = red[0];
  if (!(pAp > 0.0)) return;  // breakdown: the commit kernel reports it
  const double alpha = st->rs / pAp;
  const int Lb = L >> 1, Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const int lb = threadIdx.x / 12, l = threadIdx.x % 12;
  const int pi = l / 3, c = l - 3 * pi;
  double rr = 0.0, rz = 0.0;
  for (int b0 = b_lo + blockIdx.x * 16; b0 < b_hi; b0 += gridDim.x * 16) {
    const int b = b0 + lb;
    long long pr = -1;
    double rv = 0.0;
    if (b < b_hi) {
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
    if (b < b_hi) {
      const double zv = dist_bj_row(inv, b, l, rs + lb * 12);
      z[pr] = zv;
      rz += rv * zv;
    }
    __syncthreads();
  }
  dist_emit(st, part, out, 2, rr, rz, 0.0, sh);
}

// the all-reduced p.Ap (red[0]) and (r.r, r.z) (out) -> state: breakdown,
// convergence, beta (the tail of k_symb_bjcg_update)
__global__ void k_dist_pcg_commit(KState* st, const double* red, const double* out) {
  if (st->done) return;
  const double pAp = red[0];
  st->pAp = pAp;
  if (!(pAp > 0.0)) {
    st->breakdown = st->it + 1;
    st->done = 1;
    return;
  }
  st->alpha = st->rs / pAp;
  st->it += 1;
  const double rn = sqrt(out[0]);
  st->rnorm = rn;
  if (rn <= st->tol_abs) {
    st->done = 1;
    st->converged = 1;
  } else if (st->it >= st->max_iter) {
    st->done = 1;
    st->converged = 0;
  } else {
    st->beta = out[1] / st->rs;
    st->rs = out[1];
  }
}

// y <- y + neighbours' spill-over on the grid rows [r0, r1); out[0] = y.y partial
__global__ void __launch_bounds__(256) k_dist_fix_yy(int L, int w, double* __restrict__ y,
                                                     KState* st, double* part, double* out,
                                                     int r0, int r1) {
  __shared__ double sh[32];
  if (st->done) return;
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const long long e0 = (long long)r0 * L * 3, e1 = (long long)r1 * L * 3;
  double yy = 0.0;
  for (long long r = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < e1;
       r += (long long)gridDim.x * blockDim.x) {
    const long long pp = r / 3;
    const int c = (int)(r - pp * 3);
    const int ps = (int)(pp / L), pt = (int)(pp % L);
    const long long yi = ((long long)(ps + w) * Lpad + pt + w) * 3 + c;
    const double s = symb_fix_value(y[yi], y + npad, L, w, ps, pt, c);
    y[yi] = s;
    yy = fma(s, s, yy);
  }
  dist_emit(st, part, out, 1, yy, 0.0, 0.0, sh);
}

// power iteration: the all-reduced x.y (red[1]) and y.y (out[0]) -> lam, ynorm
__global__ void k_dist_pow_commit1(KState* st, const double* red, const double* out) {
  if (st->done) return;
  st->lam = red[1];
  st->ynorm = sqrt(out[0]);
  if (st->ynorm == 0.0) {
    st->lam = 0.0;
    st->done = 1;
  }
}

// |y - lam x|^2 partial over n contiguous elements (the strip's padded rows)
__global__ void k_dist_pow_res(long long n, const double* __restrict__ x,
                               const double* __restrict__ y, KState* st, double* part,
                               double* out) {
  __shared__ double sh[32];
  if (st->done) return;
  const double lam = st->lam;
  double rr = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double d = y[i] - lam * x[i];
    rr += d * d;
  }
  dist_emit(st, part, out, 1, rr, 0.0, 0.0, sh);
}

// residual test of the power iteration (the tail of k_pow_step)
__global__ void k_dist_pow_commit2(KState* st, const double* out, double tol) {
  if (st->done) return;
  st->res = sqrt(out[0]);
  st->it += 1;
  st->aux1 = (st->res <= 0.5 * tol * fabs(st->lam) || st->it >= st->max_iter) ? 1.0 : 0.0;
}

// Lanczos step on the grid rows [r0, r1) (k_lz_step with the spill-over of y
// completed first): alpha = x.y / bp^2 from the all-reduced red[1];
// out[0] = |u_{j+1}|^2 partial
__global__ void __launch_bounds__(256) k_dist_lz_update(int L, int w,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y,
                                                        double* __restrict__ vp, KState* st,
                                                        const double* red, double* part,
                                                        double* out, int r0, int r1) {
  __shared__ double sh[32];
  if (st->done) return;
  const int Lpad = L + 2 * w;
  const long long npad = (long long)Lpad * Lpad * 3;
  const double bp = st->aux0, ibp = 1.0 / bp;
  const double alpha = red[1] * ibp * ibp;
  const long long e0 = (long long)r0 * L * 3, e1 = (long long)r1 * L * 3;
  double uu = 0.0;
  for (long long r = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < e1;
       r += (long long)gridDim.x * blockDim.x) {
    const long long pp = r / 3;
    const int c = (int)(r - pp * 3);
    const int ps = (int)(pp / L), pt = (int)(pp % L);
    const long long yi = ((long long)(ps + w) * Lpad + pt + w) * 3 + c;
    const double yv = symb_fix_value(y[yi], y + npad, L, w, ps, pt, c);
    const double xv = x[yi];
    const double v = xv * ibp;
    const double u = (yv - alpha * xv) * ibp - bp * vp[yi];
    vp[yi] = v;
    y[yi] = u;
    uu += u * u;
  }
  dist_emit(st, part, out, 1, uu, 0.0, 0.0, sh);
}

// (alpha_j, beta_j) appended to ab; the tail of k_lz_step
__global__ void k_dist_lz_commit(KState* st, const double* red, const double* out, double* ab) {
  if (st->done) return;
  const double bp = st->aux0, ibp = 1.0 / bp;
  const double beta = sqrt(out[0]);
  ab[2 * st->it] = red[1] * ibp * ibp;
  ab[2 * st->it + 1] = beta;
  st->it += 1;
  st->aux0 = beta;
  if (!(beta > 0.0) || st->it >= st->max_iter) st->done = 1;
}

// a.b partial over n contiguous elements -> out[0] (normalizing start vectors)
__global__ void k_dist_dot(long long n, const double* __restrict__ a,
                           const double* __restrict__ b, KState* st, double* part, double* out) {
  __shared__ double sh[32];
  double d = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    d = fma(a[i], b[i], d);
  dist_emit(st, part, out, 1, d, 0.0, 0.0, sh);
}
