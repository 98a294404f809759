// 3-D localized gamblet transform (BASELINE config 4: unit cube, Q1
// trilinear, 27-point stencil, rho = 2).  The reference is 2-D only
// (grid_fem.py:1-14, hierarchy.py:1-14); these kernels follow its algorithm
// in d = 3 as restated by oracle/gamblets_oracle_nd.py:
//   2^3 children per aggregate (lexicographic offsets, axis 0 slowest),
//   pi (0/1), pibar = pi / 8, W = 7 Helmert rows per parent over its 8
//   children (Lemma 4.14), chi = 7 * ball + c.
//
// Layout ("3-D box stencil"): a level operator on an L^3 grid with nr
// components per point and half-width w stores row r = p * nr + c,
// p = (x * L + y) * L + z, columns (p + d, c') for |d|_inf <= w:
//
//     val[r * S + (((dx+w) W3 + (dy+w)) W3 + (dz+w)) * nc + c'],   W3 = 2w+1,
//     S = W3^3 * nc.
//
// Out-of-domain and dropped entries are 0.0 (the CSR export keeps != 0).
// psi^(q) rows use an origin-clamped cube window of side wd.
//
// Summation orders follow the reference's CSR products (ascending column
// index = ascending lexicographic offset), sums from 0.0.
#include "gb_common.cuh"
#include "gb_kernels.h"

namespace gb {

struct W7x8 {
  double w[7][8];
};

__host__ __device__ __forceinline__ int slot3(int w, int nc, int dx, int dy, int dz, int c) {
  const int W3 = 2 * w + 1;
  return (((dx + w) * W3 + (dy + w)) * W3 + (dz + w)) * nc + c;
}
__host__ __device__ __forceinline__ long long slots3(int w, int nc) {
  const long long W3 = 2 * w + 1;
  return W3 * W3 * W3 * nc;
}
__device__ __forceinline__ void unflat3(long long p, int L, int* x, int* y, int* z) {
  *z = (int)(p % L);
  const long long q = p / L;
  *y = (int)(q % L);
  *x = (int)(q / L);
}
__device__ __forceinline__ long long flat3(int x, int y, int z, int L) {
  return ((long long)x * L + y) * L + z;
}
__device__ __forceinline__ bool inside3(int x, int y, int z, int L) {
  return (unsigned)x < (unsigned)L && (unsigned)y < (unsigned)L && (unsigned)z < (unsigned)L;
}

// ---------------------------------------------------------------------------
// inputs: canonical CSR (27-point stencil) -> box, diagonal scaling
// ---------------------------------------------------------------------------
__global__ void k3_csr_to_box(int L, int w, const int32_t* __restrict__ indptr,
                              const int32_t* __restrict__ indices,
                              const double* __restrict__ data, double* __restrict__ box,
                              long long* status) {
  const long long n = (long long)L * L * L;
  const long long S = slots3(w, 1);
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    unflat3(r, L, &x, &y, &z);
    for (int e = indptr[r]; e < indptr[r + 1]; ++e) {
      int cx, cy, cz;
      unflat3(indices[e], L, &cx, &cy, &cz);
      const int dx = cx - x, dy = cy - y, dz = cz - z;
      if (abs(dx) > w || abs(dy) > w || abs(dz) > w) {
        raise_status(status, ST_OUTSIDE_BOX, r);
        continue;
      }
      box[r * S + slot3(w, 1, dx, dy, dz, 0)] = data[e];
    }
  }
}

// s = diag^{-1/2} (gamblet_fast.py:123-139)
__global__ void k3_box_scale(long long rows, int nr, int w, const double* __restrict__ box,
                             double* __restrict__ s, long long* status) {
  const long long S = slots3(w, nr);
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(r % nr);
    const double d = box[r * S + slot3(w, nr, 0, 0, 0, c)];
    if (!(d > 0.0)) {
      raise_status(status, ST_NONPOS_DIAG, r);
      s[r] = 0.0;
    } else {
      s[r] = 1.0 / sqrt(d);
    }
  }
}

// min over the diagonal (drop_dead_tails' d.min() <= 0 guard) and the
// symmetry statistics max|X|, max|X - X^T| (gamblet_exact.py:95-103)
__device__ __forceinline__ void atomic_min_double(double* addr, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *a, assumed;
  do {
    assumed = old;
    if (__longlong_as_double((long long)assumed) <= v) return;
    old = atomicCAS(a, assumed, (unsigned long long)__double_as_longlong(v));
  } while (old != assumed);
}

__global__ void k3_box_diag_min(long long rows, int nr, int w, const double* __restrict__ box,
                                double* dmin) {
  __shared__ double sh[32];
  const long long S = slots3(w, nr);
  double m = 1.0e308;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x)
    m = fmin(m, box[r * S + slot3(w, nr, 0, 0, 0, (int)(r % nr))]);
  m = warp_min(m);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = sh[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) t = fmin(t, sh[i]);
    atomic_min_double(dmin, t);
  }
}

// out = drop_dead(sym(raw)) (gamblet_exact.py:95-103, gamblet_fast.py:154-169):
// (x_ij + x_ji) * 0.5, off-diagonal |v| < 1e-12 sqrt(d_i d_j) dropped when
// min(d) > 0; stats[0] = max|x|, stats[1] = max|x - x^T| (non-negative bits)
__global__ void k3_box_sym_drop(int L, int nr, int w, const double* __restrict__ raw,
                                double* __restrict__ out, const double* dmin,
                                double* stats) {
  const long long rows = (long long)L * L * L * nr;
  const long long S = slots3(w, nr);
  const bool drop = *dmin > 0.0;
  double mx = 0.0, md = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < rows * S;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / S;
    const int sl = (int)(e - r * S);
    const int cp = sl % nr;
    int t = sl / nr;
    const int W3 = 2 * w + 1;
    const int dz = t % W3 - w;
    t /= W3;
    const int dy = t % W3 - w, dx = t / W3 - w;
    const long long p = r / nr;
    const int c = (int)(r - p * nr);
    int x, y, z;
    unflat3(p, L, &x, &y, &z);
    double v = 0.0;
    if (inside3(x + dx, y + dy, z + dz, L)) {
      const long long q = flat3(x + dx, y + dy, z + dz, L);
      const long long rt = q * nr + cp;
      const double a = raw[e];
      const double b = raw[rt * S + slot3(w, nr, -dx, -dy, -dz, c)];
      mx = fmax(mx, fabs(a));
      md = fmax(md, fabs(a - b));
      v = (a + b) * 0.5;
      if (drop && !(dx == 0 && dy == 0 && dz == 0 && c == cp) && v != 0.0) {
        const double di = raw[r * S + slot3(w, nr, 0, 0, 0, c)];
        const double dj = raw[rt * S + slot3(w, nr, 0, 0, 0, cp)];
        if (fabs(v) < 1e-12 * sqrt(di * dj)) v = 0.0;
      }
    }
    out[e] = v;
  }
  mx = warp_max(mx);
  md = warp_max(md);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(stats, mx);
    atomic_max_nonneg(stats + 1, md);
  }
}

// ---------------------------------------------------------------------------
// K1 mass patches, psi^(q) (gamblet_fast.py:464-498): one CTA per fine node,
// the patch (S M S)[box, box] (m <= 125 at rho = 2) packed-lower in shared
// memory, right-looking Cholesky, solve with s_i e_i, psi row = s[box] z
// ---------------------------------------------------------------------------
constexpr int k3MassThreads = 128;

__device__ __forceinline__ int type_rep3(int c, int L, int rho) {
  return (c < rho || c > L - 1 - rho) ? c : rho;
}
__device__ __forceinline__ int rep_coord3(int l, int L, int rho) {
  return l <= rho ? l : L - (2 * rho + 1) + l;
}

// mode 0: every fine node; 1: the (2 rho + 1)^3 clip-type representatives;
// 2: every node, only when *flag != 0 (M not translation invariant)
__global__ void __launch_bounds__(k3MassThreads) k3_mass_patches(
    int L, const double* __restrict__ M, const double* __restrict__ s, int rho, int wd,
    double* __restrict__ psi, long long* status, int mode, const int* __restrict__ flag) {
  if (mode == 2 && *flag == 0) return;
  extern __shared__ double sm[];
  const int R = 2 * rho + 1;
  const int mmax = R * R * R;
  double* K = sm;                                   // packed lower, mmax (mmax+1) / 2
  double* v = K + (long long)mmax * (mmax + 1) / 2;  // rhs / solution
  __shared__ int bx0, by0, bz0, nx, ny, nz, bad;
  const int tid = threadIdx.x;
  const long long N = (long long)L * L * L;
  const long long SM = slots3(1, 1);
  const long long cnt = mode == 1 ? (long long)R * R * R : N;
  for (long long ii = blockIdx.x; ii < cnt; ii += gridDim.x) {
    int x, y, z;
    if (mode == 1) {
      x = rep_coord3((int)(ii / (R * R)), L, rho);
      y = rep_coord3((int)((ii / R) % R), L, rho);
      z = rep_coord3((int)(ii % R), L, rho);
    } else {
      unflat3(ii, L, &x, &y, &z);
    }
    const long long i = flat3(x, y, z, L);
    if (tid == 0) {
      bx0 = imax(x - rho, 0);
      by0 = imax(y - rho, 0);
      bz0 = imax(z - rho, 0);
      nx = imin(x + rho, L - 1) - bx0 + 1;
      ny = imin(y + rho, L - 1) - by0 + 1;
      nz = imin(z + rho, L - 1) - bz0 + 1;
      bad = 0;
    }
    __syncthreads();
    const int m = nx * ny * nz;
    const int own = ((x - bx0) * ny + (y - by0)) * nz + (z - bz0);
    // gather: K[a][b] = (M_ab s_a) s_b for b <= a
    for (int e = tid; e < m * (m + 1) / 2; e += blockDim.x) {
      int a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (a * (a + 1) / 2 > e) --a;
      while ((a + 1) * (a + 2) / 2 <= e) ++a;
      const int b = e - a * (a + 1) / 2;
      const int az = a % nz, ay = (a / nz) % ny, ax = a / (nz * ny);
      const int bz = b % nz, by = (b / nz) % ny, bxx = b / (nz * ny);
      const int dx = bxx - ax, dy = by - ay, dz = bz - az;
      double val = 0.0;
      if (abs(dx) <= 1 && abs(dy) <= 1 && abs(dz) <= 1) {
        const long long ra = flat3(bx0 + ax, by0 + ay, bz0 + az, L);
        const long long rb = flat3(bx0 + bxx, by0 + by, bz0 + bz, L);
        val = (M[ra * SM + slot3(1, 1, dx, dy, dz, 0)] * s[ra]) * s[rb];
      }
      K[e] = val;
    }
    for (int a = tid; a < m; a += blockDim.x) v[a] = a == own ? s[i] : 0.0;
    __syncthreads();
    // right-looking Cholesky, column j
    for (int j = 0; j < m; ++j) {
      const int jj = j * (j + 1) / 2 + j;
      if (tid == 0) {
        const double d = K[jj];
        if (!(d > 0.0)) bad = 1;
        K[jj] = sqrt(d);
      }
      __syncthreads();
      if (bad) break;
      const double ljj = K[jj];
      for (int a = j + 1 + tid; a < m; a += blockDim.x) K[a * (a + 1) / 2 + j] /= ljj;
      __syncthreads();
      const int t = m - j - 1;
      for (int e = tid; e < t * (t + 1) / 2; e += blockDim.x) {
        int a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
        while (a * (a + 1) / 2 > e) --a;
        while ((a + 1) * (a + 2) / 2 <= e) ++a;
        const int b = e - a * (a + 1) / 2;
        const int ia = a + j + 1, ib = b + j + 1;
        K[ia * (ia + 1) / 2 + ib] -= K[ia * (ia + 1) / 2 + j] * K[ib * (ib + 1) / 2 + j];
      }
      __syncthreads();
    }
    if (bad) {
      if (tid == 0) raise_status(status, ST_NOT_SPD, i);
      __syncthreads();
      continue;
    }
    // forward L y = v (column oriented), back L^T z = y
    for (int j = 0; j < m; ++j) {
      if (tid == 0) v[j] /= K[j * (j + 1) / 2 + j];
      __syncthreads();
      const double yj = v[j];
      for (int a = j + 1 + tid; a < m; a += blockDim.x) v[a] -= K[a * (a + 1) / 2 + j] * yj;
      __syncthreads();
    }
    for (int j = m - 1; j >= 0; --j) {
      if (tid == 0) v[j] /= K[j * (j + 1) / 2 + j];
      __syncthreads();
      const double zj = v[j];
      const int rj = j * (j + 1) / 2;
      for (int a = tid; a < j; a += blockDim.x) v[a] -= K[rj + a] * zj;
      __syncthreads();
    }
    // psi row in the origin-clamped window
    const int ox = clampi(x - rho, 0, L - wd), oy = clampi(y - rho, 0, L - wd),
              oz = clampi(z - rho, 0, L - wd);
    const long long W3w = (long long)wd * wd * wd;
    double* row = psi + i * W3w;
    for (int e = tid; e < W3w; e += blockDim.x) {
      const int ez = e % wd, ey = (e / wd) % wd, ex = e / (wd * wd);
      const int fx = ox + ex - bx0, fy = oy + ey - by0, fz = oz + ez - bz0;
      double val = 0.0;
      if (fx >= 0 && fx < nx && fy >= 0 && fy < ny && fz >= 0 && fz < nz) {
        const int a = (fx * ny + fy) * nz + fz;
        val = s[flat3(bx0 + fx, by0 + fy, bz0 + fz, L)] * v[a];
      }
      row[e] = val;
    }
    __syncthreads();
  }
}

// M translation invariant: every in-domain stencil entry of every row equals
// the interior representative's, bit for bit (else *flag = 1)
__global__ void k3_mass_invariance(int L, const double* __restrict__ M, int* flag) {
  const long long N = (long long)L * L * L;
  const long long c = flat3(L / 2, L / 2, L / 2, L);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    unflat3(i, L, &x, &y, &z);
    bool bad = false;
    for (int d = 0; d < 27; ++d) {
      const int dx = d / 9 - 1, dy = (d / 3) % 3 - 1, dz = d % 3 - 1;
      if (inside3(x + dx, y + dy, z + dz, L) &&
          __double_as_longlong(M[i * 27 + d]) != __double_as_longlong(M[c * 27 + d]))
        bad = true;
    }
    if (bad) atomicOr(flag, 1);
  }
}

// psi row i = the row of its clip-type representative (same window content)
__global__ void k3_mass_broadcast(int L, int rho, int wd, double* __restrict__ psi,
                                  const int* __restrict__ flag) {
  if (*flag != 0) return;
  const long long W3w = (long long)wd * wd * wd;
  const long long total = (long long)L * L * L * W3w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / W3w;
    int x, y, z;
    unflat3(i, L, &x, &y, &z);
    const long long r =
        flat3(type_rep3(x, L, rho), type_rep3(y, L, rho), type_rep3(z, L, rho), L);
    if (r != i) psi[e] = psi[r * W3w + (e - i * W3w)];
  }
}

// psi window value of row i at fine node (fx, fy, fz); 0 outside the window
__device__ __forceinline__ double psi_at(const double* __restrict__ psi, long long i, int L,
                                         int lo, int wd, int cx, int cy, int cz, int fx, int fy,
                                         int fz) {
  const int ox = clampi(cx + lo, 0, L - wd), oy = clampi(cy + lo, 0, L - wd),
            oz = clampi(cz + lo, 0, L - wd);
  const int ex = fx - ox, ey = fy - oy, ez = fz - oz;
  if ((unsigned)ex >= (unsigned)wd || (unsigned)ey >= (unsigned)wd || (unsigned)ez >= (unsigned)wd)
    return 0.0;
  return psi[i * (long long)wd * wd * wd + ((long long)ex * wd + ey) * wd + ez];
}

// ---------------------------------------------------------------------------
// K2 A^(q) = psi A psi^T (gamblet_fast.py:658-665) in two stencil passes:
// X = psi A on the box of half-width rho + 1, then raw = X psi^T on 2 rho + 1
// ---------------------------------------------------------------------------
__global__ void k3_psi_stencil(int L, int rho, int wd, const double* __restrict__ psi,
                               const double* __restrict__ A, int wX, double* __restrict__ X) {
  const long long N = (long long)L * L * L;
  const long long SX = slots3(wX, 1), SA = slots3(1, 1);
  const int W3 = 2 * wX + 1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N * SX;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / SX;
    const int sl = (int)(e - i * SX);
    const int dz = sl % W3 - wX, dy = (sl / W3) % W3 - wX, dx = sl / (W3 * W3) - wX;
    int x, y, z;
    unflat3(i, L, &x, &y, &z);
    const int bx = x + dx, by = y + dy, bz = z + dz;
    double acc = 0.0;
    if (inside3(bx, by, bz, L)) {
      // a in ball(i, rho) with |b - a| <= 1, ascending
      const int ax0 = imax(imax(x - rho, bx - 1), 0), ax1 = imin(imin(x + rho, bx + 1), L - 1);
      const int ay0 = imax(imax(y - rho, by - 1), 0), ay1 = imin(imin(y + rho, by + 1), L - 1);
      const int az0 = imax(imax(z - rho, bz - 1), 0), az1 = imin(imin(z + rho, bz + 1), L - 1);
      for (int ax = ax0; ax <= ax1; ++ax)
        for (int ay = ay0; ay <= ay1; ++ay)
          for (int az = az0; az <= az1; ++az) {
            const double pv = psi_at(psi, i, L, -rho, wd, x, y, z, ax, ay, az);
            const long long ra = flat3(ax, ay, az, L);
            acc += pv * A[ra * SA + slot3(1, 1, bx - ax, by - ay, bz - az, 0)];
          }
    }
    X[e] = acc;
  }
}

__global__ void __launch_bounds__(256) k3_psi_galerkin(int L, int rho, int wd,
                                                       const double* __restrict__ psi, int wX,
                                                       const double* __restrict__ X, int wR,
                                                       double* __restrict__ raw) {
  extern __shared__ double xs[];  // X row, slots3(wX, 1)
  const long long N = (long long)L * L * L;
  const long long SX = slots3(wX, 1), SR = slots3(wR, 1);
  const int WR = 2 * wR + 1, WX = 2 * wX + 1;
  for (long long i = blockIdx.x; i < N; i += gridDim.x) {
    int x, y, z;
    unflat3(i, L, &x, &y, &z);
    for (int e = threadIdx.x; e < SX; e += blockDim.x) xs[e] = X[i * SX + e];
    __syncthreads();
    for (int sl = threadIdx.x; sl < SR; sl += blockDim.x) {
      const int dz = sl % WR - wR, dy = (sl / WR) % WR - wR, dx = sl / (WR * WR) - wR;
      const int jx = x + dx, jy = y + dy, jz = z + dz;
      double acc = 0.0;
      if (inside3(jx, jy, jz, L)) {
        const long long j = flat3(jx, jy, jz, L);
        // b in box(i, wX) and ball(j, rho), ascending
        const int b0x = imax(imax(x - wX, jx - rho), 0), b1x = imin(imin(x + wX, jx + rho), L - 1);
        const int b0y = imax(imax(y - wX, jy - rho), 0), b1y = imin(imin(y + wX, jy + rho), L - 1);
        const int b0z = imax(imax(z - wX, jz - rho), 0), b1z = imin(imin(z + wX, jz + rho), L - 1);
        for (int bx = b0x; bx <= b1x; ++bx)
          for (int by = b0y; by <= b1y; ++by)
            for (int bz = b0z; bz <= b1z; ++bz) {
              const double xv = xs[((bx - x + wX) * WX + (by - y + wX)) * WX + (bz - z + wX)];
              acc += xv * psi_at(psi, j, L, -rho, wd, jx, jy, jz, bx, by, bz);
            }
      }
      raw[i * SR + sl] = acc;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K3 B = W A W^T, G = W A pibar^T, P A P^T (gamblet_fast.py:520-544, 597-601)
// on the parent grid (Lp = Lk / 2), one thread per (p, q = p + d), |d| <= wB
// ---------------------------------------------------------------------------
__global__ void k3_level_blocks(int Lk, int wA, const double* __restrict__ A, W7x8 W, int wB,
                                double* __restrict__ Braw, double* __restrict__ G,
                                double* __restrict__ PAPt) {
  const int Lp = Lk / 2;
  const long long P = (long long)Lp * Lp * Lp;
  const int WB = 2 * wB + 1;
  const long long SBp = (long long)WB * WB * WB;
  const long long SA = slots3(wA, 1);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P * SBp;
       e += (long long)gridDim.x * blockDim.x) {
    const long long p = e / SBp;
    const int sl = (int)(e - p * SBp);
    const int dz = sl % WB - wB, dy = (sl / WB) % WB - wB, dx = sl / (WB * WB) - wB;
    int px, py, pz;
    unflat3(p, Lp, &px, &py, &pz);
    const int qx = px + dx, qy = py + dy, qz = pz + dz;
    double Xr[7][8], pa[8];
#pragma unroll
    for (int c = 0; c < 7; ++c)
#pragma unroll
      for (int b = 0; b < 8; ++b) Xr[c][b] = 0.0;
#pragma unroll
    for (int b = 0; b < 8; ++b) pa[b] = 0.0;
    const bool in = inside3(qx, qy, qz, Lp);
    if (in) {
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int ax = 2 * px + (a >> 2), ay = 2 * py + ((a >> 1) & 1), az = 2 * pz + (a & 1);
        const long long ra = flat3(ax, ay, az, Lk);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const int bx = 2 * qx + (b >> 2), by = 2 * qy + ((b >> 1) & 1), bz = 2 * qz + (b & 1);
          const int ex = bx - ax, ey = by - ay, ez = bz - az;
          double av = 0.0;
          if (abs(ex) <= wA && abs(ey) <= wA && abs(ez) <= wA)
            av = A[ra * SA + slot3(wA, 1, ex, ey, ez, 0)];
          // X = W A: sum over a ascending (children of p); P A likewise
#pragma unroll
          for (int c = 0; c < 7; ++c) Xr[c][b] += W.w[c][a] * av;
          pa[b] += av;
        }
      }
    }
    const long long SB = (long long)WB * WB * WB * 7;
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      double g = 0.0;
#pragma unroll
      for (int b = 0; b < 8; ++b) g += Xr[c][b] * 0.125;
      G[(p * 7 + c) * SBp + sl] = in ? g : 0.0;
#pragma unroll
      for (int cp = 0; cp < 7; ++cp) {
        double bv = 0.0;
#pragma unroll
        for (int b = 0; b < 8; ++b) bv += Xr[c][b] * W.w[cp][b];
        Braw[(p * 7 + c) * SB + (long long)sl * 7 + cp] = in ? bv : 0.0;
      }
    }
    double pp = 0.0;
#pragma unroll
    for (int b = 0; b < 8; ++b) pp += pa[b];
    PAPt[p * SBp + sl] = in ? pp : 0.0;
  }
}

// ---------------------------------------------------------------------------
// K4 correction patches (gamblet_fast.py:546-591): per coarse parent i, the
// dense (S B S)[chi, chi] (m <= 7 (2 rho + 1)^3 = 875) in a global-memory
// workspace slot of the CTA, blocked right-looking Cholesky (64-column
// panels: diagonal block in shared memory, warp-per-row TRSM, trailing update
// on the FP64 tensor cores, DMMA m8n8k4), the right-hand side s (-G)[chi, i]
// carried through the panels, back substitution, D^T row i = s z with the
// 1e-11 row-tail trim.  One launch per level, CTAs stride over the parents.
// ---------------------------------------------------------------------------
constexpr int k3PB = 64;    // panel width
constexpr int k3TLD = 68;   // leading dimension of the staged operand blocks (4 mod 16)

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// 16-byte global -> shared copy (LDGSTS, L2 only) and its completion wait
__device__ __forceinline__ void k3_cp16(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void k3_cp_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// stage the 64 x 64 block K[row0 + rr][j0 + kk] (rr, kk < 64) row-major into
// dst[rr * k3TLD + kk], zero beyond row m / column jb; asynchronous 16-byte
// copies (ld and j0 are even, so every pair is aligned) -- the caller waits
// (k3_cp_wait) before its barrier
__device__ __forceinline__ void k3_stage(double* dst, const double* __restrict__ K, int ld,
                                         int row0, int j0, int jb, int m, int tid) {
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int c = tid + 256 * u;
    const int rr = c >> 5, kc = (c & 31) << 1;
    double* d = dst + rr * k3TLD + kc;
    const double* src = K + (long long)(row0 + rr) * ld + j0 + kc;
    if (row0 + rr < m && kc + 2 <= jb) {
      k3_cp16(d, src);
    } else {
      const bool r = row0 + rr < m;
      d[0] = (r && kc < jb) ? src[0] : 0.0;
      d[1] = (r && kc + 1 < jb) ? src[1] : 0.0;
    }
  }
}

// one 64 x 64 x jb block product on the FP64 tensor cores: acc[ii][jj] of
// warp (wm, wn) += A[wm 32 + 8 ii + ., k] B[wn 16 + 8 jj + ., k] over k < jb,
// both operands row-major (row, k) with leading dimension k3TLD
__device__ __forceinline__ void k3_block_mma(const double* __restrict__ As,
                                             const double* __restrict__ Bs, int jb, int wm,
                                             int wn, int fr, int fk, double acc[4][2][2]) {
  const double* ap = As + (wm * 32 + fr) * k3TLD + fk;
  const double* bp = Bs + (wn * 16 + fr) * k3TLD + fk;
  for (int k4 = 0; k4 < jb; k4 += 4) {
    double af[4], bf[2];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) af[ii] = ap[ii * 8 * k3TLD + k4];
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) bf[jj] = bp[jj * 8 * k3TLD + k4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) dmma_884(acc[ii][jj][0], acc[ii][jj][1], af[ii], bf[jj]);
  }
}

__global__ void __launch_bounds__(256, 2) k3_correction_patches(
    int Lp, int wB, const double* __restrict__ B, const double* __restrict__ sB,
    const double* __restrict__ G, int rho, double* __restrict__ Dt, long long* status,
    double* __restrict__ ws, int ld) {
  extern __shared__ __align__(16) double dsm3[];
  // region 0 (64 x k3TLD doubles): the diagonal block D11 (64 x 65), y1 and
  // dinv behind it -- free during the trailing update, where it is the second
  // B-operand buffer
  double (*D11)[k3PB + 1] = reinterpret_cast<double (*)[k3PB + 1]>(dsm3);  // 64 x 65
  double* y1 = dsm3 + k3PB * (k3PB + 1);                                 // 64
  double* dinv = y1 + k3PB;                                              // 64: 1 / L_jj
  double* Bs2 = dsm3;                                                    // alias of region 0
  double* As = dsm3 + k3PB * k3TLD;                                      // 64 x k3TLD
  double* Bs = As + k3PB * k3TLD;                                        // 64 x k3TLD
  __shared__ int bx0, by0, bz0, nx, ny, nz, bad;
  __shared__ double sh[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long P = (long long)Lp * Lp * Lp;
  const int WB = 2 * wB + 1;
  const long long SB = (long long)WB * WB * WB * 7, SG = (long long)WB * WB * WB;
  const int R = 2 * rho + 1;
  const long long SD = (long long)R * R * R * 7;
  double* K = ws + (long long)blockIdx.x * ((long long)ld * ld + ld);
  double* v = K + (long long)ld * ld;
  for (long long i = blockIdx.x; i < P; i += gridDim.x) {
    int x, y, z;
    unflat3(i, Lp, &x, &y, &z);
    if (tid == 0) {
      bx0 = imax(x - rho, 0);
      by0 = imax(y - rho, 0);
      bz0 = imax(z - rho, 0);
      nx = imin(x + rho, Lp - 1) - bx0 + 1;
      ny = imin(y + rho, Lp - 1) - by0 + 1;
      nz = imin(z + rho, Lp - 1) - bz0 + 1;
      bad = 0;
    }
    __syncthreads();
    const int m = nx * ny * nz * 7;
    // gather (lower triangle and diagonal; row-major, ld): one thread per
    // (parent a, parent b <= a) pair, the 7 x 7 component block inside (the
    // 7 columns of a B row for fixed (a, c_a) are contiguous)
    const int np = nx * ny * nz;
    for (long long e = tid; e < (long long)np * np; e += blockDim.x) {
      const int pa = (int)(e / np), pb = (int)(e - (long long)pa * np);
      if (pb > pa) continue;
      const int az = pa % nz, ay = (pa / nz) % ny, ax = pa / (nz * ny);
      const int bz = pb % nz, by = (pb / nz) % ny, bxx = pb / (nz * ny);
      const int dx = bxx - ax, dy = by - ay, dz = bz - az;
      const bool in = abs(dx) <= wB && abs(dy) <= wB && abs(dz) <= wB;
      const long long qa = flat3(bx0 + ax, by0 + ay, bz0 + az, Lp);
      const long long qb = flat3(bx0 + bxx, by0 + by, bz0 + bz, Lp);
      const int sl = in ? slot3(wB, 7, dx, dy, dz, 0) : 0;
      double sb[7];
#pragma unroll
      for (int cb = 0; cb < 7; ++cb) sb[cb] = sB[qb * 7 + cb];
#pragma unroll
      for (int ca = 0; ca < 7; ++ca) {
        const long long ra = qa * 7 + ca;
        const double sa = sB[ra];
        double* krow = K + (long long)(7 * pa + ca) * ld + 7 * pb;
        const double* brow = B + ra * SB + sl;
#pragma unroll
        for (int cb = 0; cb < 7; ++cb) {
          if (pb == pa && cb > ca) break;
          krow[cb] = in ? (brow[cb] * sa) * sb[cb] : 0.0;
        }
      }
    }
    for (int a = tid; a < m; a += blockDim.x) {
      const int pa = a / 7, ca = a - 7 * pa;
      const int az = pa % nz, ay = (pa / nz) % ny, ax = pa / (nz * ny);
      const int px = bx0 + ax, py = by0 + ay, pz = bz0 + az;
      const long long ra = flat3(px, py, pz, Lp) * 7 + ca;
      double g = 0.0;
      const int dx = x - px, dy = y - py, dz = z - pz;
      if (abs(dx) <= wB && abs(dy) <= wB && abs(dz) <= wB)
        g = G[ra * SG + slot3(wB, 1, dx, dy, dz, 0)];
      v[a] = sB[ra] * (-g);
    }
    __syncthreads();
    for (int j0 = 0; j0 < m; j0 += k3PB) {
      const int jb = imin(k3PB, m - j0);
      // (a) diagonal block: factor in shared memory (warp 0), carry the rhs
      for (int e = tid; e < jb * jb; e += blockDim.x) {
        const int a = e / jb, b = e - a * jb;
        D11[a][b] = b <= a ? K[(long long)(j0 + a) * ld + j0 + b] : 0.0;
      }
      if (tid < jb) y1[tid] = v[j0 + tid];
      __syncthreads();
      // right-looking over the block's columns, all warps: column scale,
      // then the rank-1 update of the trailing triangle (pairs over threads)
      for (int j = 0; j < jb; ++j) {
        const double d = D11[j][j];
        if (!(d > 0.0)) {
          if (tid == 0) bad = 1;
          break;  // uniform: every thread read the same pivot
        }
        const double l = sqrt(d);
        const double il = 1.0 / l;
        __syncthreads();
        if (tid == 0) {
          D11[j][j] = l;
          dinv[j] = il;
        }
        for (int a = j + 1 + tid; a < jb; a += blockDim.x) D11[a][j] *= il;
        __syncthreads();
        // rank-1 update of the trailing triangle: thread (ty, tx) of a 16 x 16
        // grid owns the entries (a, b) = (ty + 16 i, tx + 16 i2), b <= a
        {
          const int ty = tid >> 4, tx = tid & 15;
          double ca[4], cb[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            ca[i] = D11[ty + 16 * i][j];
            cb[i] = D11[tx + 16 * i][j];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int a = ty + 16 * i;
            if (a <= j || a >= jb) continue;
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) {
              const int b = tx + 16 * i2;
              if (b > j && b <= a) D11[a][b] -= ca[i] * cb[i2];
            }
          }
        }
        __syncthreads();
      }
      __syncthreads();
      if (bad) break;
      if (warp == 0) {
        for (int j = 0; j < jb; ++j) {  // y1 = L11^-1 v1
          if (lane == 0) y1[j] *= dinv[j];
          __syncwarp();
          for (int a = j + 1 + lane; a < jb; a += 32) y1[a] -= D11[a][j] * y1[j];
          __syncwarp();
        }
      }
      __syncthreads();
      for (int e = tid; e < jb * jb; e += blockDim.x) {
        const int a = e / jb, b = e - a * jb;
        if (b <= a) K[(long long)(j0 + a) * ld + j0 + b] = D11[a][b];
      }
      if (tid < jb) v[j0 + tid] = y1[tid];
      const int r0 = j0 + jb;
      // (b) panel rows below: L21 = A21 L11^-T as a DMMA GEMM with the
      // explicit inverse T = L11^-1 (4 threads per column, forward
      // substitution), then v[r] -= L21[r, :] y1
      {
        double* T = Bs;  // T[c][k] stored as Bs[k * k3TLD + c] (the GEMM's B)
        for (int e = tid; e < k3PB * k3TLD; e += blockDim.x) T[e] = 0.0;
        __syncthreads();
        // column col = tid / 4 (8 per warp), its 4 threads split the sums;
        // every lane of a warp runs the same i range so the shuffles converge:
        // x_i = (delta_ic - sum_{col <= k < i} L_ik x_k) / L_ii for i >= col
        const int col = tid >> 2, q4 = tid & 3;
        for (int i = 8 * warp; i < jb; ++i) {
          const bool act = col < jb && col <= i;
          double part = 0.0;
          if (act)
            for (int k = col + q4; k < i; k += 4) part += D11[i][k] * T[k * k3TLD + col];
          part += __shfl_xor_sync(0xffffffffu, part, 1);
          part += __shfl_xor_sync(0xffffffffu, part, 2);
          if (act && q4 == 0) T[i * k3TLD + col] = ((i == col ? 1.0 : 0.0) - part) * dinv[i];
          __syncwarp();
        }
        __syncthreads();
        // T holds (row i, column c) of L11^-1 at T[i * TLD + c]; the GEMM's B
        // operand is B[k][n] = T[n][k] (L21[r][n] = sum_k A21[r][k] T[n][k])
        const int wm = warp >> 2, wn = warp & 3, fr = lane >> 2, fk = lane & 3;
        for (int rb = r0; rb < m; rb += 64) {
          k3_stage(As, K, ld, rb, j0, jb, m, tid);
          k3_cp_wait();
          __syncthreads();
          double acc[4][2][2];
#pragma unroll
          for (int ii = 0; ii < 4; ++ii)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) acc[ii][jj][0] = acc[ii][jj][1] = 0.0;
          k3_block_mma(As, T, jb, wm, wn, fr, fk, acc);
          __syncthreads();  // As is reused by the next row block
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const int gr = rb + wm * 32 + ii * 8 + fr;
            if (gr >= m) continue;
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
              for (int e2 = 0; e2 < 2; ++e2) {
                const int gc = wn * 16 + jj * 8 + 2 * fk + e2;
                if (gc < jb) K[(long long)gr * ld + j0 + gc] = acc[ii][jj][e2];
              }
          }
        }
        __syncthreads();
        for (int r = r0 + warp; r < m; r += 8) {
          const double* ar = K + (long long)r * ld + j0;
          double t = (lane < jb ? ar[lane] * y1[lane] : 0.0) +
                     (lane + 32 < jb ? ar[lane + 32] * y1[lane + 32] : 0.0);
          t = warp_sum(t);
          if (lane == 0) v[r] -= t;
        }
        __syncthreads();
      }
      // (c) trailing update K22 -= L21 L21^T (lower), 64 x 64 output blocks:
      // the row block of L21 (A operand) staged once per block row, the
      // column blocks (B operand) streamed through two buffers (the next one
      // copied asynchronously while the current one is multiplied); warp
      // (wm, wn) of a 2 x 4 grid owns 32 x 16 = 4 x 2 DMMA m8n8k4
      // accumulators.  The K entries a thread updates are loaded before its
      // products, so their latency overlaps the tensor-core work.
      const int nbk = (m - r0 + 63) / 64;
      const int wm = warp >> 2, wn = warp & 3, fr = lane >> 2, fk = lane & 3;
      for (int bi = 0; bi < nbk; ++bi) {
        const int ib = r0 + bi * 64;
        __syncthreads();  // every warp is done with the buffers of block row bi - 1
        k3_stage(As, K, ld, ib, j0, jb, m, tid);
        if (bi > 0) k3_stage(Bs, K, ld, r0, j0, jb, m, tid);  // column block 0
        for (int bj = 0; bj <= bi; ++bj) {
          const int jbase = r0 + bj * 64;
          const double* Bc = bj == bi ? As : ((bj & 1) ? Bs2 : Bs);
          k3_cp_wait();
          __syncthreads();  // block bj (and As) landed; buffer (bj + 1) & 1 is free
          if (bj + 1 < bi) k3_stage((bj & 1) ? Bs : Bs2, K, ld, jbase + 64, j0, jb, m, tid);
          double kold[4][2][2];
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const int gr = ib + wm * 32 + ii * 8 + fr;
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const int gc = jbase + wn * 16 + jj * 8 + 2 * fk;
#pragma unroll
              for (int e2 = 0; e2 < 2; ++e2)
                kold[ii][jj][e2] = (gr < m && gc + e2 < m && gc + e2 <= gr)
                                       ? __ldcg(K + (long long)gr * ld + gc + e2)
                                       : 0.0;
            }
          }
          double acc[4][2][2];
#pragma unroll
          for (int ii = 0; ii < 4; ++ii)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) acc[ii][jj][0] = acc[ii][jj][1] = 0.0;
          k3_block_mma(As, Bc, jb, wm, wn, fr, fk, acc);
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const int gr = ib + wm * 32 + ii * 8 + fr;
            if (gr >= m) continue;
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
              for (int e2 = 0; e2 < 2; ++e2) {
                const int gc = jbase + wn * 16 + jj * 8 + 2 * fk + e2;
                if (gc < m && gc <= gr)
                  K[(long long)gr * ld + gc] = kold[ii][jj][e2] - acc[ii][jj][e2];
              }
          }
        }
      }
      __syncthreads();
    }
    if (bad) {
      if (tid == 0) raise_status(status, ST_NOT_SPD, i);
      __syncthreads();
      continue;
    }
    // back substitution L^T z = y in blocks of 64 rows (row j of L is
    // contiguous): the block's own triangle by one warp on a shared-memory
    // copy, then v[a] -= sum_j L[j][a] z_j for every a above the block (one
    // thread per a, coalesced over a, no barrier inside)
    for (int jb0 = ((m - 1) / k3PB) * k3PB; jb0 >= 0; jb0 -= k3PB) {
      const int nb = imin(k3PB, m - jb0);
      for (int e = tid; e < nb * nb; e += blockDim.x) {
        const int a = e / nb, b = e - a * nb;
        D11[a][b] = b <= a ? K[(long long)(jb0 + a) * ld + jb0 + b] : 0.0;
      }
      if (tid < nb) y1[tid] = v[jb0 + tid];
      __syncthreads();
      if (warp == 0) {
        for (int j = nb - 1; j >= 0; --j) {
          if (lane == 0) y1[j] /= D11[j][j];
          __syncwarp();
          const double zj = y1[j];
          for (int a = lane; a < j; a += 32) y1[a] -= D11[j][a] * zj;
          __syncwarp();
        }
      }
      __syncthreads();
      if (tid < nb) v[jb0 + tid] = y1[tid];
      for (int a = tid; a < jb0; a += blockDim.x) {
        double acc = 0.0;
        for (int j = nb - 1; j >= 0; --j)
          acc = fma(__ldcg(K + (long long)(jb0 + j) * ld + a), y1[j], acc);
        v[a] -= acc;
      }
      __syncthreads();
    }
    // D^T row i = s z, row-tail trim (1e-11 rowmax), box slots (ball offset, c)
    double mx = 0.0;
    for (int a = tid; a < m; a += blockDim.x) {
      const int pa = a / 7, ca = a - 7 * pa;
      const int az = pa % nz, ay = (pa / nz) % ny, ax = pa / (nz * ny);
      const long long ra = flat3(bx0 + ax, by0 + ay, bz0 + az, Lp) * 7 + ca;
      const double d = sB[ra] * v[a];
      v[a] = d;
      mx = fmax(mx, fabs(d));
    }
    mx = block_max(mx, sh);
    double* row = Dt + i * SD;
    for (long long e = tid; e < SD; e += blockDim.x) {
      const int c = (int)(e % 7);
      const int t = (int)(e / 7);
      const int oz = t % R - rho, oy = (t / R) % R - rho, ox = t / (R * R) - rho;
      const int ax = x + ox - bx0, ay = y + oy - by0, az = z + oz - bz0;
      double d = 0.0;
      if (ax >= 0 && ax < nx && ay >= 0 && ay < ny && az >= 0 && az < nz) {
        d = v[((ax * ny + ay) * nz + az) * 7 + c];
        if (fabs(d) < 1e-11 * mx) d = 0.0;
      }
      row[e] = d;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K6 R = pibar + D^T W (gamblet_fast.py:581-591); rows: parents, columns: the
// 8 children of each ball member (slot (d, child))
// ---------------------------------------------------------------------------
__global__ void k3_restriction(int Lp, int rho, const double* __restrict__ Dt, W7x8 W,
                               double* __restrict__ Rv) {
  const long long P = (long long)Lp * Lp * Lp;
  const int R = 2 * rho + 1;
  const long long SR = (long long)R * R * R * 8, SD = (long long)R * R * R * 7;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P * SR;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / SR;
    const int sl = (int)(e - i * SR);
    const int j = sl & 7, t = sl >> 3;
    const int oz = t % R - rho, oy = (t / R) % R - rho, ox = t / (R * R) - rho;
    int x, y, z;
    unflat3(i, Lp, &x, &y, &z);
    double v = 0.0;
    if (inside3(x + ox, y + oy, z + oz, Lp)) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < 7; ++c) acc += Dt[i * SD + (long long)t * 7 + c] * W.w[c][j];
      v = (ox == 0 && oy == 0 && oz == 0) ? 0.125 + acc : acc;
    }
    Rv[e] = v;
  }
}

// ---------------------------------------------------------------------------
// K6 split triple product A^(k-1) = P A P^T / 64 + G^T D + D^T G + D^T B D
// (gamblet_fast.py:593-613); D[(q, c), j] = Dt[j, (q - j, c)] for |q - j| <= rho
// ---------------------------------------------------------------------------
// BD[(p, c), j], |j - p| <= wBD: sum over (q, c') of row (p, c) of B, ascending
__global__ void k3_bd(int Lp, int wB, const double* __restrict__ B, int rho,
                      const double* __restrict__ Dt, int wBD, double* __restrict__ BD) {
  const long long P = (long long)Lp * Lp * Lp;
  const int W = 2 * wBD + 1, R = 2 * rho + 1;
  const long long S = (long long)W * W * W;
  const long long SB = slots3(wB, 7), SD = (long long)R * R * R * 7;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P * 7 * S;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / S;
    const int sl = (int)(e - r * S);
    const long long p = r / 7;
    const int dz = sl % W - wBD, dy = (sl / W) % W - wBD, dx = sl / (W * W) - wBD;
    int px, py, pz;
    unflat3(p, Lp, &px, &py, &pz);
    const int jx = px + dx, jy = py + dy, jz = pz + dz;
    double acc = 0.0;
    if (inside3(jx, jy, jz, Lp)) {
      const long long j = flat3(jx, jy, jz, Lp);
      const int q0x = imax(imax(px - wB, jx - rho), 0), q1x = imin(imin(px + wB, jx + rho), Lp - 1);
      const int q0y = imax(imax(py - wB, jy - rho), 0), q1y = imin(imin(py + wB, jy + rho), Lp - 1);
      const int q0z = imax(imax(pz - wB, jz - rho), 0), q1z = imin(imin(pz + wB, jz + rho), Lp - 1);
      const double* brow = B + r * SB;
      const double* drow = Dt + j * SD;
      for (int qx = q0x; qx <= q1x; ++qx)
        for (int qy = q0y; qy <= q1y; ++qy)
          for (int qz = q0z; qz <= q1z; ++qz) {
            const int bs = slot3(wB, 7, qx - px, qy - py, qz - pz, 0);
            const int ds = slot3(rho, 7, qx - jx, qy - jy, qz - jz, 0);
#pragma unroll
            for (int c = 0; c < 7; ++c) acc += brow[bs + c] * drow[ds + c];
          }
    }
    BD[e] = acc;
  }
}

// The same BD, register tiled: a thread forms the 7 component rows of parent
// p against a run of K3_JZ consecutive column offsets along z, so a 7 x 7
// block of B serves K3_JZ columns and a 7-vector of D serves 7 rows (0.4
// loads per FMA instead of 2).  Every output is still the sequential chain
// over q ascending, c ascending from 0.0 -- bitwise the per-entry kernel.
#ifndef GB_K3_JZ
#define GB_K3_JZ 3
#endif
#ifndef GB_K3_C2U
#define GB_K3_C2U 7
#endif
constexpr int K3_JZ = GB_K3_JZ, K3_C2U = GB_K3_C2U;
__global__ void __launch_bounds__(128) k3_bd_tiled(int Lp, int wB, const double* __restrict__ B,
                                                   int rho, const double* __restrict__ Dt,
                                                   int wBD, double* __restrict__ BD) {
  const long long P = (long long)Lp * Lp * Lp;
  const int W = 2 * wBD + 1, R = 2 * rho + 1;
  const int NG = (W + K3_JZ - 1) / K3_JZ;
  const long long S = (long long)W * W * W;
  const long long SB = slots3(wB, 7), SD = (long long)R * R * R * 7;
  const long long per = (long long)W * W * NG;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P * per;
       e += (long long)gridDim.x * blockDim.x) {
    const long long p = e / per;
    const int it = (int)(e - p * per);
    const int g = it % NG, dy = (it / NG) % W - wBD, dx = it / (NG * W) - wBD;
    const int dz0 = g * K3_JZ - wBD;
    const int nz = imin(K3_JZ, wBD - dz0 + 1);  // columns of this run inside the box
    int px, py, pz;
    unflat3(p, Lp, &px, &py, &pz);
    const int jx = px + dx, jy = py + dy, jz0 = pz + dz0;
    double acc[7][K3_JZ];
#pragma unroll
    for (int c = 0; c < 7; ++c)
#pragma unroll
      for (int u = 0; u < K3_JZ; ++u) acc[c][u] = 0.0;
    if ((unsigned)jx < (unsigned)Lp && (unsigned)jy < (unsigned)Lp) {
      const int q0x = imax(imax(px - wB, jx - rho), 0), q1x = imin(imin(px + wB, jx + rho), Lp - 1);
      const int q0y = imax(imax(py - wB, jy - rho), 0), q1y = imin(imin(py + wB, jy + rho), Lp - 1);
      const int q0z = imax(imax(pz - wB, jz0 - rho), 0);
      const int q1z = imin(imin(pz + wB, jz0 + nz - 1 + rho), Lp - 1);
      const double* brow = B + p * 7 * SB;
      for (int qx = q0x; qx <= q1x; ++qx)
        for (int qy = q0y; qy <= q1y; ++qy) {
          // column j = (jx, jy, jz0 + u): Dt row and the slot of (qx, qy, .)
          const long long jrow = flat3(jx, jy, 0, Lp);
          const int dxy = ((qx - jx + rho) * R + (qy - jy + rho)) * R;
          for (int qz = q0z; qz <= q1z; ++qz) {
            const int bs = slot3(wB, 7, qx - px, qy - py, qz - pz, 0);
            bool on[K3_JZ];
            const double* dp[K3_JZ];
#pragma unroll
            for (int u = 0; u < K3_JZ; ++u) {
              const int jz = jz0 + u;
              const int dzq = qz - jz;
              on[u] = u < nz && (unsigned)jz < (unsigned)Lp && dzq >= -rho && dzq <= rho;
              dp[u] = Dt + (jrow + jz) * SD + (long long)(dxy + dzq + rho) * 7;
            }
#pragma unroll K3_C2U
            for (int c2 = 0; c2 < 7; ++c2) {
              double dv[K3_JZ];
#pragma unroll
              for (int u = 0; u < K3_JZ; ++u) dv[u] = on[u] ? dp[u][c2] : 0.0;
#pragma unroll
              for (int c = 0; c < 7; ++c) {
                const double b = brow[c * SB + bs + c2];
#pragma unroll
                for (int u = 0; u < K3_JZ; ++u)
                  if (on[u]) acc[c][u] += b * dv[u];
              }
            }
          }
        }
    }
    const long long sl0 = ((long long)(dx + wBD) * W + (dy + wBD)) * W + (dz0 + wBD);
#pragma unroll
    for (int c = 0; c < 7; ++c)
#pragma unroll
      for (int u = 0; u < K3_JZ; ++u)
        if (u < nz) BD[(p * 7 + c) * S + sl0 + u] = acc[c][u];
  }
}

// GtD[i, j], |j - i| <= wGD: sum over (p, c) ascending with G[(p,c), i] and
// D[(p,c), j] both in their boxes
__global__ void k3_gtd(int Lp, int wG, const double* __restrict__ G, int rho,
                       const double* __restrict__ Dt, int wGD, double* __restrict__ GtD) {
  const long long P = (long long)Lp * Lp * Lp;
  const int W = 2 * wGD + 1, R = 2 * rho + 1;
  const long long S = (long long)W * W * W;
  const long long SG = slots3(wG, 1), SD = (long long)R * R * R * 7;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P * S;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / S;
    const int sl = (int)(e - i * S);
    const int dz = sl % W - wGD, dy = (sl / W) % W - wGD, dx = sl / (W * W) - wGD;
    int x, y, z;
    unflat3(i, Lp, &x, &y, &z);
    const int jx = x + dx, jy = y + dy, jz = z + dz;
    double acc = 0.0;
    if (inside3(jx, jy, jz, Lp)) {
      const long long j = flat3(jx, jy, jz, Lp);
      const int p0x = imax(imax(x - wG, jx - rho), 0), p1x = imin(imin(x + wG, jx + rho), Lp - 1);
      const int p0y = imax(imax(y - wG, jy - rho), 0), p1y = imin(imin(y + wG, jy + rho), Lp - 1);
      const int p0z = imax(imax(z - wG, jz - rho), 0), p1z = imin(imin(z + wG, jz + rho), Lp - 1);
      const double* drow = Dt + j * SD;
      for (int px = p0x; px <= p1x; ++px)
        for (int py = p0y; py <= p1y; ++py)
          for (int pz = p0z; pz <= p1z; ++pz) {
            const long long pr = flat3(px, py, pz, Lp) * 7;
            const int gs = slot3(wG, 1, x - px, y - py, z - pz, 0);
            const int ds = slot3(rho, 7, px - jx, py - jy, pz - jz, 0);
#pragma unroll
            for (int c = 0; c < 7; ++c) acc += G[(pr + c) * SG + gs] * drow[ds + c];
          }
    }
    GtD[e] = acc;
  }
}

// The same GtD enumerated by column: a thread takes (j, d) and forms entry
// (i = j - d, j).  A warp then shares the D row of j (broadcast loads) and its
// G reads of row (p, c) at the consecutive columns i run through consecutive
// slots (coalesced); the per-entry kernel walked a private D row per lane.
// Same sum per entry (p ascending, c ascending, from 0.0).  Entries whose
// column lies outside the grid are never visited: the caller zeroes GtD first.
__global__ void k3_gtd_bycol(int Lp, int wG, const double* __restrict__ G, int rho,
                             const double* __restrict__ Dt, int wGD, double* __restrict__ GtD) {
  const long long P = (long long)Lp * Lp * Lp;
  const int W = 2 * wGD + 1, R = 2 * rho + 1;
  const long long S = (long long)W * W * W;
  const long long SG = slots3(wG, 1), SD = (long long)R * R * R * 7;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P * S;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / S;
    const int sl = (int)(e - j * S);
    const int dz = sl % W - wGD, dy = (sl / W) % W - wGD, dx = sl / (W * W) - wGD;
    int jx, jy, jz;
    unflat3(j, Lp, &jx, &jy, &jz);
    const int x = jx - dx, y = jy - dy, z = jz - dz;
    if (!inside3(x, y, z, Lp)) continue;
    const long long i = flat3(x, y, z, Lp);
    const int p0x = imax(imax(x - wG, jx - rho), 0), p1x = imin(imin(x + wG, jx + rho), Lp - 1);
    const int p0y = imax(imax(y - wG, jy - rho), 0), p1y = imin(imin(y + wG, jy + rho), Lp - 1);
    const int p0z = imax(imax(z - wG, jz - rho), 0), p1z = imin(imin(z + wG, jz + rho), Lp - 1);
    const double* drow = Dt + j * SD;
    double acc = 0.0;
    for (int px = p0x; px <= p1x; ++px)
      for (int py = p0y; py <= p1y; ++py)
        for (int pz = p0z; pz <= p1z; ++pz) {
          const long long pr = flat3(px, py, pz, Lp) * 7;
          const int gs = slot3(wG, 1, x - px, y - py, z - pz, 0);
          const int ds = slot3(rho, 7, px - jx, py - jy, pz - jz, 0);
#pragma unroll
          for (int c = 0; c < 7; ++c) acc += G[(pr + c) * SG + gs] * drow[ds + c];
        }
    GtD[i * S + sl] = acc;
  }
}

// raw[i, j] = ((P A P^T[i,j] / 64 + GtD[i,j]) + GtD[j,i]) + (D^T B D)[i,j],
// |j - i| <= wA2; (D^T B D)[i, j] = sum over (p, c) in chi(i) ascending of
// Dt[i, (p - i, c)] BD[(p, c), j]
__global__ void k3_coarse_raw(int Lp, int wP, const double* __restrict__ PAPt, int wGD,
                              const double* __restrict__ GtD, int rho,
                              const double* __restrict__ Dt, int wBD,
                              const double* __restrict__ BD, int wA2,
                              double* __restrict__ raw) {
  const long long P = (long long)Lp * Lp * Lp;
  const int W = 2 * wA2 + 1, R = 2 * rho + 1;
  const long long S = (long long)W * W * W;
  const long long SP = slots3(wP, 1), SGD = slots3(wGD, 1), SBD = slots3(wBD, 1);
  const long long SD = (long long)R * R * R * 7;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P * S;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / S;
    const int sl = (int)(e - i * S);
    const int dz = sl % W - wA2, dy = (sl / W) % W - wA2, dx = sl / (W * W) - wA2;
    int x, y, z;
    unflat3(i, Lp, &x, &y, &z);
    const int jx = x + dx, jy = y + dy, jz = z + dz;
    double v = 0.0;
    if (inside3(jx, jy, jz, Lp)) {
      const long long j = flat3(jx, jy, jz, Lp);
      double pap = 0.0, g1 = 0.0, g2 = 0.0;
      if (abs(dx) <= wP && abs(dy) <= wP && abs(dz) <= wP)
        pap = PAPt[i * SP + slot3(wP, 1, dx, dy, dz, 0)];
      if (abs(dx) <= wGD && abs(dy) <= wGD && abs(dz) <= wGD) {
        g1 = GtD[i * SGD + slot3(wGD, 1, dx, dy, dz, 0)];
        g2 = GtD[j * SGD + slot3(wGD, 1, -dx, -dy, -dz, 0)];
      }
      double dbd = 0.0;
      const int p0x = imax(imax(x - rho, jx - wBD), 0), p1x = imin(imin(x + rho, jx + wBD), Lp - 1);
      const int p0y = imax(imax(y - rho, jy - wBD), 0), p1y = imin(imin(y + rho, jy + wBD), Lp - 1);
      const int p0z = imax(imax(z - rho, jz - wBD), 0), p1z = imin(imin(z + rho, jz + wBD), Lp - 1);
      const double* drow = Dt + i * SD;
      for (int px = p0x; px <= p1x; ++px)
        for (int py = p0y; py <= p1y; ++py)
          for (int pz = p0z; pz <= p1z; ++pz) {
            const long long pr = flat3(px, py, pz, Lp) * 7;
            const int ds = slot3(rho, 7, px - x, py - y, pz - z, 0);
            const int bs = slot3(wBD, 1, jx - px, jy - py, jz - pz, 0);
#pragma unroll
            for (int c = 0; c < 7; ++c) dbd += drow[ds + c] * BD[(pr + c) * SBD + bs];
          }
      v = ((0.015625 * pap + g1) + g2) + dbd;
    }
    raw[e] = v;
  }
}

// The same raw, a run of K3_JZ consecutive columns along z per thread: the 7
// correction entries of (i, p) are loaded once per run and the BD entries of
// the run sit side by side.  Same sums per entry as k3_coarse_raw.
__global__ void __launch_bounds__(256) k3_coarse_raw_tiled(
    int Lp, int wP, const double* __restrict__ PAPt, int wGD, const double* __restrict__ GtD,
    int rho, const double* __restrict__ Dt, int wBD, const double* __restrict__ BD, int wA2,
    double* __restrict__ raw) {
  const long long P = (long long)Lp * Lp * Lp;
  const int W = 2 * wA2 + 1, R = 2 * rho + 1;
  const int NG = (W + K3_JZ - 1) / K3_JZ;
  const long long S = (long long)W * W * W;
  const long long SP = slots3(wP, 1), SGD = slots3(wGD, 1), SBD = slots3(wBD, 1);
  const long long SD = (long long)R * R * R * 7;
  const long long per = (long long)W * W * NG;
  const int WB = 2 * wBD + 1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P * per;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / per;
    const int it = (int)(e - i * per);
    const int g = it % NG, dy = (it / NG) % W - wA2, dx = it / (NG * W) - wA2;
    const int dz0 = g * K3_JZ - wA2;
    const int nz = imin(K3_JZ, wA2 - dz0 + 1);
    int x, y, z;
    unflat3(i, Lp, &x, &y, &z);
    const int jx = x + dx, jy = y + dy, jz0 = z + dz0;
    double dbd[K3_JZ];
    bool in[K3_JZ];
#pragma unroll
    for (int u = 0; u < K3_JZ; ++u) {
      dbd[u] = 0.0;
      in[u] = u < nz && inside3(jx, jy, jz0 + u, Lp);
    }
    if ((unsigned)jx < (unsigned)Lp && (unsigned)jy < (unsigned)Lp) {
      const int p0x = imax(imax(x - rho, jx - wBD), 0), p1x = imin(imin(x + rho, jx + wBD), Lp - 1);
      const int p0y = imax(imax(y - rho, jy - wBD), 0), p1y = imin(imin(y + rho, jy + wBD), Lp - 1);
      const int p0z = imax(imax(z - rho, jz0 - wBD), 0);
      const int p1z = imin(imin(z + rho, jz0 + nz - 1 + wBD), Lp - 1);
      const double* drow = Dt + i * SD;
      for (int px = p0x; px <= p1x; ++px)
        for (int py = p0y; py <= p1y; ++py) {
          const int bxy = ((jx - px + wBD) * WB + (jy - py + wBD)) * WB;
          for (int pz = p0z; pz <= p1z; ++pz) {
            const long long pr = flat3(px, py, pz, Lp) * 7;
            const int ds = slot3(rho, 7, px - x, py - y, pz - z, 0);
            const int bz0 = jz0 - pz + wBD;  // slot of u = 0 along z
            bool on[K3_JZ];
#pragma unroll
            for (int u = 0; u < K3_JZ; ++u) on[u] = in[u] && (unsigned)(bz0 + u) < (unsigned)WB;
#pragma unroll
            for (int c = 0; c < 7; ++c) {
              const double d = drow[ds + c];
              const double* bp = BD + (pr + c) * SBD + bxy + bz0;
#pragma unroll
              for (int u = 0; u < K3_JZ; ++u)
                if (on[u]) dbd[u] += d * bp[u];
            }
          }
        }
    }
#pragma unroll
    for (int u = 0; u < K3_JZ; ++u) {
      if (u >= nz) continue;
      const int dz = dz0 + u;
      double v = 0.0;
      if (in[u]) {
        const long long j = flat3(jx, jy, jz0 + u, Lp);
        double pap = 0.0, g1 = 0.0, g2 = 0.0;
        if (abs(dx) <= wP && abs(dy) <= wP && abs(dz) <= wP)
          pap = PAPt[i * SP + slot3(wP, 1, dx, dy, dz, 0)];
        if (abs(dx) <= wGD && abs(dy) <= wGD && abs(dz) <= wGD) {
          g1 = GtD[i * SGD + slot3(wGD, 1, dx, dy, dz, 0)];
          g2 = GtD[j * SGD + slot3(wGD, 1, -dx, -dy, -dz, 0)];
        }
        v = ((0.015625 * pap + g1) + g2) + dbd[u];
      }
      raw[i * S + ((long long)(dx + wA2) * W + (dy + wA2)) * W + (dz + wA2)] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// solve-phase transfers (gamblet_fast.py:717-765): rhs = s (W g), v = W^T w,
// g' = R g, and the prolongation u_k = R^T u_(k-1) of the increments
// ---------------------------------------------------------------------------
__global__ void k3_apply_w(int Lp, W7x8 W, const double* __restrict__ g,
                           const double* __restrict__ s, double* __restrict__ out) {
  const long long P = (long long)Lp * Lp * Lp;
  const int Lk = 2 * Lp;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P * 7;
       e += (long long)gridDim.x * blockDim.x) {
    const long long p = e / 7;
    const int c = (int)(e - p * 7);
    int x, y, z;
    unflat3(p, Lp, &x, &y, &z);
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 8; ++a)
      acc += W.w[c][a] * g[flat3(2 * x + (a >> 2), 2 * y + ((a >> 1) & 1), 2 * z + (a & 1), Lk)];
    out[e] = s ? s[e] * acc : acc;
  }
}

__global__ void k3_apply_wt(int Lp, W7x8 W, const double* __restrict__ w,
                            double* __restrict__ v) {
  const int Lk = 2 * Lp;
  const long long N = (long long)Lk * Lk * Lk;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N;
       e += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    unflat3(e, Lk, &x, &y, &z);
    const long long p = flat3(x >> 1, y >> 1, z >> 1, Lp);
    const int a = ((x & 1) << 2) | ((y & 1) << 1) | (z & 1);
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 7; ++c) acc += W.w[c][a] * w[p * 7 + c];
    v[e] = acc;
  }
}

// out[i] = sum over the row of R (ball members' children) of R[i, b] g[b]
__global__ void k3_apply_r(int Lp, int rho, const double* __restrict__ Rv,
                           const double* __restrict__ g, double* __restrict__ out) {
  const long long P = (long long)Lp * Lp * Lp;
  const int R = 2 * rho + 1, Lk = 2 * Lp;
  const long long SR = (long long)R * R * R * 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P;
       i += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    unflat3(i, Lp, &x, &y, &z);
    double acc = 0.0;
    for (int t = 0; t < R * R * R; ++t) {
      const int oz = t % R - rho, oy = (t / R) % R - rho, ox = t / (R * R) - rho;
      const int qx = x + ox, qy = y + oy, qz = z + oz;
      if (!inside3(qx, qy, qz, Lp)) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        acc += Rv[i * SR + t * 8 + j] *
               g[flat3(2 * qx + (j >> 2), 2 * qy + ((j >> 1) & 1), 2 * qz + (j & 1), Lk)];
    }
    out[i] = acc;
  }
}

// u_fine[b] = sum over parents i whose R row reaches b of R[i, b] u[i]
// (gather form of R^T u: b's parent p, ball members i = p - d)
__global__ void k3_apply_rt(int Lp, int rho, const double* __restrict__ Rv,
                            const double* __restrict__ u, double* __restrict__ out) {
  const int R = 2 * rho + 1, Lk = 2 * Lp;
  const long long N = (long long)Lk * Lk * Lk;
  const long long SR = (long long)R * R * R * 8;
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < N;
       b += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    unflat3(b, Lk, &x, &y, &z);
    const int px = x >> 1, py = y >> 1, pz = z >> 1;
    const int j = ((x & 1) << 2) | ((y & 1) << 1) | (z & 1);
    double acc = 0.0;
    for (int ix = imax(px - rho, 0); ix <= imin(px + rho, Lp - 1); ++ix)
      for (int iy = imax(py - rho, 0); iy <= imin(py + rho, Lp - 1); ++iy)
        for (int iz = imax(pz - rho, 0); iz <= imin(pz + rho, Lp - 1); ++iz) {
          const long long i = flat3(ix, iy, iz, Lp);
          const int t = ((px - ix + rho) * R + (py - iy + rho)) * R + (pz - iz + rho);
          acc += Rv[i * SR + t * 8 + j] * u[i];
        }
    out[b] = acc;
  }
}

// g^(q) = psi^(q) b (measured moments) and u = psi^(q)^T v (fine nodes)
__global__ void k3_psi_t_apply(int L, int rho, int wd, const double* __restrict__ psi,
                               const double* __restrict__ v, double* __restrict__ out) {
  const long long N = (long long)L * L * L;
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < N;
       b += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    unflat3(b, L, &x, &y, &z);
    double acc = 0.0;
    // rows i whose window contains b: |i - b| <= rho (ball), ascending i
    for (int ix = imax(x - rho, 0); ix <= imin(x + rho, L - 1); ++ix)
      for (int iy = imax(y - rho, 0); iy <= imin(y + rho, L - 1); ++iy)
        for (int iz = imax(z - rho, 0); iz <= imin(z + rho, L - 1); ++iz) {
          const long long i = flat3(ix, iy, iz, L);
          acc += psi_at(psi, i, L, -rho, wd, ix, iy, iz, x, y, z) * v[i];
        }
    out[b] = acc;
  }
}

}  // namespace gb

using namespace gb;

int g_k3_tiled = 1;  // gb_tune(6): 0 = per-entry 3-D product kernels (cross-check)

static inline int grid3(long long work, int block) {
  const long long g = (work + block - 1) / block;
  return (int)(g < 148LL * 32 ? (g > 0 ? g : 1) : 148LL * 32);
}

static W7x8 w7x8(const double* host_w) {
  W7x8 W;
  for (int c = 0; c < 7; ++c)
    for (int a = 0; a < 8; ++a) W.w[c][a] = host_w[c * 8 + a];
  return W;
}

int gbk3_csr_to_box(int L, int w, const int32_t* indptr, const int32_t* indices,
                    const double* data, double* box, long long* status, cudaStream_t s) {
  const long long n = (long long)L * L * L;
  cudaError_t e = cudaMemsetAsync(box, 0, (size_t)n * slots3(w, 1) * sizeof(double), s);
  if (e != cudaSuccess) return (int)e;
  k3_csr_to_box<<<grid3(n, 256), 256, 0, s>>>(L, w, indptr, indices, data, box, status);
  return (int)cudaGetLastError();
}
int gbk3_box_scale(long long rows, int nr, int w, const double* box, double* sv,
                   long long* status, cudaStream_t s) {
  k3_box_scale<<<grid3(rows, 256), 256, 0, s>>>(rows, nr, w, box, sv, status);
  return (int)cudaGetLastError();
}
int gbk3_box_sym_drop(int L, int nr, int w, const double* raw, double* out, double* dmin,
                      double* stats, cudaStream_t s) {
  const long long rows = (long long)L * L * L * nr;
  const double big = 1.0e308;
  cudaError_t e = cudaMemcpyAsync(dmin, &big, sizeof(double), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return (int)e;
  k3_box_diag_min<<<grid3(rows, 256), 256, 0, s>>>(rows, nr, w, raw, dmin);
  k3_box_sym_drop<<<grid3(rows * slots3(w, nr), 256), 256, 0, s>>>(L, nr, w, raw, out, dmin,
                                                                   stats);
  return (int)cudaGetLastError();
}
size_t gbk3_mass_smem(int rho) {
  const int m = (2 * rho + 1) * (2 * rho + 1) * (2 * rho + 1);
  return ((size_t)m * (m + 1) / 2 + m) * sizeof(double);
}
int gbk3_mass_patches(int L, const double* M, const double* sv, int rho, int wd, double* psi,
                      long long* status, cudaStream_t s) {
  const size_t smem = gbk3_mass_smem(rho);
  if (smem > 200 * 1024) return GB_UNSUPPORTED;
  cudaError_t e = cudaFuncSetAttribute(k3_mass_patches,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  const long long N = (long long)L * L * L;
  const int g = (int)(N < 148LL * 8 ? N : 148LL * 8);
  if (L < 2 * rho + 2) {  // no interior type: every patch
    k3_mass_patches<<<g, k3MassThreads, smem, s>>>(L, M, sv, rho, wd, psi, status, 0, nullptr);
    return (int)cudaGetLastError();
  }
  // the (2 rho + 1)^3 clip types when M is translation invariant (checked
  // on the device), else every patch; the flag is stream-ordered
  int* flag = nullptr;
  keep_default_pool();
  e = cudaMallocAsync((void**)&flag, sizeof(int), s);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemsetAsync(flag, 0, sizeof(int), s);
  if (e != cudaSuccess) return (int)e;
  k3_mass_invariance<<<grid3(N, 256), 256, 0, s>>>(L, M, flag);
  const int R = 2 * rho + 1;
  k3_mass_patches<<<R * R * R, k3MassThreads, smem, s>>>(L, M, sv, rho, wd, psi, status, 1,
                                                        flag);
  k3_mass_broadcast<<<grid3(N * wd * wd * wd, 256), 256, 0, s>>>(L, rho, wd, psi, flag);
  k3_mass_patches<<<g, k3MassThreads, smem, s>>>(L, M, sv, rho, wd, psi, status, 2, flag);
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  return (int)cudaFreeAsync(flag, s);
}
int gbk3_psi_galerkin(int L, int rho, int wd, const double* psi, const double* A, int wX,
                      double* X, int wR, double* raw, cudaStream_t s) {
  const long long N = (long long)L * L * L;
  k3_psi_stencil<<<grid3(N * slots3(wX, 1), 256), 256, 0, s>>>(L, rho, wd, psi, A, wX, X);
  const size_t smem = (size_t)slots3(wX, 1) * sizeof(double);
  const int g = (int)(N < 148LL * 16 ? N : 148LL * 16);
  k3_psi_galerkin<<<g, 256, smem, s>>>(L, rho, wd, psi, wX, X, wR, raw);
  return (int)cudaGetLastError();
}
int gbk3_level_blocks(int Lk, int wA, const double* A, const double* host_w, int wB,
                      double* Braw, double* G, double* PAPt, cudaStream_t s) {
  const long long Lp = Lk / 2;
  const long long work = Lp * Lp * Lp * (2 * wB + 1) * (2 * wB + 1) * (2 * wB + 1);
  k3_level_blocks<<<grid3(work, 128), 128, 0, s>>>(Lk, wA, A, w7x8(host_w), wB, Braw, G, PAPt);
  return (int)cudaGetLastError();
}
// leading dimension of a patch workspace: the largest patch size rounded up to a
// multiple of 4 (16-byte aligned row pairs for the asynchronous staging copies)
int gbk3_correction_ld(int rho) {
  const int m = 7 * (2 * rho + 1) * (2 * rho + 1) * (2 * rho + 1);
  return (m + 3) & ~3;
}
size_t gbk3_correction_workspace(int Lp, int rho, int ctas) {
  const long long ld = gbk3_correction_ld(rho);
  (void)Lp;
  return (size_t)ctas * (ld * ld + ld) * sizeof(double);
}
int gbk3_correction_patches(int Lp, int wB, const double* B, const double* sB, const double* G,
                            int rho, double* Dt, long long* status, double* ws, int ctas,
                            cudaStream_t s) {
  const long long P = (long long)Lp * Lp * Lp;
  const int g = (int)(P < ctas ? P : ctas);
  const size_t smem = 3 * (size_t)k3PB * k3TLD * 8;  // region 0 (D11 / B buffer 2), As, Bs
  cudaError_t e = cudaFuncSetAttribute(k3_correction_patches,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  k3_correction_patches<<<g, 256, smem, s>>>(Lp, wB, B, sB, G, rho, Dt, status, ws,
                                             gbk3_correction_ld(rho));
  return (int)cudaGetLastError();
}
int gbk3_restriction(int Lp, int rho, const double* Dt, const double* host_w, double* Rv,
                     cudaStream_t s) {
  const long long P = (long long)Lp * Lp * Lp;
  const long long R = 2 * rho + 1;
  k3_restriction<<<grid3(P * R * R * R * 8, 256), 256, 0, s>>>(Lp, rho, Dt, w7x8(host_w), Rv);
  return (int)cudaGetLastError();
}
int gbk3_triple(int Lp, int wB, const double* B, const double* G, const double* PAPt, int rho,
                const double* Dt, int wBD, double* BD, int wGD, double* GtD, int wA2,
                double* raw, cudaStream_t s) {
  const long long P = (long long)Lp * Lp * Lp;
  if (g_k3_tiled) {
    // (a D copy by rows, coalesced over the runs, was measured too: no change)
    const int W = 2 * wBD + 1;
    const long long items = P * W * W * ((W + K3_JZ - 1) / K3_JZ);
    k3_bd_tiled<<<grid3(items, 128), 128, 0, s>>>(Lp, wB, B, rho, Dt, wBD, BD);
    cudaError_t e = cudaMemsetAsync(GtD, 0, sizeof(double) * P * slots3(wGD, 1), s);
    if (e != cudaSuccess) return (int)e;
    k3_gtd_bycol<<<grid3(P * slots3(wGD, 1), 256), 256, 0, s>>>(Lp, wB, G, rho, Dt, wGD, GtD);
  } else {
    k3_bd<<<grid3(P * 7 * slots3(wBD, 1), 256), 256, 0, s>>>(Lp, wB, B, rho, Dt, wBD, BD);
    k3_gtd<<<grid3(P * slots3(wGD, 1), 256), 256, 0, s>>>(Lp, wB, G, rho, Dt, wGD, GtD);
  }
  if (g_k3_tiled) {
    const int W = 2 * wA2 + 1;
    const long long items = P * W * W * ((W + K3_JZ - 1) / K3_JZ);
    k3_coarse_raw_tiled<<<grid3(items, 256), 256, 0, s>>>(Lp, wB, PAPt, wGD, GtD, rho, Dt, wBD,
                                                           BD, wA2, raw);
  } else {
    k3_coarse_raw<<<grid3(P * slots3(wA2, 1), 256), 256, 0, s>>>(Lp, wB, PAPt, wGD, GtD, rho, Dt,
                                                                  wBD, BD, wA2, raw);
  }
  return (int)cudaGetLastError();
}
int gbk3_apply_w(int Lp, const double* host_w, const double* g, const double* sv, double* out,
                 cudaStream_t s) {
  k3_apply_w<<<grid3((long long)Lp * Lp * Lp * 7, 256), 256, 0, s>>>(Lp, w7x8(host_w), g, sv,
                                                                      out);
  return (int)cudaGetLastError();
}
int gbk3_apply_wt(int Lp, const double* host_w, const double* w, double* v, cudaStream_t s) {
  k3_apply_wt<<<grid3((long long)Lp * Lp * Lp * 8, 256), 256, 0, s>>>(Lp, w7x8(host_w), w, v);
  return (int)cudaGetLastError();
}
int gbk3_apply_r(int Lp, int rho, const double* Rv, const double* g, double* out,
                 cudaStream_t s) {
  k3_apply_r<<<grid3((long long)Lp * Lp * Lp, 128), 128, 0, s>>>(Lp, rho, Rv, g, out);
  return (int)cudaGetLastError();
}
int gbk3_apply_rt(int Lp, int rho, const double* Rv, const double* u, double* out,
                  cudaStream_t s) {
  k3_apply_rt<<<grid3((long long)Lp * Lp * Lp * 8, 128), 128, 0, s>>>(Lp, rho, Rv, u, out);
  return (int)cudaGetLastError();
}
int gbk3_psi_t_apply(int L, int rho, int wd, const double* psi, const double* v, double* out,
                     cudaStream_t s) {
  k3_psi_t_apply<<<grid3((long long)L * L * L, 128), 128, 0, s>>>(L, rho, wd, psi, v, out);
  return (int)cudaGetLastError();
}
