// Box-stencil plumbing: CSR input -> box, diagonal scaling, symmetrize + tail
// drop, row-tail drop and the box -> canonical CSR export at the API edge.
#include <cub/cub.cuh>

#include "gb_common.cuh"
#include "gb_kernels.h"

namespace gb {

// ---------------------------------------------------------------------------
// On-device Q1 assembly (grid_fem.py:189-227) straight into the box layout
// (half-width 1, slot (ds+1)*3 + (dt+1)).  The reference scatters the
// element matrices cell by cell into COO and canonicalizes; each entry is the
// sum of its cells' scale*E[r][c] in increasing flat cell order (checked
// bitwise against scipy's canonical CSR).  Products and sums are explicitly
// rounded (no FMA contraction) to reproduce the host arithmetic.
// ---------------------------------------------------------------------------
struct Elem16 {
  double e[16];
};

__global__ void k_assemble_q1(int n, const double* __restrict__ cell_scale, double const_scale,
                              Elem16 E, double* __restrict__ box) {
  const long long N = (long long)n * n;
  const int m = n + 1;
  // corner k of cell (ci, cj) is node (ci + di[k], cj + dj[k]): SW, SE, NE, NW
  const int di[4] = {0, 1, 1, 0}, dj[4] = {0, 0, 1, 1};
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < N;
       r += (long long)gridDim.x * blockDim.x) {
    const int I = (int)(r / n) + 1, J = (int)(r % n) + 1;
    double acc[9];
    bool any[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      acc[k] = 0.0;
      any[k] = false;
    }
    // the four cells around node (I, J) in increasing flat order
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int ci = I - 1 + (cc >> 1), cj = J - 1 + (cc & 1);
      const double sc = cell_scale ? cell_scale[(long long)ci * m + cj] : const_scale;
      int rl = 0;  // local corner of (I, J)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (ci + di[k] == I && cj + dj[k] == J) rl = k;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int I2 = ci + di[k], J2 = cj + dj[k];
        if (I2 < 1 || I2 > n || J2 < 1 || J2 > n) continue;  // boundary elimination
        const int slot = (I2 - I + 1) * 3 + (J2 - J + 1);
        const double v = __dmul_rn(sc, E.e[rl * 4 + k]);
        acc[slot] = any[slot] ? __dadd_rn(acc[slot], v) : v;
        any[slot] = true;
      }
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) box[r * 9 + k] = acc[k];
  }
}

// b = M g on the half-width-1 box in scipy's csr_matvec order (sorted
// columns = slot order, sum from 0, no FMA)
__global__ void k_box1_matvec(int n, const double* __restrict__ box,
                              const double* __restrict__ g, double* __restrict__ b) {
  const long long N = (long long)n * n;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < N;
       r += (long long)gridDim.x * blockDim.x) {
    const int s0 = (int)(r / n), t0 = (int)(r % n);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int s1 = s0 + k / 3 - 1, t1 = t0 + k % 3 - 1;
      if (s1 < 0 || s1 >= n || t1 < 0 || t1 >= n) continue;
      const double v = box[r * 9 + k];
      if (v == 0.0) continue;  // not stored in the canonical CSR
      acc = __dadd_rn(acc, __dmul_rn(v, g[(long long)s1 * n + t1]));
    }
    b[r] = acc;
  }
}

// ---------------------------------------------------------------------------
// CSR (fine grid, side n) -> box of half-width w
// ---------------------------------------------------------------------------
__global__ void k_csr_halfwidth(int n, const int32_t* __restrict__ indptr,
                                const int32_t* __restrict__ indices,
                                int* __restrict__ out) {
  const long long N = (long long)n * n;
  int m = 0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < N;
       r += (long long)gridDim.x * blockDim.x) {
    const int rs = (int)(r / n), rt = (int)(r % n);
    for (int e = indptr[r]; e < indptr[r + 1]; ++e) {
      const int c = indices[e];
      const int ds = c / n - rs, dt = c % n - rt;
      m = imax(m, imax(ds < 0 ? -ds : ds, dt < 0 ? -dt : dt));
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = imax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_csr_to_box(int n, int w, const int32_t* __restrict__ indptr,
                             const int32_t* __restrict__ indices,
                             const double* __restrict__ data,
                             double* __restrict__ box, long long* status, long long row0,
                             long long nrows) {
  // indptr holds nrows + 1 entries of the rows [row0, row0 + nrows); column
  // indices and the box are global
  const int S = box_slots(w, 1);
  for (long long lr = blockIdx.x * (long long)blockDim.x + threadIdx.x; lr < nrows;
       lr += (long long)gridDim.x * blockDim.x) {
    const long long r = row0 + lr;
    const int rs = (int)(r / n), rt = (int)(r % n);
    for (int e = indptr[lr]; e < indptr[lr + 1]; ++e) {
      const int c = indices[e];
      const int ds = c / n - rs, dt = c % n - rt;
      if (ds < -w || ds > w || dt < -w || dt > w) {
        raise_status(status, ST_OUTSIDE_BOX, r);
        continue;
      }
      box[r * S + slot_of(w, 1, ds, dt, 0)] += data[e];
    }
  }
}

// ---------------------------------------------------------------------------
// s = diag^-1/2 (gamblet_fast.py:123-139), nonpositive diagonal -> status
// ---------------------------------------------------------------------------
__global__ void k_box_scale(long long rows, int nr, int w,
                            const double* __restrict__ box,
                            double* __restrict__ s, long long* status) {
  const int S = box_slots(w, nr);
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(r % nr);
    const double d = box[r * S + slot_of(w, nr, 0, 0, c)];
    if (!(d > 0.0)) {
      raise_status(status, ST_NONPOS_DIAG, r);
      s[r] = 0.0;
    } else {
      s[r] = 1.0 / sqrt(d);
    }
  }
}

// min of the diagonal (the tail drop is skipped when it is <= 0,
// gamblet_fast.py:157-159); dmin must be pre-set to +inf by the caller.
__global__ void k_box_diag_min(long long rows, int nr, int w,
                               const double* __restrict__ box,
                               double* __restrict__ dmin) {
  const int S = box_slots(w, nr);
  double m = __longlong_as_double(0x7ff0000000000000ll);
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    m = fmin(m, box[r * S + slot_of(w, nr, 0, 0, (int)(r % nr))]);
  }
  m = warp_min(m);
  if ((threadIdx.x & 31) == 0) {
    // atomic min on doubles via CAS (values may be negative)
    unsigned long long* a = reinterpret_cast<unsigned long long*>(dmin);
    unsigned long long old = *a, assumed;
    do {
      assumed = old;
      if (__longlong_as_double((long long)assumed) <= m) break;
      old = atomicCAS(a, assumed, (unsigned long long)__double_as_longlong(m));
    } while (assumed != old);
  }
}

// (X + X^T) * 0.5 with the repair statistics, then the symmetric dead-tail
// drop |x| < 1e-12 sqrt(d_i d_j) off the diagonal (gamblet_exact.py:95-103,
// gamblet_fast.py:154-169).  stats[0] = max|x_ij - x_ji|, stats[1] = max|x|.
__global__ void k_box_sym_drop(int L, int nr, int w, const double* __restrict__ raw,
                               double* __restrict__ out,
                               const double* __restrict__ dmin,
                               double* __restrict__ stats, long long e0, long long e1) {
  const int S = box_slots(w, nr);
  const bool do_drop = *dmin > 0.0;
  double mdiff = 0.0, mabs = 0.0;
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / S;
    const int sl = (int)(e - r * S);
    const int cp = sl % nr;
    const int bs = sl / nr;
    const int ds = bs / (2 * w + 1) - w, dt = bs % (2 * w + 1) - w;
    const long long p = r / nr;
    const int c = (int)(r - p * nr);
    const int ps = (int)(p / L), pt = (int)(p % L);
    const int qs = ps + ds, qt = pt + dt;
    double v = 0.0;
    if (qs >= 0 && qs < L && qt >= 0 && qt < L) {
      const long long r2 = ((long long)qs * L + qt) * nr + cp;
      const double a = raw[e];
      const double b = raw[r2 * S + slot_of(w, nr, -ds, -dt, c)];
      mdiff = fmax(mdiff, fabs(a - b));
      mabs = fmax(mabs, fabs(a));
      v = (a + b) * 0.5;
      const bool diag = (r2 == r);
      if (do_drop && !diag) {
        const double di = raw[r * S + slot_of(w, nr, 0, 0, c)];
        const double dj = raw[r2 * S + slot_of(w, nr, 0, 0, cp)];
        if (!(fabs(v) >= 1e-12 * sqrt(di * dj))) v = 0.0;
      }
    }
    out[e] = v;
  }
  mdiff = warp_max(mdiff);
  mabs = warp_max(mabs);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(&stats[0], mdiff);
    atomic_max_nonneg(&stats[1], mabs);
  }
}

// ---------------------------------------------------------------------------
// row-tail drop |x| < 1e-11 * rowmax (gamblet_fast.py:172-190) on a dense row
// layout (one block per row; used for psi^(k) windows)
// ---------------------------------------------------------------------------
__global__ void k_row_tail_drop(long long rows, long long S, double* __restrict__ v) {
  __shared__ double sh[32];
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    double* row = v + r * S;
    double m = 0.0;
    for (long long j = threadIdx.x; j < S; j += blockDim.x) m = fmax(m, fabs(row[j]));
    m = block_max(m, sh);
    const double thr = 1e-11 * m;
    for (long long j = threadIdx.x; j < S; j += blockDim.x) {
      const double x = row[j];
      if (!(fabs(x) >= thr)) row[j] = 0.0;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// CSR export.  `kind` selects the slot enumeration in ascending global column
// order and the column map:
//   EXP_SQUARE : rows (p,c) on LxL x nr, cols (p+d, c') x nc
//   EXP_CHILD  : rows i on LxL, cols children of (i+d) on (2L)x(2L); slot (d, b)
//   EXP_PSI    : rows of level side L, fine window (n, lo, wd, h = n/L)
//   EXP_TDT    : D = Dt^T; rows (p,c) on LxL x3, cols i with Dt[i][(p-i, c)]
// ---------------------------------------------------------------------------
struct ExportDesc {
  int kind, L, nr, w, nc;  // box geometry (for EXP_TDT: Dt's half-width w)
  int n, lo, wd;           // psi window geometry
};

__device__ __forceinline__ bool export_entry(const ExportDesc& d,
                                             const double* __restrict__ val,
                                             long long r, long long j, double* v,
                                             int* col) {
  if (d.kind == EXP_SQUARE) {
    const int S = box_slots(d.w, d.nc);
    const int cp = (int)(j % d.nc);
    const int bs = (int)(j / d.nc);
    const int ds = bs / (2 * d.w + 1) - d.w, dt = bs % (2 * d.w + 1) - d.w;
    const long long p = r / d.nr;
    const int qs = (int)(p / d.L) + ds, qt = (int)(p % d.L) + dt;
    if (qs < 0 || qs >= d.L || qt < 0 || qt >= d.L) return false;
    *v = val[r * S + j];
    *col = (qs * d.L + qt) * d.nc + cp;
    return *v != 0.0;
  } else if (d.kind == EXP_CHILD) {
    const int W2 = 2 * d.w + 1;
    const int beta = (int)(j & 1);
    long long t = j >> 1;
    const int dti = (int)(t % W2);
    t /= W2;
    const int alpha = (int)(t & 1);
    const int dsi = (int)(t >> 1);
    const int ds = dsi - d.w, dt = dti - d.w;
    const int qs = (int)(r / d.L) + ds, qt = (int)(r % d.L) + dt;
    if (qs < 0 || qs >= d.L || qt < 0 || qt >= d.L) return false;
    const int S = W2 * W2 * 4;
    *v = val[r * S + (dsi * W2 + dti) * 4 + 2 * alpha + beta];
    *col = (2 * qs + alpha) * (2 * d.L) + 2 * qt + beta;
    return *v != 0.0;
  } else if (d.kind == EXP_PSI) {
    const int h = d.n / d.L;
    const int os = clampi((int)(r / d.L) * h + d.lo, 0, d.n - d.wd);
    const int ot = clampi((int)(r % d.L) * h + d.lo, 0, d.n - d.wd);
    const int a = (int)(j / d.wd), b = (int)(j % d.wd);
    *v = val[r * (long long)d.wd * d.wd + j];
    *col = (os + a) * d.n + (ot + b);
    return *v != 0.0;
  } else {  // EXP_TDT
    const int W2 = 2 * d.w + 1;
    const long long p = r / 3;
    const int c = (int)(r % 3);
    const int dis = (int)(j / W2) - d.w, dit = (int)(j % W2) - d.w;
    const int is = (int)(p / d.L) + dis, it = (int)(p % d.L) + dit;
    if (is < 0 || is >= d.L || it < 0 || it >= d.L) return false;
    const long long i = (long long)is * d.L + it;
    *v = val[i * (W2 * W2 * 3) + slot_of(d.w, 3, -dis, -dit, c)];
    *col = (int)i;
    return *v != 0.0;
  }
}

__global__ void k_export_count(ExportDesc d, const double* __restrict__ val,
                               long long rows, long long S,
                               long long* __restrict__ counts) {
  __shared__ double sh[32];
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    double c = 0.0;
    for (long long j = threadIdx.x; j < S; j += blockDim.x) {
      double v;
      int col;
      if (export_entry(d, val, r, j, &v, &col)) c += 1.0;
    }
    c = block_sum(c, sh);
    if (threadIdx.x == 0) counts[r] = (long long)c;
    __syncthreads();
  }
}

__global__ void k_export_emit(ExportDesc d, const double* __restrict__ val,
                              long long rows, long long S,
                              const long long* __restrict__ indptr,
                              int32_t* __restrict__ indices,
                              double* __restrict__ data) {
  typedef cub::BlockScan<int, 256> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const long long base = indptr[r];
    for (long long j0 = 0; j0 < S; j0 += 256) {
      const long long j = j0 + threadIdx.x;
      double v = 0.0;
      int col = 0;
      const int keep = (j < S) && export_entry(d, val, r, j, &v, &col);
      int pos, tot;
      Scan(tmp).ExclusiveSum(keep, pos, tot);
      if (keep) {
        indices[base + carry + pos] = col;
        data[base + carry + pos] = v;
      }
      __syncthreads();
      if (threadIdx.x == 0) carry += tot;
      __syncthreads();
    }
  }
}

}  // namespace gb

// ===========================================================================
// host launchers
// ===========================================================================
using namespace gb;

static inline int grid_for(long long work, int block, int cap = 148 * 64) {
  long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

int gbk_assemble_q1(int n, const double* cell_scale, double const_scale, const double* host_e16,
                    double* box, cudaStream_t s) {
  Elem16 E;
  for (int i = 0; i < 16; ++i) E.e[i] = host_e16[i];
  const long long N = (long long)n * n;
  k_assemble_q1<<<grid_for(N, 256), 256, 0, s>>>(n, cell_scale, const_scale, E, box);
  return (int)cudaGetLastError();
}

int gbk_box1_matvec(int n, const double* box, const double* g, double* b, cudaStream_t s) {
  const long long N = (long long)n * n;
  k_box1_matvec<<<grid_for(N, 256), 256, 0, s>>>(n, box, g, b);
  return (int)cudaGetLastError();
}

int gbk_csr_halfwidth(int n, const int32_t* indptr, const int32_t* indices,
                      int* out, cudaStream_t s) {
  const long long N = (long long)n * n;
  k_csr_halfwidth<<<grid_for(N, 256), 256, 0, s>>>(n, indptr, indices, out);
  return (int)cudaGetLastError();
}

int gbk_csr_to_box(int n, int w, const int32_t* indptr, const int32_t* indices,
                   const double* data, double* box, long long* status,
                   cudaStream_t s) {
  const long long N = (long long)n * n;
  k_csr_to_box<<<grid_for(N, 256), 256, 0, s>>>(n, w, indptr, indices, data, box,
                                                status, 0, N);
  return (int)cudaGetLastError();
}

// grid rows [r0, r1) from the CSR slice of exactly those matrix rows (local
// indptr starting at 0, global column indices) into the global box
int gbk_csr_to_box_rows(int n, int w, const int32_t* indptr, const int32_t* indices,
                        const double* data, double* box, long long* status, int r0, int r1,
                        cudaStream_t s) {
  if (r0 < 0 || r1 > n || r0 > r1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long nrows = (long long)(r1 - r0) * n;
  k_csr_to_box<<<grid_for(nrows, 256), 256, 0, s>>>(n, w, indptr, indices, data, box, status,
                                                    (long long)r0 * n, nrows);
  return (int)cudaGetLastError();
}

int gbk_box_scale(long long rows, int nr, int w, const double* box, double* sv,
                  long long* status, cudaStream_t s) {
  k_box_scale<<<grid_for(rows, 256), 256, 0, s>>>(rows, nr, w, box, sv, status);
  return (int)cudaGetLastError();
}

int gbk_box_diag_min(long long rows, int nr, int w, const double* box,
                     double* dmin, cudaStream_t s) {
  k_box_diag_min<<<grid_for(rows, 256), 256, 0, s>>>(rows, nr, w, box, dmin);
  return (int)cudaGetLastError();
}

int gbk_box_sym_drop(int L, int nr, int w, const double* raw, double* out,
                     const double* dmin, double* stats, cudaStream_t s) {
  return gbk_box_sym_drop_rows(L, nr, w, raw, out, dmin, stats, 0, L, s);
}

// grid rows [r0, r1) of the output; reads raw rows within w of the strip
int gbk_box_sym_drop_rows(int L, int nr, int w, const double* raw, double* out,
                          const double* dmin, double* stats, int r0, int r1, cudaStream_t s) {
  if (r0 < 0 || r1 > L || r0 > r1) return GB_UNSUPPORTED;
  if (r0 == r1) return 0;
  const long long per = (long long)L * nr * box_slots(w, nr);
  k_box_sym_drop<<<grid_for((r1 - r0) * per, 256), 256, 0, s>>>(L, nr, w, raw, out, dmin, stats,
                                                               r0 * per, r1 * per);
  return (int)cudaGetLastError();
}

int gbk_row_tail_drop(long long rows, long long S, double* v, cudaStream_t s) {
  const int g = (int)(rows < 65535 * 4 ? rows : 65535 * 4);
  k_row_tail_drop<<<g, 256, 0, s>>>(rows, S, v);
  return (int)cudaGetLastError();
}

int gbk_export_count(int kind, int L, int nr, int w, int nc, int n, int lo,
                     int wd, const double* val, long long rows, long long S,
                     long long* counts, cudaStream_t s) {
  ExportDesc d{kind, L, nr, w, nc, n, lo, wd};
  const int g = (int)(rows < (1ll << 30) ? rows : (1ll << 30));
  k_export_count<<<g, 256, 0, s>>>(d, val, rows, S, counts);
  return (int)cudaGetLastError();
}

int gbk_exclusive_scan(const long long* counts, long long* indptr, long long n,
                       void* tmp, size_t* tmp_bytes, cudaStream_t s) {
  // indptr has n+1 entries: exclusive scan of counts over n+1 inputs where the
  // caller guarantees counts[n] == 0.
  cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, counts, indptr,
                                                (int)(n + 1), s);
  return (int)e;
}

int gbk_export_emit(int kind, int L, int nr, int w, int nc, int n, int lo,
                    int wd, const double* val, long long rows, long long S,
                    const long long* indptr, int32_t* indices, double* data,
                    cudaStream_t s) {
  ExportDesc d{kind, L, nr, w, nc, n, lo, wd};
  const int g = (int)(rows < (1ll << 30) ? rows : (1ll << 30));
  k_export_emit<<<g, 256, 0, s>>>(d, val, rows, S, indptr, indices, data);
  return (int)cudaGetLastError();
}
