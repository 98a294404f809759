// Diagnostics on the device (diagnostics.py:40-155
// of the reference): per-cell energies and the energy-decay profile of a
// basis vector, the coefficient spectrum read off operator diagonals, the
// stable top-k selection of `compress`, and energy norms x^T A x on the box
// layout.  All reductions are two-pass with a fixed block count, so results
// are deterministic run to run.
#include <cub/cub.cuh>

#include "gb_common.cuh"
#include "gb_kernels.h"

namespace gb {

constexpr int kDiagBlocks = 148 * 4;

struct Elem16d {
  double e[16];
};

// energy of v on each cell: a_c * vals^T E vals, vals = v at the 4 corners
// (SW, SE, NE, NW; 0 on the boundary) -- diagnostics.py:40-49
__global__ void k_cell_energies(int n, const double* __restrict__ v,
                                const double* __restrict__ coef, Elem16d E,
                                double* __restrict__ out) {
  const int m = n + 1;
  const long long cells = (long long)m * m;
  const int di[4] = {0, 1, 1, 0}, dj[4] = {0, 0, 1, 1};
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < cells;
       c += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(c / m), cj = (int)(c % m);
    double vals[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int I = ci + di[k], J = cj + dj[k];
      vals[k] = (I >= 1 && I <= n && J >= 1 && J <= n) ? v[(long long)(I - 1) * n + (J - 1)]
                                                       : 0.0;
    }
    double quad = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) t += E.e[i * 4 + j] * vals[j];
      quad += vals[i] * t;
    }
    out[c] = coef[c] * quad;
  }
}

// partial sums of the energies outside each ball: part[j * gridDim.x + b] for
// radius j < nr, and the total at j = nr (diagnostics.py:58-74)
__global__ void k_decay_partial(int m, double h, const double* __restrict__ en, double cx,
                                double cy, const double* __restrict__ radii, int nr,
                                double* __restrict__ part) {
  __shared__ double sh[32];
  const long long cells = (long long)m * m;
  for (int j = 0; j <= nr; ++j) {
    const double r = j < nr ? radii[j] : 0.0;
    double acc = 0.0;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < cells;
         c += (long long)gridDim.x * blockDim.x) {
      const double x = ((double)(c / m) + 0.5) * h, y = ((double)(c % m) + 0.5) * h;
      if (j == nr || hypot(x - cx, y - cy) >= r) acc += en[c];
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[(long long)j * gridDim.x + blockIdx.x] = acc;
    __syncthreads();
  }
}

// out[j] = sum_b part[j][b] (fixed order), j = 0..nr (the last is the total)
__global__ void k_partial_rows(int rows, int nb, const double* __restrict__ part,
                               double* __restrict__ out) {
  __shared__ double sh[32];
  for (int j = blockIdx.x; j < rows; j += gridDim.x) {
    double acc = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += part[(long long)j * nb + b];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) out[j] = acc;
    __syncthreads();
  }
}

// |coef_r| * sqrt(diag_r) of a square box (nc = nr) -- diagnostics.py:97-107
__global__ void k_box_diag_spectrum(long long rows, int nr, int w, const double* __restrict__ box,
                                    const double* __restrict__ coef, double* __restrict__ out) {
  const int W2 = 2 * w + 1;
  const int S = W2 * W2 * nr;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(r % nr);
    const double d = box[r * S + (w * W2 + w) * nr + c];
    out[r] = fabs(coef[r]) * sqrt(d);
  }
}

__global__ void k_negate_iota(long long n, const double* __restrict__ mags, double* __restrict__ keys,
                              long long* __restrict__ idx) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    keys[i] = -mags[i];
    idx[i] = i;
  }
}

__global__ void k_mask_first(long long n, long long n_keep, const long long* __restrict__ order,
                             double* __restrict__ mask) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    mask[order[i]] = i < n_keep ? 1.0 : 0.0;
}

// per-block partials of x^T (A x) on a square nr = nc = 1 box of side L
__global__ void k_box_quad_partial(int L, int w, const double* __restrict__ box,
                                   const double* __restrict__ x, double* __restrict__ part) {
  __shared__ double sh[32];
  const long long N = (long long)L * L;
  const int W2 = 2 * w + 1, S = W2 * W2;
  double acc = 0.0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < N;
       r += (long long)gridDim.x * blockDim.x) {
    const int s0 = (int)(r / L), t0 = (int)(r % L);
    double y = 0.0;
    for (int ds = -w; ds <= w; ++ds) {
      const int s1 = s0 + ds;
      if (s1 < 0 || s1 >= L) continue;
      for (int dt = -w; dt <= w; ++dt) {
        const int t1 = t0 + dt;
        if (t1 < 0 || t1 >= L) continue;
        y += box[r * S + (ds + w) * W2 + (dt + w)] * x[(long long)s1 * L + t1];
      }
    }
    acc += x[r] * y;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// per-block max |x_i| (order-independent, exact)
__global__ void k_max_abs_partial(long long n, const double* __restrict__ x,
                                  double* __restrict__ part) {
  __shared__ double sh[32];
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  m = block_max(m, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

__global__ void k_max_final(int nb, const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double sh[32];
  double m = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) m = fmax(m, part[b]);
  m = block_max(m, sh);
  if (threadIdx.x == 0) *out = m;
}

}  // namespace gb

using namespace gb;

int gbk_max_abs(long long n, const double* x, double* part, double* out, cudaStream_t s) {
  k_max_abs_partial<<<kDiagBlocks, 256, 0, s>>>(n, x, part);
  k_max_final<<<1, 256, 0, s>>>(kDiagBlocks, part, out);
  return (int)cudaGetLastError();
}

int gbk_cell_energies(int n, const double* v, const double* coef, const double* host_e16,
                      double* out, cudaStream_t s) {
  Elem16d E;
  for (int i = 0; i < 16; ++i) E.e[i] = host_e16[i];
  const long long cells = (long long)(n + 1) * (n + 1);
  long long g = (cells + 255) / 256;
  k_cell_energies<<<(int)(g < kDiagBlocks ? g : kDiagBlocks), 256, 0, s>>>(n, v, coef, E, out);
  return (int)cudaGetLastError();
}

size_t gbk_decay_part_elems(int nr) { return (size_t)(nr + 1) * kDiagBlocks; }

int gbk_decay_sums(int n, double h, const double* en, double cx, double cy, const double* radii,
                   int nr, double* part, double* out, cudaStream_t s) {
  k_decay_partial<<<kDiagBlocks, 256, 0, s>>>(n + 1, h, en, cx, cy, radii, nr, part);
  k_partial_rows<<<nr + 1 < 148 ? nr + 1 : 148, 256, 0, s>>>(nr + 1, kDiagBlocks, part, out);
  return (int)cudaGetLastError();
}

int gbk_box_diag_spectrum(long long rows, int nr, int w, const double* box, const double* coef,
                          double* out, cudaStream_t s) {
  long long g = (rows + 255) / 256;
  k_box_diag_spectrum<<<(int)(g < kDiagBlocks ? g : kDiagBlocks), 256, 0, s>>>(rows, nr, w, box,
                                                                               coef, out);
  return (int)cudaGetLastError();
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

int gbk_topk_mask(long long n, const double* mags, long long n_keep, double* mask, void* work,
                  size_t* work_bytes, cudaStream_t s) {
  size_t cub_bytes = 0;
  cub::DoubleBuffer<double> dk(nullptr, nullptr);
  cub::DoubleBuffer<long long> dv(nullptr, nullptr);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, dk, dv, (int)n, 0,
                                                  sizeof(double) * 8, s);
  if (e != cudaSuccess) return (int)e;
  const size_t vec = align256(sizeof(double) * (size_t)n);
  const size_t need = 4 * vec + align256(cub_bytes);
  if (!work) {
    *work_bytes = need;
    return 0;
  }
  if (*work_bytes < need) return 1;
  char* p = (char*)work;
  double* k0 = (double*)p;
  double* k1 = (double*)(p + vec);
  long long* v0 = (long long*)(p + 2 * vec);
  long long* v1 = (long long*)(p + 3 * vec);
  void* tmp = p + 4 * vec;
  long long g = (n + 255) / 256;
  const int gb = (int)(g < kDiagBlocks ? g : kDiagBlocks);
  k_negate_iota<<<gb, 256, 0, s>>>(n, mags, k0, v0);
  cub::DoubleBuffer<double> keys(k0, k1);
  cub::DoubleBuffer<long long> vals(v0, v1);
  // LSD radix sort: stable, so equal magnitudes keep ascending index order
  // (np.argsort(-mags, kind="stable"), diagnostics.py:123-124)
  e = cub::DeviceRadixSort::SortPairs(tmp, cub_bytes, keys, vals, (int)n, 0, sizeof(double) * 8,
                                      s);
  if (e != cudaSuccess) return (int)e;
  k_mask_first<<<gb, 256, 0, s>>>(n, n_keep, vals.Current(), mask);
  return (int)cudaGetLastError();
}

size_t gbk_quad_part_elems() { return kDiagBlocks; }

int gbk_box_quadform(int L, int w, const double* box, const double* x, double* part, double* out,
                     cudaStream_t s) {
  k_box_quad_partial<<<kDiagBlocks, 256, 0, s>>>(L, w, box, x, part);
  k_partial_rows<<<1, 256, 0, s>>>(1, kDiagBlocks, part, out);
  return (int)cudaGetLastError();
}
