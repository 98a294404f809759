// extern "C" boundary of libgamblets_b200.so (declared in
// include/gamblets_b200.h).  Thin wrappers: argument checks, stream cast,
// CUDA error -> GB_ERR_CUDA with a thread-local message.
#include <stdio.h>
#include <string.h>

#include "../../include/gamblets_b200.h"
#include "gb_kernels.h"
#include "gb_lanczos.h"

int gbk_dense_gemm(int m, int n, int k, double alpha, const double* A, int lda, int ta,
                   const double* B, int ldb, int tb, double beta, double* C, int ldc,
                   cudaStream_t s);
int gbk_dense_potrf(int n, double* A, int lda, long long* status, cudaStream_t s);
int gbk_dense_potrs(int n, int nrhs, const double* L, int lda, double* X, int ldx,
                    cudaStream_t s);
int gbk_dense_sym(int n, const double* X, int ldx, double* out, double* stats,
                  cudaStream_t s);
int gbk_fp64_peak_probe(int kind, int iters, double* sink, cudaStream_t s);
int gbk_dense_build_w(int Lk, const double* w12, double* out, cudaStream_t s);
int gbk_dense_build_p(int Lk, double scale, double* out, cudaStream_t s);
int gbk_csr_to_dense(int nrows, int ncols, const int32_t* indptr, const int32_t* indices,
                     const double* data, double* out, cudaStream_t s);
int gbk_eye(int n, double* out, cudaStream_t s);

static thread_local char g_err[512];
#include <atomic>
static std::atomic<unsigned long long> g_launches{0};  // kernels launched through this ABI
#define COUNT(n) (g_launches += (unsigned long long)(n))

static int wrap(int e, const char* what) {
  if (e == 0) return GB_OK;
  snprintf(g_err, sizeof(g_err), "%s: %s", what,
           cudaGetErrorString(static_cast<cudaError_t>(e)));
  return GB_ERR_CUDA;
}

static int invalid(const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return GB_ERR_INVALID;
}

#define ST(x) reinterpret_cast<cudaStream_t>(x)
#define LL(x) reinterpret_cast<long long*>(x)

extern "C" {

int gb_abi_version(void) { return 7; }
unsigned long long gb_launch_count(void) { return g_launches.load(); }
const char* gb_last_error(void) { return g_err; }
int gb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int gb_csr_halfwidth(int n, const int32_t* indptr, const int32_t* indices,
                     int32_t* out_w, void* stream) {
  if (n <= 0) return invalid("csr_halfwidth: n <= 0");
  COUNT(1);
  return wrap(gbk_csr_halfwidth(n, indptr, indices, out_w, ST(stream)), "csr_halfwidth");
}
int gb_assemble_q1(int n, const double* cell_scale, double const_scale, const double* host_e16,
                   double* box, void* stream) {
  if (n <= 0 || !host_e16 || !box) return invalid("assemble_q1: bad arguments");
  COUNT(1);
  return wrap(gbk_assemble_q1(n, cell_scale, const_scale, host_e16, box, ST(stream)),
              "assemble_q1");
}
int gb_box1_matvec(int n, const double* box, const double* g, double* b, void* stream) {
  if (n <= 0) return invalid("box1_matvec: n <= 0");
  COUNT(1);
  return wrap(gbk_box1_matvec(n, box, g, b, ST(stream)), "box1_matvec");
}
int gb_csr_to_box(int n, int w, const int32_t* indptr, const int32_t* indices,
                  const double* data, double* box, int64_t* status, void* stream) {
  if (n <= 0 || w < 0) return invalid("csr_to_box: bad geometry");
  COUNT(1);
  return wrap(gbk_csr_to_box(n, w, indptr, indices, data, box, LL(status), ST(stream)),
              "csr_to_box");
}
int gb_box_scale(int64_t rows, int nr, int w, const double* box, double* s,
                 int64_t* status, void* stream) {
  COUNT(1);
  return wrap(gbk_box_scale(rows, nr, w, box, s, LL(status), ST(stream)), "box_scale");
}
int gb_box_diag_min(int64_t rows, int nr, int w, const double* box, double* dmin,
                    void* stream) {
  COUNT(1);
  return wrap(gbk_box_diag_min(rows, nr, w, box, dmin, ST(stream)), "box_diag_min");
}
int gb_box_sym_drop(int L, int nr, int w, const double* raw, double* out,
                    const double* dmin, double* stats, void* stream) {
  if (raw == out) return invalid("box_sym_drop: in-place not supported");
  COUNT(1);
  return wrap(gbk_box_sym_drop(L, nr, w, raw, out, dmin, stats, ST(stream)),
              "box_sym_drop");
}
int gb_row_tail_drop(int64_t rows, int64_t S, double* v, void* stream) {
  COUNT(1);
  return wrap(gbk_row_tail_drop(rows, S, v, ST(stream)), "row_tail_drop");
}

size_t gb_mass_patch_workspace(int rho, int blocks) {
  return gbk_mass_patch_workspace(rho, blocks);
}
int gb_mass_patches(int n, int wM, const double* M, const double* s, int rho, int wd,
                    double* psi, int64_t* status, double* workspace, int blocks,
                    void* stream) {
  if (rho < 0 || wd <= 0 || wd > n) return invalid("mass_patches: bad window");
  COUNT(1);
  return wrap(gbk_mass_patches(n, wM, M, s, rho, wd, psi, LL(status), workspace, blocks,
                               ST(stream)),
              "mass_patches");
}
int gb_mass_patches_v2(int n, int wM, const double* Ms, const double* s, int rho, int wd,
                       double* psi, int64_t* status, void* stream) {
  COUNT(1);
  const int rc = gbk_mass_patches_v2(n, wM, Ms, s, rho, wd, psi, LL(status), ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("mass_patches_v2: patch exceeds shared memory");
  return wrap(rc, "mass_patches_v2");
}
size_t gb_correction_patches_workspace(int Lp, int rho, int r0, int r1) {
  return gbk_correction_v3_workspace(Lp, rho, r0, r1);
}
int gb_correction_patches_v2(int Lp, int wB, const double* Bs, const double* sB, int wG,
                             const double* G, int rho, double* Dt, int64_t* status,
                             double* workspace, size_t workspace_bytes, void* stream) {
  COUNT(1);
  const int rc = gbk_correction_patches_v2(Lp, wB, Bs, sB, wG, G, rho, Dt, LL(status),
                                           workspace, workspace_bytes, ST(stream));
  if (rc == GB_UNSUPPORTED)
    return invalid("correction_patches_v2: patch exceeds shared memory or workspace too small");
  return wrap(rc, "correction_patches_v2");
}
int gb_mass_patches_rows(int n, int wM, const double* Ms, const double* s, int rho, int wd,
                         double* psi, int64_t* status, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_mass_patches_rows(n, wM, Ms, s, rho, wd, psi, LL(status), r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED)
    return invalid("mass_patches_rows: bad row range or no strip kernel for this patch");
  return wrap(rc, "mass_patches_rows");
}
int gb_psi_next_rows(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw,
                     const double* Wpsi, int rho, const double* Dt, int lo2, int wd2,
                     double* psi_next, double* rowmax, int r0, int r1, void* stream) {
  COUNT(3);
  const int rc = gbk_psi_next_rows(n, Lk, lo, hi, wd, psi, wdw, Wpsi, rho, Dt, lo2, wd2, psi_next,
                                   rowmax, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("psi_next_rows: bad row range or per-entry products mode");
  return wrap(rc, "psi_next_rows");
}
int gb_correction_patches_rows(int Lp, int wB, const double* Bs, const double* sB, int wG,
                               const double* G, int rho, double* Dt, int64_t* status, int r0,
                               int r1, double* workspace, size_t workspace_bytes, void* stream) {
  COUNT(1);
  const int rc = gbk_correction_patches_rows(Lp, wB, Bs, sB, wG, G, rho, Dt, LL(status), r0, r1,
                                             workspace, workspace_bytes, ST(stream));
  if (rc == GB_UNSUPPORTED)
    return invalid("correction_patches_rows: bad row range, no strip kernel or workspace too small");
  return wrap(rc, "correction_patches_rows");
}
int gb_psi_stencil(int n, int lo, int wd, int rho, const double* psi, int wA,
                   const double* A, int wX, double* X, void* stream) {
  COUNT(1);
  return wrap(gbk_psi_stencil(n, lo, wd, rho, psi, wA, A, wX, X, ST(stream)),
              "psi_stencil");
}
size_t gb_psi_galerkin_workspace(int n, int wd, int wX) {
  return gbk_psi_galerkin_workspace(n, wd, wX);
}
int gb_psi_galerkin_t(int n, int lo, int wd, int rho, const double* psi, int wX,
                      const double* X, int wR, double* raw, double* work, void* stream) {
  COUNT(3);
  const int rc = gbk_psi_galerkin_t(n, lo, wd, rho, psi, wX, X, wR, raw, work, ST(stream));
  if (rc == 1) return invalid("psi_galerkin_t: output block exceeds shared memory");
  return wrap(rc, "psi_galerkin_t");
}
int gb_psi_galerkin(int n, int lo, int wd, int rho, const double* psi, int wX,
                    const double* X, int wR, double* raw, void* stream) {
  COUNT(1);
  return wrap(gbk_psi_galerkin(n, lo, wd, rho, psi, wX, X, wR, raw, ST(stream)),
              "psi_galerkin");
}
int gb_level_diag(int Lk, int wA, const double* A, const double* host_w12, double* bdiag,
                  double* dmin, void* stream) {
  if (Lk < 2 || (Lk & 1)) return invalid("level_diag: bad level side");
  COUNT(1);
  return wrap(gbk_level_diag(Lk, wA, A, host_w12, bdiag, dmin, ST(stream)), "level_diag");
}
int gb_level_blocks(int Lk, int wA, const double* A, const double* host_w12, int wB,
                    const double* bdiag, const double* dmin, double* B, double* G,
                    double* PAPt, double* stats, void* stream) {
  if (Lk < 2 || (Lk & 1)) return invalid("level_blocks: bad level side");
  COUNT(1);
  return wrap(gbk_level_blocks(Lk, wA, A, host_w12, wB, bdiag, dmin, B, G, PAPt, stats,
                               ST(stream)),
              "level_blocks");
}
size_t gb_correction_workspace(int rho, int blocks) {
  return gbk_correction_workspace(rho, blocks);
}
int gb_correction_patches(int Lp, int wB, const double* B, const double* sB, int wG,
                          const double* G, int rho, double* Dt, int64_t* status,
                          double* workspace, int blocks, void* stream) {
  if (Lp < 1 || rho < 0) return invalid("correction_patches: bad geometry");
  COUNT(1);
  return wrap(gbk_correction_patches(Lp, wB, B, sB, wG, G, rho, Dt, LL(status), workspace,
                                     blocks, ST(stream)),
              "correction_patches");
}
int gb_restriction(int Lp, int rho, const double* Dt, const double* host_w12, double* R,
                   void* stream) {
  COUNT(1);
  return wrap(gbk_restriction(Lp, rho, Dt, host_w12, R, ST(stream)), "restriction");
}
int gb_bd(int Lp, int wB, const double* B, int rho, const double* Dt, int wBD,
          double* BD, void* stream) {
  COUNT(1);
  return wrap(gbk_bd(Lp, wB, B, rho, Dt, wBD, BD, ST(stream)), "bd");
}
int gb_gtd(int Lp, int wG, const double* G, int rho, const double* Dt, int wGD,
           double* GtD, void* stream) {
  COUNT(1);
  return wrap(gbk_gtd(Lp, wG, G, rho, Dt, wGD, GtD, ST(stream)), "gtd");
}
int gb_coarse_raw(int Lp, int wB, const double* PAPt, int wGD, const double* GtD,
                  int rho, const double* Dt, int wBD, const double* BD, int wA2,
                  double* raw, void* stream) {
  COUNT(1);
  return wrap(gbk_coarse_raw(Lp, wB, PAPt, wGD, GtD, rho, Dt, wBD, BD, wA2, raw,
                             ST(stream)),
              "coarse_raw");
}
int gb_wpsi(int n, int Lk, int lo, int wd, const double* host_w12, const double* psi,
            int wdw, double* Wpsi, void* stream) {
  COUNT(1);
  return wrap(gbk_wpsi(n, Lk, lo, wd, host_w12, psi, wdw, Wpsi, ST(stream)), "wpsi");
}
int gb_psi_next(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw,
                const double* Wpsi, int rho, const double* Dt, int lo2, int wd2,
                double* psi_next, double* rowmax, void* stream) {
  COUNT(2);
  return wrap(gbk_psi_next(n, Lk, lo, hi, wd, psi, wdw, Wpsi, rho, Dt, lo2, wd2, psi_next,
                           rowmax, ST(stream)),
              "psi_next");
}

int gb_products_mode(int mma) { return gbk_products_mode(mma); }
int gb_tune(int what, int value) { return gbk_tune(what, value); }
size_t gb_kstate_bytes(void) { return gbk_kstate_bytes(); }
int gb_red_blocks(void) { return gbk_red_blocks(); }
int gb_state_reset(void* state, int max_iter, void* stream) {
  COUNT(1);
  return wrap(gbk_state_reset(state, max_iter, ST(stream)), "state_reset");
}
int gb_cg_init(int64_t n, const double* b, const double* x0, const double* Ax0,
               double* x, double* r, double* p, double rel_tol, int max_iter,
               void* state, double* partials, void* stream) {
  COUNT(2);
  return wrap(gbk_cg_init(n, b, x0, Ax0, x, r, p, rel_tol, max_iter, state, partials,
                          ST(stream)),
              "cg_init");
}
int gb_cg_iterations(int L, int nr, int w, const double* B, const double* s, int mode,
                     double* x, double* r, double* p, double* Ap, int iters,
                     void* state, double* partials, void* stream) {
  COUNT(3 * (unsigned long long)iters);
  return wrap(gbk_cg_iterations(L, nr, w, B, s, mode, x, r, p, Ap, iters, state,
                                partials, ST(stream)),
              "cg_iterations");
}
int gb_pow_iterations(int L, int nr, int w, const double* B, const double* s, int mode,
                      double* x, double* y, double tol, int iters, void* state,
                      double* partials, void* stream) {
  COUNT(3 * (unsigned long long)iters);
  return wrap(gbk_pow_iterations(L, nr, w, B, s, mode, x, y, tol, iters, state,
                                 partials, ST(stream)),
              "pow_iterations");
}
int gb_scale_box(int L, int nr, int w, const double* B, const double* s, double* Bs,
                 void* stream) {
  COUNT(1);
  return wrap(gbk_scale_box(L, nr, w, B, s, Bs, ST(stream)), "scale_box");
}
int gb_pad(int L, int nr, int w, const double* src, const double* scale, double* dst,
           void* stream) {
  COUNT(1);
  return wrap(gbk_pad(L, nr, w, src, scale, dst, ST(stream)), "pad");
}
int gb_unpad(int L, int nr, int w, const double* src, const double* scale, double* dst,
             void* stream) {
  COUNT(1);
  return wrap(gbk_unpad(L, nr, w, src, scale, dst, ST(stream)), "unpad");
}
int gb_pcg_iterations(int L, int nr, int w, const double* Bs, double* x, double* r,
                      double* p, double* Ap, int iters, void* state, double* partials,
                      void* stream) {
  COUNT(3 * (unsigned long long)iters);
  return wrap(gbk_pcg_iterations(L, nr, w, Bs, x, r, p, Ap, iters, state, partials,
                                 ST(stream)),
              "pcg_iterations");
}
int gb_ppow_iterations(int L, int nr, int w, const double* Bs, double* x, double* y,
                       double tol, int iters, void* state, double* partials, void* stream) {
  COUNT(3 * (unsigned long long)iters);
  return wrap(gbk_ppow_iterations(L, nr, w, Bs, x, y, tol, iters, state, partials,
                                  ST(stream)),
              "ppow_iterations");
}
int gb_pbox_apply(int L, int nr, int w, const double* Bs, const double* x, double* y,
                  void* stream) {
  COUNT(1);
  return wrap(gbk_pbox_apply(L, nr, w, Bs, x, y, ST(stream)), "pbox_apply");
}
size_t gb_boxT_elems(int L, int nr, int w) { return gbk_boxT_elems(L, nr, w); }
// launches of one Krylov iteration: S B S application (2 kernels in the
// symmetric band layout) + update + direction
#define SPL(layout, L, nr, w) \
  (((layout) == 1 && gbk_sym_supported((L), (nr), (w))) ? 4ULL : 3ULL)
int gb_scale_box_T(int L, int nr, int w, const double* B, const double* s, double* BsT,
                   void* stream) {
  COUNT(1);
  return wrap(gbk_scale_box_T(L, nr, w, B, s, BsT, ST(stream)), "scale_box_T");
}
int gb_tcg_iterations(int L, int nr, int w, const double* BsT, double* x, double* r,
                      double* p, double* Ap, int iters, void* state, double* partials,
                      void* stream, int layout) {
  COUNT(SPL(layout, L, nr, w) * (unsigned long long)iters);
  return wrap(gbk_tcg_iterations(L, nr, w, BsT, x, r, p, Ap, iters, state, partials,
                                 ST(stream), layout),
              "tcg_iterations");
}
int gb_tpow_iterations(int L, int nr, int w, const double* BsT, double* x, double* y,
                       double tol, int iters, void* state, double* partials, void* stream,
                       int layout) {
  COUNT(SPL(layout, L, nr, w) * (unsigned long long)iters);
  return wrap(gbk_tpow_iterations(L, nr, w, BsT, x, y, tol, iters, state, partials,
                                  ST(stream), layout),
              "tpow_iterations");
}
int gb_tbox_apply(int L, int nr, int w, const double* BsT, const double* x, double* y,
                  void* stream, int layout) {
  COUNT(SPL(layout, L, nr, w) - 2);
  return wrap(gbk_tbox_apply(L, nr, w, BsT, x, y, ST(stream), layout), "tbox_apply");
}
int gb_bj_setup(int L, int w, const double* B, const double* s, float* inv, void* stream) {
  if (L < 2 || (L & 1)) return invalid("bj_setup: parent grid side must be even");
  COUNT(1);
  return wrap(gbk_bj_setup(L, w, B, s, inv, ST(stream)), "bj_setup");
}
int gb_bjcg_init(int L, int w, const double* b, const double* x0, const double* Ax0,
                 double x0_scale, double* x, double* r, double* p, double* z, const float* inv,
                 double rel_tol, int max_iter, void* state, double* partials, void* stream) {
  COUNT(1);
  return wrap(gbk_bjcg_init(L, w, b, x0, Ax0, x0_scale, x, r, p, z, inv, rel_tol, max_iter,
                            state, partials, ST(stream)),
              "bjcg_init");
}
int gb_bjcg_iterations(int L, int w, const double* BsT, const float* inv, double* x,
                       double* r, double* p, double* Ap, double* z, int iters, void* state,
                       double* partials, void* stream, int layout) {
  COUNT(3ULL * (unsigned long long)iters);  // sym layout: fused phase 2 + update
  return wrap(gbk_bjcg_iterations(L, w, BsT, inv, x, r, p, Ap, z, iters, state, partials,
                                  ST(stream), layout),
              "bjcg_iterations");
}
int gb_sync_read(const void* dev, void* host, size_t bytes, void* stream) {
  return wrap(gbk_sync_read(dev, host, bytes, ST(stream)), "sync_read");
}
int gb_tcg_solve(int L, int nr, int w, const double* BsT, double* x, double* r, double* p,
                 double* Ap, void* state, double* partials, void* host_state, int max_chunk,
                 void* stream, int layout) {
  long long n = 0;
  const int e = gbk_tcg_solve(L, nr, w, BsT, x, r, p, Ap, state, partials, host_state,
                              max_chunk, ST(stream), &n, layout);
  COUNT(n);
  return wrap(e, "tcg_solve");
}
int gb_bjcg_solve(int L, int w, const double* BsT, const float* inv, double* x, double* r,
                  double* p, double* Ap, double* z, void* state, double* partials,
                  void* host_state, int max_chunk, void* stream, int layout) {
  long long n = 0;
  const int e = gbk_bjcg_solve(L, w, BsT, inv, x, r, p, Ap, z, state, partials, host_state,
                               max_chunk, ST(stream), &n, layout);
  COUNT(n);
  return wrap(e, "bjcg_solve");
}
int gb_bjcg_solve2(int L, int w, const double* BsT, const float* inv, double* const* x,
                   double* const* r, double* const* p, double* const* Ap, double* const* z,
                   void* const* state, double* const* partials, void* const* host_state,
                   int max_chunk, void* stream) {
  if (!x || !r || !p || !Ap || !z || !state || !partials || !host_state)
    return invalid("bjcg_solve2: null pointer array");
  long long n = 0;
  const int e = gbk_bjcg_solve2(L, w, BsT, inv, x, r, p, Ap, z, state, partials, host_state,
                                max_chunk, ST(stream), &n);
  COUNT(n);
  if (e == GB_UNSUPPORTED) return invalid("bjcg_solve2: level not in the symmetric band layout");
  return wrap(e, "bjcg_solve2");
}
int gb_tpow_solve(int L, int nr, int w, const double* BsT, double* x, double* y, double tol,
                  void* state, double* partials, void* host_state, int max_chunk,
                  void* stream, int layout) {
  long long n = 0;
  const int e = gbk_tpow_solve(L, nr, w, BsT, x, y, tol, state, partials, host_state,
                               max_chunk, ST(stream), &n, layout);
  COUNT(n);
  return wrap(e, "tpow_solve");
}
size_t gb_boxsym_elems(int L, int w) { return gbk_boxsym_elems(L, w); }
size_t gb_sym_overflow_elems(int L, int w) { return gbk_sym_overflow_elems(L, w); }
int gb_sym_supported(int L, int nr, int w) { return gbk_sym_supported(L, nr, w); }
int gb_scale_box_symT(int L, int w, const double* B, const double* s, double* UsT,
                      void* stream) {
  COUNT(1);
  return wrap(gbk_scale_box_symT(L, w, B, s, UsT, ST(stream)), "scale_box_symT");
}
int gb_csr_apply(int64_t n, const int32_t* indptr, const int32_t* indices, const double* data,
                 const double* x, double* y, void* stream) {
  COUNT(1);
  return wrap(gbk_csr_apply(n, indptr, indices, data, x, y, ST(stream)), "csr_apply");
}
int gb_csr_cg_solve(int64_t n, const int32_t* indptr, const int32_t* indices,
                    const double* data, double* x, double* r, double* p, double* Ap,
                    void* state, double* partials, void* host_state, int max_chunk,
                    void* stream) {
  long long k = 0;
  const int e = gbk_csr_cg_solve(n, indptr, indices, data, x, r, p, Ap, state, partials,
                                 host_state, max_chunk, ST(stream), &k);
  COUNT(k);
  return wrap(e, "csr_cg_solve");
}
int gb_csr_pow_solve(int64_t n, const int32_t* indptr, const int32_t* indices,
                     const double* data, double* x, double* y, double tol, void* state,
                     double* partials, void* host_state, int max_chunk, void* stream) {
  long long k = 0;
  const int e = gbk_csr_pow_solve(n, indptr, indices, data, x, y, tol, state, partials,
                                  host_state, max_chunk, ST(stream), &k);
  COUNT(k);
  return wrap(e, "csr_pow_solve");
}
int gb_level_engine(gb_level_engine_args* args, void* stream) {
  long long n = 0;
  const int e = gbk_level_engine(args, ST(stream), &n);
  COUNT(n);
  return wrap(e, "level_engine");
}
int gb_lanczos_emulate(const double* ab, int m, double tol, int max_outer, double* lam,
                       int* outer, double* ritz_min, double* ritz_max) {
  if (!ab || m <= 0 || !lam || !outer) return 1;
  return gb_lz::emulate_inverse_iteration(ab, m, tol, max_outer, lam, outer, ritz_min, ritz_max);
}
int gb_lanczos_check(const double* ab, int m, double tol, int max_outer, double lz_tol,
                     double* lam, int* outer, int* stop) {
  if (!ab || m <= 0 || !lam || !outer || !stop) return 1;
  return gb_lz::lanczos_check(ab, m, tol, max_outer, lz_tol, lam, outer, stop);
}
int gb_cell_energies(int n, const double* v, const double* coef, const double* host_e16,
                     double* out, void* stream) {
  if (n <= 0 || !host_e16) return invalid("cell_energies: bad arguments");
  COUNT(1);
  return wrap(gbk_cell_energies(n, v, coef, host_e16, out, ST(stream)), "cell_energies");
}
size_t gb_decay_part_elems(int nr) { return gbk_decay_part_elems(nr); }
int gb_decay_sums(int n, double h, const double* energies, double cx, double cy,
                  const double* radii, int nr, double* part, double* out, void* stream) {
  if (n <= 0 || nr < 0) return invalid("decay_sums: bad arguments");
  COUNT(2);
  return wrap(gbk_decay_sums(n, h, energies, cx, cy, radii, nr, part, out, ST(stream)),
              "decay_sums");
}
int gb_box_diag_spectrum(int64_t rows, int nr, int w, const double* box, const double* coef,
                         double* out, void* stream) {
  if (rows < 0 || nr <= 0 || w < 0) return invalid("box_diag_spectrum: bad geometry");
  COUNT(1);
  return wrap(gbk_box_diag_spectrum(rows, nr, w, box, coef, out, ST(stream)),
              "box_diag_spectrum");
}
int gb_topk_mask(int64_t n, const double* mags, int64_t n_keep, double* mask, void* work,
                 size_t* work_bytes, void* stream) {
  if (n <= 0 || n_keep < 0 || !work_bytes) return invalid("topk_mask: bad arguments");
  if (work) COUNT(3);
  return wrap(gbk_topk_mask(n, mags, n_keep, mask, work, work_bytes, ST(stream)), "topk_mask");
}
size_t gb_quad_part_elems(void) { return gbk_quad_part_elems(); }
int gb_box_quadform(int L, int w, const double* box, const double* x, double* part, double* out,
                    void* stream) {
  if (L <= 0 || w < 0) return invalid("box_quadform: bad geometry");
  COUNT(2);
  return wrap(gbk_box_quadform(L, w, box, x, part, out, ST(stream)), "box_quadform");
}
int gb_max_abs(int64_t n, const double* x, double* part, double* out, void* stream) {
  if (n < 0) return invalid("max_abs: n < 0");
  COUNT(2);
  return wrap(gbk_max_abs(n, x, part, out, ST(stream)), "max_abs");
}
int gb_dot2(int64_t n, const double* a, const double* b, const double* c, double* out,
            void* state, double* partials, void* stream) {
  COUNT(1);
  return wrap(gbk_dot2(n, a, b, c, out, state, partials, ST(stream)), "dot2");
}
int gb_scale_by_norm(int64_t n, const double* a, const double* norm2, int which,
                     double* y, double* y2, void* stream) {
  COUNT(1);
  return wrap(gbk_scale_by_norm(n, a, norm2, which, y, y2, ST(stream)), "scale_by_norm");
}
int gb_box_apply(int L, int nr, int w, const double* B, const double* s, int mode,
                 const double* x, double* y, void* stream) {
  COUNT(1);
  return wrap(gbk_box_apply(L, nr, w, B, s, mode, x, y, ST(stream)), "box_apply");
}
int gb_apply_w(int Lp, const double* host_w12, const double* g, const double* s,
               double* out, void* stream) {
  COUNT(1);
  return wrap(gbk_apply_w(Lp, host_w12, g, s, out, ST(stream)), "apply_w");
}
int gb_apply_wt(int Lp, const double* host_w12, const double* w, double* v,
                void* stream) {
  COUNT(1);
  return wrap(gbk_apply_wt(Lp, host_w12, w, v, ST(stream)), "apply_wt");
}
int gb_apply_r(int Lp, int rho, const double* R, const double* g, double* out,
               void* stream) {
  COUNT(1);
  return wrap(gbk_apply_r(Lp, rho, R, g, out, ST(stream)), "apply_r");
}
int gb_psi_t_apply(int n, int L, int lo, int wd, const double* psi, const double* v,
                   double* inc, void* stream) {
  COUNT(1);
  return wrap(gbk_psi_t_apply(n, L, lo, wd, psi, v, inc, ST(stream)), "psi_t_apply");
}
int gb_psi_apply(int n, int L, int lo, int wd, const double* psi, const double* b,
                 double* out, void* stream) {
  COUNT(1);
  return wrap(gbk_psi_apply(n, L, lo, wd, psi, b, out, ST(stream)), "psi_apply");
}
int gb_axpby(int64_t n, double a, const double* x, double b, const double* y,
             double* out, void* stream) {
  COUNT(1);
  return wrap(gbk_axpby(n, a, x, b, y, out, ST(stream)), "axpby");
}
int gb_vmul(int64_t n, const double* a, const double* b, double* out, void* stream) {
  COUNT(1);
  return wrap(gbk_vmul(n, a, b, out, ST(stream)), "vmul");
}
int gb_vadd(int64_t n, const double* a, const double* b, double* out, void* stream) {
  COUNT(1);
  return wrap(gbk_vadd(n, a, b, out, ST(stream)), "vadd");
}

int gb_export_count(int kind, int L, int nr, int w, int nc, int n, int lo, int wd,
                    const double* val, int64_t rows, int64_t S, int64_t* counts,
                    void* stream) {
  COUNT(1);
  return wrap(gbk_export_count(kind, L, nr, w, nc, n, lo, wd, val, rows, S, LL(counts),
                               ST(stream)),
              "export_count");
}
int gb_exclusive_scan(const int64_t* counts, int64_t* indptr, int64_t n, void* tmp,
                      size_t* tmp_bytes, void* stream) {
  COUNT(1);
  return wrap(gbk_exclusive_scan(reinterpret_cast<const long long*>(counts), LL(indptr),
                                 n, tmp, tmp_bytes, ST(stream)),
              "exclusive_scan");
}
int gb_export_emit(int kind, int L, int nr, int w, int nc, int n, int lo, int wd,
                   const double* val, int64_t rows, int64_t S, const int64_t* indptr,
                   int32_t* indices, double* data, void* stream) {
  COUNT(1);
  return wrap(gbk_export_emit(kind, L, nr, w, nc, n, lo, wd, val, rows, S,
                              reinterpret_cast<const long long*>(indptr), indices, data,
                              ST(stream)),
              "export_emit");
}

int gb_dense_gemm(int m, int n, int k, double alpha, const double* A, int lda, int ta,
                  const double* B, int ldb, int tb, double beta, double* C, int ldc,
                  void* stream) {
  COUNT(1);
  return wrap(gbk_dense_gemm(m, n, k, alpha, A, lda, ta, B, ldb, tb, beta, C, ldc,
                             ST(stream)),
              "dense_gemm");
}
int gb_dense_potrf(int n, double* A, int lda, int64_t* status, void* stream) {
  COUNT(3 * ((n + 63) / 64) + 1);
  return wrap(gbk_dense_potrf(n, A, lda, LL(status), ST(stream)), "dense_potrf");
}
int gb_dense_potrs(int n, int nrhs, const double* L, int lda, double* B, int ldb,
                   void* stream) {
  COUNT(4 * ((n + 63) / 64));
  return wrap(gbk_dense_potrs(n, nrhs, L, lda, B, ldb, ST(stream)), "dense_potrs");
}
int gb_dense_sym(int n, const double* X, int ldx, double* out, double* stats,
                 void* stream) {
  COUNT(1);
  return wrap(gbk_dense_sym(n, X, ldx, out, stats, ST(stream)), "dense_sym");
}
int gb_dense_build_w(int Lk, const double* host_w12, double* out, void* stream) {
  COUNT(1);
  return wrap(gbk_dense_build_w(Lk, host_w12, out, ST(stream)), "dense_build_w");
}
int gb_dense_build_p(int Lk, double* out, double scale, void* stream) {
  COUNT(1);
  return wrap(gbk_dense_build_p(Lk, scale, out, ST(stream)), "dense_build_p");
}
int gb_csr_to_dense(int nrows, int ncols, const int32_t* indptr, const int32_t* indices,
                    const double* data, double* out, void* stream) {
  COUNT(1);
  return wrap(gbk_csr_to_dense(nrows, ncols, indptr, indices, data, out, ST(stream)),
              "csr_to_dense");
}
int gb_eye(int n, double* out, void* stream) {
  COUNT(1);
  return wrap(gbk_eye(n, out, ST(stream)), "eye");
}
int gb_fp64_peak_probe(int kind, int iters, double* sink, void* stream) {
  COUNT(1);
  return wrap(gbk_fp64_peak_probe(kind, iters, sink, ST(stream)), "fp64_peak_probe");
}


/* ---- config 4: 3-D box stencils (gb_3d.cu) ------------------------------ */
int gb3_csr_to_box(int L, int w, const int32_t* indptr, const int32_t* indices,
                   const double* data, double* box, int64_t* status, void* stream) {
  if (L <= 0 || w < 0) return invalid("gb3_csr_to_box: bad geometry");
  COUNT(1);
  return wrap(gbk3_csr_to_box(L, w, indptr, indices, data, box, LL(status), ST(stream)),
              "gb3_csr_to_box");
}
int gb3_box_scale(int64_t rows, int nr, int w, const double* box, double* s, int64_t* status,
                  void* stream) {
  COUNT(1);
  return wrap(gbk3_box_scale(rows, nr, w, box, s, LL(status), ST(stream)), "gb3_box_scale");
}
int gb3_box_sym_drop(int L, int nr, int w, const double* raw, double* out, double* dmin,
                     double* stats, void* stream) {
  if (raw == out) return invalid("gb3_box_sym_drop: in-place not supported");
  COUNT(2);
  return wrap(gbk3_box_sym_drop(L, nr, w, raw, out, dmin, stats, ST(stream)), "gb3_box_sym_drop");
}
int gb3_mass_patches(int L, const double* Ms, const double* s, int rho, int wd, double* psi,
                     int64_t* status, void* stream) {
  COUNT(1);
  const int rc = gbk3_mass_patches(L, Ms, s, rho, wd, psi, LL(status), ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("gb3_mass_patches: patch exceeds shared memory");
  return wrap(rc, "gb3_mass_patches");
}
int gb3_psi_galerkin(int L, int rho, int wd, const double* psi, const double* A, int wX,
                     double* X, int wR, double* raw, void* stream) {
  COUNT(2);
  return wrap(gbk3_psi_galerkin(L, rho, wd, psi, A, wX, X, wR, raw, ST(stream)),
              "gb3_psi_galerkin");
}
int gb3_level_blocks(int Lk, int wA, const double* A, const double* host_w, int wB, double* Braw,
                     double* G, double* PAPt, void* stream) {
  if (!host_w || Lk < 2) return invalid("gb3_level_blocks: bad arguments");
  COUNT(1);
  return wrap(gbk3_level_blocks(Lk, wA, A, host_w, wB, Braw, G, PAPt, ST(stream)),
              "gb3_level_blocks");
}
size_t gb3_correction_workspace(int Lp, int rho, int ctas) {
  return gbk3_correction_workspace(Lp, rho, ctas);
}
int gb3_correction_patches(int Lp, int wB, const double* B, const double* sB, const double* G,
                           int rho, double* Dt, int64_t* status, double* workspace, int ctas,
                           void* stream) {
  if (!workspace || ctas <= 0) return invalid("gb3_correction_patches: no workspace");
  COUNT(1);
  return wrap(gbk3_correction_patches(Lp, wB, B, sB, G, rho, Dt, LL(status), workspace, ctas,
                                      ST(stream)),
              "gb3_correction_patches");
}
int gb3_restriction(int Lp, int rho, const double* Dt, const double* host_w, double* R,
                    void* stream) {
  COUNT(1);
  return wrap(gbk3_restriction(Lp, rho, Dt, host_w, R, ST(stream)), "gb3_restriction");
}
int gb3_triple(int Lp, int wB, const double* B, const double* G, const double* PAPt, int rho,
               const double* Dt, int wBD, double* BD, int wGD, double* GtD, int wA2, double* raw,
               void* stream) {
  COUNT(3);
  return wrap(gbk3_triple(Lp, wB, B, G, PAPt, rho, Dt, wBD, BD, wGD, GtD, wA2, raw, ST(stream)),
              "gb3_triple");
}
int gb3_apply_w(int Lp, const double* host_w, const double* g, const double* s, double* out,
                void* stream) {
  COUNT(1);
  return wrap(gbk3_apply_w(Lp, host_w, g, s, out, ST(stream)), "gb3_apply_w");
}
int gb3_apply_wt(int Lp, const double* host_w, const double* w, double* v, void* stream) {
  COUNT(1);
  return wrap(gbk3_apply_wt(Lp, host_w, w, v, ST(stream)), "gb3_apply_wt");
}
int gb3_apply_r(int Lp, int rho, const double* R, const double* g, double* out, void* stream) {
  COUNT(1);
  return wrap(gbk3_apply_r(Lp, rho, R, g, out, ST(stream)), "gb3_apply_r");
}
int gb3_apply_rt(int Lp, int rho, const double* R, const double* u, double* out, void* stream) {
  COUNT(1);
  return wrap(gbk3_apply_rt(Lp, rho, R, u, out, ST(stream)), "gb3_apply_rt");
}
int gb3_psi_t_apply(int L, int rho, int wd, const double* psi, const double* v, double* out,
                    void* stream) {
  COUNT(1);
  return wrap(gbk3_psi_t_apply(L, rho, wd, psi, v, out, ST(stream)), "gb3_psi_t_apply");
}
int gb3_apply(int L, int nr, int w, const double* B, const double* s, const double* x, double* y,
              void* stream) {
  COUNT(1);
  return wrap(gbk3_apply(L, nr, w, B, s, x, y, ST(stream)), "gb3_apply");
}
int gb3_cg_solve(int L, int nr, int w, const double* B, const double* s, double* x, double* r,
                 double* p, double* Ap, void* state, double* partials, void* host_state,
                 int max_chunk, void* stream) {
  long long n = 0;
  const int e = gbk3_cg_solve(L, nr, w, B, s, x, r, p, Ap, state, partials, host_state,
                              max_chunk, ST(stream), &n);
  COUNT(n);
  return wrap(e, "gb3_cg_solve");
}
int gb3_lanczos_min(int L, int nr, int w, const double* B, const double* s, double* x,
                    double* vp, double* wv, void* state, double* partials, void* host_state,
                    double* ab, double* host_ab, int cap, double tol, int max_outer,
                    double lz_tol, double* lam, int* outer, int* its, void* stream) {
  if (!lam || !outer || !its || cap <= 0) return invalid("gb3_lanczos_min: bad arguments");
  long long n = 0;
  const int e = gbk3_lanczos_min(L, nr, w, B, s, x, vp, wv, state, partials, host_state, ab,
                                 host_ab, cap, tol, max_outer, lz_tol, lam, outer, its,
                                 ST(stream), &n);
  COUNT(n);
  if (e < 0) {
    snprintf(g_err, sizeof(g_err), "gb3_lanczos_min: %s",
             e == GB_UNSUPPORTED - 9 ? "A v_1 = 0 (inverse iteration breaks down)"
                                     : "nonpositive Ritz value or tridiagonal eigensolver failed");
    return GB_ERR_NUMERICAL;
  }
  return wrap(e, "gb3_lanczos_min");
}
int gb3_pow_solve(int L, int nr, int w, const double* B, const double* s, double* x, double* y,
                  double tol, void* state, double* partials, void* host_state, int max_chunk,
                  void* stream) {
  long long n = 0;
  const int e = gbk3_pow_solve(L, nr, w, B, s, x, y, tol, state, partials, host_state,
                               max_chunk, ST(stream), &n);
  COUNT(n);
  return wrap(e, "gb3_pow_solve");
}

// ---- row-strip entry points (multi-GPU partition) and the distributed Krylov pieces ----
size_t gb_psi_galerkin_workspace_rows(int n, int wd, int wX, int wR, int r0, int r1) {
  return gbk_psi_galerkin_workspace_rows(n, wd, wX, wR, r0, r1);
}
int gb_csr_to_box_rows(int n, int w, const int32_t* indptr, const int32_t* indices, const double* data, double* box, int64_t* status, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_csr_to_box_rows(n, w, indptr, indices, data, box, LL(status), r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("csr_to_box_rows: bad row range or unsupported configuration");
  return wrap(rc, "csr_to_box_rows");
}
int gb_box_sym_drop_rows(int L, int nr, int w, const double* raw, double* out, const double* dmin, double* stats, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_box_sym_drop_rows(L, nr, w, raw, out, dmin, stats, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("box_sym_drop_rows: bad row range or unsupported configuration");
  return wrap(rc, "box_sym_drop_rows");
}
int gb_psi_stencil_rows(int n, int lo, int wd, int rho, const double* psi, int wA, const double* A, int wX, double* X, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_psi_stencil_rows(n, lo, wd, rho, psi, wA, A, wX, X, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("psi_stencil_rows: bad row range or unsupported configuration");
  return wrap(rc, "psi_stencil_rows");
}
int gb_psi_galerkin_t_rows(int n, int lo, int wd, int rho, const double* psi, int wX, const double* X, int wR, double* raw, double* work, int r0, int r1, void* stream) {
  COUNT(3);
  const int rc = gbk_psi_galerkin_t_rows(n, lo, wd, rho, psi, wX, X, wR, raw, work, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("psi_galerkin_t_rows: bad row range or unsupported configuration");
  return wrap(rc, "psi_galerkin_t_rows");
}
int gb_level_diag_rows(int Lk, int wA, const double* A, const double* host_w12, double* bdiag, double* dmin, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_level_diag_rows(Lk, wA, A, host_w12, bdiag, dmin, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("level_diag_rows: bad row range or unsupported configuration");
  return wrap(rc, "level_diag_rows");
}
int gb_level_blocks_rows(int Lk, int wA, const double* A, const double* host_w12, int wB, const double* bdiag, const double* dmin, double* B, double* G, double* PAPt, double* stats, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_level_blocks_rows(Lk, wA, A, host_w12, wB, bdiag, dmin, B, G, PAPt, stats, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("level_blocks_rows: bad row range or unsupported configuration");
  return wrap(rc, "level_blocks_rows");
}
int gb_restriction_rows(int Lp, int rho, const double* Dt, const double* host_w12, double* R, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_restriction_rows(Lp, rho, Dt, host_w12, R, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("restriction_rows: bad row range or unsupported configuration");
  return wrap(rc, "restriction_rows");
}
int gb_bd_rows(int Lp, int wB, const double* B, int rho, const double* Dt, int wBD, double* BD, int r0, int r1, void* stream) {
  COUNT(2);
  const int rc = gbk_bd_rows(Lp, wB, B, rho, Dt, wBD, BD, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("bd_rows: bad row range or unsupported configuration");
  return wrap(rc, "bd_rows");
}
int gb_gtd_rows(int Lp, int wG, const double* G, int rho, const double* Dt, int wGD, double* GtD, int r0, int r1, void* stream) {
  COUNT(2);
  const int rc = gbk_gtd_rows(Lp, wG, G, rho, Dt, wGD, GtD, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("gtd_rows: bad row range or unsupported configuration");
  return wrap(rc, "gtd_rows");
}
int gb_coarse_raw_rows(int Lp, int wB, const double* PAPt, int wGD, const double* GtD, int rho, const double* Dt, int wBD, const double* BD, int wA2, double* raw, int r0, int r1, void* stream) {
  COUNT(2);
  const int rc = gbk_coarse_raw_rows(Lp, wB, PAPt, wGD, GtD, rho, Dt, wBD, BD, wA2, raw, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("coarse_raw_rows: bad row range or unsupported configuration");
  return wrap(rc, "coarse_raw_rows");
}
int gb_wpsi_rows(int n, int Lk, int lo, int wd, const double* host_w12, const double* psi, int wdw, double* Wpsi, int r0, int r1, int f0, int f1, void* stream) {
  COUNT(1);
  const int rc = gbk_wpsi_rows(n, Lk, lo, wd, host_w12, psi, wdw, Wpsi, r0, r1, f0, f1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("wpsi_rows: bad row range or unsupported configuration");
  return wrap(rc, "wpsi_rows");
}
int gb_psi_next_raw_rows(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw, const double* Wpsi, int rho, const double* Dt, int lo2, int wd2, double* psi_next, double* rowmax, int r0, int r1, int f0, int f1, void* stream) {
  COUNT(2);
  const int rc = gbk_psi_next_raw_rows(n, Lk, lo, hi, wd, psi, wdw, Wpsi, rho, Dt, lo2, wd2, psi_next, rowmax, r0, r1, f0, f1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("psi_next_raw_rows: bad row range or unsupported configuration");
  return wrap(rc, "psi_next_raw_rows");
}
int gb_psi_drop_rows(int n, int Lp, int lo2, int wd2, double* psi_next, const double* rowmax, int r0, int r1, int f0, int f1, void* stream) {
  COUNT(1);
  const int rc = gbk_psi_drop_rows(n, Lp, lo2, wd2, psi_next, rowmax, r0, r1, f0, f1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("psi_drop_rows: bad row range or unsupported configuration");
  return wrap(rc, "psi_drop_rows");
}
int gb_pad_rows(int L, int nr, int w, const double* src, const double* scale, double* dst, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_pad_rows(L, nr, w, src, scale, dst, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("pad_rows: bad row range or unsupported configuration");
  return wrap(rc, "pad_rows");
}
int gb_unpad_rows(int L, int nr, int w, const double* src, const double* scale, double* dst, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_unpad_rows(L, nr, w, src, scale, dst, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("unpad_rows: bad row range or unsupported configuration");
  return wrap(rc, "unpad_rows");
}
int gb_apply_w_rows(int Lp, const double* host_w12, const double* g, const double* s, double* out, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_apply_w_rows(Lp, host_w12, g, s, out, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("apply_w_rows: bad row range or unsupported configuration");
  return wrap(rc, "apply_w_rows");
}
int gb_apply_wt_rows(int Lp, const double* host_w12, const double* w, double* v, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_apply_wt_rows(Lp, host_w12, w, v, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("apply_wt_rows: bad row range or unsupported configuration");
  return wrap(rc, "apply_wt_rows");
}
int gb_apply_r_rows(int Lp, int rho, const double* R, const double* g, double* out, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_apply_r_rows(Lp, rho, R, g, out, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("apply_r_rows: bad row range or unsupported configuration");
  return wrap(rc, "apply_r_rows");
}
int gb_psi_t_apply_rows(int n, int L, int lo, int wd, const double* psi, const double* v, double* inc, int F0, int F1, int j_lo, int j_hi, void* stream) {
  COUNT(1);
  const int rc = gbk_psi_t_apply_rows(n, L, lo, wd, psi, v, inc, F0, F1, j_lo, j_hi, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("psi_t_apply_rows: bad row range or unsupported configuration");
  return wrap(rc, "psi_t_apply_rows");
}
int gb_bj_setup_rows(int L, int w, const double* B, const double* s, float* inv, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_bj_setup_rows(L, w, B, s, inv, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("bj_setup_rows: bad row range or unsupported configuration");
  return wrap(rc, "bj_setup_rows");
}
int gb_scale_box_symT_rows(int L, int w, const double* B, const double* s, double* UsT, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_scale_box_symT_rows(L, w, B, s, UsT, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("scale_box_symT_rows: bad row range or unsupported configuration");
  return wrap(rc, "scale_box_symT_rows");
}
int gb_dist_apply(int L, int w, const double* UsT, int nv, const double* x0, double* y0, void* st0, double* part0, const double* x1, double* y1, void* st1, double* part1, double* red, int r0, int r1, void* stream) {
  COUNT(2);
  const int rc = gbk_dist_apply(L, w, UsT, nv, x0, y0, st0, part0, x1, y1, st1, part1, red, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_apply: bad row range or unsupported configuration");
  return wrap(rc, "dist_apply");
}
int gb_dist_pcg_init(int L, int w, const double* b, double* x, double* r, double* p, double* z, const float* inv, void* st, double* part, double* out, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_dist_pcg_init(L, w, b, x, r, p, z, inv, st, part, out, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_pcg_init: bad row range or unsupported configuration");
  return wrap(rc, "dist_pcg_init");
}
int gb_dist_pcg_init_commit(void* st, const double* out, double rel_tol, int max_iter, void* stream) {
  COUNT(1);
  const int rc = gbk_dist_pcg_init_commit(st, out, rel_tol, max_iter, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_pcg_init_commit: bad row range or unsupported configuration");
  return wrap(rc, "dist_pcg_init_commit");
}
int gb_dist_pcg_update(int L, int w, double* x, double* r, const double* p, const double* Ap, double* z, const float* inv, void* st, const double* red, double* part, double* out, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_dist_pcg_update(L, w, x, r, p, Ap, z, inv, st, red, part, out, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_pcg_update: bad row range or unsupported configuration");
  return wrap(rc, "dist_pcg_update");
}
int gb_dist_pcg_commit_dir(int L, int w, void* st, const double* red, const double* out, const double* z, double* p, int r0, int r1, void* stream) {
  COUNT(2);
  const int rc = gbk_dist_pcg_commit_dir(L, w, st, red, out, z, p, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_pcg_commit_dir: bad row range or unsupported configuration");
  return wrap(rc, "dist_pcg_commit_dir");
}
int gb_dist_fix_yy(int L, int w, double* y, void* st, double* part, double* out, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_dist_fix_yy(L, w, y, st, part, out, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_fix_yy: bad row range or unsupported configuration");
  return wrap(rc, "dist_fix_yy");
}
int gb_dist_pow_step(int L, int w, double* x, const double* y, void* st, const double* red, const double* out_yy, double* out_res, double* part, double tol, int r0, int r1, int stage, void* stream) {
  COUNT(2);
  const int rc = gbk_dist_pow_step(L, w, x, y, st, red, out_yy, out_res, part, tol, r0, r1, stage, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_pow_step: bad row range or unsupported configuration");
  return wrap(rc, "dist_pow_step");
}
int gb_dist_lz_update(int L, int w, const double* x, double* y, double* vp, void* st, const double* red, double* part, double* out, int r0, int r1, void* stream) {
  COUNT(1);
  const int rc = gbk_dist_lz_update(L, w, x, y, vp, st, red, part, out, r0, r1, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_lz_update: bad row range or unsupported configuration");
  return wrap(rc, "dist_lz_update");
}
int gb_dist_lz_commit(void* st, const double* red, const double* out, double* ab, void* stream) {
  COUNT(1);
  const int rc = gbk_dist_lz_commit(st, red, out, ab, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_lz_commit: bad row range or unsupported configuration");
  return wrap(rc, "dist_lz_commit");
}
int gb_dist_lz_begin(void* st, int cap, void* stream) {
  COUNT(2);
  const int rc = gbk_dist_lz_begin(st, cap, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_lz_begin: bad row range or unsupported configuration");
  return wrap(rc, "dist_lz_begin");
}
int gb_dist_dot(int64_t n, const double* a, const double* b, void* st, double* part, double* out, void* stream) {
  COUNT(1);
  const int rc = gbk_dist_dot(n, a, b, st, part, out, ST(stream));
  if (rc == GB_UNSUPPORTED) return invalid("dist_dot: bad row range or unsupported configuration");
  return wrap(rc, "dist_dot");
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Host -> device upload of pageable host memory (the API's scipy inputs):
// chunks are copied into a process-wide pinned staging ring by several host
// threads and DMA'd asynchronously on `stream`, the next chunk's host copy
// overlapping the previous chunk's DMA.  A pageable cudaMemcpy is bounded by
// one driver memcpy thread.
// ---------------------------------------------------------------------------
#include <stdint.h>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace {
constexpr size_t kStageChunk = 16u << 20;
constexpr int kStageSlots = 3;
std::mutex g_stage_mu;
char* g_stage = nullptr;
cudaEvent_t g_stage_ev[kStageSlots];

// Persistent host threads of the staging copies: a job is a function of the
// piece index, pieces are handed out under the pool's lock, the caller takes
// pieces too and returns when all are done.  (Spawning threads per 16 MB chunk
// cost more than the chunk's copy: 23 GB/s; the pool reaches the DMA rate.)
class StagePool {
 public:
  static StagePool& get() {
    static StagePool* p = new StagePool();  // never destroyed: no join at exit
    return *p;
  }
  template <class F>
  void run(int pieces, int nthreads, F&& f) {
    if (pieces <= 1 || nthreads <= 1) {
      for (int i = 0; i < pieces; ++i) f(i);
      return;
    }
    grow(nthreads - 1);
    std::function<void(int)> fn = f;
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &fn;
      next_ = 0;
      total_ = pieces;
      left_ = pieces;
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    work(&fn);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return left_ == 0; });
    job_ = nullptr;
  }

 private:
  void grow(int n) {
    std::lock_guard<std::mutex> lk(mu_);
    while ((int)th_.size() < n && th_.size() < 32) {
      th_.emplace_back([this] { loop(); });
      th_.back().detach();
    }
  }
  // take pieces of the current job until none is left
  void work(std::function<void(int)>* fn) {
    for (;;) {
      int i;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (job_ != fn || next_ >= total_) return;
        i = next_++;
      }
      (*fn)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--left_ == 0) done_.notify_all();
    }
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      // a transfer issues its chunks back to back: spin for the next one
      // (~0.5 ms) before sleeping, a condition-variable wake-up costs as
      // much as a chunk's copy on these hosts
      for (int spin = 0; spin < 20000 && gen_.load(std::memory_order_acquire) == seen; ++spin)
        cpu_relax();
      std::function<void(int)>* fn;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load(std::memory_order_relaxed) != seen; });
        seen = gen_.load(std::memory_order_relaxed);
        fn = job_;
      }
      if (fn) work(fn);
    }
  }
  static void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#else
    std::this_thread::yield();
#endif
  }
  std::mutex mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> th_;
  std::function<void(int)>* job_ = nullptr;
  int next_ = 0, total_ = 0, left_ = 0;
  std::atomic<unsigned long long> gen_{0};
};

constexpr size_t kStagePiece = 1u << 20;  // bytes per piece of a staging copy

void par_memcpy(char* dst, const char* src, size_t bytes, int nthreads) {
  if (nthreads <= 1 || bytes < (1u << 20)) {
    memcpy(dst, src, bytes);
    return;
  }
  const int pieces = (int)((bytes + kStagePiece - 1) / kStagePiece);
  StagePool::get().run(pieces, nthreads, [=](int i) {
    const size_t off = (size_t)i * kStagePiece;
    memcpy(dst + off, src + off, off + kStagePiece <= bytes ? kStagePiece : bytes - off);
  });
}
}  // namespace

// narrowing copy int64 -> int32 by several threads; false if a value does not fit
bool par_narrow(int32_t* dst, const int64_t* src, size_t count, int nthreads) {
  const size_t per = kStagePiece / sizeof(int32_t);
  const int pieces = (int)((count + per - 1) / per);
  std::vector<char> okv((size_t)(pieces > 0 ? pieces : 1), 1);
  char* ok = okv.data();
  StagePool::get().run(pieces, nthreads < 1 ? 1 : nthreads, [=](int p) {
    const size_t off = (size_t)p * per;
    const size_t len = off + per <= count ? per : count - off;
    bool good = true;
    for (size_t i = 0; i < len; ++i) {
      const int64_t v = src[off + i];
      good = good && v >= INT32_MIN && v <= INT32_MAX;
      dst[off + i] = (int32_t)v;
    }
    ok[p] = good;
  });
  for (char c : okv)
    if (!c) return false;
  return true;
}

static int h2d_staged(void* dst, const void* src, int64_t count, int elem_in, int elem_out,
                      int nthreads, void* stream);

int gb_h2d_staged(void* dst, const void* src, int64_t bytes, int nthreads, void* stream) {
  return h2d_staged(dst, src, bytes, 1, 1, nthreads, stream);
}

int gb_h2d_staged_i64_i32(int32_t* dst, const int64_t* src, int64_t count, int nthreads,
                          void* stream) {
  return h2d_staged(dst, src, count, 8, 4, nthreads, stream);
}

// count elements of elem_in bytes -> elem_out bytes (1/1: raw bytes, 8/4: int64 -> int32)
static int h2d_staged(void* dst, const void* src, int64_t count, int elem_in, int elem_out,
                      int nthreads, void* stream) {
  if (count < 0 || (count > 0 && (!dst || !src))) return invalid("h2d_staged: bad arguments");
  if (nthreads < 1) nthreads = 1;
  std::lock_guard<std::mutex> lock(g_stage_mu);
  cudaError_t e;
  if (!g_stage) {
    e = cudaHostAlloc((void**)&g_stage, kStageChunk * kStageSlots, cudaHostAllocDefault);
    if (e != cudaSuccess) return wrap((int)e, "h2d_staged: cudaHostAlloc");
    for (int i = 0; i < kStageSlots; ++i) {
      e = cudaEventCreateWithFlags(&g_stage_ev[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return wrap((int)e, "h2d_staged: event");
      cudaEventRecord(g_stage_ev[i], 0);
    }
  }
  int slot = 0;
  const int64_t chunk = (int64_t)(kStageChunk / (size_t)elem_out);  // elements per chunk
  for (int64_t off = 0; off < count; off += chunk, slot = (slot + 1) % kStageSlots) {
    const int64_t cnt = count - off < chunk ? count - off : chunk;
    const size_t len = (size_t)cnt * (size_t)elem_out;
    char* buf = g_stage + (size_t)slot * kStageChunk;
    e = cudaEventSynchronize(g_stage_ev[slot]);  // the slot's previous DMA is done
    if (e != cudaSuccess) return wrap((int)e, "h2d_staged: sync");
    if (elem_in == elem_out) {
      par_memcpy(buf, (const char*)src + off * elem_in, len, nthreads);
    } else if (!par_narrow((int32_t*)buf, (const int64_t*)src + off, (size_t)cnt, nthreads)) {
      return invalid("h2d_staged: index does not fit in int32");
    }
    e = cudaMemcpyAsync((char*)dst + off * elem_out, buf, len, cudaMemcpyHostToDevice,
                        ST(stream));
    if (e != cudaSuccess) return wrap((int)e, "h2d_staged: copy");
    e = cudaEventRecord(g_stage_ev[slot], ST(stream));
    if (e != cudaSuccess) return wrap((int)e, "h2d_staged: record");
  }
  return 0;
}
