// Internal launcher prototypes (C++ linkage); the public C ABI wraps these in
// gb_capi.cu and is declared in include/gamblets_b200.h.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

// launcher status: 0 ok, > 0 a cudaError_t, GB_UNSUPPORTED when no kernel of
// the family covers the arguments (the caller picks another variant)
#define GB_UNSUPPORTED (-1)

enum { EXP_SQUARE = 0, EXP_CHILD = 1, EXP_PSI = 2, EXP_TDT = 3 };

// gb_box.cu
int gbk_assemble_q1(int n, const double* cell_scale, double const_scale, const double* host_e16,
                    double* box, cudaStream_t s);
int gbk_box1_matvec(int n, const double* box, const double* g, double* b, cudaStream_t s);
int gbk_csr_halfwidth(int n, const int32_t* indptr, const int32_t* indices, int* out,
                      cudaStream_t s);
int gbk_csr_to_box(int n, int w, const int32_t* indptr, const int32_t* indices,
                   const double* data, double* box, long long* status, cudaStream_t s);
int gbk_box_scale(long long rows, int nr, int w, const double* box, double* sv,
                  long long* status, cudaStream_t s);
int gbk_box_diag_min(long long rows, int nr, int w, const double* box, double* dmin,
                     cudaStream_t s);
int gbk_box_sym_drop(int L, int nr, int w, const double* raw, double* out,
                     const double* dmin, double* stats, cudaStream_t s);
int gbk_row_tail_drop(long long rows, long long S, double* v, cudaStream_t s);
int gbk_export_count(int kind, int L, int nr, int w, int nc, int n, int lo, int wd,
                     const double* val, long long rows, long long S, long long* counts,
                     cudaStream_t s);
int gbk_exclusive_scan(const long long* counts, long long* indptr, long long n, void* tmp,
                       size_t* tmp_bytes, cudaStream_t s);
int gbk_export_emit(int kind, int L, int nr, int w, int nc, int n, int lo, int wd,
                    const double* val, long long rows, long long S,
                    const long long* indptr, int32_t* indices, double* data,
                    cudaStream_t s);

// gb_patch.cu
size_t gbk_mass_patch_workspace(int rho, int blocks);
int gbk_mass_patches(int n, int wM, const double* M, const double* s, int rho, int wd,
                     double* psi, long long* status, double* gws, int blocks,
                     cudaStream_t st);
size_t gbk_correction_workspace(int rho, int blocks);
int gbk_correction_patches(int Lp, int wB, const double* B, const double* sB, int wG,
                           const double* G, int rho, double* Dt, long long* status,
                           double* gws, int blocks, cudaStream_t st);

// gb_products.cu
int gbk_psi_stencil(int n, int lo, int wd, int rho, const double* psi, int wA,
                    const double* A, int wX, double* X, cudaStream_t s);
size_t gbk_psi_galerkin_workspace(int n, int wd, int wX);
size_t gbk_psi_galerkin_workspace_rows(int n, int wd, int wX, int wR, int r0, int r1);
int gbk_psi_galerkin_t(int n, int lo, int wd, int rho, const double* psi, int wX,
                       const double* X, int wR, double* raw, double* work, cudaStream_t s);
int gbk_psi_galerkin(int n, int lo, int wd, int rho, const double* psi, int wX,
                     const double* X, int wR, double* raw, cudaStream_t s);
int gbk_level_diag(int Lk, int wA, const double* A, const double* w12, double* bdiag,
                   double* dmin, cudaStream_t s);
int gbk_level_blocks(int Lk, int wA, const double* A, const double* w12, int wB,
                     const double* bdiag, const double* dmin, double* B, double* G,
                     double* PAPt, double* stats, cudaStream_t s);
int gbk_restriction(int Lp, int rho, const double* Dt, const double* w12, double* R,
                    cudaStream_t s);
int gbk_bd(int Lp, int wB, const double* B, int rho, const double* Dt, int wBD,
           double* BD, cudaStream_t s);
int gbk_gtd(int Lp, int wG, const double* G, int rho, const double* Dt, int wGD,
            double* GtD, cudaStream_t s);
int gbk_coarse_raw(int Lp, int wB, const double* PAPt, int wGD, const double* GtD,
                   int rho, const double* Dt, int wBD, const double* BD, int wA2,
                   double* raw, cudaStream_t s);
int gbk_wpsi(int n, int Lk, int lo, int wd, const double* w12, const double* psi,
             int wdw, double* Wpsi, cudaStream_t s);
int gbk_psi_next(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw,
                 const double* Wpsi, int rho, const double* Dt, int lo2, int wd2,
                 double* psi_next, double* rowmax, cudaStream_t s);

// gb_krylov.cu
size_t gbk_kstate_bytes();
int gbk_red_blocks();
int gbk_state_reset(void* st, int max_iter, cudaStream_t s);
int gbk_cg_init(long long n, const double* b, const double* x0, const double* Ax0,
                double* x, double* r, double* p, double rel_tol, int max_iter, void* st,
                double* part, cudaStream_t s);
int gbk_cg_iterations(int L, int nr, int w, const double* B, const double* sv, int mode,
                      double* x, double* r, double* p, double* Ap, int iters, void* st,
                      double* part, cudaStream_t s);
int gbk_pow_iterations(int L, int nr, int w, const double* B, const double* sv, int mode,
                       double* x, double* y, double tol, int iters, void* st,
                       double* part, cudaStream_t s);
int gbk_dot2(long long n, const double* a, const double* b, const double* c, double* out,
             void* st, double* part, cudaStream_t s);
int gbk_scale_by_norm(long long n, const double* a, const double* norm2, int which,
                      double* y, double* y2, cudaStream_t s);
int gbk_box_apply(int L, int nr, int w, const double* B, const double* sv, int mode,
                  const double* x, double* y, cudaStream_t s);
int gbk_apply_w(int Lp, const double* w12, const double* g, const double* sv, double* out,
                cudaStream_t s);
int gbk_apply_wt(int Lp, const double* w12, const double* w, double* v, cudaStream_t s);
int gbk_apply_r(int Lp, int rho, const double* R, const double* g, double* out,
                cudaStream_t s);
int gbk_psi_t_apply(int n, int L, int lo, int wd, const double* psi, const double* v,
                    double* inc, cudaStream_t s);
int gbk_axpby(long long n, double a, const double* x, double b, const double* y,
              double* out, cudaStream_t s);
int gbk_vmul(long long n, const double* a, const double* b, double* out, cudaStream_t s);
int gbk_vadd(long long n, const double* a, const double* b, double* out, cudaStream_t s);
int gbk_psi_apply(int n, int L, int lo, int wd, const double* psi, const double* b,
                  double* out, cudaStream_t s);
int gbk_scale_box(int L, int nr, int w, const double* B, const double* sv, double* Bs,
                  cudaStream_t s);
int gbk_pad(int L, int nr, int w, const double* src, const double* scale, double* dst,
            cudaStream_t s);
int gbk_unpad(int L, int nr, int w, const double* src, const double* scale, double* dst,
              cudaStream_t s);
int gbk_pcg_iterations(int L, int nr, int w, const double* Bs, double* x, double* r,
                       double* p, double* Ap, int iters, void* st, double* part,
                       cudaStream_t s);
int gbk_ppow_iterations(int L, int nr, int w, const double* Bs, double* x, double* y,
                        double tol, int iters, void* st, double* part, cudaStream_t s);
int gbk_pbox_apply(int L, int nr, int w, const double* Bs, const double* x, double* y,
                   cudaStream_t s);
int gbk_psi_next_rows(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw,
                      const double* Wpsi, int rho, const double* Dt, int lo2, int wd2,
                      double* psi_next, double* rowmax, int r0, int r1, cudaStream_t s);
int gbk_correction_patches_rows(int Lp, int wB, const double* B, const double* sB, int wG,
                                const double* G, int rho, double* Dt, long long* status, int r0,
                                int r1, double* ws, size_t ws_bytes, cudaStream_t st);
size_t gbk_correction_v3_workspace(int Lp, int rho, int r0, int r1);
int gbk_mass_patches_rows(int n, int wM, const double* M, const double* s, int rho, int wd,
                          double* psi, long long* status, int r0, int r1, cudaStream_t st);
int gbk_correction_patches_v2(int Lp, int wB, const double* Bs, const double* sB, int wG,
                              const double* G, int rho, double* Dt, long long* status,
                              double* ws, size_t ws_bytes, cudaStream_t st);
int gbk_mass_patches_v2(int n, int wM, const double* Ms, const double* s, int rho, int wd,
                        double* psi, long long* status, cudaStream_t st);
int gbk_scale_box_T(int L, int nr, int w, const double* B, const double* sv, double* BsT,
                    cudaStream_t s);
int gbk_tcg_iterations(int L, int nr, int w, const double* BsT, double* x, double* r,
                       double* p, double* Ap, int iters, void* st, double* part,
                       cudaStream_t s, int layout);
int gbk_tpow_iterations(int L, int nr, int w, const double* BsT, double* x, double* y,
                        double tol, int iters, void* st, double* part, cudaStream_t s,
                        int layout);
int gbk_tbox_apply(int L, int nr, int w, const double* BsT, const double* x, double* y,
                   cudaStream_t s, int layout);
size_t gbk_boxT_elems(int L, int nr, int w);
int gbk_bj_setup(int L, int w, const double* B, const double* sv, float* inv,
                 cudaStream_t s);
int gbk_bjcg_init(int L, int w, const double* b, const double* x0, const double* Ax0,
                  double x0_scale, double* x, double* r, double* p, double* z, const float* inv,
                  double rel_tol, int max_iter, void* st, double* part, cudaStream_t s);
int gbk_bjcg_iterations(int L, int w, const double* BsT, const float* inv, double* x,
                        double* r, double* p, double* Ap, double* z, int iters, void* st,
                        double* part, cudaStream_t s, int layout);
int gbk_sync_read(const void* dev, void* host, size_t bytes, cudaStream_t s);
int gbk_tcg_solve(int L, int nr, int w, const double* BsT, double* x, double* r, double* p,
                  double* Ap, void* st, double* part, void* host_state, int max_chunk,
                  cudaStream_t s, long long* launches, int layout);
int gbk_bjcg_solve2(int L, int w, const double* BsT, const float* inv, double* const* x,
                    double* const* r, double* const* p, double* const* Ap, double* const* z,
                    void* const* st, double* const* part, void* const* host_state,
                    int max_chunk, cudaStream_t s, long long* launches);
int gbk_bjcg_solve(int L, int w, const double* BsT, const float* inv, double* x, double* r,
                   double* p, double* Ap, double* z, void* st, double* part, void* host_state,
                   int max_chunk, cudaStream_t s, long long* launches, int layout);
int gbk_tpow_solve(int L, int nr, int w, const double* BsT, double* x, double* y, double tol,
                   void* st, double* part, void* host_state, int max_chunk, cudaStream_t s,
                   long long* launches, int layout);
size_t gbk_boxsym_elems(int L, int w);
size_t gbk_sym_overflow_elems(int L, int w);
int gbk_sym_supported(int L, int nr, int w);
int gbk_scale_box_symT(int L, int w, const double* B, const double* sv, double* UsT,
                       cudaStream_t s);
int gbk_csr_apply(long long n, const int32_t* indptr, const int32_t* indices,
                  const double* data, const double* x, double* y, cudaStream_t s);
int gbk_csr_cg_solve(long long n, const int32_t* indptr, const int32_t* indices,
                     const double* data, double* x, double* r, double* p, double* Ap,
                     void* st, double* part, void* host_state, int max_chunk, cudaStream_t s,
                     long long* launches);
int gbk_csr_pow_solve(long long n, const int32_t* indptr, const int32_t* indices,
                      const double* data, double* x, double* y, double tol, void* st,
                      double* part, void* host_state, int max_chunk, cudaStream_t s,
                      long long* launches);
#include "gb_engine.h"
int gbk_level_engine(gb_level_engine_args* e, cudaStream_t s, long long* launches);
int gbk_products_mode(int mma);
int gbk_tune(int what, int value);

// row-strip variants (gb_box.cu, gb_products.cu, gb_krylov.cu) and gb_dist.cuh launchers
int gbk_csr_to_box_rows(int n, int w, const int32_t* indptr, const int32_t* indices, const double* data, double* box, long long* status, int r0, int r1, cudaStream_t st_);
int gbk_box_sym_drop_rows(int L, int nr, int w, const double* raw, double* out, const double* dmin, double* stats, int r0, int r1, cudaStream_t st_);
int gbk_psi_stencil_rows(int n, int lo, int wd, int rho, const double* psi, int wA, const double* A, int wX, double* X, int r0, int r1, cudaStream_t st_);
int gbk_psi_galerkin_t_rows(int n, int lo, int wd, int rho, const double* psi, int wX, const double* X, int wR, double* raw, double* work, int r0, int r1, cudaStream_t st_);
int gbk_level_diag_rows(int Lk, int wA, const double* A, const double* host_w12, double* bdiag, double* dmin, int r0, int r1, cudaStream_t st_);
int gbk_level_blocks_rows(int Lk, int wA, const double* A, const double* host_w12, int wB, const double* bdiag, const double* dmin, double* B, double* G, double* PAPt, double* stats, int r0, int r1, cudaStream_t st_);
int gbk_restriction_rows(int Lp, int rho, const double* Dt, const double* host_w12, double* R, int r0, int r1, cudaStream_t st_);
int gbk_bd_rows(int Lp, int wB, const double* B, int rho, const double* Dt, int wBD, double* BD, int r0, int r1, cudaStream_t st_);
int gbk_gtd_rows(int Lp, int wG, const double* G, int rho, const double* Dt, int wGD, double* GtD, int r0, int r1, cudaStream_t st_);
int gbk_coarse_raw_rows(int Lp, int wB, const double* PAPt, int wGD, const double* GtD, int rho, const double* Dt, int wBD, const double* BD, int wA2, double* raw, int r0, int r1, cudaStream_t st_);
int gbk_wpsi_rows(int n, int Lk, int lo, int wd, const double* host_w12, const double* psi, int wdw, double* Wpsi, int r0, int r1, int f0, int f1, cudaStream_t st_);
int gbk_psi_next_raw_rows(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw, const double* Wpsi, int rho, const double* Dt, int lo2, int wd2, double* psi_next, double* rowmax, int r0, int r1, int f0, int f1, cudaStream_t st_);
int gbk_psi_drop_rows(int n, int Lp, int lo2, int wd2, double* psi_next, const double* rowmax, int r0, int r1, int f0, int f1, cudaStream_t st_);
int gbk_pad_rows(int L, int nr, int w, const double* src, const double* scale, double* dst, int r0, int r1, cudaStream_t st_);
int gbk_unpad_rows(int L, int nr, int w, const double* src, const double* scale, double* dst, int r0, int r1, cudaStream_t st_);
int gbk_apply_w_rows(int Lp, const double* host_w12, const double* g, const double* s, double* out, int r0, int r1, cudaStream_t st_);
int gbk_apply_wt_rows(int Lp, const double* host_w12, const double* w, double* v, int r0, int r1, cudaStream_t st_);
int gbk_apply_r_rows(int Lp, int rho, const double* R, const double* g, double* out, int r0, int r1, cudaStream_t st_);
int gbk_psi_t_apply_rows(int n, int L, int lo, int wd, const double* psi, const double* v, double* inc, int F0, int F1, int j_lo, int j_hi, cudaStream_t st_);
int gbk_bj_setup_rows(int L, int w, const double* B, const double* s, float* inv, int r0, int r1, cudaStream_t st_);
int gbk_scale_box_symT_rows(int L, int w, const double* B, const double* s, double* UsT, int r0, int r1, cudaStream_t st_);
int gbk_dist_apply(int L, int w, const double* UsT, int nv, const double* x0, double* y0, void* st0, double* part0, const double* x1, double* y1, void* st1, double* part1, double* red, int r0, int r1, cudaStream_t st_);
int gbk_dist_pcg_init(int L, int w, const double* b, double* x, double* r, double* p, double* z, const float* inv, void* st, double* part, double* out, int r0, int r1, cudaStream_t st_);
int gbk_dist_pcg_init_commit(void* st, const double* out, double rel_tol, int max_iter, cudaStream_t st_);
int gbk_dist_pcg_update(int L, int w, double* x, double* r, const double* p, const double* Ap, double* z, const float* inv, void* st, const double* red, double* part, double* out, int r0, int r1, cudaStream_t st_);
int gbk_dist_pcg_commit_dir(int L, int w, void* st, const double* red, const double* out, const double* z, double* p, int r0, int r1, cudaStream_t st_);
int gbk_dist_fix_yy(int L, int w, double* y, void* st, double* part, double* out, int r0, int r1, cudaStream_t st_);
int gbk_dist_pow_step(int L, int w, double* x, const double* y, void* st, const double* red, const double* out_yy, double* out_res, double* part, double tol, int r0, int r1, int stage, cudaStream_t st_);
int gbk_dist_lz_update(int L, int w, const double* x, double* y, double* vp, void* st, const double* red, double* part, double* out, int r0, int r1, cudaStream_t st_);
int gbk_dist_lz_commit(void* st, const double* red, const double* out, double* ab, cudaStream_t st_);
int gbk_dist_lz_begin(void* st, int cap, cudaStream_t st_);
int gbk_dist_dot(long long n, const double* a, const double* b, void* st, double* part, double* out, cudaStream_t st_);

// gb_diag.cu
int gbk_cell_energies(int n, const double* v, const double* coef, const double* host_e16,
                      double* out, cudaStream_t s);
size_t gbk_decay_part_elems(int nr);
int gbk_decay_sums(int n, double h, const double* en, double cx, double cy, const double* radii,
                   int nr, double* part, double* out, cudaStream_t s);
int gbk_box_diag_spectrum(long long rows, int nr, int w, const double* box, const double* coef,
                          double* out, cudaStream_t s);
int gbk_topk_mask(long long n, const double* mags, long long n_keep, double* mask, void* work,
                  size_t* work_bytes, cudaStream_t s);
size_t gbk_quad_part_elems();
int gbk_box_quadform(int L, int w, const double* box, const double* x, double* part, double* out,
                     cudaStream_t s);
int gbk_max_abs(long long n, const double* x, double* part, double* out, cudaStream_t s);

// gb_3d.cu (config 4, 3-D box stencils) and the 3-D operator of gb_krylov.cu
int gbk3_csr_to_box(int L, int w, const int32_t* indptr, const int32_t* indices,
                    const double* data, double* box, long long* status, cudaStream_t s);
int gbk3_box_scale(long long rows, int nr, int w, const double* box, double* sv,
                   long long* status, cudaStream_t s);
int gbk3_box_sym_drop(int L, int nr, int w, const double* raw, double* out, double* dmin,
                      double* stats, cudaStream_t s);
size_t gbk3_mass_smem(int rho);
int gbk3_mass_patches(int L, const double* M, const double* sv, int rho, int wd, double* psi,
                      long long* status, cudaStream_t s);
int gbk3_psi_galerkin(int L, int rho, int wd, const double* psi, const double* A, int wX,
                      double* X, int wR, double* raw, cudaStream_t s);
int gbk3_level_blocks(int Lk, int wA, const double* A, const double* host_w, int wB,
                      double* Braw, double* G, double* PAPt, cudaStream_t s);
int gbk3_correction_ld(int rho);
size_t gbk3_correction_workspace(int Lp, int rho, int ctas);
int gbk3_correction_patches(int Lp, int wB, const double* B, const double* sB, const double* G,
                            int rho, double* Dt, long long* status, double* ws, int ctas,
                            cudaStream_t s);
int gbk3_restriction(int Lp, int rho, const double* Dt, const double* host_w, double* Rv,
                     cudaStream_t s);
int gbk3_triple(int Lp, int wB, const double* B, const double* G, const double* PAPt, int rho,
                const double* Dt, int wBD, double* BD, int wGD, double* GtD, int wA2,
                double* raw, cudaStream_t s);
int gbk3_apply_w(int Lp, const double* host_w, const double* g, const double* sv, double* out,
                 cudaStream_t s);
int gbk3_apply_wt(int Lp, const double* host_w, const double* w, double* v, cudaStream_t s);
int gbk3_apply_r(int Lp, int rho, const double* Rv, const double* g, double* out,
                 cudaStream_t s);
int gbk3_apply_rt(int Lp, int rho, const double* Rv, const double* u, double* out,
                  cudaStream_t s);
int gbk3_psi_t_apply(int L, int rho, int wd, const double* psi, const double* v, double* out,
                     cudaStream_t s);
int gbk3_apply(int L, int nr, int w, const double* B, const double* sv, const double* x,
               double* y, cudaStream_t s);
int gbk3_cg_solve(int L, int nr, int w, const double* B, const double* sv, double* x, double* r,
                  double* p, double* Ap, void* st, double* part, void* host_state, int max_chunk,
                  cudaStream_t s, long long* launches);
int gbk3_pow_solve(int L, int nr, int w, const double* B, const double* sv, double* x,
                   double* y, double tol, void* st, double* part, void* host_state,
                   int max_chunk, cudaStream_t s, long long* launches);
int gbk3_lanczos_min(int L, int nr, int w, const double* B, const double* sv, double* x,
                     double* vp, double* wv, void* st, double* part, void* host_state,
                     double* ab, double* hab, int cap, double tol, int max_outer,
                     double lz_tol, double* lam_out, int* outer_out, int* its_out,
                     cudaStream_t s, long long* launches);
