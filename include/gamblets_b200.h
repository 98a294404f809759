/* C ABI of libgamblets_b200.so -- the drop-in boundary of the B200 gamblet
 * hot path (arXiv 1503.03467; reference: /root/reference/pkg/src/gamblets).
 *
 * The reference is a pure-Python package with no FFI of its own; its boundary
 * is the Python API re-exported in gamblets/__init__.py:10-94.  This library
 * sits *under* a Python shim (paper_1503_03467_b200) that keeps those
 * signatures and binds these symbols with ctypes.  Each
 * entry point below names the reference call site it replaces.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer (cudaMalloc / torch storage) unless
 *     named host_*; sizes are plain ints; `stream` is a cudaStream_t passed
 *     as void*; calls are asynchronous on that stream.
 *   - return value: GB_OK, GB_ERR_INVALID (bad argument, the shim raises
 *     InvalidArgumentError) or GB_ERR_CUDA (launch failure; message in
 *     gb_last_error()).  Numerical failures found on the device (nonpositive
 *     diagonal, non-SPD patch, CG breakdown) are written to the caller's
 *     int64 status block {code, detail}; the shim raises NumericalError.
 *   - box-stencil layout of every level operator: see
 *     paper_1503_03467_b200/csrc/gb_common.cuh and DESIGN.md section 3.
 */
#ifndef GAMBLETS_B200_H
#define GAMBLETS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GB_OK 0
#define GB_ERR_INVALID 1
#define GB_ERR_NUMERICAL 2
#define GB_ERR_CUDA 3

/* device status codes (status[0]) */
#define GB_ST_NONPOS_DIAG 1
#define GB_ST_NOT_SPD 2
#define GB_ST_OUTSIDE_BOX 3
#define GB_ST_CG_BREAKDOWN 4

/* CSR export kinds */
#define GB_EXP_SQUARE 0
#define GB_EXP_CHILD 1
#define GB_EXP_PSI 2
#define GB_EXP_TDT 3

int gb_abi_version(void);
/* kernels launched through this ABI since load (for the bench's gpu_launches) */
unsigned long long gb_launch_count(void);
const char* gb_last_error(void);
int gb_device_count(void);

/* ---- input conversion: canonical CSR (fine grid side n) -> box ----------
 * replaces as_csr(M)/as_csr(A) in fast_transform (gamblet_fast.py:645-646)
 * and the implicit 9-point stencil of grid_fem._assemble (grid_fem.py:205-214) */
int gb_csr_halfwidth(int n, const int32_t* indptr, const int32_t* indices,
                     int32_t* out_w, void* stream);
int gb_csr_to_box(int n, int w, const int32_t* indptr, const int32_t* indices,
                  const double* data, double* box, int64_t* status, void* stream);

/* ---- host input upload -------------------------------------------------
 * bytes of pageable host memory -> device, staged through a pinned ring by
 * nthreads host threads, DMA asynchronous on `stream` (ordered before later
 * work on that stream). */
int gb_h2d_staged(void* dst, const void* src, int64_t bytes, int nthreads, void* stream);
/* the same for count int64 host indices narrowed to int32 on the way (scipy
 * int64 CSR indices; 1 = a value outside int32) */
int gb_h2d_staged_i64_i32(int32_t* dst, const int64_t* src, int64_t count, int nthreads,
                          void* stream);

/* ---- on-device Q1 assembly (replaces grid_fem.py:189-227 _assemble /
 * assemble_mass / assemble_stiffness and the b = M g of assemble_load,
 * grid_fem.py:238-245) ---------------------------------------------------
 * box: n*n rows x 9 slots (half-width-1 box, slot (ds+1)*3 + (dt+1)); entry =
 * sum over the adjacent cells in increasing flat cell order of
 * scale[cell] * E[r][c] (cell_scale == NULL: const_scale for every cell),
 * host_e16 = the 4x4 element matrix (corners SW, SE, NE, NW), row major.
 * Bitwise equal to the reference's canonical CSR values. */
int gb_assemble_q1(int n, const double* cell_scale, double const_scale, const double* host_e16,
                   double* box, void* stream);
/* b = M g for a half-width-1 box in scipy csr_matvec order (bitwise) */
int gb_box1_matvec(int n, const double* box, const double* g, double* b, void* stream);

/* ---- unit-diagonal congruence s = diag^-1/2 (gamblet_fast.py:123-139) ---- */
int gb_box_scale(int64_t rows, int nr, int w, const double* box, double* s,
                 int64_t* status, void* stream);

/* ---- symmetrize + dead-tail drop (gamblet_exact.py:95-103,
 *      gamblet_fast.py:154-169); dmin preset to +inf, stats to 0 ------------ */
int gb_box_diag_min(int64_t rows, int nr, int w, const double* box, double* dmin,
                    void* stream);
int gb_box_sym_drop(int L, int nr, int w, const double* raw, double* out,
                    const double* dmin, double* stats, void* stream);
/* row-tail drop (gamblet_fast.py:172-190) on dense row windows */
int gb_row_tail_drop(int64_t rows, int64_t S, double* v, void* stream);

/* ---- K1 mass patches: local_mass_inverse (gamblet_fast.py:464-498) ------- */
size_t gb_mass_patch_workspace(int rho, int blocks);
int gb_mass_patches(int n, int wM, const double* M, const double* s, int rho, int wd,
                    double* psi, int64_t* status, double* workspace, int blocks,
                    void* stream);

/* v2: tiled DMMA Cholesky in shared memory on the pre-scaled S M S box
 * (gb_scale_box); GB_ERR_INVALID when the patch does not fit (use v1) */
int gb_mass_patches_v2(int n, int wM, const double* Ms, const double* s, int rho, int wd,
                       double* psi, int64_t* status, void* stream);

/* spatial strips (multi-GPU row partition): the same
 * patch solves restricted to grid rows [r0, r1) of the patch centres
 * (fine rows for the mass patches, parent rows for the correction
 * patches); output rows outside the strip are not written.  The union of
 * the strips of a partition equals the whole-level call bitwise. */
int gb_mass_patches_rows(int n, int wM, const double* Ms, const double* s, int rho, int wd,
                         double* psi, int64_t* status, int r0, int r1, void* stream);
int gb_correction_patches_rows(int Lp, int wB, const double* Bs, const double* sB, int wG,
                               const double* G, int rho, double* Dt, int64_t* status, int r0,
                               int r1, double* workspace, size_t workspace_bytes, void* stream);
/* psi^(k-1) rows of the parents in rows [r0, r1) (gb_psi_next, strip form) */
int gb_psi_next_rows(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw,
                     const double* Wpsi, int rho, const double* Dt, int lo2, int wd2,
                     double* psi_next, double* rowmax, int r0, int r1, void* stream);

/* ---- K2 A^(q) = psi A psi^T (gamblet_fast.py:658-665) -------------------- */
int gb_psi_stencil(int n, int lo, int wd, int rho, const double* psi, int wA,
                   const double* A, int wX, double* X, void* stream);
int gb_psi_galerkin(int n, int lo, int wd, int rho, const double* psi, int wX,
                    const double* X, int wR, double* raw, void* stream);
/* coalesced form of gb_psi_galerkin (same sums): psi and X transposed to
 * plane-major into `work` (gb_psi_galerkin_workspace bytes), a CTA per
 * 32 fine nodes of a grid row, outputs staged in shared memory */
size_t gb_psi_galerkin_workspace(int n, int wd, int wX);
int gb_psi_galerkin_t(int n, int lo, int wd, int rho, const double* psi, int wX,
                      const double* X, int wR, double* raw, double* work, void* stream);

/* ---- K3 B = W A W^T, G = W A pibar^T, P A P^T (gamblet_fast.py:520-544,
 *      597-601); w12 = the 3x4 null-basis template (hierarchy.py:31-42) ----- */
int gb_level_diag(int Lk, int wA, const double* A, const double* host_w12,
                  double* bdiag, double* dmin, void* stream);
int gb_level_blocks(int Lk, int wA, const double* A, const double* host_w12, int wB,
                    const double* bdiag, const double* dmin, double* B, double* G,
                    double* PAPt, double* stats, void* stream);

/* ---- K4 correction patches (gamblet_fast.py:546-591) --------------------- */
size_t gb_correction_workspace(int rho, int blocks);
int gb_correction_patches(int Lp, int wB, const double* B, const double* sB, int wG,
                          const double* G, int rho, double* Dt, int64_t* status,
                          double* workspace, int blocks, void* stream);

/* v2/v3: tiled DMMA Cholesky on the pre-scaled S B S box.  The v3 kernel
 * streams finished L columns through a caller-owned scratch of
 * gb_correction_patches_workspace(Lp, rho, r0, r1) bytes (0: v3 does not run,
 * pass NULL); the scratch must not be shared by concurrent calls.
 * GB_ERR_INVALID when no tiled kernel covers the patch (use v1). */
size_t gb_correction_patches_workspace(int Lp, int rho, int r0, int r1);
int gb_correction_patches_v2(int Lp, int wB, const double* Bs, const double* sB, int wG,
                             const double* G, int rho, double* Dt, int64_t* status,
                             double* workspace, size_t workspace_bytes, void* stream);

/* ---- K6 R, split triple product, psi^(k-1) (gamblet_fast.py:587-624) ----- */
int gb_restriction(int Lp, int rho, const double* Dt, const double* host_w12,
                   double* R, void* stream);
int gb_bd(int Lp, int wB, const double* B, int rho, const double* Dt, int wBD,
          double* BD, void* stream);
int gb_gtd(int Lp, int wG, const double* G, int rho, const double* Dt, int wGD,
           double* GtD, void* stream);
int gb_coarse_raw(int Lp, int wB, const double* PAPt, int wGD, const double* GtD,
                  int rho, const double* Dt, int wBD, const double* BD, int wA2,
                  double* raw, void* stream);
int gb_wpsi(int n, int Lk, int lo, int wd, const double* host_w12, const double* psi,
            int wdw, double* Wpsi, void* stream);
/* psi^(k-1) = drop_row(0.25 P psi + Dt (W psi)) (gamblet_fast.py:615-622),
 * row-tail drop included; rowmax: (Lk/2)^2 doubles of workspace.
 * gb_products_mode selects the kernels of psi_next, gb_bd, gb_gtd and
 * gb_coarse_raw: 1 (default) tensor-core block GEMMs, 0 per-entry gathers;
 * both accumulate in the reference's order (ascending CSR column), -1
 * queries; returns the previous mode. */
int gb_products_mode(int mma);
/* launch tuning (tests and tools only): what = 0 -> total CTAs of the v2
 * correction-patch grid (0 = auto); 1 -> correction kernel (1 = v3, default;
 * 0 = v2); 2 -> mass patches (0 = banded, default; 1 = dense tiled); 3 -> CTA cap
 * of the persistent symmetric-band SpMV pass (0 = one per SM); 4 -> mass patches by
 * clip type when M is translation invariant (1, default; 0 = every patch); 5 -> phase-1
 * kernel of the symmetric-band SpMV (1 = warp-specialized, default; 0 =
 * register-pipelined).  value
 * < 0 queries.  Returns the previous value (-1: unknown key). */
int gb_tune(int what, int value);
int gb_psi_next(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw,
                const double* Wpsi, int rho, const double* Dt, int lo2, int wd2,
                double* psi_next, double* rowmax, void* stream);

/* ---- K7/K8 Krylov (sparse_core.py:126-165, 232-278;
 *      gamblet_fast.py:380-387, 717-760) ---------------------------------- */
size_t gb_kstate_bytes(void);
int gb_red_blocks(void);
int gb_state_reset(void* state, int max_iter, void* stream);
int gb_cg_init(int64_t n, const double* b, const double* x0, const double* Ax0,
               double* x, double* r, double* p, double rel_tol, int max_iter,
               void* state, double* partials, void* stream);
int gb_cg_iterations(int L, int nr, int w, const double* B, const double* s, int mode,
                     double* x, double* r, double* p, double* Ap, int iters,
                     void* state, double* partials, void* stream);
int gb_pow_iterations(int L, int nr, int w, const double* B, const double* s, int mode,
                      double* x, double* y, double tol, int iters, void* state,
                      double* partials, void* stream);
/* v2 operator: pre-scaled Bs = S B S on zero-halo padded vectors */
int gb_scale_box(int L, int nr, int w, const double* B, const double* s, double* Bs,
                 void* stream);
int gb_pad(int L, int nr, int w, const double* src, const double* scale, double* dst,
           void* stream);
int gb_unpad(int L, int nr, int w, const double* src, const double* scale, double* dst,
             void* stream);
int gb_pcg_iterations(int L, int nr, int w, const double* Bs, double* x, double* r,
                      double* p, double* Ap, int iters, void* state, double* partials,
                      void* stream);
int gb_ppow_iterations(int L, int nr, int w, const double* Bs, double* x, double* y,
                       double tol, int iters, void* state, double* partials, void* stream);
int gb_pbox_apply(int L, int nr, int w, const double* Bs, const double* x, double* y,
                  void* stream);
/* layout argument of the Krylov entries: 0 = full blocked slot-major box
 * (gb_scale_box_T), 1 = symmetric band: upper 3x3 blocks per parent
 * (gb_scale_box_symT; tiled levels only, gb_sym_supported).  In layout 1
 * every OUTPUT vector of an S B S application (Ap, y) must have
 * (L+2w)^2*3 + gb_sym_overflow_elems(L, w) doubles: the tail holds the
 * tiles' spill-over between the two passes of one application. */
size_t gb_boxsym_elems(int L, int w);
size_t gb_sym_overflow_elems(int L, int w);
int gb_sym_supported(int L, int nr, int w);
int gb_scale_box_symT(int L, int w, const double* B, const double* s, double* UsT,
                      void* stream);
/* v3 operator: blocked slot-major S B S (BsT[(r/32)*S*32 + j*32 + r%32]),
 * one thread per row; gb_boxT_elems gives the allocation size in doubles */
size_t gb_boxT_elems(int L, int nr, int w);
int gb_scale_box_T(int L, int nr, int w, const double* B, const double* s, double* BsT,
                   void* stream);
int gb_tcg_iterations(int L, int nr, int w, const double* BsT, double* x, double* r,
                      double* p, double* Ap, int iters, void* state, double* partials,
                      void* stream, int layout);
int gb_tpow_iterations(int L, int nr, int w, const double* BsT, double* x, double* y,
                       double tol, int iters, void* state, double* partials, void* stream, int layout);
int gb_tbox_apply(int L, int nr, int w, const double* BsT, const double* x, double* y,
                  void* stream, int layout);
/* block-Jacobi (2x2 parents = 12x12 blocks) PCG for the subband systems */
int gb_bj_setup(int L, int w, const double* B, const double* s, float* inv, void* stream);
/* x = x0_scale * x0 (x0, Ax0 = A x0 nullable: zero start) */
int gb_bjcg_init(int L, int w, const double* b, const double* x0, const double* Ax0,
                 double x0_scale, double* x, double* r, double* p, double* z, const float* inv,
                 double rel_tol, int max_iter, void* state, double* partials, void* stream);
int gb_bjcg_iterations(int L, int w, const double* BsT, const float* inv, double* x,
                       double* r, double* p, double* Ap, double* z, int iters, void* state,
                       double* partials, void* stream, int layout);
/* whole Krylov loops driven from C (chunked launches, pinned state reads);
 * host_state: pinned host buffer of gb_kstate_bytes() bytes */
int gb_sync_read(const void* dev, void* host, size_t bytes, void* stream);
int gb_tcg_solve(int L, int nr, int w, const double* BsT, double* x, double* r, double* p,
                 double* Ap, void* state, double* partials, void* host_state, int max_chunk,
                 void* stream, int layout);
int gb_bjcg_solve(int L, int w, const double* BsT, const float* inv, double* x, double* r,
                  double* p, double* Ap, double* z, void* state, double* partials,
                  void* host_state, int max_chunk, void* stream, int layout);
/* two independent block-Jacobi PCG solves in lockstep sharing every operator
 * pass (batched repeat solves of solve_with_transform, gamblet_fast.py:
 * 717-760): each argument is a 2-array (vector 0, vector 1), both initialised
 * by gb_bjcg_init; each result is bitwise the single solve's.  Symmetric band
 * layout with the warp-specialized pass for one and two vectors only
 * (GB_ERR_INVALID otherwise). */
int gb_bjcg_solve2(int L, int w, const double* BsT, const float* inv, double* const* x,
                   double* const* r, double* const* p, double* const* Ap, double* const* z,
                   void* const* state, double* const* partials, void* const* host_state,
                   int max_chunk, void* stream);
int gb_tpow_solve(int L, int nr, int w, const double* BsT, double* x, double* y, double tol,
                  void* state, double* partials, void* host_state, int max_chunk,
                  void* stream, int layout);
int gb_dot2(int64_t n, const double* a, const double* b, const double* c, double* out,
            void* state, double* partials, void* stream);
int gb_scale_by_norm(int64_t n, const double* a, const double* norm2, int which,
                     double* y, double* y2, void* stream);
int gb_box_apply(int L, int nr, int w, const double* B, const double* s, int mode,
                 const double* x, double* y, void* stream);

/* general CSR operator: sparse_core.cg_solve / eig_extremes (sparse_core.py:
 * 126-165, 232-278) on any SPD canonical CSR matrix in device memory */
int gb_csr_apply(int64_t n, const int32_t* indptr, const int32_t* indices, const double* data,
                 const double* x, double* y, void* stream);
int gb_csr_cg_solve(int64_t n, const int32_t* indptr, const int32_t* indices,
                    const double* data, double* x, double* r, double* p, double* Ap,
                    void* state, double* partials, void* host_state, int max_chunk,
                    void* stream);
int gb_csr_pow_solve(int64_t n, const int32_t* indptr, const int32_t* indices,
                     const double* data, double* x, double* y, double tol, void* state,
                     double* partials, void* host_state, int max_chunk, void* stream);

/* level engine: lambda estimates of S B S (power + inverse iteration, the
 * reference algorithm) paired with the subband PCG, one S B S pass per pair
 * of iterations (argument block: paper_1503_03467_b200/csrc/gb_engine.h) */
struct gb_level_engine_args;
int gb_level_engine(struct gb_level_engine_args* args, void* stream);

/* host-only: lambda_min of the reference's inverse iteration
 * (sparse_core.py:258-277, stopping test at `tol`) evaluated from m Lanczos
 * coefficient pairs ab = (alpha_0, beta_0, ...) of the unit start vector --
 * the level engine's spectral mode 1 (csrc/gb_lanczos.h).  Outputs the
 * estimate, the outer iteration at which the reference would stop, and the
 * extreme Ritz values.  Returns 0, 1 (QL failure), 2 (nonpositive Ritz value). */
int gb_lanczos_emulate(const double* ab, int m, double tol, int max_outer, double* lam,
                       int* outer, double* ritz_min, double* ritz_max);
/* host-only: the engines' convergence check after m Lanczos steps.  The same
 * estimate by the inverse iteration run on T_m itself (LDL^T solves, O(m) per
 * outer step), and *stop = 1 once the estimates on T_m, T_{m-16}, T_{m-32}
 * share the stopping index and the geometric tail of their differences is
 * below lz_tol |lam|.  Returns 0, 1 (bad arguments), 2 (T_m not positive
 * definite). */
int gb_lanczos_check(const double* ab, int m, double tol, int max_outer, double lz_tol,
                     double* lam, int* outer, int* stop);

/* ---- diagnostics on the device (replaces diagnostics.py:40-155) --------
 * cell energies a_c * v_c^T E v_c of a fine vector (diagnostics.py:40-49);
 * decay sums: out[j] = sum of energies of the cells whose centre lies at
 * distance >= radii[j] from (cx, cy), out[nr] = total (diagnostics.py:58-74),
 * part = gb_decay_part_elems(nr) doubles; |coef_r| sqrt(diag_r) of a square
 * box (coefficient_spectrum, diagnostics.py:97-107); stable top-n_keep mask
 * of mags (compress, diagnostics.py:110-142; work NULL = size query);
 * x^T A x on a square half-width-w box (energy_norm, grid_fem.py:248-257),
 * part = gb_quad_part_elems() doubles. */
int gb_cell_energies(int n, const double* v, const double* coef, const double* host_e16,
                     double* out, void* stream);
size_t gb_decay_part_elems(int nr);
int gb_decay_sums(int n, double h, const double* energies, double cx, double cy,
                  const double* radii, int nr, double* part, double* out, void* stream);
int gb_box_diag_spectrum(int64_t rows, int nr, int w, const double* box, const double* coef,
                         double* out, void* stream);
int gb_topk_mask(int64_t n, const double* mags, int64_t n_keep, double* mask, void* work,
                 size_t* work_bytes, void* stream);
size_t gb_quad_part_elems(void);
int gb_box_quadform(int L, int w, const double* box, const double* x, double* part, double* out,
                    void* stream);
/* max_i |x_i| (part = gb_quad_part_elems() doubles) */
int gb_max_abs(int64_t n, const double* x, double* part, double* out, void* stream);

/* ---- K9 load-dependent transfers (gamblet_fast.py:726-765) --------------- */
int gb_apply_w(int Lp, const double* host_w12, const double* g, const double* s,
               double* out, void* stream);
int gb_apply_wt(int Lp, const double* host_w12, const double* w, double* v,
                void* stream);
int gb_apply_r(int Lp, int rho, const double* R, const double* g, double* out,
               void* stream);
int gb_psi_t_apply(int n, int L, int lo, int wd, const double* psi, const double* v,
                   double* inc, void* stream);
int gb_psi_apply(int n, int L, int lo, int wd, const double* psi, const double* b,
                 double* out, void* stream);
int gb_axpby(int64_t n, double a, const double* x, double b, const double* y,
             double* out, void* stream);
int gb_vmul(int64_t n, const double* a, const double* b, double* out, void* stream);
int gb_vadd(int64_t n, const double* a, const double* b, double* out, void* stream);

/* ---- CSR export at the API edge (the .stiffness/.subband/... attributes,
 *      gamblet_fast.py:626-632; canonical form of sparse_core.py:47-67) ---- */
int gb_export_count(int kind, int L, int nr, int w, int nc, int n, int lo, int wd,
                    const double* val, int64_t rows, int64_t S, int64_t* counts,
                    void* stream);
int gb_exclusive_scan(const int64_t* counts, int64_t* indptr, int64_t n, void* tmp,
                      size_t* tmp_bytes, void* stream);
int gb_export_emit(int kind, int L, int nr, int w, int nc, int n, int lo, int wd,
                   const double* val, int64_t rows, int64_t S, const int64_t* indptr,
                   int32_t* indices, double* data, void* stream);

/* ---- K10 exact path, dense (gamblet_exact.py:115-263) -------------------- */
int gb_dense_gemm(int m, int n, int k, double alpha, const double* A, int lda, int ta,
                  const double* B, int ldb, int tb, double beta, double* C, int ldc,
                  void* stream);
int gb_dense_potrf(int n, double* A, int lda, int64_t* status, void* stream);
int gb_dense_potrs(int n, int nrhs, const double* L, int lda, double* B, int ldb,
                   void* stream);
int gb_dense_sym(int n, const double* X, int ldx, double* out, double* stats,
                 void* stream);

int gb_csr_to_dense(int nrows, int ncols, const int32_t* indptr, const int32_t* indices,
                    const double* data, double* out, void* stream);
int gb_eye(int n, double* out, void* stream);
int gb_dense_build_w(int Lk, const double* host_w12, double* out, void* stream);
int gb_dense_build_p(int Lk, double* out, double scale, void* stream);

/* ---- FP64 peak probes (DFMA / DMMA) used for the roofline denominators --- */
int gb_fp64_peak_probe(int kind, int iters, double* sink, void* stream);


/* ---- config 4 (BASELINE.json configs[4]): the 3-D localized transform on
 *      3-D box stencils (csrc/gb_3d.cu); the reference is 2-D only, the
 *      algorithm is gamblet_fast.py:464-775 in d = 3 (8 children, 7 Helmert
 *      W rows per parent, pibar = pi/8), restated by
 *      oracle/gamblets_oracle_nd.py.  host_w: 7 x 8 row-major W template. */
int gb3_csr_to_box(int L, int w, const int32_t* indptr, const int32_t* indices,
                   const double* data, double* box, int64_t* status, void* stream);
int gb3_box_scale(int64_t rows, int nr, int w, const double* box, double* s, int64_t* status,
                  void* stream);
int gb3_box_sym_drop(int L, int nr, int w, const double* raw, double* out, double* dmin,
                     double* stats, void* stream);
int gb3_mass_patches(int L, const double* Ms, const double* s, int rho, int wd, double* psi,
                     int64_t* status, void* stream);
int gb3_psi_galerkin(int L, int rho, int wd, const double* psi, const double* A, int wX,
                     double* X, int wR, double* raw, void* stream);
int gb3_level_blocks(int Lk, int wA, const double* A, const double* host_w, int wB, double* Braw,
                     double* G, double* PAPt, void* stream);
size_t gb3_correction_workspace(int Lp, int rho, int ctas);
int gb3_correction_patches(int Lp, int wB, const double* B, const double* sB, const double* G,
                           int rho, double* Dt, int64_t* status, double* workspace, int ctas,
                           void* stream);
int gb3_restriction(int Lp, int rho, const double* Dt, const double* host_w, double* R,
                    void* stream);
int gb3_triple(int Lp, int wB, const double* B, const double* G, const double* PAPt, int rho,
               const double* Dt, int wBD, double* BD, int wGD, double* GtD, int wA2, double* raw,
               void* stream);
int gb3_apply_w(int Lp, const double* host_w, const double* g, const double* s, double* out,
                void* stream);
int gb3_apply_wt(int Lp, const double* host_w, const double* w, double* v, void* stream);
int gb3_apply_r(int Lp, int rho, const double* R, const double* g, double* out, void* stream);
int gb3_apply_rt(int Lp, int rho, const double* R, const double* u, double* out, void* stream);
int gb3_psi_t_apply(int L, int rho, int wd, const double* psi, const double* v, double* out,
                    void* stream);
int gb3_apply(int L, int nr, int w, const double* B, const double* s, const double* x, double* y,
              void* stream);
int gb3_cg_solve(int L, int nr, int w, const double* B, const double* s, double* x, double* r,
                 double* p, double* Ap, void* state, double* partials, void* host_state,
                 int max_chunk, void* stream);
/* lambda_min of S B S (3-D box) by the Lanczos moments of the unit start
 * vector x: the reference's inverse-iteration sequence (sparse_core.py:
 * 258-277) evaluated from T_m, stop by gb_lanczos_check at lz_tol.  x is overwritten; vp, wv: work n-vectors; ab /
 * host_ab: 2 cap doubles (device / pinned host). */
int gb3_lanczos_min(int L, int nr, int w, const double* B, const double* s, double* x,
                    double* vp, double* wv, void* state, double* partials, void* host_state,
                    double* ab, double* host_ab, int cap, double tol, int max_outer,
                    double lz_tol, double* lam, int* outer, int* its, void* stream);
int gb3_pow_solve(int L, int nr, int w, const double* B, const double* s, double* x, double* y,
                  double tol, void* state, double* partials, void* host_state, int max_chunk,
                  void* stream);

/* ---- Row strips (multi-GPU spatial partition) --------------
 * Every `_rows` entry computes the grid rows [r0, r1) of its output only and
 * reads its inputs at global indices, so a rank passes the same base pointers
 * as the whole-level call and provides the halo rows named in each comment
 * (exchanged by paper_1503_03467_b200/comm.py).  The whole-level entry points
 * are the [0, L) instances: the union of a partition's strips is bitwise the
 * whole level.  Patches are independent given the level operator
 * (gamblet_fast.py:464-498, 546-580).
 * The `gb_dist_*` entries are the rank-local pieces of the distributed
 * block-Jacobi PCG / power iteration / Lanczos recurrence on a strip of a
 * tiled level (rows multiples of 4): every reduction stops at the strip's
 * partial sum, the caller all-reduces it, a commit entry applies it to the
 * iteration state (sparse_core.py:126-165, 232-278 split at the reductions). */
/* bytes of the gb_psi_galerkin_t_rows workspace for the strip [r0, r1) */
size_t gb_psi_galerkin_workspace_rows(int n, int wd, int wX, int wR, int r0, int r1);
/* grid rows [r0, r1) of a box from the CSR slice of exactly those matrix rows (local indptr, global columns) */
int gb_csr_to_box_rows(int n, int w, const int32_t* indptr, const int32_t* indices, const double* data, double* box, int64_t* status, int r0, int r1, void* stream);
/* gb_box_sym_drop on the grid rows [r0, r1); reads raw rows within w of the strip */
int gb_box_sym_drop_rows(int L, int nr, int w, const double* raw, double* out, const double* dmin, double* stats, int r0, int r1, void* stream);
/* X = psi A, fine rows [r0, r1); reads A rows within rho */
int gb_psi_stencil_rows(int n, int lo, int wd, int rho, const double* psi, int wA, const double* A, int wX, double* X, int r0, int r1, void* stream);
/* raw = X psi^T, fine rows [r0, r1); reads psi rows within wR */
int gb_psi_galerkin_t_rows(int n, int lo, int wd, int rho, const double* psi, int wX, const double* X, int wR, double* raw, double* work, int r0, int r1, void* stream);
/* diag(B) of the parents in rows [r0, r1) and their running minimum */
int gb_level_diag_rows(int Lk, int wA, const double* A, const double* host_w12, double* bdiag, double* dmin, int r0, int r1, void* stream);
/* B, G, P A P^T rows of the parents in rows [r0, r1); reads A rows of parents within wB, bdiag within wB */
int gb_level_blocks_rows(int Lk, int wA, const double* A, const double* host_w12, int wB, const double* bdiag, const double* dmin, double* B, double* G, double* PAPt, double* stats, int r0, int r1, void* stream);
/* R rows [r0, r1) from the same rows of D^T */
int gb_restriction_rows(int Lp, int rho, const double* Dt, const double* host_w12, double* R, int r0, int r1, void* stream);
/* B D rows [r0, r1); reads D^T rows within wBD */
int gb_bd_rows(int Lp, int wB, const double* B, int rho, const double* Dt, int wBD, double* BD, int r0, int r1, void* stream);
/* G^T D rows [r0, r1); reads G rows within wG and D^T rows within wGD */
int gb_gtd_rows(int Lp, int wG, const double* G, int rho, const double* Dt, int wGD, double* GtD, int r0, int r1, void* stream);
/* raw A^(k-1) rows [r0, r1); reads G^T D rows within wGD and B D rows within rho */
int gb_coarse_raw_rows(int Lp, int wB, const double* PAPt, int wGD, const double* GtD, int rho, const double* Dt, int wBD, const double* BD, int wA2, double* raw, int r0, int r1, void* stream);
/* W psi rows of the parents in rows [r0, r1), window points with fine row in [f0, f1) only */
int gb_wpsi_rows(int n, int Lk, int lo, int wd, const double* host_w12, const double* psi, int wdw, double* Wpsi, int r0, int r1, int f0, int f1, void* stream);
/* raw psi^(k-1) rows [r0, r1) and their maxima, window points with fine row in [f0, f1) only (no drop) */
int gb_psi_next_raw_rows(int n, int Lk, int lo, int hi, int wd, const double* psi, int wdw, const double* Wpsi, int rho, const double* Dt, int lo2, int wd2, double* psi_next, double* rowmax, int r0, int r1, int f0, int f1, void* stream);
/* the row-tail drop of psi rows [r0, r1) given their (all-reduced) maxima */
int gb_psi_drop_rows(int n, int Lp, int lo2, int wd2, double* psi_next, const double* rowmax, int r0, int r1, int f0, int f1, void* stream);
/* gb_pad on grid rows [r0, r1) */
int gb_pad_rows(int L, int nr, int w, const double* src, const double* scale, double* dst, int r0, int r1, void* stream);
/* gb_unpad on grid rows [r0, r1) */
int gb_unpad_rows(int L, int nr, int w, const double* src, const double* scale, double* dst, int r0, int r1, void* stream);
/* gb_apply_w on parent rows [r0, r1) */
int gb_apply_w_rows(int Lp, const double* host_w12, const double* g, const double* s, double* out, int r0, int r1, void* stream);
/* gb_apply_wt on parent rows [r0, r1) */
int gb_apply_wt_rows(int Lp, const double* host_w12, const double* w, double* v, int r0, int r1, void* stream);
/* gb_apply_r on parent rows [r0, r1); reads g within 2 rho + 1 child rows */
int gb_apply_r_rows(int Lp, int rho, const double* R, const double* g, double* out, int r0, int r1, void* stream);
/* fine rows [F0, F1) of psi^T v summed over the psi rows in grid rows [j_lo, j_hi) only */
int gb_psi_t_apply_rows(int n, int L, int lo, int wd, const double* psi, const double* v, double* inc, int F0, int F1, int j_lo, int j_hi, void* stream);
/* block-Jacobi inverses of the 2x2-parent blocks in rows [r0, r1) */
int gb_bj_setup_rows(int L, int w, const double* B, const double* s, float* inv, int r0, int r1, void* stream);
/* rows [r0, r1) of the symmetric band copy of S B S; reads s within w rows below */
int gb_scale_box_symT_rows(int L, int w, const double* B, const double* s, double* UsT, int r0, int r1, void* stream);
/* phase 1 of the symmetric SpMV on the strip's tiles for nv vectors; red[v] = strip partial of x_v.(A x_v) */
int gb_dist_apply(int L, int w, const double* UsT, int nv, const double* x0, double* y0, void* st0, double* part0, const double* x1, double* y1, void* st1, double* part1, double* red, int r0, int r1, void* stream);
/* x = 0, r = b, z = p = Minv r on the strip; out = (r.r, r.z, b.b) partials */
int gb_dist_pcg_init(int L, int w, const double* b, double* x, double* r, double* p, double* z, const float* inv, void* st, double* part, double* out, int r0, int r1, void* stream);
/* all-reduced init sums -> iteration state */
int gb_dist_pcg_init_commit(void* st, const double* out, double rel_tol, int max_iter, void* stream);
/* PCG update on the strip with alpha = rs / red[0]; out = (r.r, r.z) partials */
int gb_dist_pcg_update(int L, int w, double* x, double* r, const double* p, const double* Ap, double* z, const float* inv, void* st, const double* red, double* part, double* out, int r0, int r1, void* stream);
/* all-reduced sums -> state (convergence, beta), then p = z + beta p on the strip */
int gb_dist_pcg_commit_dir(int L, int w, void* st, const double* red, const double* out, const double* z, double* p, int r0, int r1, void* stream);
/* y += spill-over on the strip; out[0] = y.y partial */
int gb_dist_fix_yy(int L, int w, double* y, void* st, double* part, double* out, int r0, int r1, void* stream);
/* power iteration between its reductions (stage 0: lam, ynorm, residual partial; stage 1: test, x = y / ynorm) */
int gb_dist_pow_step(int L, int w, double* x, const double* y, void* st, const double* red, const double* out_yy, double* out_res, double* part, double tol, int r0, int r1, int stage, void* stream);
/* Lanczos recurrence on the strip; out[0] = |u|^2 partial */
int gb_dist_lz_update(int L, int w, const double* x, double* y, double* vp, void* st, const double* red, double* part, double* out, int r0, int r1, void* stream);
/* all-reduced |u|^2 -> (alpha_j, beta_j) appended, state advanced */
int gb_dist_lz_commit(void* st, const double* red, const double* out, double* ab, void* stream);
/* reset the state for a Lanczos sequence of at most cap steps */
int gb_dist_lz_begin(void* st, int cap, void* stream);
/* out[0] = a.b over n contiguous elements (strip partial) */
int gb_dist_dot(int64_t n, const double* a, const double* b, void* st, double* part, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GAMBLETS_B200_H */
