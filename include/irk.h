/*
 * irk.h — C ABI of libirk, the sm_100a kernel library behind the
 * paper_2403_08084_b200 drop-in for the `implicitrk` stage-coupled solve path.
 *
 * Conventions
 *  - Every entry point returns an irk_status (0 = ok).  No C++ exception ever
 *    crosses this boundary.  The message of the most recent failure on the
 *    calling host thread is available from irk_last_error().
 *  - Pointers named *_dev are device pointers; *_host are host pointers.
 *    Sizes are int64_t element counts.  No torch (or any other framework) type
 *    appears in a signature.
 *  - All device work is ordered on the context's stream (irk_ctx_set_stream).
 *    Calls are asynchronous unless they return host scalars (documented per
 *    call: the Krylov/CG solvers return iteration counts and residuals).
 *  - A context is NOT thread-safe; use one context per host thread / stream.
 *  - Stage vectors use the stage-INTERLEAVED layout: element (row r, stage i)
 *    of an m-by-s stage block lives at  Y[r*s + i].  The reference stores the
 *    same data stage-major, v[i*m + r] (implicitrk/sparsela.py:226).
 *  - Sign convention of the reference: M u' + K u = f with K positive
 *    semidefinite; stage operator  C1 (x) M + dt * C2 (x) K
 *    (implicitrk/sparsela.py:194-235).
 *
 * Every function cites the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/implicitrk/).
 */
#ifndef IRK_H
#define IRK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  IRK_OK = 0,
  IRK_EINVAL = 1,      /* invalid argument        -> ValueError            */
  IRK_ECUDA = 2,       /* CUDA runtime failure    -> RuntimeError          */
  IRK_ENOCONV = 3,     /* iteration cap reached   -> NonConvergenceError   */
  IRK_ENONFINITE = 4,  /* non-finite data seen    -> ValueError / divergence */
  IRK_ESINGULAR = 5    /* zero pivot / breakdown  -> FactorizationError    */
} irk_status;

typedef struct irk_ctx irk_ctx;
typedef struct irk_mat irk_mat;

/* ---------------------------------------------------------------- context */

/* Create a context on `device`; work is issued on the legacy default stream
 * until irk_ctx_set_stream is called. */
int irk_ctx_create(int device, irk_ctx** out);
int irk_ctx_destroy(irk_ctx* ctx);
/* `stream` is a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream). */
int irk_ctx_set_stream(irk_ctx* ctx, void* stream);
int irk_ctx_synchronize(irk_ctx* ctx);
/* Number of kernels this context has launched so far (bench accounting). */
int64_t irk_ctx_launch_count(const irk_ctx* ctx);
/* Deferred inner-solve status.  While enabled, irk_pcg / irk_cocg /
 * irk_mg_pcg called with its_host == relres_host == NULL return IRK_OK
 * without synchronising and append (iterations, code 0 ok / 1 cap /
 * 2 breakdown, executed loop passes, kernels per loop pass) to a device log;
 * irk_ctx_log_take copies the entries in call order (synchronous) and
 * clears the log.  Enabling also clears it.  The log grows on demand;
 * irk_ctx_log_size reports the number of pending entries. */
int irk_ctx_log_enable(irk_ctx* ctx, int on);
int irk_ctx_log_size(const irk_ctx* ctx, int64_t* n_out);
int irk_ctx_log_take(irk_ctx* ctx, int* out_host, int max_entries, int* n_out);
const char* irk_last_error(void);
/* Library version string. */
const char* irk_version(void);

/* --------------------------------------------------------------- matrices
 * An irk_mat is a device CSR matrix (int32 row offsets / column indices,
 * float64 values) plus a sliced-ELL (SELL-32, column-major within a slice of
 * 32 rows) copy of the same entries used by every kernel.  Matrices created by
 * irk_mat_assemble_p1, irk_mat_combine, irk_mat_constrain and irk_mat_union
 * share one pattern object with their sources.
 * Replaces: SparseMatrix (sparsela.py:43-115). */

/* Upload host CSR (int64 indices as the reference stores them,
 * sparsela.py:53-55).  Rows must be strictly increasing (validated by the
 * Python layer, sparsela.py:61-78). */
int irk_mat_from_csr(irk_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                     const int64_t* row_offsets_host, const int64_t* col_indices_host,
                     const double* values_host, irk_mat** out);

/* On-device assembly of the P1 mass and stiffness matrices on the structured
 * unit grid with N cells per direction: dim 1 (intervals), dim 2 (each square
 * split into two right triangles along (i,j)-(i+1,j+1)), dim 3 (Kuhn split of
 * each cube into 6 tetrahedra sharing the (0,0,0)-(1,1,1) diagonal).  Vertices
 * are numbered lexicographically, x fastest (problems.py:25-64).  M and K share
 * one pattern; explicit zeros of K are kept.  Replaces assemble_heat
 * (problems.py:80-99), which builds 1D P1 / 2D Q1 only. */
int irk_mat_assemble_p1(irk_ctx* ctx, int dim, int64_t N, irk_mat** M, irk_mat** K);

/* Q1 (bilinear) 2D operators M1(x)M1, K1(x)M1 + M1(x)K1 of the reference's
 * assemble_heat (problems.py:93-95), assembled on device on one pattern. */
int irk_mat_assemble_q1(irk_ctx* ctx, int64_t N, irk_mat** M, irk_mat** K);

int irk_mat_info(const irk_mat* A, int64_t* nrows, int64_t* ncols, int64_t* nnz);
/* 1 when A and B are stored on the same pattern object. */
int irk_mat_same_pattern(const irk_mat* A, const irk_mat* B);
/* Copy to host CSR (int64 indices).  Synchronous. */
int irk_mat_download(irk_ctx* ctx, const irk_mat* A, int64_t* row_offsets_host,
                     int64_t* col_indices_host, double* values_host);
int irk_mat_destroy(irk_mat* A);

/* Re-express A and B on the union of their patterns (new handles). */
int irk_mat_union(irk_ctx* ctx, const irk_mat* A, const irk_mat* B,
                  irk_mat** A_out, irk_mat** B_out);

/* C = alpha*A + beta*B on their shared pattern (explicit zeros kept).
 * Replaces the sparse add inside factorize_block (sparsela.py:181). */
int irk_mat_combine(irk_ctx* ctx, double alpha, const irk_mat* A, double beta,
                    const irk_mat* B, irk_mat** C);

/* Rows and columns flagged in mask_dev (uint8, length nrows) are zeroed and
 * the diagonal set to diag_value; the pattern is kept.  Replaces
 * dirichlet_constrain (sparsela.py:126-146), which rebuilds the pattern. */
int irk_mat_constrain(irk_ctx* ctx, const irk_mat* A, const uint8_t* mask_dev,
                      double diag_value, irk_mat** out);

/* Express X on T's pattern (every stored entry of X must exist in T). */
int irk_mat_on_pattern(irk_ctx* ctx, const irk_mat* X, const irk_mat* T, irk_mat** out);

/* out = kscale*K + M diag(d) on their shared pattern: the Jacobian of the
 * semilinear residual M u' + kscale*K u + M g(u) with d = g'(u), read as
 * d[c*ld + off] (stepper.py:550; tests/test_stepper.py:297-300). */
int irk_mat_semilinear_jacobian(irk_ctx* ctx, const irk_mat* M, const irk_mat* K, double kscale,
                                const double* d_dev, int64_t ld, int64_t off, irk_mat** out);

/* diag_dev[r] = A[r,r] (0 when absent). */
int irk_mat_diagonal(irk_ctx* ctx, const irk_mat* A, double* diag_dev);
/* Row sums (lumped mass), rowsum_dev[r] = sum_c A[r,c]. */
int irk_mat_rowsum(irk_ctx* ctx, const irk_mat* A, double* rowsum_dev);
/* out[r] = sum_c |A[r,c]| (Gershgorin radii of D^-1 A with irk_mat_diagonal;
 * the Chebyshev block solver's bounds). */
int irk_mat_absrowsum(irk_ctx* ctx, const irk_mat* A, double* out_dev);
/* Dense row-major n x n copy of a square matrix into device memory (the
 * direct block solver's setup; replaces a host to_dense + copy). */
int irk_mat_to_dense(irk_ctx* ctx, const irk_mat* A, double* dense_dev);

/* y = A x (k right-hand sides, interleaved: x[c*k + j]).  Replaces spmv
 * (sparsela.py:118-123). */
int irk_spmv(irk_ctx* ctx, const irk_mat* A, int k, const double* x_dev, double* y_dev);
/* y[r*ldy] = sum_c A[r,c] x[c*ldx], A dense row-major n x n on the device
 * (the direct solve of small blocks: A = the precomputed block inverse). */
int irk_dense_gemv(irk_ctx* ctx, int64_t n, const double* A_dev, const double* x_dev,
                   int64_t ldx, double* y_dev, int64_t ldy);

/* ------------------------------------------------------ stage operator (K2)
 * Out = (C1 (x) M + dt * C2 (x) K) Y on interleaved m-by-s blocks, computed
 * as  Out_r = C1 (M Y)_r + dt * C2 (K Y)_r  with the s-by-s mix in registers.
 * Ks holds nK = 1 matrix or nK = s per-stage matrices (row-indexed: stage row
 * i uses Ks[i], sparsela.py:230-234); all on M's pattern.
 * If rowmask_dev is non-NULL the constrained form is applied: flagged rows
 * are identity (bcs.py:99-120); the column elimination is carried by the
 * matrices, which the caller passes with flagged rows and columns zeroed
 * (irk_mat_constrain(..., diag_value = 0)).
 * Replaces KroneckerStageOperator.apply (sparsela.py:222-235) and
 * ConstrainedStageOperator.apply (bcs.py:114-120). */
int irk_stage_apply(irk_ctx* ctx, int s, const double* C1_host, const double* C2_host,
                    double dt, const irk_mat* M, const irk_mat* const* Ks, int nK,
                    const uint8_t* rowmask_dev, const double* Y_dev, double* Out_dev);

/* Semilinear Jacobian variant: stage row i uses
 *   K_i = kscale*K + M diag(D[:, i])          (D interleaved m-by-s)
 * the per-stage Jacobian of  F(u, u') = M u' + kscale*K u + M g(u)
 * (the reference's per-stage Jacobian operator, stepper.py:550-551, for the
 * cubic-reaction recipe of tests/test_stepper.py:282-334). */
int irk_stage_apply_semilinear(irk_ctx* ctx, int s, const double* C1_host,
                               const double* C2_host, double dt, const irk_mat* M,
                               const irk_mat* K, double kscale, const double* D_dev,
                               const uint8_t* rowmask_dev, const double* Y_dev,
                               double* Out_dev);

/* Y_r = Q X_r for every row r: Q is s_out-by-s_in (host, row-major), X is
 * m-by-s_in and Y m-by-s_out, both interleaved (in place allowed when
 * s_in == s_out).  Used for (A^-1 (x) I), (Q^T (x) I) Schur transforms, ... */
int irk_stage_mix(irk_ctx* ctx, int64_t m, int s_out, int s_in, const double* Q_host,
                  const double* X_dev, double* Y_dev);

/* Gauss-Seidel stage coupling of the block preconditioner
 * (StagePreconditioner.apply, precond.py:104-115):
 *   out[r*ld_out] = R[r*s + i] - sum_c C[r,c] * sum_j coef[j] X[c*s + j]
 * flagged rows are left at R; C must come with flagged columns zeroed
 * (irk_mat_constrain). */
int irk_stage_couple(irk_ctx* ctx, int s, int i, const double* coef_host, const irk_mat* C,
                     const uint8_t* rowmask_dev, const double* R_dev, const double* X_dev,
                     double* out_dev, int64_t ld_out);

/* Out_r,i = a * (B u)_r + sum_j G[i,j] * F[r,j]   (B may be NULL: then B is
 * the identity when u is given, else the term is dropped; F may be NULL).  Builds the linear stage right-hand sides of
 * assemble_linear_stage_system (stepper.py:291-293) and
 * _stage_value_system (stepper.py:309-311). */
int irk_stage_rhs(irk_ctx* ctx, int64_t m, int s, double a, const irk_mat* B,
                  const double* u_dev, const double* G_host, const double* F_dev,
                  double* Out_dev);

/* u_next_r = a*u_r + sum_i w[i]*X_r,i  (fused Runge-Kutta update,
 * stepper.py:352-361, :421).  If copy_stage >= 0, u_next = X[:, copy_stage]
 * bit for bit (stiffly accurate stage-value update, stepper.py:354). */
int irk_stage_update(irk_ctx* ctx, int64_t m, int s, double a, const double* u_dev,
                     const double* w_host, int copy_stage, const double* X_dev,
                     double* u_next_dev);

/* out[r*s + i] = w[i] * v[r] * D[r*s + i]  (D may be NULL: read as 1).
 * Builds the lumped reaction shifts of the semilinear block surrogate. */
int irk_stage_scale(irk_ctx* ctx, int64_t m, int s, const double* w_host, const double* v_dev,
                    const double* D_dev, double* out_dev);

/* Column extract / insert between an interleaved m-by-s block and a
 * contiguous m vector, and stage-major <-> interleaved permutations. */
int irk_stage_get(irk_ctx* ctx, int64_t m, int s, int i, const double* X_dev, double* x_dev);
int irk_stage_set(irk_ctx* ctx, int64_t m, int s, int i, const double* x_dev, double* X_dev);
int irk_to_interleaved(irk_ctx* ctx, int64_t m, int s, const double* stage_major_dev,
                       double* interleaved_dev);
int irk_to_stage_major(irk_ctx* ctx, int64_t m, int s, const double* interleaved_dev,
                       double* stage_major_dev);

/* Boundary handling on an interleaved block with the dof list idx_dev
 * (int64, length nb):
 *  scatter:  X[idx[k]*s + i] = V[i*nb + k]   (V stage-major, s-by-nb)
 *  gather:   V[k] = x[idx[k]]                 (single vector)
 *  zero:     X[idx[k]*s + i] = 0
 * Used by constrain_stage_system (bcs.py:123-142), _solve_constrained
 * (stepper.py:334-336) and the Newton increment masking (stepper.py:558-559). */
int irk_bc_scatter(irk_ctx* ctx, int s, int64_t nb, const int64_t* idx_dev,
                   const double* V_dev, double* X_dev);
int irk_bc_gather(irk_ctx* ctx, int64_t nb, const int64_t* idx_dev, const double* x_dev,
                  double* v_dev);
int irk_bc_zero(irk_ctx* ctx, int s, int64_t nb, const int64_t* idx_dev, double* X_dev);
/* DAE stage boundary values from the device state (stage_bc_values,
 * bcs.py:76-87): out[i*nb+k] = (G[i*nb+k] - u[idx[k]]) / dt (Ainv_host NULL:
 * the W unknowns), or sum_j Ainv[i][j] (G[j*nb+k] - u[idx[k]]) / dt (the
 * stage derivatives; Ainv row-major s x s on the host). */
int irk_bc_dae_values(irk_ctx* ctx, int s, int64_t nb, const int64_t* idx_dev,
                      const double* G_dev, const double* u_dev, double dt,
                      const double* Ainv_host, double* out_dev);
/* mask_dev[idx[k]] = 1, others 0 (length m). */
int irk_bc_mask(irk_ctx* ctx, int64_t m, int64_t nb, const int64_t* idx_dev, uint8_t* mask_dev);

/* ------------------------------------------------ Krylov building blocks (K3)
 * Vectors are contiguous float64 of length n; a basis V holds k vectors
 * V + i*ldv.  All results stay on the device unless stated.
 * Replace the numpy MGS/Givens arithmetic of fgmres (sparsela.py:355-394). */

/* h[i] = <V_i, w>, i < k (classical Gram-Schmidt projections, one fused pass
 * over w and the basis). */
int irk_multidot(irk_ctx* ctx, int64_t n, int k, const double* V_dev, int64_t ldv,
                 const double* w_dev, double* h_dev);
/* w -= sum_i h[i] V_i ; then h[k] = ||w||_2 (device).  With reorth != 0 a
 * second classical pass (CGS2) is made and its coefficients are added to h.
 * h_dev must provide 128 doubles of storage (the second half is scratch). */
int irk_orth_update(irk_ctx* ctx, int64_t n, int k, const double* V_dev, int64_t ldv,
                    double* h_dev, double* w_dev, int reorth);
/* x += sum_i y[i] Z_i (y on host, k <= 64). */
int irk_lincomb(irk_ctx* ctx, int64_t n, int k, const double* Z_dev, int64_t ldz,
                const double* y_host, double* x_dev);
/* y = a*x + b*y ; y = a*x (b = 0 ignores y's old content, NaN-safe). */
int irk_axpby(irk_ctx* ctx, int64_t n, double a, const double* x_dev, double b, double* y_dev);
/* y = a*x + b*y with a,b read from device scalars  a = num/den (den != 0). */
int irk_scale_dev(irk_ctx* ctx, int64_t n, const double* num_dev, const double* den_dev,
                  const double* x_dev, double* y_dev);
/* out = ||x||_2 (device scalar) and <x,y> (device scalar). */
int irk_norm2(irk_ctx* ctx, int64_t n, const double* x_dev, double* out_dev);
int irk_dot(irk_ctx* ctx, int64_t n, const double* x_dev, const double* y_dev, double* out_dev);
/* 1 if every entry is finite (synchronous). */
int irk_all_finite(irk_ctx* ctx, int64_t n, const double* x_dev, int* result_host);

/* ------------------------------------------ device-resident FGMRES cycle
 * The Arnoldi loop of fgmres (sparsela.py:355-403) without a host round trip
 * per iteration: one CUDA graph runs a whole restart cycle (a conditional
 * WHILE node; Givens rotations and the stop tests on the device).
 * step_graph (a cudaGraph_t, cloned) computes w from v_j on fixed buffers:
 * right preconditioning z_j = P v_j, w = A z_j (Z != NULL: Z_j = z_j is
 * stored), or w = A v_j (Z == NULL, the solution update uses V).  work
 * holds irk_fgmres_work_doubles(cycle) doubles, st_dev 8 ints.  The graph
 * bakes in the context scratch: irk_fgmres_graph_run fails with
 * IRK_EINVAL if that scratch was reallocated since (re-create it).
 * irk_fgmres_graph_run: one cycle of at most cap <= cycle steps from the
 * residual r (beta = ||r||): V_0 = r / beta, ..., x += Z y; writes the
 * steps taken, the convergence flag (residual <= target or breakdown
 * h_{j+1,j} < breakdown) and the residual estimates hist[0..k]
 * (synchronous). */
typedef struct irk_fgraph irk_fgraph;
size_t irk_fgmres_work_doubles(int cycle);
int irk_fgmres_graph_create(irk_ctx* ctx, void* step_graph, int64_t n, int cycle, int reorth,
                            double* V, int64_t ldv, double* Z, int64_t ldz, double* vj,
                            const double* zj, double* w, double* work, int* st_dev,
                            irk_fgraph** out);
int irk_fgmres_graph_run(irk_ctx* ctx, irk_fgraph* fg, int cap, const double* r, double beta,
                         double target, double breakdown, double* x, int* k_host,
                         int* conv_host, double* hist_host);
int irk_fgmres_graph_destroy(irk_fgraph* fg);

/* ------------------------------------------------------ inner block solves
 * Jacobi-preconditioned CG on nb independent SPD systems stored interleaved
 * (m-by-nb).  System k is
 *      B_k = alpha[k]*A + beta[k]*Bm + diag(shift[:, k])
 * (Bm and shift may be NULL); rows flagged in rowmask_dev are identity rows
 * and the caller passes A, Bm with the flagged columns eliminated
 * (irk_mat_constrain), the treatment factorize_block gives its blocks
 * (sparsela.py:181-183).  A pre-combined, constrained block needs no mask.  Solves start from x = 0 and stop
 * per system when ||r_k|| <= max(rtol*||b_k||, atol) or after maxit
 * iterations; all loop control stays on the device.
 * its_host[k] / relres_host[k] receive the iteration count and final
 * relative residual.  Returns IRK_ENOCONV if a system hit maxit.
 * Replaces BlockFactorization.solve / splu (sparsela.py:149-191), which the
 * north_star swaps for Jacobi-PCG. */
int irk_pcg(irk_ctx* ctx, int nb, const double* alpha_host, const double* beta_host,
            const irk_mat* A, const irk_mat* Bm, const double* shift_dev,
            const uint8_t* rowmask_dev, const double* rhs_dev, int64_t ld_rhs,
            double* x_dev, int64_t ld_x, double rtol, double atol, int maxit,
            int* its_host, double* relres_host);

/* Jacobi-preconditioned COCG on np complex-symmetric systems
 *     (alpha[k] * A + beta[k] * Bm) z_k = b_k,  alpha, beta complex
 * stored interleaved as (re, im) pairs: z_k at X[r*ld + 2k], X[r*ld + 2k+1].
 * Used for the 2x2 real-Schur blocks of the transformed stage preconditioner
 * (new; the reference declines the Schur preconditioner). */
int irk_cocg(irk_ctx* ctx, int np, const double* alpha_re_host, const double* alpha_im_host,
             const double* beta_re_host, const double* beta_im_host, const irk_mat* A,
             const irk_mat* Bm, const uint8_t* rowmask_dev, const double* rhs_dev,
             int64_t ld_rhs, double* x_dev, int64_t ld_x, double rtol, double atol,
             int maxit, int* its_host, double* relres_host);

/* Jacobi-Chebyshev iteration (no inner products) with eigenvalue bounds
 * [lmin, lmax] of D^-1 B_k; same system definition as irk_pcg; fixed
 * iteration count `iters`. */
int irk_chebyshev(irk_ctx* ctx, int nb, const double* alpha_host, const double* beta_host,
                  const irk_mat* A, const irk_mat* Bm, const double* shift_dev,
                  const uint8_t* rowmask_dev, const double* lmin_host,
                  const double* lmax_host, const double* rhs_dev, int64_t ld_rhs,
                  double* x_dev, int64_t ld_x, int iters);

/* ------------------------------------------------------ semilinear kernels
 * Residual of the stacked stage system for F(u, u') = M u' + kscale*K u +
 * M g(u) - f, g(u) = sum_p coef[p] u^p (p < ncoef <= 8), on interleaved
 * blocks:  U = u + dt * (A (x) I) X  (stage-derivative unknowns),
 *          R_i = M X_i + kscale*K U_i + M g(U_i)  (- F_i if F given)
 *          D_i = g'(U_i)                         (Jacobian diagonal weights)
 * Constrained rows (rowmask) of R are zeroed (stepper.py:516-524). */
int irk_semilinear_residual(irk_ctx* ctx, int s, const double* A_host, double dt,
                            const irk_mat* M, const irk_mat* K, double kscale,
                            int ncoef, const double* coef_host, const double* u_dev,
                            const double* X_dev, const double* F_dev,
                            const uint8_t* rowmask_dev, double* R_dev, double* D_dev);

/* ---- finite-element load vectors and error norms (SURVEY §8 f) ---------
 * Structured grids of the manufactured-solution problems: dim 1 (P1
 * intervals) or 2 (Q1 squares), N cells per direction, 2-point Gauss rule
 * per direction (problems.py:158-191).  Quadrature data are q-major:
 * value at point q of element e at [q*nelem + e].  */
/* out = (f, phi_v) element by element, in the reference's accumulation
 * order (assemble_load, problems.py:194-202): bitwise equal for equal f. */
int irk_fe_load(irk_ctx* ctx, int dim, int64_t N, const double* f_dev, double* out_dev);
/* f at the quadrature points of the built-in manufactured solutions:
 * kind 1 = heat_mms_1d, 2 = heat_mms_2d (problems.py:113-149). */
int irk_fe_mms_forcing(irk_ctx* ctx, int kind, int64_t N, double t, double* f_dev);
/* sum_q w_q sum_e [(u_h - uex)^2 + |grad u_h - gex|^2] (gradient part when
 * gex_dev != NULL, layout [(q*dim + d)*nelem + e]; uex_dev NULL = 0):
 * squared l2_error / h1_error (problems.py:205-232).  Synchronous. */
int irk_fe_error_sq(irk_ctx* ctx, int dim, int64_t N, const double* u_dev, const double* uex_dev,
                    const double* gex_dev, double* result_host);

/* ---- geometric multigrid for the P1 stage blocks ------------------------
 * Replaces the exact block factorisations (sparsela.py:149-191) for blocks
 * assembled on structured grids: level l is the block re-assembled with
 * N_l = N_0 / 2^l cells per direction ((N_l+1)^dim rows, identity rows at
 * masks[l] != 0); prolongation = P1 interpolation on the nested grids,
 * restriction its transpose, Chebyshev smoothing (nu steps pre/post; nu = 0
 * picks 2) and
 * `ncoarse` Chebyshev steps on the coarsest level.  The handle keeps
 * pointers to the level matrices and masks (they must outlive it). */
typedef struct irk_mg irk_mg;
int irk_mg_create(irk_ctx* ctx, int dim, int nlev, const int64_t* N_host,
                  const irk_mat* const* A_levels, const uint8_t* const* masks, int nu,
                  int ncoarse, irk_mg** out);
int irk_mg_destroy(irk_mg* mg);
/* z = V(r): one V-cycle from a zero start (r != z). */
int irk_mg_vcycle(irk_ctx* ctx, irk_mg* mg, const double* r_dev, double* z_dev);
/* Structured 2D path (matrix-free stencil tile kernels, chosen at create
 * time when every level is a verified 2D grid stencil with the full-boundary
 * Dirichlet set and 2 <= nu <= 4; env IRK_MG_GENERIC disables it): switch it on
 * (IRK_EINVAL when unavailable) or off, and query the hierarchy. */
int irk_mg_set_structured(irk_mg* mg, int on);
int irk_mg_info(const irk_mg* mg, int* nlev, int* structured);
/* Fast sine-transform preconditioner of the level-0 block (replaces the
 * V-cycle inside irk_mg_pcg when on): the reflection-symmetrised level-0
 * stencil inverted exactly by 2D DST-I (shared-memory FFTs of length 2N),
 * B_s^-1 = (2/N)^2 S Lambda^-1 S.  Available for verified 2D grid stencils
 * with the full-boundary Dirichlet set, N a power of two in [32, 2048].
 * Replaces the reference's exact block solve (sparsela.py:171-191) like
 * the V-cycle does: CG on the block to the requested tolerance. */
int irk_mg_set_dst(irk_mg* mg, int on);
int irk_mg_dst_info(const irk_mg* mg, int* available, int* on);
/* CG on the level-0 block preconditioned by one V-cycle per iteration;
 * strided rhs/x as irk_pcg; status as irk_pcg. */
int irk_mg_pcg(irk_ctx* ctx, irk_mg* mg, const double* rhs_dev, int64_t ld_rhs, double* x_dev,
               int64_t ld_x, double rtol, double atol, int maxit, int* its_host,
               double* relres_host);
/* n independent block solves (system k: mgs[k], rhs_dev + k*rhs_step,
 * x_dev + k*x_step; steps in doubles): the block-Jacobi preconditioner's
 * diagonal blocks (precond.py:97-117 with no coupling terms).  Deferred
 * solves run concurrently on auxiliary streams (see irk_mgc_cocg_multi). */
int irk_mg_pcg_multi(irk_ctx* ctx, int n, irk_mg* const* mgs, const double* rhs_dev,
                     int64_t ld_rhs, int64_t rhs_step, double* x_dev, int64_t ld_x,
                     int64_t x_step, double rtol, double atol, int maxit, int* its_host,
                     double* relres_host);

/* ---- complex multigrid for the Schur-pair blocks ------------------------
 * alpha M + beta K with complex alpha, beta (the 2x2 real-Schur pairs of the
 * transformed stage preconditioner): levels M_l, K_l on N_l = N_0 / 2^l
 * grids sharing one pattern per level, masked rows identity and masked
 * columns eliminated (the caller passes eliminated copies); Chebyshev
 * smoothing on D^-1 A with complex D over a real interval.  Replaces the
 * batched Jacobi-COCG of irk_cocg for P1 grid blocks. */
typedef struct irk_mgc irk_mgc;
int irk_mgc_create(irk_ctx* ctx, int dim, int nlev, const int64_t* N_host,
                   const irk_mat* const* M_levels, const irk_mat* const* K_levels,
                   const uint8_t* const* masks, double alpha_re, double alpha_im, double beta_re,
                   double beta_im, int nu, int ncoarse, irk_mgc** out);
int irk_mgc_destroy(irk_mgc* mg);
/* Structured 3D path (matrix-free Kuhn-stencil tile kernels, chosen at
 * create time for 3D levels with the full-boundary Dirichlet set and nu = 2;
 * env IRK_MG_GENERIC disables it): switch it on (IRK_EINVAL when unavailable)
 * or off, and query the hierarchy. */
int irk_mgc_set_structured(irk_mgc* mg, int on);
int irk_mgc_info(const irk_mgc* mg, int* nlev, int* structured);
/* Fast sine-transform preconditioner of the level-0 pair block (replaces the
 * complex V-cycle inside irk_mgc_cocg when on): the level-0 3x3x3 stencil,
 * averaged over the reflections of every offset, inverted exactly by 3D
 * DST-I (shared-memory mixed-radix FFTs of length 2N, five line-transform
 * launches), B_s^-1 = (2/N)^3 F Lambda^-1 F with complex Lambda.  Available
 * for verified 3D grid stencils with the full-boundary Dirichlet set and
 * 2N = 2^a or 3 * 2^a in [24, 384].  Stands where the reference's exact
 * block solve does (sparsela.py:171-191): COCG on the block to the requested
 * tolerance. */
int irk_mgc_set_dst(irk_mgc* mg, int on);
/* One application z = P^-1 r of the pair block's preconditioner (the V-cycle,
 * or the sine transform when on); r, z interleaved complex, contiguous,
 * 16-byte aligned, r != z. */
int irk_mgc_vcycle(irk_ctx* ctx, irk_mgc* mg, const double* r_dev, double* z_dev);
int irk_mgc_dst_info(const irk_mgc* mg, int* available, int* on);
/* COCG on the level-0 block preconditioned by one complex V-cycle per
 * iteration; rhs/x interleaved complex (re, im) with leading dimensions in
 * doubles (even), 16-byte aligned; status and deferred logging as irk_pcg. */
int irk_mgc_cocg(irk_ctx* ctx, irk_mgc* mg, const double* rhs_dev, int64_t ld_rhs,
                 double* x_dev, int64_t ld_x, double rtol, double atol, int maxit,
                 int* its_host, double* relres_host);
/* n independent pair solves (system k: mgs[k], rhs_dev + k*rhs_step,
 * x_dev + k*x_step; steps in doubles, even): the transformed
 * block-diagonal preconditioner's pair blocks (precond.py:120-157 solves its
 * blocks one by one).  Deferred solves (NULL its/relres, log enabled) run
 * concurrently on auxiliary streams forked from and joined into the context
 * stream; otherwise one after another.  its_host/relres_host: n entries. */
int irk_mgc_cocg_multi(irk_ctx* ctx, int n, irk_mgc* const* mgs, const double* rhs_dev,
                       int64_t ld_rhs, int64_t rhs_step, double* x_dev, int64_t ld_x,
                       int64_t x_step, double rtol, double atol, int maxit, int* its_host,
                       double* relres_host);

#ifdef __cplusplus
}
#endif
#endif /* IRK_H */
