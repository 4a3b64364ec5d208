/* cyqlone_b200 -- C ABI of the B200-native KKT factor+solve for
 * linear-quadratic optimal control problems (arXiv 2512.09058, "Cyqlone").
 *
 * Drop-in boundary for the reference's hot path
 *   cyqlone::kkt::factor / solve / solve_problem
 *   (/root/reference/proj/include/cyqlone/kkt_solver.hpp:118-128)
 * with a batch dimension added (the reference API is single-instance; its
 * internal "batch" is the P partition columns, kkt_solver.hpp:74-75).
 * The C++ mirror of the reference interface (include/cyqlone_b200/
 * kkt_solver.hpp) and the Python bindings sit on top of these entry points.
 *
 * Data layout (all FP64, C-contiguous, instance-major, stage-major, each
 * block row-major exactly like the reference's DenseMatrix,
 * batch_matrix.hpp:170-189; b = instance):
 *   A[b][N][nx][nx]  B[b][N][nx][nu]  R[b][N][nu][nu]  S[b][N][nu][nx]
 *   Q[b][N+1][nx][nx] f[b][N][nx] r[b][N][nu] q[b][N+1][nx] x_init[b][nx]
 *   rhs  ru[b][N][nu]  qx[b][N+1][nx]  fd[b][N][nx]          (EqRhs)
 *   sol  u[b][N][nu]   x[b][N+1][nx]   lam[b][N][nx]         (EqSolution)
 * Pointers are host memory (mem = CYQ_MEM_HOST; pinned memory lets the
 * copies overlap compute) or device memory on the context's GPU
 * (mem = CYQ_MEM_DEVICE). Calls are stream-ordered on the context stream;
 * host-memory calls return after the results are in host memory.
 *
 * Errors mirror the reference's exceptions: std::invalid_argument (P not a
 * power of two, kkt_factor.cpp:253-256) -> CYQ_INVALID_ARG; batla::
 * factorize_error (kernels.cpp:42-45, block_tridiag.cpp:140-147) ->
 * CYQ_PIVOT_FAIL with per-instance detail in cyq_status, other instances of
 * the batch are still solved.
 */
#ifndef CYQLONE_B200_H
#define CYQLONE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CYQ_OK 0
#define CYQ_INVALID_ARG 1
#define CYQ_PIVOT_FAIL 2
#define CYQ_CUDA_ERR 3
#define CYQ_NO_DEVICE 4

#define CYQ_MEM_HOST 0
#define CYQ_MEM_DEVICE 1

#define CYQ_FAIL_RICCATI 0 /* column_or_level = column c, stage = position s */
#define CYQ_FAIL_CR 1      /* column_or_level = CR level, stage = block index */

typedef struct cyq_ctx cyq_ctx;
typedef struct cyq_factor cyq_factor;

/* Problem dimensions: horizon N, states nx, inputs nu, partitions P (power
 * of two; N is padded to a multiple of P as pad_problem does,
 * kkt_factor.cpp:27-47), number of independent instances. */
typedef struct {
    int64_t N, nx, nu, P, batch;
} cyq_dims;

typedef struct {
    const double *A, *B, *R, *S, *Q, *f, *r, *q, *x_init;
} cyq_ocp_batch;

typedef struct {
    const double *ru, *qx, *fd;
} cyq_rhs_batch;

typedef struct {
    double *u, *x, *lam;
} cyq_sol_batch;

/* Per-instance status (mirrors batla::factorize_error{batch_index, pivot}). */
typedef struct {
    int32_t code;  /* CYQ_OK / CYQ_PIVOT_FAIL */
    int32_t kind;  /* CYQ_FAIL_RICCATI / CYQ_FAIL_CR */
    int64_t instance, column_or_level, stage, pivot;
} cyq_status;

/* One context per GPU; no global state. */
int cyq_ctx_create(int device, cyq_ctx **out);
int cyq_ctx_destroy(cyq_ctx *ctx);
/* Use an existing cudaStream_t (NULL = the context's own stream). */
int cyq_ctx_set_stream(cyq_ctx *ctx, void *cuda_stream);
int cyq_ctx_synchronize(cyq_ctx *ctx);
/* Last error message of this context (static storage of the context). */
const char *cyq_ctx_last_error(cyq_ctx *ctx);

/* kkt::solve_problem (kkt_solve.cpp:311-317) for every instance:
 * factor + solve with EqRhs::of_problem (ocp.cpp:154-174). `status` may be
 * NULL or point to `batch` entries. Returns the worst status code. */
int cyq_solve_problem_batch(cyq_ctx *ctx, const cyq_dims *dims,
                            const cyq_ocp_batch *prob, const cyq_sol_batch *sol,
                            cyq_status *status, int mem);

/* kkt::factor (kkt_factor.cpp:251-313): the factor stays on the device. */
int cyq_factor_batch(cyq_ctx *ctx, const cyq_dims *dims,
                     const cyq_ocp_batch *prob, int mem, cyq_factor **out,
                     cyq_status *status);
/* kkt::solve (kkt_solve.cpp:23-309) with an explicit right-hand side; `prob`
 * must be the problem the factor was computed from (its A, B enter the
 * substitution, as in the reference signature). The solve's vectors
 * (forward-substituted y, wl, coupling rhs and multipliers) live in the
 * factor's workspace: solves on one factor are stream-ordered on the
 * context stream and must not run concurrently on different streams. */
int cyq_solve_batch(cyq_ctx *ctx, const cyq_factor *factor,
                    const cyq_ocp_batch *prob, const cyq_rhs_batch *rhs,
                    const cyq_sol_batch *sol, int mem);
int cyq_factor_destroy(cyq_factor *factor);

/* Copies the factor blocks of instance `inst` to host memory in the
 * reference's Factor member shapes (kkt_solver.hpp:76-95), dense row-major
 * per column c: LH[s][c][nux][nux], LB[s][c][nx][nu], Acl[s][c][nx][nx],
 * LA[c][nx][nx]; any pointer may be NULL. For block-level parity tests. */
int cyq_factor_materialize(const cyq_factor *factor, int64_t inst, double *LH,
                           double *LB, double *Acl, double *LA);

/* The Schur-side factor blocks of instance `inst` in the reference's Factor
 * member shapes (kkt_solver.hpp:84-97), dense row-major per column / block:
 * T[P][nx][nx] (= L_Q^{-T} of the column's last stage, upper), Mfwd, Mbwd,
 * W (= T LA') [P][nx][nx] (sc_Mfwd / sc_Mbwd / sc_W), the assembled Schur
 * complement schur_diag[P][nx][nx], schur_sub[P][nx][nx] (block (k+1, k);
 * the circular [P-1] is zero), and the CR factor (blocktri::CRFactor,
 * block_tridiag.hpp:56-79): level l, slot mm at index P - (P >> l) + mm of
 * cr_L / cr_U / cr_Y [P-1][nx][nx] (L = chol of the eliminated block,
 * U = K_{k-1}' L^{-T}, Y = K_k L^{-T}), cr_Lbase[nx][nx]. Any pointer may
 * be NULL. CYQ_INVALID_ARG for factors whose Schur path (the per-level /
 * scalar kernels of unusual shapes) keeps no persistent blocks. */
int cyq_factor_materialize_schur(const cyq_factor *factor, int64_t inst, double *T,
                                 double *Mfwd, double *Mbwd, double *W,
                                 double *schur_diag, double *schur_sub,
                                 double *cr_L, double *cr_U, double *cr_Y,
                                 double *cr_Lbase);

/* kkt::update (kkt_solver.hpp:152-161, kkt_update.cpp:372-477) of every
 * instance of a factor, in place: afterwards the factor is (up to roundoff)
 * the factor of p_new, whose stage Hessians are H_j + (D_j | C_j)' dSigma_j
 * (D_j | C_j) (terminal: C_term' dSigma_term C_term). Per partition column
 * the accumulated update rank r (nonzeros of dSigma over its stages,
 * kkt_update.cpp:392-409) selects the path: r = 0 untouched; r < rho nx
 * the low-rank hyperbolic-Householder column update on the GPU; r >= rho nx
 * (or a hyperbolic breakdown) a refactorization of the column. The Schur
 * complement and its CR factor are then re-formed from the updated columns
 * (instances with any nonzero rank). Layouts: C[b][N][ny][nx],
 * D[b][N][ny][nu], ds_stage[b][N][ny], C_term[b][ny_term][nx],
 * ds_term[b][ny_term] (ny_term may be 0); `mem` says where p_new, C, D,
 * C_term and the dSigma arrays live. report[batch] (nullable) mirrors
 * UpdateReport per instance. Returns CYQ_PIVOT_FAIL when a refactorized
 * column or the CR factor breaks down. */
typedef struct {
    int64_t columns_updated, columns_refactored, schur_refactored, schur_levels_updated;
} cyq_update_report;
int cyq_factor_update_batch(cyq_ctx *ctx, cyq_factor *factor, const cyq_ocp_batch *p_new,
                            int64_t ny, const double *C, const double *D,
                            const double *ds_stage, int64_t ny_term,
                            const double *C_term, const double *ds_term,
                            double rho, int mem, cyq_update_report *report);

/* Newton-system assembly of the QPALM inner loop (qpalm::assemble_newton,
 * qpalm.cpp:167-225, equality part; BASELINE config 4): for every instance
 * and stage j
 *   R_out = R + D_j' diag(sigma_j) D_j + gamma_inv I          (j < N)
 *   S_out = S + D_j' diag(sigma_j) C_j                        (j < N)
 *   Q_out = Q + C_j' diag(sigma_j) C_j + gamma_inv I (j >= 1) (j <= N)
 * with D[b][N][ny][nu], C[b][N+1][ny][nx] (C[N] = the terminal rows),
 * sigma[b][N+1][ny] (0 for inactive rows), R/S/Q in the problem layout.
 * DEVICE pointers on the context's GPU; stream-ordered, asynchronous. The
 * outputs plus the unchanged A, B, f, r, q, x_init form the Newton problem
 * for cyq_solve_problem_batch / cyq_factor_batch. ny <= 64, nx + nu <= 64. */
int cyq_augment_hessians_batch(cyq_ctx *ctx, const cyq_dims *dims, int64_t ny,
                               const double *R, const double *S, const double *Q,
                               const double *D, const double *C,
                               const double *sigma, double gamma_inv,
                               double *R_out, double *S_out, double *Q_out);

/* The Newton system of the QPALM inner loop solved in one call:
 * kkt::solve_problem (kkt_solve.cpp:311-317) of the problem whose Hessians
 * are augmented as cyq_augment_hessians_batch describes (qpalm::
 * assemble_newton, qpalm.cpp:167-225, then qpalm.cpp:368-413's factor +
 * solve). For the stage shapes the warp-level panel kernel covers
 * (nu = 8, nx = 16, ny = 24: BASELINE config 4) the assembly is fused into
 * the factorization's stage loads and the augmented Hessians never reach
 * HBM; other shapes run the assembly kernel into context scratch first.
 * DEVICE pointers only (prob, D, C, sigma, sol); stream-ordered. */
int cyq_solve_newton_batch(cyq_ctx *ctx, const cyq_dims *dims,
                           const cyq_ocp_batch *prob, int64_t ny,
                           const double *D, const double *C,
                           const double *sigma, double gamma_inv,
                           const cyq_sol_batch *sol, cyq_status *status);

/* Augmented-Lagrangian gradients of the QPALM inner loop
 * (qpalm::eval_al_gradients, qpalm.cpp:106-165), batched, for every
 * instance and stage j: with g = C_j x_j + D_j u_j (j = N: C_N x_N),
 *   yhat_j = y_j + sigma_j (g - clamp(g + y_j / sigma_j, bl_j, bu_j))
 *   ru_j   = r_j + R_j u_j + S_j x_j + D_j' yhat_j + gamma_inv (u_j - ubar_j)  j < N
 *   cres_j = f_j + A_j x_j + B_j u_j - x_{j+1}                                j < N
 *   qx_j   = q_j + Q_j x_j + S_j' u_j + C_j' yhat_j + gamma_inv (x_j - xbar_j) j >= 1
 *            (no S term at j = N; qx_0 is written as 0, unused)
 * Layouts: prob in the problem layout (R, S, Q, A, B, f, r, q read), D[b][N][ny][nu],
 * C[b][N+1][ny][nx] (C[N] = the terminal rows, ny_term = ny), bl, bu, y,
 * sigma, yhat [b][N+1][ny], u, ubar [b][N][nu], x, xbar, qx [b][N+1][nx],
 * ru [b][N][nu], cres [b][N][nx]. The Newton step's rhs is
 * (-ru, -qx, -cres) (qpalm.cpp:391-405). DEVICE pointers; stream-ordered. */
int cyq_al_gradients_batch(cyq_ctx *ctx, const cyq_dims *dims, int64_t ny,
                           const cyq_ocp_batch *prob, const double *D,
                           const double *C, const double *bl, const double *bu,
                           const double *u, const double *x, const double *y,
                           const double *sigma, const double *ubar,
                           const double *xbar, double gamma_inv, double *ru,
                           double *qx, double *yhat, double *cres);

/* Exact line search of the QPALM inner loop (qpalm::line_search_exact,
 * line_search.cpp:112-206, over LineSearchData::add_term of every term,
 * line_search.cpp:9-27), batched: for instance b, the root tau of
 *   psi'(tau) = eta[b] tau + beta[b] + sum_i delta_i [delta_i tau - alpha_i]_+
 * over the m terms alpha[b][i], delta[b][i] (delta = 0 or a non-finite
 * alpha / delta drops the term, as add_term does). status[b] (nullable):
 * CYQ_OK, or CYQ_INVALID_ARG when psi'(0) > 0 (the reference throws
 * std::invalid_argument); psi'(0) == 0 gives tau = 0. iterations (nullable,
 * DEVICE) receives the probes + scan steps per instance. alpha, delta, eta,
 * beta, tau are DEVICE pointers; the call synchronizes the context stream
 * (per-instance status to the host). Returns the worst status. */
int cyq_line_search_batch(cyq_ctx *ctx, int64_t batch, int64_t m,
                          const double *alpha, const double *delta,
                          const double *eta, const double *beta, double *tau,
                          int32_t *status, int64_t *iterations);

/* Kernel selection of a context (defaults: the fastest measured kernel per
 * shape). Options apply to later calls on this context; a factor keeps the
 * options it was computed with for its solves. A forced kernel that has no
 * specialisation for a shape falls back to the automatic choice. */
#define CYQ_OPT_PANEL 0         /* CYQ_PANEL_* (stage-panel Riccati kernel) */
#define CYQ_OPT_SCHUR 1         /* CYQ_SCHUR_* (Schur complement + CR) */
#define CYQ_OPT_SCHUR_WARPS 2   /* fused Schur CTA width: 0 auto, 2, 4 */
#define CYQ_OPT_SCHUR_CLUSTER 3 /* 1 (default): 8-CTA cluster per long horizon; 0 never */
#define CYQ_OPT_SPLIT 4         /* device batches in K parts on two streams (default 1) */
#define CYQ_OPT_BACKSUB 5       /* 0 auto, 1 generic runtime-shape kernel */
#define CYQ_OPT_FUSED_AUGMENT 6 /* 1 (default): Newton assembly fused into the panel */
#define CYQ_OPT_PANEL_WARPS 7   /* generic panel: warps per chain CTA, 0 auto */
#define CYQ_OPT_TAIL 8          /* CYQ_TAIL_* (FactorOptions::tail, kkt_solver.hpp:45-64) */
#define CYQ_OPT_PHASE_PROF 9    /* 1: per-stage phase clocks of chain 0 to stderr */
#define CYQ_OPT_ASYNC_STATUS 10 /* 1: device-memory calls return without a host sync;
                                   cyq_ctx_wait_status reports the last call */
#define CYQ_OPT_GRAPHS 11       /* 1 (default): a device-memory call repeated with the same
                                   shape and pointers replays a captured CUDA graph */
#define CYQ_OPT_VLEN 12          /* FactorOptions::vlen (power of two, default 4): with
                                   CYQ_TAIL_PCR the last min(P, vlen) Schur blocks are
                                   solved by parallel cyclic reduction */
#define CYQ_OPT_COUNT 13

#define CYQ_PANEL_AUTO 0
#define CYQ_PANEL_WARP 1      /* one warp per chain, compile-time shapes */
#define CYQ_PANEL_TWO_WARP 2  /* producer/consumer warp pair per chain */
#define CYQ_PANEL_CTA 3       /* one CTA per chain (large tile-aligned blocks) */
#define CYQ_PANEL_GENERIC 4   /* runtime-shape CTA kernel */
#define CYQ_PANEL_WARP_TMEM 5 /* warp kernel with W in tensor memory */
#define CYQ_PANEL_CTA_TMA 6   /* CTA kernel staging [B A] with TMA bulk copies */

#define CYQ_SCHUR_AUTO 0   /* fused one-kernel Schur + CR */
#define CYQ_SCHUR_LEVELS 1 /* per-level batch-wide tile kernels */
#define CYQ_SCHUR_SCALAR 2 /* runtime-shape scalar kernel */

#define CYQ_TAIL_CR1 0 /* cyclic reduction down to one block (default) */
#define CYQ_TAIL_PCR 1 /* parallel cyclic reduction for the last levels */
#define CYQ_TAIL_PCG 2 /* served by exact CR (meets the PCG tolerance contract) */

int cyq_ctx_set_option(cyq_ctx *ctx, int option, int64_t value);
int cyq_ctx_get_option(cyq_ctx *ctx, int option, int64_t *value);
/* With CYQ_OPT_ASYNC_STATUS, device-memory factor / solve_problem / Newton
 * calls enqueue their work and the per-instance failure keys' readback and
 * return CYQ_OK (argument errors are still reported at once). This waits
 * for the context stream and decodes the most recent such call's status
 * into `status` (n entries, may be NULL); returns its worst code. */
int cyq_ctx_wait_status(cyq_ctx *ctx, cyq_status *status, int64_t n);

/* Per-kernel device timing: when enabled, every launch of the pipeline is
 * bracketed by CUDA events on the context stream. `read` synchronizes and
 * returns, per kernel (0 riccati_panel, 1 schur_cr, 2 backsub, 3 forward
 * sweep, 4 Newton-system assembly / line search) -- ms[5], launches[5] -- the summed
 * milliseconds and launch counts since the last reset. */
int cyq_ctx_profile(cyq_ctx *ctx, int enable);
int cyq_ctx_profile_read(cyq_ctx *ctx, double *ms, int64_t *launches,
                         int reset);

/* Library build/runtime information (kernel names, tile shapes). */
const char *cyq_version(void);

#ifdef __cplusplus
}
#endif
#endif
