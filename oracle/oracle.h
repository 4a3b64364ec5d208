/* TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * Shared C declarations of the CPU oracles for the KKT factor+solve path:
 *   - oracle/cyq_oracle.c : plain-C restatement of the reference algorithm
 *                           (liboracle.so, "port" CPU baseline);
 *   - oracle/ref_shim.cpp : extern "C" wrapper around the reference's own
 *                           sources compiled from /root/reference into
 *                           oracle/_ref/libcyqref.so ("reference" baseline).
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load them.
 *
 * Array layouts (all row-major, instance-major, stage-major; "b" = instance):
 *   A[b][N][nx][nx]  B[b][N][nx][nu]  R[b][N][nu][nu]  S[b][N][nu][nx]
 *   Q[b][N+1][nx][nx] f[b][N][nx] r[b][N][nu] q[b][N+1][nx] x_init[b][nx]
 *   rhs: ru[b][N][nu] qx[b][N+1][nx] fd[b][N][nx]
 *   sol: u[b][N][nu]  x[b][N+1][nx]  lam[b][N][nx]
 * This is the reference's EqOCP / EqRhs / EqSolution
 * (proj/include/cyqlone/ocp.hpp:24-59) with each std::vector<DenseMatrix>
 * flattened (DenseMatrix is row-major, batch_matrix.hpp:170-189).
 */
#ifndef CYQ_ORACLE_H
#define CYQ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t N, nx, nu, P, batch;
} oc_dims;

typedef struct {
    const double *A, *B, *R, *S, *Q, *f, *r, *q, *x_init;
} oc_ocp;

typedef struct {
    const double *ru, *qx, *fd;
} oc_rhs;

typedef struct {
    double *u, *x, *lam;
} oc_sol;

/* Factor blocks of one instance, in the reference's public Factor members
 * (kkt_solver.hpp:69-105), unpacked per column c to dense row-major:
 *   LH[s][c][nux][nux] (lower, upper part zero), LB[s][c][nx][nu],
 *   Acl[s][c][nx][nx], LA[c][nx][nx], T[c][nx][nx] (upper),
 *   Mfwd/Mbwd[c][nx][nx] (full symmetric), W[c][nx][nx],
 *   schur_diag[c][nx][nx] (full symmetric), schur_sub[c][nx][nx]. */
typedef struct {
    double *LH, *LB, *Acl, *LA, *T, *Mfwd, *Mbwd, *W, *schur_diag, *schur_sub;
} oc_factor_blocks;

/* Status mirroring batla::factorize_error (kernels.hpp:11-16):
 * code 0 ok, 1 invalid argument, 2 pivot failure. */
typedef struct {
    int32_t code, kind; /* kind 0: Riccati column, 1: cyclic reduction */
    int64_t instance, column_or_level, stage, pivot;
} oc_status;

/* ---- plain-C restatement (liboracle.so) ------------------------------- */
int oc_solve_problem(const oc_dims *d, const oc_ocp *p, oc_sol *out,
                     oc_status *st);
int oc_solve(const oc_dims *d, const oc_ocp *p, const oc_rhs *rhs,
             oc_sol *out, oc_status *st);
int oc_factor_export(const oc_dims *d, const oc_ocp *p, oc_factor_blocks *o,
                     oc_status *st);
/* EqRhs::of_problem (ocp.cpp:154-174) for every instance of the batch. */
void oc_rhs_of_problem(const oc_dims *d, const oc_ocp *p, double *ru,
                       double *qx, double *fd);
/* kkt_residual_eq (ocp.cpp:180-230): out[b*4 + {stat_u,stat_x,dyn,term}]. */
void oc_kkt_residual(const oc_dims *d, const oc_ocp *p, const oc_rhs *rhs,
                     const oc_sol *s, double *out);
/* Multiply-add counts of factor and solve (batla::flops semantics,
 * kernels.cpp:8-15), for one instance: out[0] factor, out[1] solve. */
void oc_fma_counts(const oc_dims *d, uint64_t *out);
/* Batched solve_problem on `threads` pthreads, instance-parallel; returns
 * elapsed seconds of the factor+solve work (rhs formed before timing). */
double oc_bench_solve_problem(const oc_dims *d, const oc_ocp *p,
                              int64_t n_solves, int threads, oc_sol *out);

/* Exact line search (qpalm::line_search_exact, line_search.cpp:112-206)
 * of psi'(tau) = eta tau + beta + sum_i delta_i [delta_i tau - alpha_i]_+
 * over m terms registered as LineSearchData::add_term (line_search.cpp:
 * 9-27). Returns 0 (tau set), 1 when psi'(0) > 0 (not a descent direction;
 * the reference throws std::invalid_argument). */
int oc_line_search(int64_t m, const double *alpha, const double *delta,
                   double eta, double beta, double *tau);
/* Batched line search on `threads` pthreads; returns elapsed seconds. */
double oc_bench_line_search(int64_t batch, int64_t m, const double *alpha,
                            const double *delta, const double *eta,
                            const double *beta, double *tau, int threads);

/* ---- reference shim (oracle/_ref/libcyqref.so) ------------------------ */
int ref_line_search(int64_t m, const double *alpha, const double *delta,
                    double eta, double beta, double *tau, int64_t *iters);
double ref_bench_line_search(int64_t batch, int64_t m, const double *alpha,
                             const double *delta, const double *eta,
                             const double *beta, double *tau, int threads);
int ref_solve_problem(const oc_dims *d, const oc_ocp *p, int64_t vlen,
                      int threads, oc_sol *out, double *resid,
                      oc_status *st);
int ref_solve(const oc_dims *d, const oc_ocp *p, const oc_rhs *rhs,
              int64_t vlen, oc_sol *out, oc_status *st);
int ref_factor_export(const oc_dims *d, const oc_ocp *p, int64_t vlen,
                      oc_factor_blocks *o, oc_status *st);
void ref_kkt_residual(const oc_dims *d, const oc_ocp *p, const oc_rhs *rhs,
                      const oc_sol *s, double *out);
void ref_fma_counts(const oc_dims *d, uint64_t *out);
/* random_eq_ocp (ocp.cpp:566-603) into caller-provided arrays. */
void ref_random_eq_ocp(int64_t N, int64_t nx, int64_t nu, uint64_t seed,
                       double conditioning, double *A, double *B, double *R,
                       double *S, double *Q, double *f, double *r, double *q,
                       double *x_init);
/* factor(p_old) -> kkt::update(p_new, C, D, C_term, dSigma) -> solve, instance 0 */
int ref_update_solve(const oc_dims *d, const oc_ocp *p_old, const oc_ocp *p_new, int64_t ny,
                     const double *D, const double *C, int64_t ny_term, const double *C_term,
                     const double *ds_stage, const double *ds_term, double rho, oc_sol *out,
                     int64_t *report);
double ref_bench_solve_problem(const oc_dims *d, const oc_ocp *p,
                               int64_t vlen, int64_t n_solves, int threads);

#ifdef __cplusplus
}
#endif
#endif
