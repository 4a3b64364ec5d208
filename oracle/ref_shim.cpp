// TEST INFRASTRUCTURE ONLY — the reference checker, never the product.
//
// extern "C" shim over the reference's own factor+solve path, compiled
// together with the unmodified reference sources under /root/reference
// (see oracle/Makefile) into oracle/_ref/libcyqref.so. The shim only converts
// the flat instance-major arrays of oracle/oracle.h to and from the
// reference's EqOCP / EqRhs / EqSolution (proj/include/cyqlone/ocp.hpp:24-59)
// and calls:
//   cyqlone::kkt::factor / solve / solve_problem   (kkt_solver.hpp:118-128)
//   cyqlone::ocp::kkt_residual_eq                  (ocp.cpp:180-230)
//   cyqlone::ocp::random_eq_ocp                    (ocp.cpp:566-603)
//   cyqlone::batla::flops::{reset,total}           (kernels.cpp:8-15)
#include "oracle.h"

#include <cyqlone/kkt_solver.hpp>
#include <cyqlone/qpalm.hpp>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

using namespace cyqlone;
using batla::index_t;
using cyqlone::kkt::Factor;
using cyqlone::kkt::FactorOptions;
using cyqlone::ocp::EqOCP;
using cyqlone::ocp::EqRhs;
using cyqlone::ocp::EqSolution;
using cyqlone::ocp::Mat;
using cyqlone::ocp::Vec;

namespace {

Mat mat_from(const double *p, index_t m, index_t n) {
    Mat a(m, n);
    std::copy_n(p, m * n, a.a.data());
    return a;
}
Vec vec_from(const double *p, index_t n) { return Vec(p, p + n); }

EqOCP make_ocp(const oc_dims *d, const oc_ocp *p, index_t b) {
    const index_t N = d->N, nx = d->nx, nu = d->nu;
    EqOCP o;
    o.N  = N;
    o.nx = nx;
    o.nu = nu;
    o.resize();
    for (index_t j = 0; j < N; ++j) {
        auto ju = static_cast<std::size_t>(j);
        o.A[ju] = mat_from(p->A + ((b * N + j) * nx * nx), nx, nx);
        o.B[ju] = mat_from(p->B + ((b * N + j) * nx * nu), nx, nu);
        o.R[ju] = mat_from(p->R + ((b * N + j) * nu * nu), nu, nu);
        o.S[ju] = mat_from(p->S + ((b * N + j) * nu * nx), nu, nx);
        o.f[ju] = vec_from(p->f + (b * N + j) * nx, nx);
        o.r[ju] = vec_from(p->r + (b * N + j) * nu, nu);
    }
    for (index_t j = 0; j <= N; ++j) {
        auto ju = static_cast<std::size_t>(j);
        o.Q[ju] = mat_from(p->Q + ((b * (N + 1) + j) * nx * nx), nx, nx);
        o.q[ju] = vec_from(p->q + (b * (N + 1) + j) * nx, nx);
    }
    o.x_init = vec_from(p->x_init + b * nx, nx);
    return o;
}

EqRhs make_rhs(const oc_dims *d, const oc_rhs *r, index_t b) {
    const index_t N = d->N, nx = d->nx, nu = d->nu;
    EqRhs o;
    for (index_t j = 0; j < N; ++j) {
        o.ru.push_back(vec_from(r->ru + (b * N + j) * nu, nu));
        o.fd.push_back(vec_from(r->fd + (b * N + j) * nx, nx));
    }
    for (index_t j = 0; j <= N; ++j)
        o.qx.push_back(vec_from(r->qx + (b * (N + 1) + j) * nx, nx));
    return o;
}

EqSolution make_sol(const oc_dims *d, const oc_sol *s, index_t b) {
    const index_t N = d->N, nx = d->nx, nu = d->nu;
    EqSolution o;
    for (index_t j = 0; j < N; ++j) {
        o.u.push_back(vec_from(s->u + (b * N + j) * nu, nu));
        o.lam.push_back(vec_from(s->lam + (b * N + j) * nx, nx));
    }
    for (index_t j = 0; j <= N; ++j)
        o.x.push_back(vec_from(s->x + (b * (N + 1) + j) * nx, nx));
    return o;
}

void store_sol(const oc_dims *d, const EqSolution &s, oc_sol *o, index_t b) {
    const index_t N = d->N, nx = d->nx, nu = d->nu;
    for (index_t j = 0; j < N; ++j) {
        auto ju = static_cast<std::size_t>(j);
        std::copy_n(s.u[ju].data(), nu, o->u + (b * N + j) * nu);
        std::copy_n(s.lam[ju].data(), nx, o->lam + (b * N + j) * nx);
    }
    for (index_t j = 0; j <= N; ++j)
        std::copy_n(s.x[static_cast<std::size_t>(j)].data(), nx,
                    o->x + (b * (N + 1) + j) * nx);
}

void set_status(oc_status *st, int code, int kind, index_t inst, index_t col,
                index_t stage, index_t piv) {
    if (!st)
        return;
    st->code            = code;
    st->kind            = kind;
    st->instance        = inst;
    st->column_or_level = col;
    st->stage           = stage;
    st->pivot           = piv;
}

int g_tail = 0; // ref_set_tail: 0 cr1, 1 pcr, 2 pcg

FactorOptions opts_of(const oc_dims *d, int64_t vlen) {
    FactorOptions o;
    o.P       = d->P;
    o.vlen    = vlen;
    o.workers = 1;
    o.tail    = g_tail == 1 ? kkt::Tail::pcr : g_tail == 2 ? kkt::Tail::pcg : kkt::Tail::cr1;
    return o;
}

template <class F> int guarded(oc_status *st, index_t b, F &&fn) {
    try {
        fn();
        set_status(st, 0, 0, b, 0, 0, 0);
        return 0;
    } catch (const batla::factorize_error &e) {
        set_status(st, 2, std::strstr(e.what(), "cyclic") ? 1 : 0, b,
                   e.batch_index, 0, e.pivot);
        return 2;
    } catch (const std::invalid_argument &) {
        set_status(st, 1, 0, b, 0, 0, 0);
        return 1;
    }
}

void dense_of(const batla::BatchMatrix &m, index_t lane, double *out) {
    for (index_t r = 0; r < m.rows(); ++r)
        for (index_t c = 0; c < m.cols(); ++c)
            out[r * m.cols() + c] = m(lane, r, c);
}

} // namespace

extern "C" {

// FactorOptions::tail of every following call (kkt_solver.hpp:45-57)
void ref_set_tail(int tail) { g_tail = tail; }

int ref_solve_problem(const oc_dims *d, const oc_ocp *p, int64_t vlen,
                      int threads, oc_sol *out, double *resid,
                      oc_status *st) {
    std::atomic<int> worst{0};
    const index_t B = d->batch;
    threads         = std::max(1, std::min<int>(threads, (int)B));
    auto work = [&](int w) {
        for (index_t b = w; b < B; b += threads) {
            int rc = guarded(st ? st + b : nullptr, b, [&] {
                EqOCP o = make_ocp(d, p, b);
                EqSolution s = kkt::solve_problem(o, opts_of(d, vlen));
                store_sol(d, s, out, b);
                if (resid)
                    resid[b] = ocp::kkt_residual_eq(
                                   o, EqRhs::of_problem(o), s)
                                   .max();
            });
            int cur = worst.load();
            while (rc > cur && !worst.compare_exchange_weak(cur, rc)) {
            }
        }
    };
    std::vector<std::thread> ts;
    for (int w = 1; w < threads; ++w)
        ts.emplace_back(work, w);
    work(0);
    for (auto &t : ts)
        t.join();
    return worst.load();
}

int ref_solve(const oc_dims *d, const oc_ocp *p, const oc_rhs *rhs,
              int64_t vlen, oc_sol *out, oc_status *st) {
    int worst = 0;
    for (index_t b = 0; b < d->batch; ++b) {
        int rc = guarded(st ? st + b : nullptr, b, [&] {
            EqOCP o = make_ocp(d, p, b);
            Factor f = kkt::factor(o, opts_of(d, vlen));
            EqSolution s = kkt::solve(f, o, make_rhs(d, rhs, b));
            store_sol(d, s, out, b);
        });
        worst = std::max(worst, rc);
    }
    return worst;
}

// kkt::factor(p_old) -> kkt::update(p_new, C, D, C_term, dSigma) -> kkt::solve
// (EqRhs::of_problem(p_new)) of instance 0 (kkt_update.cpp:372-477):
// D[N][ny][nu], C[N][ny][nx] (stage rows), C_term[ny_term][nx],
// ds_stage[N][ny], ds_term[ny_term]; report[4] = UpdateReport fields.
int ref_update_solve(const oc_dims *d, const oc_ocp *p_old, const oc_ocp *p_new, int64_t ny,
                     const double *D, const double *C, int64_t ny_term, const double *C_term,
                     const double *ds_stage, const double *ds_term, double rho, oc_sol *out,
                     int64_t *report) {
    return guarded(nullptr, 0, [&] {
        const index_t N = d->N, nx = d->nx, nu = d->nu;
        EqOCP o0 = make_ocp(d, p_old, 0), o1 = make_ocp(d, p_new, 0);
        kkt::FactorOptions opts = opts_of(d, 4);
        opts.rho = rho;
        Factor f = kkt::factor(o0, opts);
        std::vector<batla::DenseMatrix> Cm, Dm;
        kkt::SigmaDelta ds;
        for (index_t j = 0; j < N; ++j) {
            batla::DenseMatrix dj(ny, nu), cj(ny, nx);
            for (index_t i = 0; i < ny; ++i) {
                for (index_t a = 0; a < nu; ++a)
                    dj(i, a) = D[(j * ny + i) * nu + a];
                for (index_t a = 0; a < nx; ++a)
                    cj(i, a) = C[(j * ny + i) * nx + a];
            }
            Dm.push_back(dj);
            Cm.push_back(cj);
            ds.stage.emplace_back(ds_stage + j * ny, ds_stage + (j + 1) * ny);
        }
        batla::DenseMatrix ct(ny_term, nx);
        for (index_t i = 0; i < ny_term; ++i)
            for (index_t a = 0; a < nx; ++a)
                ct(i, a) = C_term[i * nx + a];
        ds.terminal.assign(ds_term, ds_term + ny_term);
        kkt::UpdateReport r = kkt::update(f, o1, Cm, Dm, ct, ds);
        report[0] = r.columns_updated;
        report[1] = r.columns_refactored;
        report[2] = r.schur_refactored ? 1 : 0;
        report[3] = r.schur_levels_updated;
        EqSolution s = kkt::solve(f, o1, ocp::EqRhs::of_problem(o1));
        store_sol(d, s, out, 0);
    });
}

int ref_factor_export(const oc_dims *d, const oc_ocp *p, int64_t vlen,
                      oc_factor_blocks *o, oc_status *st) {
    return guarded(st, 0, [&] {
        EqOCP pr = make_ocp(d, p, 0);
        Factor f = kkt::factor(pr, opts_of(d, vlen));
        const index_t nx = d->nx, nu = d->nu, nux = nx + nu, P = d->P;
        const index_t n = f.part.n_per;
        for (index_t s = 0; s < n; ++s)
            for (index_t c = 0; c < P; ++c) {
                auto su = static_cast<std::size_t>(s);
                double *lh = o->LH + (s * P + c) * nux * nux;
                dense_of(f.LH[su], c, lh);
                for (index_t r = 0; r < nux; ++r) // LH is lower triangular
                    for (index_t k = r + 1; k < nux; ++k)
                        lh[r * nux + k] = 0;
                dense_of(f.LB[su], c, o->LB + (s * P + c) * nx * nu);
                dense_of(f.Acl[su], c, o->Acl + (s * P + c) * nx * nx);
            }
        for (index_t c = 0; c < P; ++c) {
            dense_of(f.LA, c, o->LA + c * nx * nx);
            dense_of(f.T, c, o->T + c * nx * nx);
            dense_of(f.sc_W, c, o->W + c * nx * nx);
            double *mf = o->Mfwd + c * nx * nx, *mb = o->Mbwd + c * nx * nx,
                   *sd = o->schur_diag + c * nx * nx;
            dense_of(f.sc_Mfwd, c, mf);
            dense_of(f.sc_Mbwd, c, mb);
            dense_of(f.schur.diag, c, sd);
            dense_of(f.schur.subdiag, c, o->schur_sub + c * nx * nx);
            // symmetric_lower kinds: the lower triangle is authoritative
            for (index_t r = 0; r < nx; ++r)
                for (index_t k = r + 1; k < nx; ++k) {
                    mf[r * nx + k] = mf[k * nx + r];
                    mb[r * nx + k] = mb[k * nx + r];
                    sd[r * nx + k] = sd[k * nx + r];
                }
        }
    });
}

// The CR factor of the Schur complement (Factor::schur_cr,
// block_tridiag.hpp:56-79) of instance 0: level l, slot mm at index
// P - (P >> l) + mm of L / U / Y [P-1][nx][nx] (dense row-major), L_base.
int ref_factor_export_cr(const oc_dims *d, const oc_ocp *p, int64_t vlen, double *L, double *U,
                         double *Y, double *Lbase, oc_status *st) {
    return guarded(st, 0, [&] {
        EqOCP pr = make_ocp(d, p, 0);
        Factor f = kkt::factor(pr, opts_of(d, vlen));
        const index_t nx = d->nx, P = d->P;
        const auto &cr = f.schur_cr;
        for (index_t l = 0; l + 1 < cr.n_levels; ++l) {
            const index_t half = (P >> l) / 2, o0 = P - (P >> l);
            for (index_t mm = 0; mm < half; ++mm) {
                const auto lu = static_cast<std::size_t>(l);
                double *lo = L + (o0 + mm) * nx * nx;
                dense_of(cr.L[lu], mm, lo);
                for (index_t r = 0; r < nx; ++r)
                    for (index_t k = r + 1; k < nx; ++k)
                        lo[r * nx + k] = 0;
                dense_of(cr.U[lu], mm, U + (o0 + mm) * nx * nx);
                dense_of(cr.Y[lu], mm, Y + (o0 + mm) * nx * nx);
            }
        }
        if (cr.L_base.batch() > 0) {
            dense_of(cr.L_base, 0, Lbase);
            for (index_t r = 0; r < nx; ++r)
                for (index_t k = r + 1; k < nx; ++k)
                    Lbase[r * nx + k] = 0;
        }
    });
}

void ref_kkt_residual(const oc_dims *d, const oc_ocp *p, const oc_rhs *rhs,
                      const oc_sol *s, double *out) {
    for (index_t b = 0; b < d->batch; ++b) {
        EqOCP o = make_ocp(d, p, b);
        auto r  = ocp::kkt_residual_eq(o, make_rhs(d, rhs, b),
                                       make_sol(d, s, b));
        out[b * 4 + 0] = r.stat_u;
        out[b * 4 + 1] = r.stat_x;
        out[b * 4 + 2] = r.dynamics;
        out[b * 4 + 3] = r.terminal;
    }
}

void ref_fma_counts(const oc_dims *d, uint64_t *out) {
    EqOCP o = ocp::random_eq_ocp(d->N, d->nx, d->nu, 1);
    batla::flops::reset();
    Factor f = kkt::factor(o, opts_of(d, 1));
    out[0]   = batla::flops::total();
    batla::flops::reset();
    EqSolution s = kkt::solve(f, o, EqRhs::of_problem(o));
    out[1]       = batla::flops::total();
    (void)s;
}

void ref_random_eq_ocp(int64_t N, int64_t nx, int64_t nu, uint64_t seed,
                       double conditioning, double *A, double *B, double *R,
                       double *S, double *Q, double *f, double *r, double *q,
                       double *x_init) {
    EqOCP o = ocp::random_eq_ocp(N, nx, nu, seed, conditioning);
    for (index_t j = 0; j < N; ++j) {
        auto ju = static_cast<std::size_t>(j);
        std::copy_n(o.A[ju].a.data(), nx * nx, A + j * nx * nx);
        std::copy_n(o.B[ju].a.data(), nx * nu, B + j * nx * nu);
        std::copy_n(o.R[ju].a.data(), nu * nu, R + j * nu * nu);
        std::copy_n(o.S[ju].a.data(), nu * nx, S + j * nu * nx);
        std::copy_n(o.f[ju].data(), nx, f + j * nx);
        std::copy_n(o.r[ju].data(), nu, r + j * nu);
    }
    for (index_t j = 0; j <= N; ++j) {
        auto ju = static_cast<std::size_t>(j);
        std::copy_n(o.Q[ju].a.data(), nx * nx, Q + j * nx * nx);
        std::copy_n(o.q[ju].data(), nx, q + j * nx);
    }
    std::copy_n(o.x_init.data(), nx, x_init);
}

double ref_bench_solve_problem(const oc_dims *d, const oc_ocp *p,
                               int64_t vlen, int64_t n_solves, int threads) {
    // Problems and right-hand sides are built before the clock starts
    // (generation and EqRhs::of_problem are excluded); the
    // timed region is kkt::factor + kkt::solve only, instance-parallel, one
    // std::thread per core, workers = 1 inside each solve.
    const index_t B = d->batch;
    std::vector<EqOCP> probs;
    std::vector<EqRhs> rhss;
    for (index_t b = 0; b < B; ++b) {
        probs.push_back(make_ocp(d, p, b));
        rhss.push_back(EqRhs::of_problem(probs.back()));
    }
    threads = std::max(1, threads);
    std::atomic<int64_t> next{0};
    std::atomic<int> failed{0};
    auto work = [&] {
        for (;;) {
            int64_t i = next.fetch_add(1);
            if (i >= n_solves)
                break;
            auto bu = static_cast<std::size_t>(i % B);
            try {
                Factor f     = kkt::factor(probs[bu], opts_of(d, vlen));
                EqSolution s = kkt::solve(f, probs[bu], rhss[bu]);
                if (s.u.empty())
                    failed = 1;
            } catch (...) {
                failed = 1;
            }
        }
    };
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ts;
    for (int w = 1; w < threads; ++w)
        ts.emplace_back(work);
    work();
    for (auto &t : ts)
        t.join();
    auto t1 = std::chrono::steady_clock::now();
    if (failed)
        return -1.0;
    return std::chrono::duration<double>(t1 - t0).count();
}

// qpalm::eval_al_gradients (qpalm.cpp:106-165) of every instance: the
// reference's own code on an OCPProblem built from the ABI layout (D
// [b][N][ny][nu], C [b][N+1][ny][nx] with C[N] = C_term, bl / bu / y /
// sigma [b][N+1][ny], u [b][N][nu], x [b][N+1][nx], ubar, xbar alike),
// QPALMSettings::gamma = 1 / gamma_inv. Outputs ru [b][N][nu],
// qx [b][N+1][nx] (qx[0] = 0, unused), yhat [b][N+1][ny], cres [b][N][nx].
int ref_al_gradients(const oc_dims *d, const oc_ocp *p, int64_t ny, const double *D, const double *C,
                     const double *bl, const double *bu, const double *u, const double *x,
                     const double *y, const double *sigma, const double *ubar, const double *xbar,
                     double gamma_inv, double *ru, double *qx, double *yhat, double *cres) {
    const index_t N = d->N, nx = d->nx, nu = d->nu;
    try {
        for (index_t b = 0; b < d->batch; ++b) {
            EqOCP e = make_ocp(d, p, b);
            ocp::OCPProblem pr;
            pr.N = N, pr.nx = nx, pr.nu = nu, pr.ny = ny, pr.ny_term = ny;
            pr.A = e.A, pr.B = e.B, pr.f = e.f, pr.R = e.R, pr.S = e.S, pr.Q = e.Q, pr.q = e.q, pr.r = e.r;
            pr.x_init = e.x_init;
            qpalm::ALMState st;
            for (index_t j = 0; j < N; ++j) {
                pr.D.push_back(mat_from(D + (b * N + j) * ny * nu, ny, nu));
                pr.C.push_back(mat_from(C + (b * (N + 1) + j) * ny * nx, ny, nx));
                st.u.push_back(vec_from(u + (b * N + j) * nu, nu));
                st.ubar.push_back(vec_from(ubar + (b * N + j) * nu, nu));
            }
            pr.C_term = mat_from(C + (b * (N + 1) + N) * ny * nx, ny, nx);
            for (index_t j = 0; j <= N; ++j) {
                const index_t o = (b * (N + 1) + j) * ny;
                pr.bl.push_back(vec_from(bl + o, ny));
                pr.bu.push_back(vec_from(bu + o, ny));
                st.y.push_back(vec_from(y + o, ny));
                st.sigma.push_back(vec_from(sigma + o, ny));
                st.x.push_back(vec_from(x + (b * (N + 1) + j) * nx, nx));
                st.xbar.push_back(vec_from(xbar + (b * (N + 1) + j) * nx, nx));
            }
            qpalm::QPALMSettings s;
            s.gamma = 1.0 / gamma_inv;
            const qpalm::AlGradients g = qpalm::eval_al_gradients(pr, st, s);
            for (index_t j = 0; j <= N; ++j) {
                const auto ju = static_cast<std::size_t>(j);
                std::copy_n(g.yhat[ju].data(), ny, yhat + (b * (N + 1) + j) * ny);
                if (j >= 1)
                    std::copy_n(g.qx[ju].data(), nx, qx + (b * (N + 1) + j) * nx);
                else
                    std::fill_n(qx + b * (N + 1) * nx, nx, 0.0);
                if (j < N) {
                    std::copy_n(g.ru[ju].data(), nu, ru + (b * N + j) * nu);
                    std::copy_n(g.cres[ju].data(), nx, cres + (b * N + j) * nx);
                }
            }
        }
    } catch (...) {
        return 1;
    }
    return 0;
}

// Single-instance latency: kkt::factor +
// kkt::solve of instance 0 with FactorOptions{P, vlen, workers}, repeated
// `reps` times after one warm-up; returns the best time per solve (s).
double ref_bench_latency(const oc_dims *d, const oc_ocp *p, int64_t vlen, int64_t workers,
                         int64_t reps) {
    EqOCP prob = make_ocp(d, p, 0);
    EqRhs rhs  = EqRhs::of_problem(prob);
    FactorOptions o = opts_of(d, vlen);
    o.workers       = std::max<int64_t>(1, workers);
    double best     = 1e300;
    try {
        for (int64_t r = 0; r <= reps; ++r) {
            auto t0      = std::chrono::steady_clock::now();
            Factor f     = kkt::factor(prob, o);
            EqSolution s = kkt::solve(f, prob, rhs);
            auto t1      = std::chrono::steady_clock::now();
            if (s.u.empty())
                return -1.0;
            if (r > 0)
                best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
        }
    } catch (...) {
        return -1.0;
    }
    return best;
}

} // extern "C"


// ---- exact line search: the reference's qpalm::line_search_exact --------
#include <cyqlone/line_search.hpp>

#include <chrono>
#include <stdexcept>
#include <thread>

extern "C" int ref_line_search(int64_t m, const double *alpha, const double *delta, double eta,
                               double beta, double *tau, int64_t *iters) {
    cyqlone::qpalm::LineSearchData ls;
    ls.eta = eta;
    ls.beta = beta;
    for (int64_t i = 0; i < m; ++i)
        ls.add_term(alpha[i], delta[i]);
    ls.finalize();
    try {
        auto r = cyqlone::qpalm::line_search_exact(ls);
        *tau = r.tau;
        if (iters)
            *iters = r.iterations;
        return 0;
    } catch (const std::invalid_argument &) {
        *tau = 0;
        return 1;
    }
}

extern "C" double ref_bench_line_search(int64_t batch, int64_t m, const double *alpha,
                                        const double *delta, const double *eta,
                                        const double *beta, double *tau, int threads) {
    if (threads < 1)
        threads = 1;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int k = 0; k < threads; ++k)
        th.emplace_back([=] {
            for (int64_t b = batch * k / threads; b < batch * (k + 1) / threads; ++b)
                ref_line_search(m, alpha + b * m, delta + b * m, eta[b], beta[b], tau + b, nullptr);
        });
    for (auto &t : th)
        t.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
