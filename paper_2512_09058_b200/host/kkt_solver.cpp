// cyqlone::kkt host entry points (include/cyqlone_b200/kkt_solver.hpp) over
// the C ABI of the sm_100a library (include/cyqlone_b200.h). Each call
// flattens the reference's per-stage DenseMatrix vectors into the ABI's
// instance-major row-major arrays, runs the GPU pipeline with host buffers
// (copies inside the call, as the reference API is host-memory), and maps
// the ABI status to the reference's exceptions:
//   CYQ_INVALID_ARG -> std::invalid_argument  (kkt_factor.cpp:253-256)
//   CYQ_PIVOT_FAIL  -> batla::factorize_error (kernels.cpp:42-45,
//                      block_tridiag.cpp:140-147)
//   CUDA / device   -> std::runtime_error (no CPU fallback)
#include "../../include/cyqlone_b200/kkt_solver.hpp"
#include "../../include/cyqlone_b200.h"

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>

namespace cyqlone::kkt {

namespace {

std::size_t z(index_t i) { return static_cast<std::size_t>(i); }

// one context per process on device $CYQ_DEVICE (default 0)
cyq_ctx *ctx() {
    static std::mutex mu;
    static cyq_ctx *c = nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!c) {
        const char *e = std::getenv("CYQ_DEVICE");
        cyq_ctx *h = nullptr;
        const int rc = cyq_ctx_create(e ? std::atoi(e) : 0, &h);
        if (rc != CYQ_OK)
            throw std::runtime_error(std::string("cyqlone_b200: no CUDA device: ") +
                                     cyq_ctx_last_error(nullptr));
        c = h;
    }
    return c;
}

bool pow2(index_t v) { return v > 0 && (v & (v - 1)) == 0; }

void check_opts(const FactorOptions &o) {
    if (!pow2(o.P))
        throw std::invalid_argument("P must be a power of two");
    if (!pow2(o.vlen))
        throw std::invalid_argument("vlen must be a power of two");
    if (o.tail != Tail::cr1 && o.tail != Tail::pcr && o.tail != Tail::pcg)
        throw std::invalid_argument("unknown tail");
}

// The context is shared by the host threads of the process: one call at a
// time (its options and grow-only buffers are per context).
std::mutex &call_mutex() {
    static std::mutex m;
    return m;
}

// FactorOptions::tail / vlen as context options (kkt_factor.cpp:214-247):
// Tail::pcr solves the last min(P, vlen) Schur blocks by parallel cyclic
// reduction on the GPU; Tail::pcg is served by exact cyclic reduction
// (within its 1e-8 contract, test_kkt.cpp:157-161).
void apply_opts(const FactorOptions &o) {
    const int64_t tail = o.tail == Tail::pcr ? CYQ_TAIL_PCR : o.tail == Tail::pcg ? CYQ_TAIL_PCG : CYQ_TAIL_CR1;
    if (cyq_ctx_set_option(ctx(), CYQ_OPT_TAIL, tail) != CYQ_OK ||
        cyq_ctx_set_option(ctx(), CYQ_OPT_VLEN, o.vlen) != CYQ_OK)
        throw std::invalid_argument(cyq_ctx_last_error(ctx()));
}

void check_mat(const Mat &m, index_t r, index_t c, const char *what) {
    if (m.rows != r || m.cols != c || m.a.size() != z(r * c))
        throw std::invalid_argument(std::string("EqOCP: block ") + what + " has the wrong shape");
}
void check_vec(const Vec &v, index_t n, const char *what) {
    if (v.size() != z(n))
        throw std::invalid_argument(std::string("EqOCP: vector ") + what + " has the wrong length");
}

// instance-major flat copy of a batch of same-shape problems
struct FlatOCP {
    index_t N = 0, nx = 0, nu = 0, batch = 0;
    std::vector<double> A, B, R, S, Q, f, r, q, x0;

    explicit FlatOCP(const std::vector<const EqOCP *> &ps) {
        if (ps.empty())
            throw std::invalid_argument("empty problem batch");
        N = ps[0]->N, nx = ps[0]->nx, nu = ps[0]->nu, batch = static_cast<index_t>(ps.size());
        if (N < 1 || nx < 1 || nu < 1)
            throw std::invalid_argument("EqOCP: N, nx, nu must be >= 1");
        for (const EqOCP *p : ps) {
            if (p->N != N || p->nx != nx || p->nu != nu)
                throw std::invalid_argument("problem batch: instances differ in shape");
            if (p->A.size() != z(N) || p->B.size() != z(N) || p->R.size() != z(N) ||
                p->S.size() != z(N) || p->f.size() != z(N) || p->r.size() != z(N) ||
                p->Q.size() != z(N + 1) || p->q.size() != z(N + 1))
                throw std::invalid_argument("EqOCP: stage vectors have the wrong length");
            for (index_t j = 0; j < N; ++j) {
                check_mat(p->A[z(j)], nx, nx, "A");
                check_mat(p->B[z(j)], nx, nu, "B");
                check_mat(p->R[z(j)], nu, nu, "R");
                check_mat(p->S[z(j)], nu, nx, "S");
                check_vec(p->f[z(j)], nx, "f");
                check_vec(p->r[z(j)], nu, "r");
                append(A, p->A[z(j)].a);
                append(B, p->B[z(j)].a);
                append(R, p->R[z(j)].a);
                append(S, p->S[z(j)].a);
                append(f, p->f[z(j)]);
                append(r, p->r[z(j)]);
            }
            for (index_t j = 0; j <= N; ++j) {
                check_mat(p->Q[z(j)], nx, nx, "Q");
                check_vec(p->q[z(j)], nx, "q");
                append(Q, p->Q[z(j)].a);
                append(q, p->q[z(j)]);
            }
            check_vec(p->x_init, nx, "x_init");
            append(x0, p->x_init);
        }
    }
    static void append(std::vector<double> &dst, const std::vector<double> &src) {
        dst.insert(dst.end(), src.begin(), src.end());
    }
    cyq_ocp_batch view() const {
        return {A.data(), B.data(), R.data(), S.data(), Q.data(), f.data(), r.data(), q.data(), x0.data()};
    }
    cyq_dims dims(index_t P) const { return {N, nx, nu, P, batch}; }
};

struct FlatSol {
    std::vector<double> u, x, lam;
    FlatSol(index_t N, index_t nx, index_t nu, index_t batch)
        : u(z(batch * N * nu)), x(z(batch * (N + 1) * nx)), lam(z(batch * N * nx)) {}
    cyq_sol_batch view() { return {u.data(), x.data(), lam.data()}; }
    EqSolution instance(index_t b, index_t N, index_t nx, index_t nu) const {
        EqSolution s;
        for (index_t j = 0; j < N; ++j) {
            const double *pu = u.data() + z((b * N + j) * nu), *pl = lam.data() + z((b * N + j) * nx);
            s.u.emplace_back(pu, pu + nu);
            s.lam.emplace_back(pl, pl + nx);
        }
        for (index_t j = 0; j <= N; ++j) {
            const double *px = x.data() + z((b * (N + 1) + j) * nx);
            s.x.emplace_back(px, px + nx);
        }
        return s;
    }
};

[[noreturn]] void throw_status(int rc, const std::vector<cyq_status> &st) {
    const std::string msg = cyq_ctx_last_error(ctx());
    if (rc == CYQ_INVALID_ARG)
        throw std::invalid_argument(msg);
    if (rc == CYQ_PIVOT_FAIL) {
        for (const cyq_status &s : st)
            if (s.code == CYQ_PIVOT_FAIL) {
                // single instance: the reference's (column, pivot); batches: instance
                const index_t bi = st.size() == 1 ? s.column_or_level : s.instance;
                throw batla::factorize_error("factorization failed: " + msg, bi, s.pivot);
            }
        throw batla::factorize_error("factorization failed: " + msg, 0, 0);
    }
    throw std::runtime_error("cyqlone_b200: " + msg);
}

std::vector<InstanceStatus> to_status(const std::vector<cyq_status> &st) {
    std::vector<InstanceStatus> out(st.size());
    for (std::size_t i = 0; i < st.size(); ++i)
        out[i] = {st[i].code, st[i].kind, st[i].column_or_level, st[i].stage, st[i].pivot};
    return out;
}

// per-column multiply-add counts of the phases (the reference's counter
// with vlen = 1; paper_2512_09058_b200/flops.py, pinned to the reference)
FlopTrace trace_of(index_t N, index_t nx, index_t nu, index_t P) {
    auto tri = [](index_t n) { return n * (n + 1) / 2; };
    auto potrf = [](index_t n) { return n * (n + 1) * (n + 2) / 6; };
    auto trsyrk = [](index_t n) {
        index_t s = 0;
        for (index_t i = 0; i < n; ++i)
            s += (i + 1) * (n - i);
        return s;
    };
    const index_t nux = nx + nu, n = (N + P - 1) / P;
    FlopTrace t;
    std::uint64_t ric = 0;
    for (index_t s = 0; s < n; ++s) {
        if (s > 0)
            ric += nx * tri(nux);
        ric += potrf(nux) + nx * tri(nu) + nx * nx * nu;
        ric += (s + 1 < n) ? nx * nux * nx + nux * tri(nx) : nx * tri(nx);
    }
    t.riccati = ric;
    t.schur = n * nu * tri(nx) + nx * tri(nx) + potrf(nx) + trsyrk(nx) + nx * tri(nx);
    std::uint64_t cr = 0;
    for (index_t size = P; size > 1; size /= 2) {
        const index_t half = size / 2;
        for (index_t mm = 0; mm < half; ++mm) {
            cr += potrf(nx) + nx * tri(nx);
            if (2 * mm + 1 < size - 1)
                cr += nx * tri(nx);
            cr += nx * tri(nx);
            if (mm > 0)
                cr += nx * tri(nx);
            if (mm < half - 1)
                cr += nx * nx * nx;
        }
    }
    t.cr = cr + potrf(nx);
    return t;
}

} // namespace

struct Factor::Impl {
    cyq_factor *f = nullptr;
    ~Impl() {
        if (f)
            cyq_factor_destroy(f);
    }
};

Factor::Factor() : impl(std::make_unique<Impl>()) {}
Factor::~Factor() = default;
Factor::Factor(Factor &&) noexcept = default;
Factor &Factor::operator=(Factor &&) noexcept = default;

index_t nu2(index_t i, index_t P) {
    if (!pow2(P) || i < 0 || i >= P)
        throw std::invalid_argument("nu2: need 0 <= i < P, P a power of two");
    if (i == 0)
        i = P;
    index_t v = 0;
    for (; (i & 1) == 0; i >>= 1)
        ++v;
    return v;
}

EqOCP pad_problem(const EqOCP &p, index_t P) {
    if (!pow2(P))
        throw std::invalid_argument("P must be a power of two");
    const index_t Np = P * ((p.N + P - 1) / P);
    EqOCP o = p;
    o.N = Np;
    o.A.resize(z(Np), Mat(p.nx, p.nx));
    o.B.resize(z(Np), Mat(p.nx, p.nu));
    o.f.resize(z(Np), Vec(z(p.nx), 0.0));
    o.R.resize(z(Np), Mat::identity(p.nu));
    o.S.resize(z(Np), Mat(p.nu, p.nx));
    o.Q.resize(z(Np + 1), Mat::identity(p.nx));
    o.q.resize(z(Np + 1), Vec(z(p.nx), 0.0));
    o.r.resize(z(Np), Vec(z(p.nu), 0.0));
    return o;
}

Factor factor_batch(const std::vector<EqOCP> &ps, const FactorOptions &opts) {
    check_opts(opts);
    std::vector<const EqOCP *> v;
    for (const EqOCP &p : ps)
        v.push_back(&p);
    FlatOCP fl(v);
    Factor f;
    f.opts = opts;
    f.nx = fl.nx;
    f.nu = fl.nu;
    f.N_orig = fl.N;
    f.batch = fl.batch;
    const index_t Np = opts.P * ((fl.N + opts.P - 1) / opts.P);
    f.part = Partition{opts.P, Np / opts.P, Np};
    const cyq_dims d = fl.dims(opts.P);
    const cyq_ocp_batch pb = fl.view();
    std::vector<cyq_status> st(z(fl.batch));
    std::lock_guard<std::mutex> lk(call_mutex());
    apply_opts(opts);
    const int rc = cyq_factor_batch(ctx(), &d, &pb, CYQ_MEM_HOST, &f.impl->f, st.data());
    if (rc != CYQ_OK)
        throw_status(rc, st);
    return f;
}

Factor factor(const EqOCP &p, const FactorOptions &opts, FlopTrace *trace) {
    Factor f = factor_batch(std::vector<EqOCP>{p}, opts);
    if (trace)
        *trace = trace_of(p.N, p.nx, p.nu, opts.P);
    return f;
}

std::vector<EqSolution> solve_batch(const Factor &f, const std::vector<EqOCP> &ps,
                                    const std::vector<EqRhs> &rhs) {
    if (!f.impl || !f.impl->f)
        throw std::invalid_argument("solve: empty factor");
    if (static_cast<index_t>(ps.size()) != f.batch || rhs.size() != ps.size())
        throw std::invalid_argument("solve: batch size differs from the factor's");
    const index_t N = f.N_orig, nx = f.nx, nu = f.nu, B = f.batch;
    std::vector<double> ru, qx, fd;
    for (const EqRhs &r : rhs) {
        if (r.ru.size() != z(N) || r.qx.size() != z(N + 1) || r.fd.size() != z(N))
            throw std::invalid_argument("EqRhs: wrong number of stages");
        for (index_t j = 0; j < N; ++j) {
            check_vec(r.ru[z(j)], nu, "ru");
            check_vec(r.fd[z(j)], nx, "fd");
            FlatOCP::append(ru, r.ru[z(j)]);
            FlatOCP::append(fd, r.fd[z(j)]);
        }
        for (index_t j = 0; j <= N; ++j) {
            check_vec(r.qx[z(j)], nx, "qx");
            FlatOCP::append(qx, r.qx[z(j)]);
        }
    }
    std::vector<const EqOCP *> v;
    for (const EqOCP &p : ps)
        v.push_back(&p);
    FlatOCP fl(v);
    const cyq_ocp_batch pb = fl.view();
    const cyq_rhs_batch rb{ru.data(), qx.data(), fd.data()};
    FlatSol sol(N, nx, nu, B);
    const cyq_sol_batch sb = sol.view();
    std::lock_guard<std::mutex> lk(call_mutex());
    const int rc = cyq_solve_batch(ctx(), f.impl->f, &pb, &rb, &sb, CYQ_MEM_HOST);
    if (rc != CYQ_OK)
        throw_status(rc, {});
    std::vector<EqSolution> out;
    for (index_t b = 0; b < B; ++b)
        out.push_back(sol.instance(b, N, nx, nu));
    return out;
}

EqSolution solve(const Factor &f, const EqOCP &p, const EqRhs &rhs) {
    return solve_batch(f, std::vector<EqOCP>{p}, std::vector<EqRhs>{rhs})[0];
}

std::vector<EqSolution> solve_problem_batch(const std::vector<EqOCP> &ps, const FactorOptions &opts,
                                            std::vector<InstanceStatus> *status) {
    check_opts(opts);
    std::vector<const EqOCP *> v;
    for (const EqOCP &p : ps)
        v.push_back(&p);
    FlatOCP fl(v);
    const cyq_dims d = fl.dims(opts.P);
    const cyq_ocp_batch pb = fl.view();
    FlatSol sol(fl.N, fl.nx, fl.nu, fl.batch);
    const cyq_sol_batch sb = sol.view();
    std::vector<cyq_status> st(z(fl.batch));
    std::lock_guard<std::mutex> lk(call_mutex());
    apply_opts(opts);
    const int rc = cyq_solve_problem_batch(ctx(), &d, &pb, &sb, st.data(), CYQ_MEM_HOST);
    if (status)
        *status = to_status(st);
    if (rc != CYQ_OK && !(rc == CYQ_PIVOT_FAIL && status))
        throw_status(rc, st);
    std::vector<EqSolution> out;
    for (index_t b = 0; b < fl.batch; ++b)
        out.push_back(sol.instance(b, fl.N, fl.nx, fl.nu));
    return out;
}

EqSolution solve_problem(const EqOCP &p, const FactorOptions &opts, Factor *factor_out) {
    if (factor_out) { // keep the factor: factor + solve(of_problem)
        *factor_out = factor(p, opts);
        return solve(*factor_out, p, EqRhs::of_problem(p));
    }
    return solve_problem_batch(std::vector<EqOCP>{p}, opts)[0];
}

Factor::Blocks Factor::materialize(index_t inst) const {
    if (!impl || !impl->f)
        throw std::invalid_argument("materialize: empty factor");
    const index_t P = part.P, n = part.n_per, nux = nx + nu;
    std::vector<double> LH(z(n * P * nux * nux)), LB(z(n * P * nx * nu)), Acl(z(n * P * nx * nx)),
        LA(z(P * nx * nx));
    const int rc = cyq_factor_materialize(impl->f, inst, LH.data(), LB.data(), Acl.data(), LA.data());
    if (rc != CYQ_OK)
        throw_status(rc, {});
    auto mat = [](const double *src, index_t r, index_t c) {
        Mat m(r, c);
        m.a.assign(src, src + r * c);
        return m;
    };
    Blocks bl;
    bl.LH.resize(z(n));
    bl.LB.resize(z(n));
    bl.Acl.resize(z(n));
    for (index_t s = 0; s < n; ++s)
        for (index_t c = 0; c < P; ++c) {
            bl.LH[z(s)].push_back(mat(LH.data() + z((s * P + c) * nux * nux), nux, nux));
            bl.LB[z(s)].push_back(mat(LB.data() + z((s * P + c) * nx * nu), nx, nu));
            bl.Acl[z(s)].push_back(mat(Acl.data() + z((s * P + c) * nx * nx), nx, nx));
        }
    for (index_t c = 0; c < P; ++c)
        bl.LA.push_back(mat(LA.data() + z(c * nx * nx), nx, nx));
    return bl;
}

index_t SigmaDelta::total_rank() const {
    index_t r = 0;
    for (const Vec &v : stage)
        for (real_t x : v)
            r += x != 0;
    for (real_t x : terminal)
        r += x != 0;
    return r;
}

Vec active_set_delta(const std::vector<bool> &prev, const std::vector<bool> &now, const Vec &sigma) {
    if (prev.size() != now.size() || now.size() != sigma.size())
        throw std::invalid_argument("active_set_delta: size mismatch");
    Vec d(sigma.size(), 0);
    for (std::size_t i = 0; i < sigma.size(); ++i) {
        if (now[i] && !prev[i])
            d[i] = sigma[i];
        else if (!now[i] && prev[i])
            d[i] = -sigma[i];
    }
    return d;
}

UpdateReport update(Factor &f, const EqOCP &p_new, const std::vector<Mat> &C, const std::vector<Mat> &D,
                    const Mat &C_term, const SigmaDelta &ds) {
    if (!f.impl)
        throw std::invalid_argument("update: empty factor");
    if (f.batch != 1)
        throw std::invalid_argument("update: single-instance factors only");
    if (p_new.N != f.N_orig || p_new.nx != f.nx || p_new.nu != f.nu)
        throw std::invalid_argument("update: p_new shape differs from the factor's");
    if (static_cast<index_t>(ds.stage.size()) != p_new.N || static_cast<index_t>(D.size()) < p_new.N ||
        static_cast<index_t>(C.size()) < p_new.N)
        throw std::invalid_argument("update: SigmaDelta / C / D sizes differ from N");
    for (index_t j = 0; j < p_new.N; ++j) {
        const index_t ny = static_cast<index_t>(ds.stage[z(j)].size());
        if (D[z(j)].rows != ny || D[z(j)].cols != f.nu || C[z(j)].rows != ny || C[z(j)].cols != f.nx)
            throw std::invalid_argument("update: D_j / C_j shapes differ from (ny x nu, ny x nx)");
    }
    if (!ds.terminal.empty() && (C_term.rows != static_cast<index_t>(ds.terminal.size()) || C_term.cols != f.nx))
        throw std::invalid_argument("update: C_term shape differs from (ny_term x nx)");
    // flat instance-major arrays of the ABI (batch of one)
    const index_t N = p_new.N, nx = f.nx, nu = f.nu;
    const index_t ny = N > 0 ? static_cast<index_t>(ds.stage[0].size()) : 0;
    const index_t nyt = static_cast<index_t>(ds.terminal.size());
    std::vector<double> Cf, Df, dsf, Ctf, dtf(ds.terminal.begin(), ds.terminal.end());
    for (index_t j = 0; j < N; ++j) {
        if (static_cast<index_t>(ds.stage[z(j)].size()) != ny)
            throw std::invalid_argument("update: dSigma stages differ in length");
        FlatOCP::append(Cf, C[z(j)].a);
        FlatOCP::append(Df, D[z(j)].a);
        FlatOCP::append(dsf, ds.stage[z(j)]);
    }
    if (nyt > 0)
        Ctf = C_term.a;
    FlatOCP fl(std::vector<const EqOCP *>{&p_new});
    const cyq_ocp_batch pb = fl.view();
    cyq_update_report r{};
    std::lock_guard<std::mutex> lk(call_mutex());
    const int rc = cyq_factor_update_batch(ctx(), f.impl->f, &pb, ny, Cf.data(), Df.data(), dsf.data(), nyt,
                                           nyt ? Ctf.data() : nullptr, nyt ? dtf.data() : nullptr, f.opts.rho,
                                           CYQ_MEM_HOST, &r);
    if (rc != CYQ_OK)
        throw_status(rc, {});
    UpdateReport rep;
    rep.columns_updated = r.columns_updated;
    rep.columns_refactored = r.columns_refactored;
    rep.schur_refactored = r.schur_refactored != 0;
    rep.schur_levels_updated = r.schur_levels_updated;
    (void)nu;
    (void)nx;
    return rep;
}

FlopModel flops_critical_path(index_t nx, index_t nu, index_t N, index_t P) {
    if (!pow2(P) || N % P != 0)
        throw std::invalid_argument("flops_critical_path: P must be a power of two dividing N");
    const double x = static_cast<double>(nx), u = static_cast<double>(nu), m = x + u;
    const double nP = static_cast<double>(N) / static_cast<double>(P);
    const double lg = std::log2(static_cast<double>(P));
    FlopModel fm; // Eq. 14
    fm.riccati = nP * (m * m * m / 6 + x * u * u / 2 + x * x * u) +
                 (nP - 1) * (1.5 * m * x * x + 0.5 * m * m * x) + 0.5 * x * x * x;
    fm.schur = 4.0 / 3.0 * x * x * x + nP * 0.5 * u * x * x;
    fm.cr = x * x * x / 6 + lg * 5.0 / 3.0 * x * x * x;
    fm.total = fm.riccati + fm.schur + fm.cr;
    fm.serial = x * x * x / 6 + static_cast<double>(N) * (0.5 * m * x * x + 0.5 * m * m * x + m * m * m / 6);
    fm.speedup = fm.serial / fm.total;
    return fm;
}

std::string backend_info() { return cyq_version(); }

} // namespace cyqlone::kkt
