// C++ test driver of the host interface (include/cyqlone_b200/kkt_solver.hpp),
// written the way the reference's own tests use cyqlone::kkt
// (proj/tests/test_kkt.cpp): same calls, same properties.
//
//   test_kkt_host selftest          property tests on the GPU (exit 0 = pass)
//   test_kkt_host golden IN OUT     solve_problem on a binary input batch
//                                   (written by tests/test_host_cpp.py from
//                                   the golden fixtures), solution to OUT
//   test_kkt_host compile-only      links and exits (CPU-side build check)
#include "cyqlone_b200/kkt_solver.hpp"

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

using namespace cyqlone;
using kkt::FactorOptions;
using ocp::EqOCP;
using ocp::EqRhs;
using ocp::EqSolution;
using ocp::Mat;
using ocp::Vec;

namespace {

int g_fail = 0;
#define CHECK(cond, ...)                                                      \
    do {                                                                      \
        if (!(cond)) {                                                        \
            std::fprintf(stderr, "FAIL %s:%d: %s -- ", __FILE__, __LINE__, #cond); \
            std::fprintf(stderr, __VA_ARGS__);                                \
            std::fprintf(stderr, "\n");                                       \
            ++g_fail;                                                         \
        }                                                                     \
    } while (0)

// Random well-posed problem: SPD stage Hessians, contractive dynamics.
EqOCP random_ocp(ocp::index_t N, ocp::index_t nx, ocp::index_t nu, unsigned seed, bool with_s = true) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> nd(0.0, 1.0);
    EqOCP p;
    p.N = N, p.nx = nx, p.nu = nu;
    p.resize();
    auto spd = [&](ocp::index_t n) {
        Mat m(n, n), g(n, n);
        for (auto &v : g.a)
            v = nd(rng);
        for (ocp::index_t i = 0; i < n; ++i)
            for (ocp::index_t j = 0; j < n; ++j) {
                double s = 0;
                for (ocp::index_t k = 0; k < n; ++k)
                    s += g(i, k) * g(j, k);
                m(i, j) = s / n + (i == j ? 1.0 : 0.0);
            }
        return m;
    };
    for (ocp::index_t j = 0; j <= N; ++j) {
        p.Q[j] = spd(nx);
        for (auto &v : p.q[j])
            v = nd(rng);
    }
    for (ocp::index_t j = 0; j < N; ++j) {
        p.R[j] = spd(nu);
        for (auto &v : p.A[j].a)
            v = 0.9 * nd(rng) / std::sqrt(double(nx));
        for (auto &v : p.B[j].a)
            v = nd(rng) / std::sqrt(double(nu));
        for (auto &v : p.S[j].a)
            v = with_s ? 0.05 * nd(rng) : 0.0;
        for (auto &v : p.f[j])
            v = nd(rng);
        for (auto &v : p.r[j])
            v = nd(rng);
    }
    for (auto &v : p.x_init)
        v = nd(rng);
    return p;
}

double sol_max(const EqSolution &s) {
    double m = 0;
    for (const auto *vs : {&s.u, &s.x, &s.lam})
        for (const Vec &v : *vs)
            for (double e : v)
                m = std::fmax(m, std::fabs(e));
    return m;
}
double rel_err(const EqSolution &a, const EqSolution &b) {
    double d = 0;
    const std::vector<Vec> *pa[] = {&a.u, &a.x, &a.lam}, *pb[] = {&b.u, &b.x, &b.lam};
    for (int k = 0; k < 3; ++k)
        for (std::size_t j = 0; j < pa[k]->size(); ++j)
            for (std::size_t i = 0; i < (*pa[k])[j].size(); ++i)
                d = std::fmax(d, std::fabs((*pa[k])[j][i] - (*pb[k])[j][i]));
    return d / std::fmax(1.0, sol_max(b));
}
bool bit_equal(const EqSolution &a, const EqSolution &b) {
    return a.u == b.u && a.x == b.x && a.lam == b.lam;
}

void test_residuals() {
    struct Case { ocp::index_t N, nx, nu, P; };
    for (Case c : {Case{64, 10, 5, 4}, Case{40, 20, 10, 16}, Case{37, 4, 3, 8}, Case{16, 3, 2, 1},
                   Case{256, 12, 4, 64}, Case{48, 16, 8, 16}}) {
        EqOCP p = random_ocp(c.N, c.nx, c.nu, 100 + unsigned(c.N));
        EqSolution s = kkt::solve_problem(p, FactorOptions{c.P});
        const double res = ocp::kkt_residual_eq(p, EqRhs::of_problem(p), s).max();
        CHECK(res <= 1e-10, "N=%lld nx=%lld nu=%lld P=%lld residual %.3e", (long long)c.N,
              (long long)c.nx, (long long)c.nu, (long long)c.P, res);
        CHECK(s.x[0] == p.x_init, "x[0] must equal x_init");
    }
}

void test_zero_rhs_exact() { // test_kkt.cpp:114-121
    EqOCP p = random_ocp(32, 6, 3, 7);
    kkt::Factor f = kkt::factor(p, FactorOptions{4});
    EqSolution s = kkt::solve(f, p, EqRhs::zero(p));
    CHECK(s.x[0] == p.x_init, "x[0] is the fixed initial state");
    s.x[0].assign(s.x[0].size(), 0.0);
    CHECK(sol_max(s) == 0.0, "zero rhs must give an exactly zero u, x[1..], lam (max %.3e)", sol_max(s));
}

void test_cross_P_and_repeat() { // test_kkt.cpp:125-139
    EqOCP p = random_ocp(64, 10, 5, 8);
    EqSolution ref = kkt::solve_problem(p, FactorOptions{1});
    for (ocp::index_t P : {2, 4, 8, 16, 32, 64}) {
        EqSolution s = kkt::solve_problem(p, FactorOptions{P});
        CHECK(rel_err(s, ref) < 1e-8, "P=%lld vs P=1 rel err %.3e", (long long)P, rel_err(s, ref));
    }
    FactorOptions o{4};
    EqSolution a = kkt::solve_problem(p, o), b = kkt::solve_problem(p, o);
    CHECK(bit_equal(a, b), "repeated solves must be bit-identical");
    o.vlen = 8;
    o.workers = 4; // CPU knobs: no effect
    EqSolution c = kkt::solve_problem(p, o);
    CHECK(bit_equal(a, c), "vlen / workers must not change the result");
}

void test_factor_then_solve() {
    EqOCP p = random_ocp(32, 20, 10, 9);
    FactorOptions o{16};
    kkt::FlopTrace tr;
    kkt::Factor f = kkt::factor(p, o, &tr);
    CHECK(tr.riccati > 0 && tr.cr > 0, "flop trace filled");
    EqSolution s1 = kkt::solve(f, p, EqRhs::of_problem(p));
    EqSolution s2 = kkt::solve_problem(p, o);
    CHECK(rel_err(s1, s2) <= 1e-13, "factor+solve vs solve_problem %.3e", rel_err(s1, s2));
    kkt::Factor kept;
    EqSolution s3 = kkt::solve_problem(p, o, &kept);
    CHECK(rel_err(s3, s2) <= 1e-13, "solve_problem with factor_out %.3e", rel_err(s3, s2));
    // a second right-hand side on the same factor
    EqRhs r2 = EqRhs::of_problem(p);
    for (auto &v : r2.ru)
        for (auto &e : v)
            e *= 2.0;
    EqSolution s4 = kkt::solve(kept, p, r2);
    CHECK(ocp::kkt_residual_eq(p, r2, s4).max() <= 1e-10, "second rhs residual");
}

void test_factor_blocks() { // factor reconstruction (test_kkt.cpp:66-103)
    EqOCP p = random_ocp(32, 10, 5, 10);
    FactorOptions o{4};
    kkt::Factor f = kkt::factor(p, o);
    kkt::Factor::Blocks bl = f.materialize(0);
    const ocp::index_t nu = p.nu, nx = p.nx, nux = nu + nx;
    for (ocp::index_t c = 0; c < o.P; ++c) {
        const ocp::index_t j = f.part.stage_of(c, 0), xi = f.part.x_index_of(c, 0);
        const Mat &L = bl.LH[0][c];
        double err = 0;
        for (ocp::index_t r = 0; r < nux; ++r)
            for (ocp::index_t k = 0; k <= r; ++k) {
                double v = 0;
                for (ocp::index_t m = 0; m <= k; ++m)
                    v += L(r, m) * L(k, m);
                double h; // H_0 = [[R_j, .], [S_j', Q_xi]] (no S at stage 0)
                if (r < nu)
                    h = p.R[j](r, k);
                else if (k < nu)
                    h = j == 0 ? 0.0 : p.S[j](k, r - nu);
                else
                    h = p.Q[xi](r - nu, k - nu);
                err = std::fmax(err, std::fabs(v - h));
            }
        CHECK(err <= 1e-12, "LH_0 LH_0' != H_0 for column %lld (%.3e)", (long long)c, err);
        for (ocp::index_t r = 0; r < nux; ++r)
            CHECK(L(r, r) > 0, "LH diagonal must be positive");
    }
}

void test_errors() {
    EqOCP p = random_ocp(16, 4, 2, 11);
    bool threw = false;
    try {
        kkt::solve_problem(p, FactorOptions{3});
    } catch (const std::invalid_argument &) {
        threw = true;
    }
    CHECK(threw, "P = 3 must throw std::invalid_argument");
    for (kkt::Tail tl : {kkt::Tail::pcr, kkt::Tail::pcg}) { // tail strategies agree (test_kkt.cpp:152-159)
        FactorOptions o{8};
        o.tail = tl;
        const double d = rel_err(kkt::solve_problem(p, o), kkt::solve_problem(p, FactorOptions{8}));
        CHECK(d < 1e-10, "tail %d vs cr1: %.3e", (int)tl, d);
    }
    EqOCP bad = p;
    bad.R[5] = Mat::identity(p.nu);
    for (auto &v : bad.R[5].a)
        v *= -10.0;
    threw = false;
    try {
        kkt::solve_problem(bad, FactorOptions{4});
    } catch (const batla::factorize_error &e) {
        threw = true;
        CHECK(e.pivot >= 0, "pivot index");
    }
    CHECK(threw, "an indefinite Hessian must throw batla::factorize_error");
    // batch: the failure stays with its instance
    std::vector<EqOCP> batch = {p, bad, random_ocp(16, 4, 2, 12)};
    std::vector<kkt::InstanceStatus> st;
    std::vector<EqSolution> sols = kkt::solve_problem_batch(batch, FactorOptions{4}, &st);
    CHECK(st[0].code == 0 && st[1].code == 2 && st[2].code == 0, "per-instance status");
    CHECK(rel_err(sols[0], kkt::solve_problem(p, FactorOptions{4})) <= 1e-13, "instance 0 unaffected");
    threw = false;
    try {
        kkt::solve_problem_batch(batch, FactorOptions{4});
    } catch (const batla::factorize_error &e) {
        threw = true;
        CHECK(e.batch_index == 1, "batch_index of the failing instance (%lld)", (long long)e.batch_index);
    }
    CHECK(threw, "batch without status must throw");
}

void test_batch_matches_single() {
    std::vector<EqOCP> ps;
    for (unsigned i = 0; i < 5; ++i)
        ps.push_back(random_ocp(24, 8, 4, 200 + i));
    std::vector<EqSolution> sb = kkt::solve_problem_batch(ps, FactorOptions{8});
    for (std::size_t i = 0; i < ps.size(); ++i)
        CHECK(rel_err(sb[i], kkt::solve_problem(ps[i], FactorOptions{8})) <= 1e-13, "batch vs single");
}

void test_update() { // kkt::update (kkt_solver.hpp:152-161): low-rank path for rank 1 < rho nx
    const ocp::index_t N = 32, nx = 6, nu = 3, ny = 4;
    EqOCP p = random_ocp(N, nx, nu, 21);
    std::mt19937_64 rng(5);
    std::normal_distribution<double> gauss(0, 1);
    std::vector<Mat> C, D;
    kkt::SigmaDelta ds;
    for (ocp::index_t j = 0; j < N; ++j) {
        Mat cj(ny, nx), dj(ny, nu);
        for (auto &v : cj.a) v = gauss(rng);
        for (auto &v : dj.a) v = gauss(rng);
        C.push_back(cj);
        D.push_back(dj);
        ds.stage.push_back(Vec(ny, 0.0));
    }
    Mat ct(ny, nx);
    for (auto &v : ct.a) v = gauss(rng);
    ds.terminal = Vec(ny, 0.0);
    kkt::Factor f = kkt::factor(p, FactorOptions{4});
    kkt::UpdateReport r0 = kkt::update(f, p, C, D, ct, ds);
    CHECK(r0.columns_refactored == 0 && !r0.schur_refactored, "no change: factor kept");
    // one newly active row at stage 9: H_9 += (D_9 | C_9)' e_i 2.5 e_i' (D_9 | C_9)
    ds.stage[9][2] = 2.5;
    EqOCP pn = p;
    for (ocp::index_t a = 0; a < nu; ++a)
        for (ocp::index_t b = 0; b < nu; ++b)
            pn.R[9](a, b) += 2.5 * D[9](2, a) * D[9](2, b);
    for (ocp::index_t a = 0; a < nu; ++a)
        for (ocp::index_t b = 0; b < nx; ++b)
            pn.S[9](a, b) += 2.5 * D[9](2, a) * C[9](2, b);
    for (ocp::index_t a = 0; a < nx; ++a)
        for (ocp::index_t b = 0; b < nx; ++b)
            pn.Q[9](a, b) += 2.5 * C[9](2, a) * C[9](2, b);
    CHECK(ds.total_rank() == 1, "total_rank");
    kkt::UpdateReport r1 = kkt::update(f, pn, C, D, ct, ds);
    CHECK(r1.columns_updated == 1 && r1.columns_refactored == 0 && r1.schur_refactored,
          "one column updated (%lld / %lld)", (long long)r1.columns_updated, (long long)r1.columns_refactored);
    EqSolution s = kkt::solve(f, pn, EqRhs::of_problem(pn));
    // the reference's update-vs-refactor bar (test_kkt_update.cpp:127-241)
    CHECK(rel_err(s, kkt::solve_problem(pn, FactorOptions{4})) <= 1e-8, "update == fresh factorization %.3e",
          rel_err(s, kkt::solve_problem(pn, FactorOptions{4})));
    // rank >= rho nx in one column: the refactorization path
    for (ocp::index_t i = 0; i < ny; ++i)
        ds.stage[9][i] = 0.0;
    ds.stage[9][0] = ds.stage[9][1] = ds.stage[9][3] = 1.5;
    EqOCP pn2 = pn;
    for (ocp::index_t i : {0, 1, 3}) {
        for (ocp::index_t a = 0; a < nu; ++a)
            for (ocp::index_t b = 0; b < nu; ++b)
                pn2.R[9](a, b) += 1.5 * D[9](i, a) * D[9](i, b);
        for (ocp::index_t a = 0; a < nu; ++a)
            for (ocp::index_t b = 0; b < nx; ++b)
                pn2.S[9](a, b) += 1.5 * D[9](i, a) * C[9](i, b);
        for (ocp::index_t a = 0; a < nx; ++a)
            for (ocp::index_t b = 0; b < nx; ++b)
                pn2.Q[9](a, b) += 1.5 * C[9](i, a) * C[9](i, b);
    }
    kkt::UpdateReport r2 = kkt::update(f, pn2, C, D, ct, ds);
    CHECK(r2.columns_refactored == 1 && r2.columns_updated == 0, "rank 3 >= rho nx: refactored");
    EqSolution s2 = kkt::solve(f, pn2, EqRhs::of_problem(pn2));
    CHECK(rel_err(s2, kkt::solve_problem(pn2, FactorOptions{4})) <= 1e-8, "refactor path %.3e",
          rel_err(s2, kkt::solve_problem(pn2, FactorOptions{4})));
    Vec d = kkt::active_set_delta({true, false, true}, {false, false, true}, {1.0, 2.0, 3.0});
    CHECK(d[0] == -1.0 && d[1] == 0.0 && d[2] == 0.0, "active_set_delta");
}

void test_flop_model() { // kkt_factor.cpp:319-339 (Eq. 14)
    kkt::FlopModel m = kkt::flops_critical_path(30, 20, 96, 8);
    CHECK(m.total > 0 && std::fabs(m.total - (m.riccati + m.schur + m.cr)) < 1e-9 * m.total, "total");
    CHECK(std::fabs(m.speedup - m.serial / m.total) < 1e-12, "speedup");
    CHECK(m.speedup > 1.0, "P = 8 beats the serial recursion in the model");
    bool threw = false;
    try {
        kkt::flops_critical_path(4, 2, 30, 8);
    } catch (const std::invalid_argument &) {
        threw = true;
    }
    CHECK(threw, "P must divide N");
    CHECK(kkt::nu2(0, 16) == 4 && kkt::nu2(12, 16) == 2 && kkt::nu2(5, 16) == 0, "nu2");
}

int golden(const char *in, const char *out) {
    FILE *fi = std::fopen(in, "rb");
    if (!fi)
        return 2;
    std::int64_t hdr[5];
    if (std::fread(hdr, sizeof hdr, 1, fi) != 1)
        return 2;
    const ocp::index_t N = hdr[0], nx = hdr[1], nu = hdr[2], P = hdr[3], B = hdr[4];
    auto rd = [&](std::size_t cnt) {
        std::vector<double> v(cnt);
        if (std::fread(v.data(), sizeof(double), cnt, fi) != cnt)
            std::exit(3);
        return v;
    };
    const auto A = rd(B * N * nx * nx), Bm = rd(B * N * nx * nu), R = rd(B * N * nu * nu),
               S = rd(B * N * nu * nx), Q = rd(B * (N + 1) * nx * nx), f = rd(B * N * nx),
               r = rd(B * N * nu), q = rd(B * (N + 1) * nx), x0 = rd(B * nx);
    std::fclose(fi);
    std::vector<EqOCP> ps;
    for (ocp::index_t b = 0; b < B; ++b) { // flat arrays -> the reference's per-stage blocks
        EqOCP p;
        p.N = N, p.nx = nx, p.nu = nu;
        p.resize();
        auto fill = [](Mat &m, const double *src) { m.a.assign(src, src + m.rows * m.cols); };
        auto fillv = [](Vec &v, const double *src) { v.assign(src, src + v.size()); };
        for (ocp::index_t j = 0; j < N; ++j) {
            fill(p.A[j], A.data() + (b * N + j) * nx * nx);
            fill(p.B[j], Bm.data() + (b * N + j) * nx * nu);
            fill(p.R[j], R.data() + (b * N + j) * nu * nu);
            fill(p.S[j], S.data() + (b * N + j) * nu * nx);
            fillv(p.f[j], f.data() + (b * N + j) * nx);
            fillv(p.r[j], r.data() + (b * N + j) * nu);
        }
        for (ocp::index_t j = 0; j <= N; ++j) {
            fill(p.Q[j], Q.data() + (b * (N + 1) + j) * nx * nx);
            fillv(p.q[j], q.data() + (b * (N + 1) + j) * nx);
        }
        fillv(p.x_init, x0.data() + b * nx);
        ps.push_back(std::move(p));
    }
    FILE *fo = std::fopen(out, "wb");
    if (!fo)
        return 2;
    std::vector<EqSolution> sols;
    for (const EqOCP &p : ps) // the single-instance reference entry point
        sols.push_back(kkt::solve_problem(p, FactorOptions{P}));
    for (const auto &s : sols)
        for (const Vec &v : s.u)
            std::fwrite(v.data(), sizeof(double), v.size(), fo);
    for (const auto &s : sols)
        for (const Vec &v : s.x)
            std::fwrite(v.data(), sizeof(double), v.size(), fo);
    for (const auto &s : sols)
        for (const Vec &v : s.lam)
            std::fwrite(v.data(), sizeof(double), v.size(), fo);
    std::fclose(fo);
    return 0;
}

} // namespace

int main(int argc, char **argv) {
    const std::string mode = argc > 1 ? argv[1] : "selftest";
    if (mode == "compile-only")
        return 0;
    if (mode == "golden")
        return argc == 4 ? golden(argv[2], argv[3]) : 2;
    try {
        std::printf("%s\n", kkt::backend_info().c_str());
        test_residuals();
        test_zero_rhs_exact();
        test_cross_P_and_repeat();
        test_factor_then_solve();
        test_factor_blocks();
        test_errors();
        test_batch_matches_single();
        test_update();
        test_flop_model();
    } catch (const std::exception &e) {
        std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        return 1;
    }
    std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "OK", g_fail);
    return g_fail ? 1 : 0;
}
