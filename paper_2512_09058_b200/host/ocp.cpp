// cyqlone::ocp host types (include/cyqlone_b200/ocp.hpp): allocation, the
// objective, the right-hand-side convention and the KKT residual of the
// reference API (/root/reference/proj/src/ocp.cpp:96-230), restated as plain
// loops over the row-major DenseMatrix blocks.
#include "../../include/cyqlone_b200/ocp.hpp"

#include <algorithm>
#include <cmath>

namespace cyqlone::ocp {

namespace {

// y[i] += alpha * sum_k op(M)[i][k] x[k], op = transpose when `trans`
void gemv_acc(Vec &y, const Mat &m, const Vec &x, real_t alpha = 1.0, bool trans = false) {
    const index_t rows = trans ? m.cols : m.rows, inner = trans ? m.rows : m.cols;
    for (index_t i = 0; i < rows; ++i) {
        real_t acc = 0.0;
        for (index_t k = 0; k < inner; ++k)
            acc += (trans ? m(k, i) : m(i, k)) * x[static_cast<std::size_t>(k)];
        y[static_cast<std::size_t>(i)] += alpha * acc;
    }
}

real_t max_abs(const Vec &v) {
    real_t m = 0.0;
    for (real_t e : v)
        m = std::max(m, std::fabs(e));
    return m;
}

Vec negated(const Vec &v) {
    Vec w(v.size());
    for (std::size_t i = 0; i < v.size(); ++i)
        w[i] = -v[i];
    return w;
}

std::size_t z(index_t i) { return static_cast<std::size_t>(i); }

} // namespace

void EqOCP::resize() {
    A.assign(z(N), Mat(nx, nx));
    B.assign(z(N), Mat(nx, nu));
    f.assign(z(N), Vec(z(nx), 0.0));
    R.assign(z(N), Mat(nu, nu));
    S.assign(z(N), Mat(nu, nx));
    Q.assign(z(N + 1), Mat(nx, nx));
    q.assign(z(N + 1), Vec(z(nx), 0.0));
    r.assign(z(N), Vec(z(nu), 0.0));
    x_init.assign(z(nx), 0.0);
}

// sum_j (u'R u / 2 + u'S x + x'Q x / 2 + r'u + q'x) + terminal (ocp.cpp:109-143)
real_t EqOCP::objective(const std::vector<Vec> &u, const std::vector<Vec> &x) const {
    real_t obj = 0.0;
    for (index_t j = 0; j <= N; ++j) {
        const Vec &xj = x[z(j)];
        Vec qx(z(nx), 0.0);
        gemv_acc(qx, Q[z(j)], xj);
        for (index_t i = 0; i < nx; ++i)
            obj += (0.5 * qx[z(i)] + q[z(j)][z(i)]) * xj[z(i)];
        if (j == N)
            break;
        const Vec &uj = u[z(j)];
        Vec ru(z(nu), 0.0);
        gemv_acc(ru, R[z(j)], uj);
        gemv_acc(ru, S[z(j)], xj);
        for (index_t i = 0; i < nu; ++i)
            obj += (0.5 * ru[z(i)] + r[z(j)][z(i)]) * uj[z(i)];
        Vec su(z(nx), 0.0); // the other half of the cross term
        gemv_acc(su, S[z(j)], uj, 1.0, true);
        for (index_t i = 0; i < nx; ++i)
            obj += 0.5 * su[z(i)] * xj[z(i)];
    }
    return obj;
}

EqRhs EqRhs::zero(const EqOCP &p) {
    EqRhs rhs;
    rhs.ru.assign(z(p.N), Vec(z(p.nu), 0.0));
    rhs.qx.assign(z(p.N + 1), Vec(z(p.nx), 0.0));
    rhs.fd.assign(z(p.N), Vec(z(p.nx), 0.0));
    return rhs;
}

EqRhs EqRhs::of_problem(const EqOCP &p) {
    EqRhs rhs = zero(p);
    for (index_t j = 0; j < p.N; ++j) {
        rhs.ru[z(j)] = negated(p.r[z(j)]);
        rhs.fd[z(j)] = negated(p.f[z(j)]);
    }
    for (index_t j = 1; j <= p.N; ++j)
        rhs.qx[z(j)] = negated(p.q[z(j)]);
    if (p.N > 0) { // the eliminated x^0: ru[0] -= S_0 x_init, fd[0] -= A_0 x_init
        gemv_acc(rhs.ru[0], p.S[0], p.x_init, -1.0);
        gemv_acc(rhs.fd[0], p.A[0], p.x_init, -1.0);
    }
    return rhs;
}

real_t EqResiduals::max() const { return std::max(std::max(stat_u, stat_x), std::max(dynamics, terminal)); }

EqResiduals kkt_residual_eq(const EqOCP &p, const EqRhs &rhs, const EqSolution &s) {
    EqResiduals res;
    for (index_t j = 0; j < p.N; ++j) {
        // stationarity in u^j: R u + S x + B' lam - ru
        Vec g = negated(rhs.ru[z(j)]);
        gemv_acc(g, p.R[z(j)], s.u[z(j)]);
        if (j > 0)
            gemv_acc(g, p.S[z(j)], s.x[z(j)]);
        gemv_acc(g, p.B[z(j)], s.lam[z(j)], 1.0, true);
        res.stat_u = std::max(res.stat_u, max_abs(g));
        // dynamics: B u + A x - x_next - fd
        Vec c = negated(rhs.fd[z(j)]);
        gemv_acc(c, p.B[z(j)], s.u[z(j)]);
        if (j > 0)
            gemv_acc(c, p.A[z(j)], s.x[z(j)]);
        for (index_t i = 0; i < p.nx; ++i)
            c[z(i)] -= s.x[z(j + 1)][z(i)];
        res.dynamics = std::max(res.dynamics, max_abs(c));
    }
    for (index_t j = 1; j < p.N; ++j) { // stationarity in x^j
        Vec g = negated(rhs.qx[z(j)]);
        gemv_acc(g, p.S[z(j)], s.u[z(j)], 1.0, true);
        gemv_acc(g, p.Q[z(j)], s.x[z(j)]);
        gemv_acc(g, p.A[z(j)], s.lam[z(j)], 1.0, true);
        for (index_t i = 0; i < p.nx; ++i)
            g[z(i)] -= s.lam[z(j - 1)][z(i)];
        res.stat_x = std::max(res.stat_x, max_abs(g));
    }
    if (p.N > 0) { // terminal: Q_N x_N - lam_{N-1} - qx_N
        Vec g = negated(rhs.qx[z(p.N)]);
        gemv_acc(g, p.Q[z(p.N)], s.x[z(p.N)]);
        for (index_t i = 0; i < p.nx; ++i)
            g[z(i)] -= s.lam[z(p.N - 1)][z(i)];
        res.terminal = max_abs(g);
    }
    return res;
}

} // namespace cyqlone::ocp
