// cyqlone_b200 C++ host interface -- problem / right-hand side / solution
// types of the equality-constrained LQ optimal control problem, mirroring
// the reference's cyqlone::ocp API (/root/reference/proj/include/cyqlone/
// ocp.hpp:24-69; DenseMatrix: batch_matrix.hpp:170-189) so reference callers
// compile against this header unchanged. Host-only C++ (no CUDA types); the
// solver behind it is the sm_100a library reached through the C ABI
// (include/cyqlone_b200.h).
#pragma once

#include <cstdint>
#include <limits>
#include <vector>

namespace cyqlone {
namespace batla {
using index_t = std::int64_t;
using real_t = double;

/// Dense row-major matrix used at the API boundary (batch_matrix.hpp:170-189).
struct DenseMatrix {
    index_t rows = 0, cols = 0;
    std::vector<real_t> a;

    DenseMatrix() = default;
    DenseMatrix(index_t m, index_t n) : rows(m), cols(n), a(static_cast<std::size_t>(m * n), 0.0) {}
    real_t &operator()(index_t r, index_t c) { return a[static_cast<std::size_t>(r * cols + c)]; }
    real_t operator()(index_t r, index_t c) const { return a[static_cast<std::size_t>(r * cols + c)]; }
    static DenseMatrix identity(index_t n) {
        DenseMatrix m(n, n);
        for (index_t i = 0; i < n; ++i)
            m(i, i) = 1;
        return m;
    }
};
} // namespace batla

namespace ocp {
using batla::DenseMatrix;
using batla::index_t;
using batla::real_t;
using Mat = DenseMatrix;
using Vec = std::vector<real_t>;

constexpr real_t inf = std::numeric_limits<real_t>::infinity();

/// Stage costs (u, x)' [[R, S], [S', Q]] (u, x) / 2 + r'u + q'x, dynamics
/// x^{j+1} = A_j x^j + B_j u^j + f^j, fixed x^0 = x_init (ocp.hpp:20-38).
/// Q[j], q[j] weigh x^j (1..N); Q[0] is unused, S_0 / A_0 only enter through
/// the eliminated initial state.
struct EqOCP {
    index_t N = 0, nx = 0, nu = 0;
    std::vector<Mat> A, B; ///< size N
    std::vector<Vec> f;    ///< size N
    std::vector<Mat> R, S; ///< size N (S is nu-by-nx)
    std::vector<Mat> Q;    ///< size N+1
    std::vector<Vec> q;    ///< size N+1
    std::vector<Vec> r;    ///< size N
    Vec x_init;

    /// Allocates every block with the current N, nx, nu (zero-filled).
    void resize();
    /// Objective value of a trajectory (u, x) with x[0] = x_init.
    real_t objective(const std::vector<Vec> &u, const std::vector<Vec> &x) const;
};

/// Right-hand side convention of the optimality system (ocp.hpp:40-53):
///   R u + S x + B' lam            = ru
///   S'u + Q x + A' lam - lam_prev = qx
///   B u + A x - x_next            = fd
struct EqRhs {
    std::vector<Vec> ru; ///< size N
    std::vector<Vec> qx; ///< size N+1, qx[0] unused
    std::vector<Vec> fd; ///< size N

    static EqRhs zero(const EqOCP &p);
    /// Negated gradients of p, with ru[0] -= S_0 x_init, fd[0] -= A_0 x_init.
    static EqRhs of_problem(const EqOCP &p);
};

struct EqSolution {
    std::vector<Vec> u;   ///< size N
    std::vector<Vec> x;   ///< size N+1, x[0] = x_init
    std::vector<Vec> lam; ///< size N
};

struct EqResiduals {
    real_t stat_u = 0, stat_x = 0, dynamics = 0, terminal = 0;
    real_t max() const;
};

/// Infinity norms of the residual groups of the optimality system
/// (ocp.cpp:180-230) -- the parity metric of the reference's tests.
EqResiduals kkt_residual_eq(const EqOCP &p, const EqRhs &rhs, const EqSolution &s);

} // namespace ocp
} // namespace cyqlone
