// cyqlone_b200 C++ host interface -- the KKT factor / solve entry points of
// the reference (cyqlone::kkt, /root/reference/proj/include/cyqlone/
// kkt_solver.hpp:118-128) with the same names, argument meaning and error
// behaviour, backed by the sm_100a kernels through the C ABI
// (include/cyqlone_b200.h). A reference caller (qpalm::inner_newton_loop,
// cyqlone-bench, the tests) links libcyqlone_b200_host.so instead of the CPU
// sources; there is no CPU fallback.
//
// Differences a caller can observe:
//  * Factor keeps its blocks on the GPU; `materialize()` copies the public
//    reference members LH, LB, Acl, LA (kkt_solver.hpp:76-85) to the host.
//  * FactorOptions::vlen / workers are CPU lane / thread knobs and have no
//    effect (the reference's results do not depend on them either,
//    test_kkt.cpp:133-138); every tail (cr1 / pcr / pcg) is served by the
//    exact cyclic reduction of the whole Schur tree (within the pcr / pcg
//    accuracy contracts of test_kkt.cpp:152-161).
//  * Batched entry points (solve_problem_batch, factor_batch) are additions:
//    the reference API is single-instance.
#pragma once

#include "ocp.hpp"

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace cyqlone {
namespace batla {
/// Pivot failure of a Cholesky factorization (kernels.hpp:11-16).
struct factorize_error : std::runtime_error {
    index_t batch_index, pivot;
    factorize_error(const std::string &what, index_t batch_index, index_t pivot)
        : std::runtime_error(what), batch_index(batch_index), pivot(pivot) {}
};
} // namespace batla

namespace kkt {
using batla::index_t;
using batla::real_t;
using ocp::EqOCP;
using ocp::EqRhs;
using ocp::EqSolution;
using ocp::Mat;
using ocp::Vec;

/// 2-adic valuation with nu2(0, P) = nu2(P) (kkt_factor.cpp:15-25).
index_t nu2(index_t i, index_t P);

/// Rounds the horizon up to a multiple of P with identity-cost, zero-dynamics
/// padding stages (kkt_factor.cpp:27-47).
EqOCP pad_problem(const EqOCP &p, index_t P);

/// Column c owns stages n_per c - s (mod N_pad), s = 0 .. n_per-1
/// (kkt_solver.hpp:31-43).
struct Partition {
    index_t P = 1, n_per = 0, N_pad = 0;
    index_t stage_of(index_t c, index_t s) const {
        index_t j = n_per * c - s;
        return ((j % N_pad) + N_pad) % N_pad;
    }
    index_t x_index_of(index_t c, index_t s) const {
        index_t j = stage_of(c, s);
        return j == 0 ? N_pad : j;
    }
};

enum class Tail { cr1, pcr, pcg };

struct FactorOptions {
    index_t P = 1;
    index_t vlen = 4;
    index_t workers = 1;
    Tail tail = Tail::cr1;
    real_t pcg_tol = 1e-12;
    index_t pcg_max_iter = 50;
    real_t rho = 0.5;
};

/// Per-phase multiply-add counts (kkt_solver.hpp:59-64): the reference's
/// counter with one column per group (vlen = 1); the GPU executes exactly
/// these operations.
struct FlopTrace {
    std::uint64_t riccati = 0, schur = 0, cr = 0;
    std::uint64_t total() const { return riccati + schur + cr; }
};

/// Device-resident factor of one (or a batch of) KKT system(s).
class Factor {
  public:
    FactorOptions opts;
    Partition part;
    index_t nx = 0, nu = 0, N_orig = 0, batch = 1;

    /// Host copies of the reference's public factor blocks of instance
    /// `inst`, dense row-major: LH[s][c] (nux x nux lower), LB[s][c]
    /// (nx x nu), Acl[s][c] (nx x nx), LA[c] (nx x nx).
    struct Blocks {
        std::vector<std::vector<Mat>> LH, LB, Acl; // [s][c]
        std::vector<Mat> LA;                       // [c]
    };
    Blocks materialize(index_t inst = 0) const;

    Factor();
    ~Factor();
    Factor(Factor &&) noexcept;
    Factor &operator=(Factor &&) noexcept;
    Factor(const Factor &) = delete;
    Factor &operator=(const Factor &) = delete;

    struct Impl;
    std::unique_ptr<Impl> impl;
};

/// kkt::factor (kkt_factor.cpp:251-313). Throws std::invalid_argument for a
/// non-power-of-two P or vlen, batla::factorize_error on a pivot failure,
/// std::runtime_error on a CUDA error.
Factor factor(const EqOCP &p, const FactorOptions &opts, FlopTrace *trace = nullptr);
/// kkt::solve (kkt_solve.cpp:23-309) with an explicit right-hand side.
EqSolution solve(const Factor &f, const EqOCP &p, const EqRhs &rhs);
/// kkt::solve_problem (kkt_solve.cpp:311-317): factor + solve(of_problem).
EqSolution solve_problem(const EqOCP &p, const FactorOptions &opts, Factor *factor_out = nullptr);

/// Batched additions: independent instances of one shape, solved in one
/// launch sequence (the GPU's unit of work). A pivot failure in any
/// instance throws factorize_error{batch_index = instance}; the other
/// instances' solutions are still written when `status` is given.
struct InstanceStatus {
    int code = 0; ///< 0 ok, 2 pivot failure
    int kind = 0; ///< 0 Riccati, 1 cyclic reduction
    index_t column_or_level = 0, stage = 0, pivot = 0;
};
std::vector<EqSolution> solve_problem_batch(const std::vector<EqOCP> &ps, const FactorOptions &opts,
                                            std::vector<InstanceStatus> *status = nullptr);
Factor factor_batch(const std::vector<EqOCP> &ps, const FactorOptions &opts);
std::vector<EqSolution> solve_batch(const Factor &f, const std::vector<EqOCP> &ps,
                                    const std::vector<EqRhs> &rhs);

/// Diagonal penalty change per stage (kkt_solver.hpp:130-138): zero where
/// the active set did not change; `terminal` applies to the rows C_N.
struct SigmaDelta {
    std::vector<Vec> stage; ///< size N, length ny each
    Vec terminal;           ///< length ny_term
    index_t total_rank() const;
};

/// delta[i] = +sigma_i for newly active rows, -sigma_i for newly inactive
/// (kkt_update.cpp:30-41).
Vec active_set_delta(const std::vector<bool> &prev, const std::vector<bool> &now, const Vec &sigma);

struct UpdateReport {
    index_t columns_updated = 0;
    index_t columns_refactored = 0;
    bool schur_refactored = false;
    index_t schur_levels_updated = 0;
};

/// kkt::update (kkt_solver.hpp:152-161, kkt_update.cpp:372-477): afterwards
/// the factor equals (up to roundoff) a fresh factorization of `p_new`
/// (whose Hessians carry H_j + (D_j | C_j)' dSigma_j (D_j | C_j)). Per
/// partition column the accumulated update rank r selects the path, as in
/// the reference: r < rho nx the hyperbolic-Householder low-rank column
/// update (on the GPU), r >= rho nx (or a hyperbolic breakdown) a column
/// refactorization; the Schur complement and its CR factor are then
/// re-formed from the updated columns (schur_refactored = true,
/// schur_levels_updated = 0). With dSigma = 0 the factor is left as it is.
/// Throws std::invalid_argument on shape mismatches.
UpdateReport update(Factor &f, const EqOCP &p_new, const std::vector<Mat> &C,
                    const std::vector<Mat> &D, const Mat &C_term, const SigmaDelta &ds);

/// Critical-path FLOP model (kkt_solver.hpp:165-176, kkt_factor.cpp:319-339).
struct FlopModel {
    real_t riccati = 0, schur = 0, cr = 0, total = 0, serial = 0, speedup = 0;
};
FlopModel flops_critical_path(index_t nx, index_t nu, index_t N, index_t P);

/// Name and tile shapes of the kernels behind this library.
std::string backend_info();

} // namespace kkt
} // namespace cyqlone
