// Kernel argument blocks and launch helpers shared by the C ABI.
#pragma once

#include <atomic>
#include <mutex>
#include <utility>

#include "kkt_common.cuh"

#include <cuda_runtime.h>

struct cyq_ctx; // include/cyqlone_b200.h

namespace cyqb {

// One-time per-device launch setup (function attributes, constant-memory
// tables are per device; a context per GPU may live in one process,
// include/cyqlone_b200.h). `setup()` runs under a lock, at most once per
// device once it succeeded: a second host thread never launches before the
// attributes are set, and a failed setup is retried on the next call (the
// launch itself then reports the error).
struct DeviceOnce {
    std::mutex m;
    std::atomic<unsigned long long> done{0};
};
template <class F> cudaError_t once_per_device(DeviceOnce &o, F &&setup) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    if (o.done.load(std::memory_order_acquire) & bit)
        return cudaSuccess;
    std::lock_guard<std::mutex> lk(o.m);
    if (o.done.load(std::memory_order_relaxed) & bit)
        return cudaSuccess;
    const cudaError_t e = setup();
    if (e == cudaSuccess)
        o.done.fetch_or(bit, std::memory_order_release);
    return e;
}

// Launch with programmatic stream serialization (PDL, see griddep_wait in
// kkt_common.cuh); `cluster` > 1 adds a thread-block cluster dimension.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                       Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    int na = 1;
    if (cluster > 1) {
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = cluster;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        na = 2;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Kernel selection of a context (cyq_ctx_set_option, include/cyqlone_b200.h);
// the defaults pick the fastest measured kernel per shape.
struct LaunchOpts {
    int panel = 0;         // CYQ_PANEL_*: 0 auto, 1 warp, 2 two-warp, 3 CTA, 4 generic, 5 warp + TMEM, 6 CTA + TMA
    int schur = 0;         // CYQ_SCHUR_*: 0 auto (fused / big), 1 per-level tile kernels, 2 scalar
    int schur_warps = 0;   // fused Schur CTA width: 0 auto, 2 or 4 warps
    int schur_cluster = 1; // 8-CTA cluster for a few long horizons (0: never)
    int split = 1;         // device batches in K parts on two streams
    int backsub = 0;       // 0 auto, 1 generic runtime-shape kernel
    int fused_aug = 1;     // Newton-system assembly fused into the panel (0: assembly kernel)
    int panel_warps = 0;   // generic panel: warps per chain CTA (0 auto)
    int tail = 0;          // CYQ_TAIL_*: Schur tail (0 cr1 / 2 pcg: exact CR, 1 pcr)
    int vlen = 4;          // FactorOptions::vlen: the pcr tail has min(P, vlen) blocks
    int phase_prof = 0;    // per-stage phase clocks of chain 0 (profiling aid)
    int async_status = 0;  // device calls return without a host sync (cyq_ctx_wait_status)
    int graphs = 1;        // repeated identical device calls replay a captured CUDA graph
    int sms = 148;         // multiprocessors of the context's device
};

// Device workspace of one factorization of a batch (all chains).
struct FactorWS {
    double *fac;   // [chain][s][NPT][64]   stored pivot tiles (LH | LB ALQ | y')
    double *y;     // [chain][s][nux]       forward-substituted [u; x] per stage
    double *wl;    // [chain][s][nx]        interior multipliers after the forward sweep
    double *trail; // [chain][NTT][64]      -Mfwd (coupling) and -fwd (rhs row)
    double *schur; // [batch][SCH]          CR factor + scratch (see schur_layout)
    double *lamc;  // [batch][P][nx]        coupling multipliers lambda^{n i}
    unsigned long long *fail; // [batch]    first failure key, ~0 = ok
    double *consts;           // identity / zero constants (generic kernel)
};

struct RiccatiArgs {
    Geo g;
    ProbView p;
    double *fac, *y, *wl, *trail;
    unsigned long long *fail;
    const double *consts; // I_nu | I_nx | zeros (direct-mode generic kernel)
    int staged;           // generic kernel: stage data staged in smem
    long long *phase;     // optional per-stage phase clocks of chain 0 (profiling)
    // optional: factor only the listed chains (instance * P + column), n_list
    // of them, one per grid slot (kkt::update's refactorized columns)
    const int *chain_list = nullptr;
    int n_list = 0;
    // number of chains the grid covers
    __host__ __device__ int grid_chains() const { return chain_list ? n_list : g.batch * g.P; }
    __device__ int chain_of(int slot) const { return chain_list ? chain_list[slot] : slot; }
};

struct SchurArgs {
    Geo g;
    ProbView p;
    const double *fac, *y, *trail;
    double *schur, *lamc;
    double *lam_out; // solution lam (nullable)
    unsigned long long *fail;
    int do_factor, do_solve;
    long long *phase = nullptr; // optional phase clocks of instance 0 (profiling)
};

struct BacksubArgs {
    Geo g;
    ProbView p;
    const double *fac, *y, *wl, *lamc;
    SolView sol;
};

// Per-instance Schur workspace layout (doubles), nx x nx blocks:
//   D[P], K[P]            level-0 block tridiagonal (diag, subdiag)
//   Mb[P], Z[P]           Mbwd and L_Q^{-1} per column (scratch)
//   bn[P * nx]            bwd_neg = T x' per column (scratch)
//   per level l: L[half], U[half], Y[half], M[half], Kn[half], CY[half]
//   Lbase                 base Cholesky factor
//   rhs[P * nx]
struct SchurLayout {
    long long D, K, Mb, Z, bn, lvl0, Lbase, rhs, total;
    int levels;
    __host__ __device__ static SchurLayout make(int P, int nx) {
        SchurLayout s;
        const long long nn = (long long)nx * nx;
        int lg = 0;
        while ((1 << lg) < P)
            ++lg;
        s.levels = lg;
        s.D = 0;
        s.K = s.D + P * nn;
        s.Mb = s.K + P * nn;
        s.Z = s.Mb + P * nn;
        s.bn = s.Z + P * nn;
        s.lvl0 = s.bn + (long long)P * nx;
        long long off = s.lvl0;
        int sz = P;
        for (int l = 0; l < lg; ++l, sz /= 2)
            off += 6LL * (sz / 2) * nn;
        s.Lbase = off;
        s.rhs = s.Lbase + nn;
        s.total = s.rhs + (long long)P * nx;
        return s;
    }
    // level l arrays (half = P >> (l+1) blocks each)
    __host__ __device__ long long level(int l, int P, int nx, int which) const {
        const long long nn = (long long)nx * nx;
        long long off = lvl0;
        int sz = P;
        for (int k = 0; k < l; ++k, sz /= 2)
            off += 6LL * (sz / 2) * nn;
        return off + (long long)which * (sz / 2) * nn;
    }
};

template <int MAXT> __global__ void riccati_panel_kernel_t(RiccatiArgs a);
// compile-time (nu, nx) warp-per-chain fast path; false if not instantiated
// exact QPALM line search (linesearch.cu), one CTA per instance
struct LineSearchArgs {
    long long batch, m;
    const double *alpha, *delta, *eta, *beta; // [batch][m], [batch][m], [batch], [batch]
    double *tau;                              // [batch]
    int *status;                              // [batch]: 0 ok, 1 not a descent direction
    long long *iters;                         // [batch] probes + scan steps (nullable)
    double *scratch;                          // [batch][m][2] breakpoints (t, w)
};
void launch_line_search(cudaStream_t st, const LineSearchArgs &a);
// augmented-Lagrangian gradients of the QPALM inner loop (gradients.cu)
struct GradArgs {
    int batch, N, nx, nu, ny;
    const double *R, *S, *Q, *A, *B, *f, *r, *q;                 // problem (ABI layout)
    const double *D, *C, *bl, *bu, *u, *x, *y, *sigma, *ubar, *xbar; // QPALM data and state
    double gamma_inv;
    double *ru, *qx, *yhat, *cres;                               // outputs
};
bool launch_al_gradients(cudaStream_t st, const GradArgs &a);
// kkt::update's column path (update.cu): listed chains, in place
struct UpdateArgs {
    Geo g;
    ProbView p;           // the updated problem ([B A] for the propagation)
    double *fac, *trail;  // factor tiles and -Mfwd, updated in place
    const int *chains;    // chains to update (instance * P + column)
    int n;
    const double *D, *C;  // [b][N][ny][nu], [b][N][ny][nx]
    const double *C_term; // [b][ny_term][nx]
    const double *ds, *ds_term; // [b][N][ny], [b][ny_term]
    int ny, ny_term, cap; // cap: max update columns of a listed chain
    int *breakdown;       // [n]: 1 = hyperbolic breakdown / over cap -> refactorize
};
bool launch_update_columns(cudaStream_t st, const UpdateArgs &a);
size_t update_smem_bytes(int nx, int nu, int cap);

bool launch_riccati_warp(const Geo &g, cudaStream_t st, const RiccatiArgs &ra, const LaunchOpts &o);
// true when the warp kernel has a fused Newton-system augmentation variant
// for this stage shape and ny (ProbView::aD path)
bool riccati_warp_fuses_aug(const Geo &g, int ny, const LaunchOpts &o);
// CTA-per-chain kernel for large tile-aligned panels (riccati_cta.cu); false if n/a
bool launch_riccati_cta(const Geo &g, cudaStream_t st, const RiccatiArgs &ra, bool tma = false);
// producer/consumer two-warp-per-chain kernel (riccati_pc.cu); false if n/a
bool launch_riccati_pc(const Geo &g, cudaStream_t st, const RiccatiArgs &ra);
// tile-based Schur assembly + CR factorization (compile-time nx); false if n/a
bool launch_schur_tiles(const Geo &g, cudaStream_t st, const SchurArgs &sa);
// fused Schur + CR factor (+ solve) kernel, one CTA per instance (schur_fused.cu);
// false if the shape / batch is not served (the caller falls back)
bool schur_fused_ok(const Geo &g, const LaunchOpts &o);
bool launch_schur_fused(const Geo &g, cudaStream_t st, const SchurArgs &sa, const LaunchOpts &o);
size_t schur_fused_doubles(const Geo &g);
// CTA-level Schur + CR for large tile-aligned nx (schur_big.cu); false if n/a
bool launch_schur_big(const Geo &g, cudaStream_t st, const SchurArgs &sa);
size_t schur_big_doubles(const Geo &g);
// compile-time (nu, nx) warp-per-chain back substitution; false if n/a
bool launch_backsub_warp(const Geo &g, cudaStream_t st, const BacksubArgs &ba);
// warp-per-chain back substitution streaming tiles from global (tile-aligned large shapes)
bool launch_backsub_tile(const Geo &g, cudaStream_t st, const BacksubArgs &ba);
// forward substitution over a stored factor (kkt::solve with a new rhs)
__global__ void forward_kernel(BacksubArgs a, double *y_out, double *wl_out, double *trail);
__host__ __device__ size_t forward_smem_per_warp(const Geo &g);
__global__ void schur_cr_kernel(SchurArgs a);
__global__ void backsub_kernel(BacksubArgs a);

// Where the Schur-side factor blocks of one instance live in its workspace
// slice (doubles), for cyq_factor_materialize_schur: 8x8-tile-ordered
// blocks, `full` = XT x XT tiles (else lower tiles i(i+1)/2 + j, and T_c as
// upper tiles at slot T(j, i)); tt_is_inverse: the slot holds L_Q^{-1}
// (T = its transpose) instead of T. Li / Lb are L^{-1} of the CR pivots.
struct SchurBlocks {
    long long Tt, Li, U, Y, Lb, Mb, total;
    bool full, tt_is_inverse;
    int cr_levels; // CR levels stored (below a PCR tail)
};
bool schur_fused_blocks(const Geo &g, SchurBlocks &out);
bool schur_big_blocks(const Geo &g, SchurBlocks &out);

size_t riccati_smem_bytes(const Geo &g);
// context helpers for entry points outside capi.cu: selects the context's
// device, returns its stream
cudaStream_t ctx_prepare(::cyq_ctx *ctx);
// Newton-system assembly (augment.cu); false if the shape is not supported
bool launch_augment(cudaStream_t st, int batch, int N, int nx, int nu, int ny, const double *R,
                    const double *S, const double *Q, const double *D, const double *C,
                    const double *sigma, double gamma_inv, double *R_out, double *S_out,
                    double *Q_out);
bool riccati_staged(const Geo &g);
size_t riccati_consts_doubles(const Geo &g);
size_t backsub_smem_bytes(const Geo &g);
constexpr int BACKSUB_WPB = 4; // chains (warps) per back-substitution CTA (max)
int backsub_wpb(const Geo &g);
size_t schur_smem_bytes(const Geo &g);
int schur_warps(const Geo &g);
int schur_warps_solve(const Geo &g);
size_t schur_smem_for(const Geo &g, int nw);

} // namespace cyqb
