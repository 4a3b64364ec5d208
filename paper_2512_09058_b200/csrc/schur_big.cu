// Schur complement + cyclic reduction (factor and solve) for LARGE,
// tile-aligned nx (nx % 8 == 0, nx >= 32; BASELINE config 3: 64 x 64
// blocks): one CTA per OCP instance, every block operation spread over the
// CTA's warps (cta_tiles.cuh). Same algorithm and workspace semantics as the
// register-tile fused kernel for small nx (schur_fused.cu):
//   kkt_factor.cpp:163-178    T = L_Q^{-T}, Mbwd = T T', W = T LA'
//   kkt_factor.cpp:194-212    assemble_schur
//   block_tridiag.cpp:126-238 cr_level / cr_factor_base
//   kkt_solve.cpp:137-182     Schur rhs, CRFactor::forward / backward
// with explicit inverse factors Li = L^{-1} (so U, Y are DMMA GEMMs and the
// CR solve is matrix-vector products) and the forward CR sweep fused into
// the factor levels when the rhs is known (solve_problem).
#include "cta_tiles.cuh"
#include "kernels.h"

#include <cstdlib>

namespace cyqb {

namespace {

// Per-instance workspace, full XT x XT tile blocks (NF tiles):
//   Tt[P]  L_Q^{-1} per column (T = Tt')          (persistent)
//   Li[P-1], U[P-1], Y[P-1], Lb                    (persistent)
//   D[P], Mb[P], K[P]                              (scratch, CR in place)
//   S1, S2                                         (scratch blocks; S1 unused since
//                                                    the working blocks moved to shared memory)
struct SBLayout {
    long long Tt, Li, U, Y, Lb, D, Mb, K, S1, S2, total;
    int levels;
    __host__ __device__ static SBLayout make(int P, int nx) {
        SBLayout s;
        const long long tf = 64LL * (nx / 8) * (nx / 8);
        int lg = 0;
        while ((1 << lg) < P)
            ++lg;
        s.levels = lg;
        long long o = 0;
        s.Tt = o; o += P * tf;
        s.Li = o; o += (P - 1) * tf;
        s.U = o; o += (P - 1) * tf;
        s.Y = o; o += (P - 1) * tf;
        s.Lb = o; o += tf;
        s.D = o; o += P * tf;
        s.Mb = o; o += P * tf;
        s.K = o; o += P * tf;
        s.S1 = o; o += tf;
        s.S2 = o; o += tf;
        s.total = o;
        return s;
    }
};

template <int XT, int NW>
__device__ __forceinline__ void blk_zero(double *C, int warp, int lane) {
    for (int t = warp; t < XT * XT; t += NW)
        st_frag(C + t * kTileElems, lane, Frag{0.0, 0.0});
}
// C = A + sgn B over the lower tiles (B nullable)
template <int XT, int NW>
__device__ __forceinline__ void blk_axpy_lower(double *C, const double *A, const double *B, double sgn,
                                               int warp, int lane) {
    for (int o = warp; o < XT * (XT + 1) / 2; o += NW) {
        int i = 0;
        while ((i + 1) * (i + 2) / 2 <= o)
            ++i;
        const int t = i * XT + (o - i * (i + 1) / 2);
        Frag f = ld_frag(A + t * kTileElems, lane);
        if (B) {
            const Frag h = ld_frag(B + t * kTileElems, lane);
            f.a += sgn * h.a;
            f.b += sgn * h.b;
        }
        st_frag(C + t * kTileElems, lane, f);
    }
}

// C = A over all XT x XT tiles (shared -> global stream-out of a block)
template <int XT, int NW>
__device__ __forceinline__ void blk_copy(double *C, const double *A, int warp, int lane) {
    for (int t = warp; t < XT * XT; t += NW)
        st_frag(C + t * kTileElems, lane, ld_frag(A + t * kTileElems, lane));
}
// the lower tiles of A, zero upper tiles
template <int XT, int NW>
__device__ __forceinline__ void blk_copy_lower(double *C, const double *A, int warp, int lane) {
    for (int t = warp; t < XT * XT; t += NW)
        st_frag(C + t * kTileElems, lane, t % XT <= t / XT ? ld_frag(A + t * kTileElems, lane) : Frag{0.0, 0.0});
}

// shared-memory layout (doubles): per-warp scratch, the solve vectors (the
// CR contributions cu / cy alias bwd_neg, dead once the rhs is assembled)
// and two 64 x 64 working blocks: the pivot block (factored in place) and
// L^{-1} of each elimination (T of each column in phase 1), the operands
// the block ops read most, stay in shared memory; L^{-1} / T are streamed
// out to the persistent factor. Two CTAs of 8 warps per SM (measured:
// 2.57 -> 2.44 ms at config 3; four shared blocks at one 16- or 8-warp CTA
// per SM: 3.29 / 3.88 ms -- two instances per SM hide each other's barriers)
template <int NX, int NW> struct SBSmem {
    static constexpr int XT = NX / 8, BLK = XT * XT * kTileElems;
    __host__ __device__ static size_t vec(int P) {
        const size_t bn = (size_t)P * NX > (size_t)(P / 2 + 1) * NX * 2 ? (size_t)P * NX : (size_t)(P / 2 + 1) * NX * 2;
        return (size_t)NW * kTileElems + (size_t)P * NX + bn + 2 * NX;
    }
    __host__ __device__ static size_t total(int P) { return vec(P) + 2 * (size_t)BLK; }
};

template <int NX, int NW>
__global__ void __launch_bounds__(32 * NW, 2) schur_big_kernel(SchurArgs a) {
    constexpr int XT = NX / 8, NF = XT * XT;
    constexpr long long TF = 64LL * NF;
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = g.P, nu = g.nu, n = g.n, CT = g.CT;
    griddep_launch();
    griddep_wait(); // the stage panel's factor tiles
    const SBLayout Lo = SBLayout::make(P, NX);
    double *ws = a.schur + (size_t)b * Lo.total;
    double *Tt = ws + Lo.Tt, *D = ws + Lo.D, *Mb = ws + Lo.Mb, *K = ws + Lo.K, *S1 = ws + Lo.S1,
           *S2 = ws + Lo.S2;
    using SB = SBSmem<NX, NW>;
    double *scr = sm;                       // NW x 64
    double *xs = scr + NW * kTileElems;     // P x NX
    double *bns = xs + (size_t)P * NX;      // P x NX (then cu / cy)
    double *cu = bns;                       // P/2 x NX
    double *cy = cu + (size_t)(P / 2 + 1) * NX;
    double *v1 = sm + SB::vec(P) - 2 * NX, *v2 = v1 + NX; // NX each
    double *B0 = sm + SB::vec(P), *B1 = B0 + SB::BLK;
    (void)S1;
    const bool fwd_fused = a.do_factor && a.do_solve;
    int fail = -1, fail_l = 0, fail_k = 0;

    long long *ph = (a.phase && b == 0 && threadIdx.x == 0) ? a.phase : nullptr;
    int php = 0;
    if (ph) ph[php++] = clock64();
    // ---- phase 1: per column T, Mbwd, K, Mfwd, bwd_neg ------------------
    for (int c = 0; c < P; ++c) {
        const size_t chain = (size_t)b * P + c;
        const double *st = a.fac + (chain * n + (n - 1)) * g.NPT * kTileElems;
        auto ftile = [&](int i, int j) { // stored pivot tile (i, j < CT)
            return st + (i < CT ? tri_index(i, j) : CT * (CT + 1) / 2 + (i - CT) * CT + j) * kTileElems;
        };
        const int xt0 = nu / 8;
        double *Tc = Tt + c * TF;
        if (a.do_factor) {
            // L_Q -> B0 (lower), LA -> B1 (full), -Mfwd -> D[c] (lower)
            const double *tr = a.trail + chain * g.NTT * kTileElems;
            double *LAb = S2, *Tb = B1; // LA (global scratch), T (shared)
            for (int t = warp; t < NF; t += NW) {
                const int i = t / XT, j = t % XT;
                st_frag(LAb + t * kTileElems, lane, ld_frag_g(ftile(CT + i, xt0 + j), lane));
                if (j <= i) {
                    st_frag(B0 + t * kTileElems, lane, ld_frag_g(ftile(xt0 + i, xt0 + j), lane));
                    Frag m = ld_frag_g(tr + tri_index(i, j) * kTileElems, lane);
                    st_frag(D + c * TF + t * kTileElems, lane, Frag{-m.a, -m.b});
                }
            }
            __syncthreads();
            ctat::cta_trtri<XT, NW>(B0, Tb, scr, warp, lane); // Tt = L_Q^{-1} (shared)
            // Mbwd = T T' (T(i,k) = Tt(k,i)', upper) ; K[c-1] = -LA T'
            ctat::cta_gemm<XT, NW, true, true, ctat::kGeMaxIJ, true>(Mb + c * TF, nullptr, 1.0, Tb, Tb, warp, lane);
            double *Kc = K + (size_t)((c + P - 1) % P) * TF;
            if (c > 0)
                ctat::cta_gemm<XT, NW, false, true, ctat::kGeJ, false>(Kc, nullptr, -1.0, LAb, Tb, warp, lane);
            else
                blk_zero<XT, NW>(Kc, warp, lane);
            if (!a.do_solve) // persistent T: read again only by kkt::solve on a kept factor
                blk_copy_lower<XT, NW>(Tc, Tb, warp, lane); // (upper tiles zero)
        }
        if (a.do_solve) { // bwd_neg_c = T x'_{n-1} = Tt' x'
            const double *yv = a.y + (chain * n + (n - 1)) * g.nux + nu;
            for (int k = tid; k < NX; k += 32 * NW)
                v1[k] = __ldg(yv + k);
            __syncthreads();
            ctat::cta_matvec<XT, NW, true, true>(a.do_factor ? B1 : Tc, v1, bns + c * NX, 1.0, false, warp, lane);
        }
        __syncthreads();
    }

    if (ph) ph[php++] = clock64();
    // ---- Schur rhs b_i = fd[n i] - fwd_i + bwd_neg_{(i+1) % P} ------------
    if (a.do_solve) {
        ProbAcc pa{a.p, g, b};
        for (int e = tid; e < P * NX; e += 32 * NW) {
            const int i = e / NX, k = e % NX, jst = n * i;
            double v = pa.fd(jst, k);
            if (jst == 0 && a.p.fd == nullptr) {
                double ax = 0.0;
                for (int m = 0; m < NX; ++m)
                    ax = fma(pa.A(0, k, m), __ldg(a.p.x_init + (size_t)b * NX + m), ax);
                v -= ax;
            }
            const double *tr = a.trail + ((size_t)b * P + i) * g.NTT * kTileElems;
            v += __ldg(tr + tri_index(XT, k / 8) * kTileElems + k % 8);
            v += bns[((i + 1) % P) * NX + k];
            xs[e] = v;
        }
        __syncthreads();
    }

    if (ph) ph[php++] = clock64();
    // ---- CR levels (in place in D / K, as schur_fused.cu) -----------------
    if (a.do_factor) {
        for (int l = 0, s = P; l < Lo.levels; ++l, s >>= 1) {
            if (ph && l > 0) ph[php++] = clock64();
            const int half = s / 2, hcy = l > 0 ? 1 << (l - 1) : 0;
            const long long out0 = P - (P >> l);
            auto assemble = [&](double *dst, int i) { // level-l diagonal block i -> dst
                if (l == 0)
                    blk_axpy_lower<XT, NW>(dst, D + i * TF, Mb + ((i + 1) % P) * TF, 1.0, warp, lane);
                else
                    blk_axpy_lower<XT, NW>(dst, D + (size_t)(i << l) * TF,
                                           i > 0 ? D + (size_t)((i << l) - hcy) * TF : nullptr, -1.0,
                                           warp, lane);
            };
            for (int mm = 0; mm < half; ++mm) {
                const int k = 2 * mm + 1;
                const bool has_y = k < s - 1, last = mm == half - 1;
                double *Lig = ws + Lo.Li + (out0 + mm) * TF, *Ug = ws + Lo.U + (out0 + mm) * TF;
                double *Yg = ws + Lo.Y + (out0 + mm) * TF;
                double *Li = B1, *U = Ug, *Y = Yg; // L^{-1} in shared memory
                const double *Kp = K + (size_t)((k - 1) << l) * TF, *Kk = K + (size_t)(k << l) * TF;
                assemble(B0, k);
                __syncthreads();
                int f = -1;
                ctat::cta_potrf_inv<XT, NW>(B0, Li, scr, NX, warp, lane, tid, f);
                if (warp == 0 && f >= 0 && fail < 0) {
                    fail = f;
                    fail_l = l;
                    fail_k = k;
                }
                // U = K_{k-1}' Li', Y = K_k Li' (Li lower: k-range <= j)
                ctat::cta_gemm<XT, NW, true, false, ctat::kLeJ, false>(U, nullptr, 1.0, Kp, Li, warp, lane);
                if (has_y)
                    ctat::cta_gemm<XT, NW, false, false, ctat::kLeJ, false>(Y, nullptr, 1.0, Kk, Li, warp, lane);
                else
                    blk_zero<XT, NW>(Y, warp, lane);
                __syncthreads();
                blk_copy<XT, NW>(Lig, Li, warp, lane); // persistent CR factor
                assemble(B0, 2 * mm); // the even block (B0's L is dead)
                if (fwd_fused) { // x_k <- Li x_k ; contributions U x_k, Y x_k
                    double *xk = xs + (size_t)(k << l) * NX;
                    ctat::cta_matvec<XT, NW, false, true>(Li, xk, v1, 1.0, false, warp, lane);
                    __syncthreads();
                    for (int e = tid; e < NX; e += 32 * NW)
                        xk[e] = v1[e];
                    __syncthreads();
                    ctat::cta_matvec<XT, NW, false, false>(U, xk, cu + mm * NX, 1.0, false, warp, lane);
                    ctat::cta_matvec<XT, NW, false, false>(Y, xk, cy + mm * NX, 1.0, false, warp, lane);
                }
                // M' = M_2mm - U U' -> D[2mm << l]; CY = Y Y' -> D[k << l]; K' = -Y U' -> K[2mm << l]
                __syncthreads();
                ctat::cta_gemm<XT, NW, false, false, ctat::kAll, true>(D + (size_t)((2 * mm) << l) * TF, B0, -1.0,
                                                                      U, U, warp, lane);
                ctat::cta_gemm<XT, NW, false, false, ctat::kAll, true>(D + (size_t)(k << l) * TF, nullptr, 1.0, Y,
                                                                      Y, warp, lane);
                if (!last)
                    ctat::cta_gemm<XT, NW, false, false, ctat::kAll, false>(K + (size_t)((2 * mm) << l) * TF,
                                                                           nullptr, -1.0, Y, U, warp, lane);
                else
                    blk_zero<XT, NW>(K + (size_t)((2 * mm) << l) * TF, warp, lane);
                __syncthreads();
            }
            if (fwd_fused) { // x_{2mm} -= U_mm x_{2mm+1} + Y_{mm-1} x_{2mm-1}
                for (int e = tid; e < half * NX; e += 32 * NW) {
                    const int mm = e / NX, r = e % NX;
                    double d = cu[e];
                    if (mm > 0)
                        d += cy[e - NX];
                    xs[(size_t)((2 * mm) << l) * NX + r] -= d;
                }
                __syncthreads();
            }
        }
        // cr_factor_base
        if (Lo.levels == 0)
            blk_axpy_lower<XT, NW>(B0, D, Mb, 1.0, warp, lane);
        else
            blk_axpy_lower<XT, NW>(B0, D, nullptr, 0.0, warp, lane);
        __syncthreads();
        int f = -1;
        ctat::cta_potrf_inv<XT, NW>(B0, B1, scr, NX, warp, lane, tid, f);
        __syncthreads();
        blk_copy<XT, NW>(ws + Lo.Lb, B1, warp, lane);
        if (warp == 0 && f >= 0 && fail < 0) {
            fail = f;
            fail_l = Lo.levels;
            fail_k = 0;
        }
        __syncthreads();
    }

    // ---- CR solve over the stored factor, negate --------------------------
    if (a.do_solve) {
        if (!fwd_fused) {
            for (int l = 0, s = P; l < Lo.levels; ++l, s >>= 1) {
                const int half = s / 2, stride = P / s;
                const long long o0 = P - (P >> l);
                for (int mm = 0; mm < half; ++mm) {
                    double *xk = xs + (size_t)(2 * mm + 1) * stride * NX;
                    ctat::cta_matvec<XT, NW, false, true>(ws + Lo.Li + (o0 + mm) * TF, xk, v1, 1.0, false, warp,
                                                         lane);
                    __syncthreads();
                    for (int e = tid; e < NX; e += 32 * NW)
                        xk[e] = v1[e];
                    __syncthreads();
                }
                for (int mm = 0; mm < half; ++mm) {
                    double *xe = xs + (size_t)2 * mm * stride * NX;
                    ctat::cta_matvec<XT, NW, false, false>(ws + Lo.U + (o0 + mm) * TF,
                                                          xs + (size_t)(2 * mm + 1) * stride * NX, v1, 1.0, false,
                                                          warp, lane);
                    if (mm > 0)
                        ctat::cta_matvec<XT, NW, false, false>(ws + Lo.Y + (o0 + mm - 1) * TF,
                                                              xs + (size_t)(2 * mm - 1) * stride * NX, v1, 1.0,
                                                              true, warp, lane);
                    __syncthreads();
                    for (int e = tid; e < NX; e += 32 * NW)
                        xe[e] -= v1[e];
                    __syncthreads();
                }
            }
        }
        if (ph) ph[php++] = clock64();
        // base: x_0 <- Lb^{-T} Lb^{-1} x_0
        ctat::cta_matvec<XT, NW, false, true>(ws + Lo.Lb, xs, v1, 1.0, false, warp, lane);
        __syncthreads();
        ctat::cta_matvec<XT, NW, true, true>(ws + Lo.Lb, v1, xs, 1.0, false, warp, lane);
        __syncthreads();
        // CRFactor::backward
        for (int l = Lo.levels - 1; l >= 0; --l) {
            const int sl = P >> l, half = sl / 2, stride = P / sl;
            const long long o0 = P - (P >> l);
            for (int mm = 0; mm < half; ++mm) {
                double *xo = xs + (size_t)(2 * mm + 1) * stride * NX;
                ctat::cta_matvec<XT, NW, true, false>(ws + Lo.U + (o0 + mm) * TF,
                                                     xs + (size_t)2 * mm * stride * NX, v1, 1.0, false, warp, lane);
                if (2 * mm + 2 < sl)
                    ctat::cta_matvec<XT, NW, true, false>(ws + Lo.Y + (o0 + mm) * TF,
                                                         xs + (size_t)((2 * mm + 2) * stride % P) * NX, v1, 1.0,
                                                         true, warp, lane);
                __syncthreads();
                for (int e = tid; e < NX; e += 32 * NW)
                    v2[e] = xo[e] - v1[e];
                __syncthreads();
                ctat::cta_matvec<XT, NW, true, true>(ws + Lo.Li + (o0 + mm) * TF, v2, xo, 1.0, false, warp, lane);
                __syncthreads();
            }
        }
        for (int e = tid; e < P * NX; e += 32 * NW) {
            const int i = e / NX, k = e % NX;
            const double lam = -xs[e];
            a.lamc[(size_t)b * P * NX + e] = lam;
            if (a.lam_out && n * i < g.N)
                a.lam_out[((size_t)b * g.N + n * i) * NX + k] = lam;
        }
    }
    if (ph) {
        ph[php++] = clock64();
        ph[31] = php;
    }
    if (warp == 0 && lane == 0 && fail >= 0)
        atomicMin(a.fail + b, fail_key(kKindCR, fail_l, fail_k, fail));
}

template <int NX> bool launch_sb(const Geo &g, cudaStream_t st, const SchurArgs &sa) {
    if (g.nx != NX)
        return false;
    // 16 warps per instance CTA (two CTAs per SM, 64 registers): the block
    // operations are chains of dependent DMMAs per tile, so more warps per
    // block shorten every step (config 3: 8 / 12 / 16 warps 2.44 / 2.31 /
    // 2.27 ms)
#ifndef CYQ_SB_NW
#define CYQ_SB_NW 16
#endif
    constexpr int NW = CYQ_SB_NW;
    const size_t smem = SBSmem<NX, NW>::total(g.P) * sizeof(double);
    if (smem > 227 * 1024)
        return false;
    static DeviceOnce once;
    once_per_device(once, [&] {
        return cudaFuncSetAttribute(schur_big_kernel<NX, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    launch_pdl(schur_big_kernel<NX, NW>, dim3(g.batch), dim3(32 * NW), smem, st, 1, sa);
    return true;
}

} // namespace

bool schur_big_blocks(const Geo &g, SchurBlocks &out) {
    if (g.nx % 8 != 0)
        return false;
    const SBLayout L = SBLayout::make(g.P, g.nx);
    out = SchurBlocks{L.Tt, L.Li, L.U, L.Y, L.Lb, L.Mb, L.total, true, true, L.levels};
    return true;
}

size_t schur_big_doubles(const Geo &g) {
    return (g.nx % 8 == 0) ? (size_t)SBLayout::make(g.P, g.nx).total : 0;
}

bool launch_schur_big(const Geo &g, cudaStream_t st, const SchurArgs &sa) {
    if (g.nu % 8 != 0)
        return false;
    return launch_sb<64>(g, st, sa) || launch_sb<32>(g, st, sa);
}

} // namespace cyqb
