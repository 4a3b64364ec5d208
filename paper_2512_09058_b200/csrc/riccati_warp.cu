// Warp-per-chain stage-panel Riccati kernel, specialised at compile time on
// (nu, nx): the fast path for stage blocks up to nux = 32 (BASELINE configs
// 0, 1, 2, 4). Same algorithm and outputs as riccati.cu (the runtime-shape
// CTA kernel used for every other shape):
//   kkt_factor.cpp:125-158  modified Riccati recursion (LH, LB, Acl, LA)
//   kkt_factor.cpp:163-185  Mfwd = sum LB LB' + LA LA' (trailing block)
//   kkt_solve.cpp:72-134    forward substitution + coupling rows (rhs row)
//
// One warp owns one partition column. The whole extended panel lives in the
// warp's registers as 8x8 DMMA C-fragments (tile indices are compile-time,
// so all index arithmetic folds away); the rank-8 block updates are DMMAs
// whose A/B operands are the register tiles themselves (k permuted, no
// shuffles).
//
// Shared memory per warp:
//  * the next stage's data, staged by cp.async straight into the layouts the
//    compute reads: R and Q land in a tile-ordered image of the panel's
//    pivot block (padding diagonal preset once), so initialising a panel
//    tile is one 16-byte shared load per lane; [B A] lands as one padded
//    row-major block (the A operand of V = BA' L_Q, no selects); S (its
//    transpose fills the S' tiles), [r; q] and f as plain vectors;
//  * W = [V; ALQ; -wl] with its x-columns COMPACTED and permuted (the last
//    partial tile's columns on even positions), so W W' and V run over
//    ceil(nx/4) k-slices instead of the panel's x-tile span (5 instead of 6
//    at config 1) -- W W' is invariant under a column permutation;
//  * L_Q as a row-major x-space block (the B operand of V).
#include "kkt_common.cuh"
#include "kernels.h"

#include "riccati_common.cuh"
#include "riccati_stage.cuh"

#include <cstdlib>
#include <type_traits>

namespace cyqb {

using namespace cyqb::ric;

namespace {

template <int NU, int NX, int NY = 0, bool TM = false> struct WS : PanelShape<NU, NX> {
    using P_ = PanelShape<NU, NX>;
    static constexpr int TT = P_::TT, NXC = P_::NXC, NXR = P_::NXR, NIMG = P_::NIMG, PW = P_::PW;
    // per-warp shared memory (doubles); every offset is even (16-byte aligned).
    // TM: W lives in tensor memory instead (natural x-tile layout, no shared copy)
    static constexpr int O_W = 0;
    static constexpr int O_LQ = O_W + (TM ? 0 : TT * NXC * kTileElems);
    static constexpr int O_IMG = O_LQ + NXR * NX;
    static constexpr int O_IMR = O_IMG + NIMG * kTileElems;
    static constexpr int O_S = O_IMR + PW;
    static constexpr int O_BA = O_S + ((NU * NX + 1) & ~1);
    static constexpr int O_F = O_BA + NXR * PW;
    static constexpr int O_RU0 = O_F + ((NX + 1) & ~1);
    static constexpr int O_SCR = O_RU0 + ((NU + 1) & ~1);
    // Newton-system augmentation (NY > 0): [D_j C_xi] rows (NY x nux),
    // sigma of the u rows and of the x rows
    static constexpr int NUX_ = NU + NX, NYP = (NY + 7) / 8 * 8;
    static constexpr int O_X = O_SCR + kTileElems;
    static constexpr int O_SGU = O_X + ((NY * NUX_ + 1) & ~1);
    static constexpr int O_SGX = O_SGU + NYP;
    // per-lane copy plan: R / Q only (stage_H_plan; 576 B at config 1, inside
    // the 8-chains-per-SM shared-memory budget), plus [B A] (stage_BA_plan)
    // when the kernel is register-limited anyway (NY > 0)
    static constexpr bool PLAN_BA = NY > 0;
    static constexpr int O_TAB = NY > 0 ? O_SGX + NYP : O_SCR + kTileElems;
    static constexpr int SMEM = O_TAB + (PLAN_BA ? CopyPlan<NU, NX>::DOUBLES : CopyPlan<NU, NX>::DOUBLES_H);
    static_assert((O_LQ | O_IMG | O_IMR | O_S | O_BA | O_F | O_RU0 | O_SCR | O_X | O_SGU | O_SGX | O_TAB | SMEM) % 2 == 0,
                  "align");
};

// Newton-system augmentation rows of stage position (j, xi): X[k][0..nu) =
// D_j row k (j < N), X[k][nu..nux) = C_xi row k (1 <= xi <= N), and their
// sigma vectors (zero rows / sigma where a block does not apply)
template <int NU, int NX, int NY>
__device__ __forceinline__ void stage_aug(const Geo &g, const ProbView &p, int b, int j, int xi, double *X,
                                          double *sgu, double *sgx) {
    constexpr int NUX = NU + NX;
    const int N = g.N;
    const int lane = lane_v();
    const bool du = j < N, dx = xi >= 1 && xi <= N;
    const double *Dj = du ? p.aD + ((size_t)b * N + j) * NY * NU : nullptr;
    const double *Cj = dx ? p.aC + ((size_t)b * (N + 1) + xi) * NY * NX : nullptr;
    constexpr bool V2 = NU % 2 == 0 && NX % 2 == 0;
    if (Dj && V2 && aligned16(Dj)) {
#pragma unroll
        for (int e = 2 * lane; e < NY * NU; e += 64)
            cp16(X + (e / NU) * NUX + e % NU, Dj + e);
    } else {
#pragma unroll
        for (int e = lane; e < NY * NU; e += 32) {
            double *d = X + (e / NU) * NUX + e % NU;
            if (Dj)
                cp8(d, Dj + e);
            else
                *d = 0.0;
        }
    }
    if (Cj && V2 && aligned16(Cj)) {
#pragma unroll
        for (int e = 2 * lane; e < NY * NX; e += 64)
            cp16(X + (e / NX) * NUX + NU + e % NX, Cj + e);
    } else {
#pragma unroll
        for (int e = lane; e < NY * NX; e += 32) {
            double *d = X + (e / NX) * NUX + NU + e % NX;
            if (Cj)
                cp8(d, Cj + e);
            else
                *d = 0.0;
        }
    }
    wcopy<NY, 0>(sgu, du ? p.asig + ((size_t)b * (N + 1) + j) * NY : nullptr, lane);
    wcopy<NY, 0>(sgx, dx ? p.asig + ((size_t)b * (N + 1) + xi) * NY : nullptr, lane);
}

} // namespace

// ---- tensor memory as a per-lane store (TM variant) --------------------------
// W = [V; ALQ; -wl] is the one panel-sized operand that lives across a stage
// boundary; keeping it in TMEM (each warp owns its 32-lane sub-partition
// slice, a tile fragment = 4 consecutive 32-bit columns of the lane) frees
// 10.75 KB of shared memory per chain at config 1, enough for 12 resident
// chains per SM instead of 8. tcgen05.ld results are valid only after
// tcgen05.wait::ld, which therefore takes them as in/out operands.
__device__ __forceinline__ void tm_st4(uint32_t addr, Frag f) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr),
                 "r"(__double2loint(f.a)), "r"(__double2hiint(f.a)), "r"(__double2loint(f.b)),
                 "r"(__double2hiint(f.b))
                 : "memory");
}
template <int NTL> struct TmFrags {
    uint32_t r[4 * NTL];
};
// NTL consecutive tile fragments (4 columns each) starting at addr
template <int NTL> __device__ __forceinline__ void tm_ld(uint32_t addr, TmFrags<NTL> &t) {
    static_assert(NTL == 8, "x32 load");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                 "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(t.r[0]), "=r"(t.r[1]), "=r"(t.r[2]), "=r"(t.r[3]), "=r"(t.r[4]), "=r"(t.r[5]),
                   "=r"(t.r[6]), "=r"(t.r[7]), "=r"(t.r[8]), "=r"(t.r[9]), "=r"(t.r[10]), "=r"(t.r[11]),
                   "=r"(t.r[12]), "=r"(t.r[13]), "=r"(t.r[14]), "=r"(t.r[15]), "=r"(t.r[16]), "=r"(t.r[17]),
                   "=r"(t.r[18]), "=r"(t.r[19]), "=r"(t.r[20]), "=r"(t.r[21]), "=r"(t.r[22]), "=r"(t.r[23]),
                   "=r"(t.r[24]), "=r"(t.r[25]), "=r"(t.r[26]), "=r"(t.r[27]), "=r"(t.r[28]), "=r"(t.r[29]),
                   "=r"(t.r[30]), "=r"(t.r[31])
                 : "r"(addr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(t.r[0]), "+r"(t.r[1]), "+r"(t.r[2]), "+r"(t.r[3]), "+r"(t.r[4]), "+r"(t.r[5]),
                   "+r"(t.r[6]), "+r"(t.r[7]), "+r"(t.r[8]), "+r"(t.r[9]), "+r"(t.r[10]), "+r"(t.r[11]),
                   "+r"(t.r[12]), "+r"(t.r[13]), "+r"(t.r[14]), "+r"(t.r[15]), "+r"(t.r[16]), "+r"(t.r[17]),
                   "+r"(t.r[18]), "+r"(t.r[19]), "+r"(t.r[20]), "+r"(t.r[21]), "+r"(t.r[22]), "+r"(t.r[23]),
                   "+r"(t.r[24]), "+r"(t.r[25]), "+r"(t.r[26]), "+r"(t.r[27]), "+r"(t.r[28]), "+r"(t.r[29]),
                   "+r"(t.r[30]), "+r"(t.r[31])
                 :
                 : "memory");
}
template <int NTL> __device__ __forceinline__ Frag tm_frag(const TmFrags<NTL> &t, int i) {
    return Frag{__hiloint2double(t.r[4 * i + 1], t.r[4 * i]), __hiloint2double(t.r[4 * i + 3], t.r[4 * i + 2])};
}

template <int NU, int NX, int WPB, int NY, bool TM>
__device__ __forceinline__ void riccati_warp_body(const RiccatiArgs &a, int chain, uint32_t tmw, double *sm);

template <int NU, int NX, int WPB, int NY, bool TM>
__global__ void __launch_bounds__(32 * WPB, TM ? 3 : 1) riccati_warp_kernel(RiccatiArgs a) {
    using S = Shp<NU, NX>;
    static_assert(!TM || (WPB == 4 && S::TT <= 8 && S::NXT * S::TT * 4 <= 128), "TM layout");
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int wib = threadIdx.x >> 5;
    const int chain = blockIdx.x * WPB + wib;
    griddep_launch();
    uint32_t tmw = 0; // TM: this warp's TMEM base (lane offset 32 wib, column 0)
    __shared__ uint32_t s_taddr;
    if constexpr (TM) {
        if (wib == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(&s_taddr)))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tmw = s_taddr + ((32u * (uint32_t)(wib & 3)) << 16);
    }
    if (chain < a.grid_chains())
        riccati_warp_body<NU, NX, WPB, NY, TM>(a, a.chain_of(chain), tmw, sm);
    if constexpr (TM) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (wib == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(s_taddr) : "memory");
        }
    }
}

// "Pure" coupling tiles: trailing tiles whose rows and columns are all
// coupling rows (tile rows CT .. RT-1; tile row RT holds the rhs row).
// Their ALQ_s ALQ_s' terms cancel between stage s's trailing update and
// stage s+1's W W' (only LB LB' and the last stage's LA LA' remain in
// -Mfwd, kkt_factor.cpp:179-184), so both are skipped and LA LA' is
// subtracted once after the last stage.
template <int NU, int NX, int WPB, int NY, bool TM>
__device__ __forceinline__ void riccati_warp_body(const RiccatiArgs &a, int chain, uint32_t tmw, double *sm) {
    (void)tmw;
    using S = Shp<NU, NX>;
    using W = WS<NU, NX, NY, TM>;
    constexpr int RT_ = S::RHS / 8;
    auto pure = [](int ti, int tj) constexpr { return ti >= S::CT && tj >= S::CT && ti < RT_ && tj < RT_; };
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int b = chain / g.P, c = chain % g.P, n = g.n;
    const int rq = lane >> 2, cq = 2 * (lane & 3), q2 = lane & 3;

    double *base = sm + (size_t)wib * W::SMEM;
    double *Wsm = base + W::O_W, *LQ = base + W::O_LQ, *img = base + W::O_IMG;
    double *imr = base + W::O_IMR, *Sb = base + W::O_S, *BA = base + W::O_BA;
    double *fb = base + W::O_F, *ru0 = base + W::O_RU0, *tscr = base + W::O_SCR;
    double *Xa = base + W::O_X, *sgu = base + W::O_SGU, *sgx = base + W::O_SGX; // NY > 0 only
    short *ctab = reinterpret_cast<short *>(base + W::O_TAB);
    const bool implicit_rhs = (a.p.ru == nullptr);
    const double sgn = implicit_rhs ? -1.0 : 1.0;
    int fail_piv = -1, fail_stage = 0;

    // one-time init: everything zero, unit padding diagonal in the image
    // (the stage copies never touch padding / permutation-gap positions)
    for (int i = lane; i < W::SMEM; i += 32)
        base[i] = 0.0;
    __syncwarp();
    if (lane < W::PW - W::NUX) {
        const int r = W::NUX + lane;
        img[S::T(r / 8, r / 8) * kTileElems + (r % 8) * 9] = 1.0;
    }
    CopyPlan<NU, NX>::build(ctab, lane, W::PLAN_BA);
    __syncwarp();

    // prologue: H_0, BA_0 and the x_init term of ru[0]
    {
        const int j0 = g.stage_of(c, 0);
        stage_H<NU, NX>(g, a.p, b, j0, g.x_index_of(c, 0), img, imr, Sb);
        stage_BA<NU, NX>(g, a.p, b, j0, BA, fb);
        if constexpr (NY > 0)
            stage_aug<NU, NX, NY>(g, a.p, b, j0, g.x_index_of(c, 0), Xa, sgu, sgx);
        cp_commit();
        if constexpr (NY > 0) {
            // augmented S_0 = S_0 + D_0' Σ_0 C_0 enters ru[0] through S_0 x_init:
            // tscr[m] = σ_0[m] (C_0 x_init)[m]
            if (implicit_rhs && c == 0) {
                for (int m = lane; m < NY; m += 32) {
                    double t = 0;
                    for (int k = 0; k < NX; ++k)
                        t += __ldg(a.p.aC + (size_t)b * (g.N + 1) * NY * NX + m * NX + k) *
                             __ldg(a.p.x_init + (size_t)b * NX + k);
                    tscr[m] = t * __ldg(a.p.asig + (size_t)b * (g.N + 1) * NY + m);
                }
                __syncwarp();
            }
        }
        if (implicit_rhs && c == 0 && lane < NU) {
            double s0 = 0;
            for (int k = 0; k < NX; ++k)
                s0 += __ldg(a.p.S + (size_t)b * g.N * NU * NX + lane * NX + k) *
                      __ldg(a.p.x_init + (size_t)b * NX + k);
            if constexpr (NY > 0)
                for (int m = 0; m < NY; ++m)
                    s0 += __ldg(a.p.aD + (size_t)b * g.N * NY * NU + m * NU + lane) * tscr[m];
            ru0[lane] = s0;
        }
        cp_wait<0>();
        __syncwarp();
    }

    Frag P[S::NT];
#pragma unroll
    for (int t = 0; t < S::NT; ++t)
        P[t] = Frag{0.0, 0.0};

    long long *ph = (a.phase && chain == 0 && lane == 0) ? a.phase : nullptr;
    for (int s = 0; s < n; ++s) {
        if (ph) ph[s * 8 + 0] = clock64();
        const int j = g.stage_of(c, s);
        const bool j0 = j == 0;
        const double *ru0p = (implicit_rhs && j0) ? ru0 : nullptr;
        if (s > 0) {
            cp_wait<1>(); // H_s has landed (the newest group may still fly)
            __syncwarp();
        }
        // ---- init: H_s image (+ S' gather), BA_0 rows at s = 0, rhs row ----
#pragma unroll
        for (int ti = 0; ti < S::TT; ++ti)
#pragma unroll
            for (int tj = 0; tj <= ti && tj < S::CT; ++tj) {
                Frag f{0.0, 0.0};
                if (8 * ti < S::TOP) {
                    f = ld_frag(img + S::T(ti, tj) * kTileElems, lane);
                    if (8 * ti + 7 >= NU && 8 * tj < NU && !j0) { // tile meets the S' block
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int r = 8 * ti + rq, col = 8 * tj + cq + h;
                            const bool isS = r >= NU && r < S::NUX && col < NU;
                            const double v = Sb[isS ? col * NX + (r - NU) : 0];
                            (h ? f.b : f.a) += isS ? v : 0.0;
                        }
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int rb = 8 * ti + rq - S::TOP, col = 8 * tj + cq + h;
                        double v = 0.0;
                        if (s == 0 && rb < NX)
                            v = BA[rb * W::PW + col];
                        if (rb == NX)
                            v = sgn * imr[col] - ((ru0p && col < NU) ? ru0p[col] : 0.0);
                        (h ? f.b : f.a) = v;
                    }
                }
                P[S::T(ti, tj)] = f;
            }
        if constexpr (NY > 0) {
            // Newton-system augmentation of the pivot block, fused into the
            // stage load: += X' diag(σ) X (qpalm.cpp:184-221) on DMMA tiles,
            // A operand = σ-scaled X' tiles, B operand = X' tiles (the
            // reference's D'(ΣD) association). Stage j != 0 < N: one pass
            // over [D_j C_j] with σ_j (R, S', Q blocks). Otherwise the u
            // and x rows come from different stages (j = 0: D_0 and the
            // terminal C_N) and take one pass each, no cross block.
            const bool cross = j < g.N && !j0;
            constexpr int KT = (NY + 7) / 8;
            for (int pass = 0; pass < (cross ? 1 : 2); ++pass) {
                const int c0 = (cross || pass == 0) ? 0 : NU, c1 = (!cross && pass == 0) ? NU : S::NUX;
                const double *sg = (cross || pass == 0) ? sgu : sgx;
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) {
                    const int k0 = 8 * kt + cq;
                    const double s0 = k0 < NY ? sg[k0] : 0.0, s1 = k0 + 1 < NY ? sg[k0 + 1] : 0.0;
                    Frag y[S::CT], ys[S::CT];
#pragma unroll
                    for (int ti = 0; ti < S::CT; ++ti) {
                        const int col = 8 * ti + rq;
                        const bool in = col >= c0 && col < c1;
                        const double v0 = (in && k0 < NY) ? Xa[(k0 < NY ? k0 : 0) * S::NUX + (in ? col : 0)] : 0.0;
                        const double v1 =
                            (in && k0 + 1 < NY) ? Xa[(k0 + 1 < NY ? k0 + 1 : 0) * S::NUX + (in ? col : 0)] : 0.0;
                        y[ti] = Frag{v0, v1};
                        ys[ti] = Frag{v0 * s0, v1 * s1};
                    }
#pragma unroll
                    for (int ti = 0; ti < S::CT; ++ti)
#pragma unroll
                        for (int tj = 0; tj <= ti; ++tj)
                            tile_gemm_nt(P[S::T(ti, tj)], ys[ti], y[tj]);
                }
            }
            if (a.p.gamma_inv != 0.0) { // + gamma^-1 I on R (j < N) and Q (1 <= xi <= N)
                const int xi = g.x_index_of(c, s);
                const double gu = j < g.N ? a.p.gamma_inv : 0.0;
                const double gx = (xi >= 1 && xi <= g.N) ? a.p.gamma_inv : 0.0;
#pragma unroll
                for (int kb = 0; kb < S::CT; ++kb) {
                    const int r = 8 * kb + rq;
                    const double gv = r < NU ? gu : (r < S::NUX ? gx : 0.0);
                    P[S::T(kb, kb)].a += rq == cq ? gv : 0.0;
                    P[S::T(kb, kb)].b += rq == cq + 1 ? gv : 0.0;
                }
            }
        }
        if (TM && s > 0) {
            // += W W' from tensor memory: natural x-tile columns XT0 .. CT-1,
            // one 32-column load per k-slice pair (all TT row tiles)
#pragma unroll
            for (int kt = 0; kt < S::NXT; ++kt) {
                TmFrags<8> t;
                tm_ld<8>(tmw + (uint32_t)(kt * S::TT * 4), t);
                Frag w[S::TT];
#pragma unroll
                for (int i = 0; i < S::TT; ++i)
                    w[i] = tm_frag(t, i);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    // skip k-slices without an x column (u columns are zero in W)
                    constexpr int dummy = 0;
                    (void)dummy;
                    bool has_x = false;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int col = 8 * (S::XT0 + kt) + 2 * q + h;
                        has_x = has_x || (col >= NU && col < S::NUX);
                    }
                    if (!has_x)
                        continue;
#pragma unroll
                    for (int ti = 0; ti < S::TT; ++ti)
#pragma unroll
                        for (int tj = 0; tj <= ti; ++tj)
                            if (!pure(ti, tj))
                                dmma(P[S::T(ti, tj)], h ? w[ti].b : w[ti].a, h ? w[tj].b : w[tj].a);
                }
            }
        }
        if (!TM && s > 0) {
            // += W W' over the compact x-columns: k-slice outer, tiles inner
            // (consecutive DMMAs hit different accumulators)
#pragma unroll
            for (int kt = 0; kt < W::NXC; ++kt) {
                Frag w[S::TT];
#pragma unroll
                for (int i = 0; i < S::TT; ++i)
                    w[i] = ld_frag(Wsm + (i * W::NXC + kt) * kTileElems, lane);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (kt == W::NXF && W::HALF && h == 1)
                        continue; // odd positions of the last tile are empty
#pragma unroll
                    for (int ti = 0; ti < S::TT; ++ti)
#pragma unroll
                        for (int tj = 0; tj <= ti; ++tj)
                            if (!pure(ti, tj)) // ALQ ALQ': cancels (see pure)
                                dmma(P[S::T(ti, tj)], h ? w[ti].b : w[ti].a, h ? w[tj].b : w[tj].a);
                }
            }
        }
        __syncwarp();
        // the H buffers are free: prefetch H_{s+1} (and BA_1 at s = 0)
        if (s + 1 < n) {
            stage_H_plan<NU, NX>(g, a.p, b, g.stage_of(c, s + 1), g.x_index_of(c, s + 1), img, imr, Sb, ctab);
            if constexpr (NY > 0)
                stage_aug<NU, NX, NY>(g, a.p, b, g.stage_of(c, s + 1), g.x_index_of(c, s + 1), Xa, sgu, sgx);
            if (s == 0)
                stage_BA<NU, NX>(g, a.p, b, g.stage_of(c, 1), BA, fb);
        }
        cp_commit();

        if (ph) ph[s * 8 + 1] = clock64();
        // ---- pivot floor: max |diag| of H_s + V V' (kernels.cpp:21-29) ----
        double dmax = 0.0;
#pragma unroll
        for (int kb = 0; kb < S::CT; ++kb) {
            const Frag &d = P[S::T(kb, kb)];
            const double v = (rq & 1) ? d.b : d.a;
            if ((lane & 3) == rq / 2 && 8 * kb + rq < S::NUX)
                dmax = fmax(dmax, fabs(v));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        const double dfloor = 1e-14 * dmax;

        // ---- blocked Cholesky of the pivot columns -------------------------
        // The diagonal tile's pivot steps carry an identity tile (ends as
        // L_kk^{-T}); the sub-diagonal tiles are then solved by two DMMAs
        // each against L_kk^{-1}, and the trailing updates are DMMAs.
        // (Issuing the trailing / W W' DMMAs between the pivot steps instead
        // was measured slower: the DMMA pipe, shared by the SM sub-partition's
        // two resident warps, then throttles the pivot chain's issue.)
#pragma unroll
        for (int kb = 0; kb < S::CT; ++kb) {
            Frag &dg = P[S::T(kb, kb)];
            Frag idt{rq == cq ? 1.0 : 0.0, rq == cq + 1 ? 1.0 : 0.0};
            // The next pivot is computed in every lane from the values
            // shuffled at this step (d = (k+1, k+1) and u = (k+1, k) before
            // this step's update): pv' = d - (u iv)^2, exactly the owner
            // lane's fma -- so the pivot chain is rsqrt -> mul -> fma, with
            // no shuffle on it (bit-identical to shuffling the updated value)
            double pvn = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (8 * kb + k >= S::NUX)
                    break; // padding pivots: the identity tile stays as it is
                constexpr unsigned FULL = 0xffffffffu;
                const int src = k / 2;
                const double vk = (k & 1) ? dg.b : dg.a;
                const double pv = k == 0 ? __shfl_sync(FULL, vk, 4 * k + src) : pvn;
                const double urk = __shfl_sync(FULL, vk, 4 * rq + src);
                const double uc0 = __shfl_sync(FULL, vk, 4 * cq + src);
                const double uc1 = __shfl_sync(FULL, vk, 4 * (cq + 1) + src);
                double dn = 0.0, un = 0.0;
                if (k + 1 < 8 && 8 * kb + k + 1 < S::NUX) {
                    dn = __shfl_sync(FULL, ((k + 1) & 1) ? dg.b : dg.a, 4 * (k + 1) + (k + 1) / 2);
                    un = __shfl_sync(FULL, vk, 4 * (k + 1) + src);
                }
                if (8 * kb + k < S::NUX) { // potrf pivot check (off the critical path)
                    const bool first = !(pv > dfloor && isfinite(pv)) && fail_piv < 0;
                    fail_piv = first ? 8 * kb + k : fail_piv;
                    fail_stage = first ? s : fail_stage;
                }
                const double iv = rsqrt_nr(pv);
                if (k + 1 < 8) {
                    const double l = un * iv;
                    pvn = fma(-l, l, dn);
                }
                const double lc0 = (cq > k) ? uc0 * iv : 0.0;
                const double lc1 = (cq + 1 > k) ? uc1 * iv : 0.0;
                const double lrk = urk * iv;
                const double nv = (rq == k) ? pv * iv : lrk;
                if (k & 1)
                    dg.b = (q2 == src) ? nv : dg.b;
                else
                    dg.a = (q2 == src) ? nv : dg.a;
                dg.a = fma(-lrk, lc0, dg.a);
                dg.b = fma(-lrk, lc1, dg.b);
                const double vq = (k & 1) ? idt.b : idt.a;
                const double xrq = __shfl_sync(FULL, vq, 4 * rq + src) * iv;
                if (k & 1)
                    idt.b = (q2 == src) ? xrq : idt.b;
                else
                    idt.a = (q2 == src) ? xrq : idt.a;
                idt.a -= xrq * lc0;
                idt.b -= xrq * lc1;
            }
            if (cq > rq) dg.a = 0.0;
            if (cq + 1 > rq) dg.b = 0.0;
            // L^{-1} = (L^{-T})' through a shared-memory transpose, then every
            // sub-diagonal tile at once: X <- X L^{-T} = X (L^{-1})'
            st_frag(tscr, lane, idt);
            __syncwarp();
            Frag linv;
            linv.a = tscr[cq * 8 + rq];
            linv.b = tscr[(cq + 1) * 8 + rq];
            __syncwarp();
#pragma unroll
            for (int ti = kb + 1; ti < S::TT; ++ti) {
                Frag x = P[S::T(ti, kb)], r{0.0, 0.0};
                tile_gemm_nt(r, x, linv);
                P[S::T(ti, kb)] = r;
            }
            // trailing update C(ti,tj) -= L(ti,kb) L(tj,kb)': the next diagonal
            // tile first (its factorization can start early), then both k
            // slices over all tiles so consecutive DMMAs are independent
            if (kb + 1 < S::CT) // a pivot diagonal tile (trailing ones: the loop below)
                tile_gemm_nt_sub(P[S::T(kb + 1, kb + 1)], P[S::T(kb + 1, kb)], P[S::T(kb + 1, kb)]);
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int tj = kb + 1; tj < S::TT; ++tj)
#pragma unroll
                    for (int ti = tj; ti < S::TT; ++ti)
                        if (!(ti == kb + 1 && tj == kb + 1 && kb + 1 < S::CT)) {
                            const Frag &li = P[S::T(ti, kb)], &lj = P[S::T(tj, kb)];
                            if (!pure(ti, tj) || 8 * kb + 7 < NU) {
                                dmma(P[S::T(ti, tj)], h ? -li.b : -li.a, h ? lj.b : lj.a);
                            } else if (8 * kb < NU) { // u columns only (LB LB')
                                const double m = (h ? -li.b : -li.a);
                                dmma(P[S::T(ti, tj)], (8 * kb + cq + h < NU) ? m : 0.0, h ? lj.b : lj.a);
                            } // x columns: ALQ ALQ' cancels
                        }
        }

        if (ph) ph[s * 8 + 2] = clock64();
        // ---- store the factor tiles and y_s' ---------------------------------
        {
            double *dst = a.fac + ((size_t)chain * n + s) * S::NPT * kTileElems;
            int o = 0;
#pragma unroll
            for (int ti = 0; ti < S::TT; ++ti)
#pragma unroll
                for (int tj = 0; tj < S::CT; ++tj)
                    if (tj <= ti) {
                        st_frag(dst + o * kTileElems, lane, P[S::T(ti, tj)]);
                        ++o;
                    }
            if (rq == W::RR) {
                double *yv = a.y + ((size_t)chain * n + s) * S::NUX;
#pragma unroll
                for (int tj = 0; tj < S::CT; ++tj) {
                    const int col = 8 * tj + cq;
                    if (col < S::NUX) yv[col] = P[S::T(W::RT, tj)].a;
                    if (col + 1 < S::NUX) yv[col + 1] = P[S::T(W::RT, tj)].b;
                }
            }
        }

        if (s + 1 < n) {
            if (ph) ph[s * 8 + 3] = clock64();
            // ---- W for stage s+1 -------------------------------------------
            if (s == 0) cp_wait<0>();
            else cp_wait<1>();   // BA_{s+1} has landed
            __syncwarp();
            // -wl_new = L_Q' wl + x'  (kkt_solve.cpp:85-90), column-wise
            // reduction over the 8 rows of each tile row group
            double mw[S::NXT][2];
#pragma unroll
            for (int kt = 0; kt < S::NXT; ++kt) {
                const int ct = S::XT0 + kt;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int C = 8 * ct + cq + e;
                    double acc = 0.0;
#pragma unroll
                    for (int ti = ct; ti < S::CT; ++ti) {
                        const int K = 8 * ti + rq;
                        const double lv = e ? P[S::T(ti, ct)].b : P[S::T(ti, ct)].a;
                        if (K >= NU && K < S::NUX && K >= C && C >= NU && C < S::NUX)
                            acc += lv * (sgn * fb[K - NU]);
                    }
                    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 8);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
                    const double xr = e ? P[S::T(W::RT, ct)].b : P[S::T(W::RT, ct)].a;
                    const double xp = __shfl_sync(0xffffffffu, xr, 4 * W::RR + (lane & 3));
                    mw[kt][e] = (C >= NU && C < S::NUX) ? acc + xp : 0.0;
                }
            }
            if (rq == 0) {
                double *wl = a.wl + ((size_t)chain * n + s) * NX;
#pragma unroll
                for (int kt = 0; kt < S::NXT; ++kt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int C = 8 * (S::XT0 + kt) + cq + e;
                        if (C >= NU && C < S::NUX)
                            wl[C - NU] = -mw[kt][e];
                    }
            }
            if constexpr (TM) {
                // W bottom rows in TMEM, natural x tiles: ALQ (x columns of the
                // coupling rows), the rhs row -wl (mw), zero u / padding columns
                // and rows past the rhs row
#pragma unroll
                for (int ti = S::CT; ti < S::TT; ++ti)
#pragma unroll
                    for (int kt = 0; kt < S::NXT; ++kt) {
                        const int ct = S::XT0 + kt, r = 8 * ti + rq;
                        Frag f = P[S::T(ti, ct)];
                        const int C0 = 8 * ct + cq;
                        f.a = (C0 >= NU && C0 < S::NUX) ? f.a : 0.0;
                        f.b = (C0 + 1 >= NU && C0 + 1 < S::NUX) ? f.b : 0.0;
                        if (r == S::RHS)
                            f = Frag{mw[kt][0], mw[kt][1]};
                        else if (r > S::RHS)
                            f = Frag{0.0, 0.0};
                        tm_st4(tmw + (uint32_t)((kt * S::TT + ti) * 4), f);
                    }
            }
            // W bottom rows: ALQ (x columns of the coupling rows) and the rhs
            // row -wl, scattered to the compact column positions; L_Q -> LQ
            {
            const int lv = lane_v(), rq = lv >> 2, cq = 2 * (lv & 3);
#pragma unroll
            for (int ti = S::CT; ti < (TM ? S::CT : S::TT); ++ti)
#pragma unroll
                for (int kt = 0; kt < S::NXT; ++kt) {
                    const int ct = S::XT0 + kt, r = 8 * ti + rq;
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int C = 8 * ct + cq + e;
                        if (C >= NU && C < S::NUX && r <= S::RHS) {
                            const double v = (r == S::RHS) ? mw[kt][e]
                                                           : (e ? P[S::T(ti, ct)].b : P[S::T(ti, ct)].a);
                            const int p = W::pos(C - NU);
                            Wsm[(ti * W::NXC + p / 8) * kTileElems + (r % 8) * 8 + p % 8] = v;
                        }
                    }
                }
#pragma unroll
            for (int u = 0; u < S::NXT; ++u)
#pragma unroll
                for (int v = 0; v <= u; ++v) {
                    const Frag w = P[S::T(S::XT0 + u, S::XT0 + v)];
                    const int K = 8 * (S::XT0 + u) + rq;
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int C = 8 * (S::XT0 + v) + cq + e;
                        if (K >= NU && K < S::NUX && C >= NU && C <= K)
                            LQ[(K - NU) * NX + (C - NU)] = e ? w.b : w.a;
                    }
                }
            }
            __syncwarp();
            if (ph) ph[s * 8 + 4] = clock64();
            // V = BA_{s+1}' L_Q : rows 0..nux-1 of W (DMMA over x rows K)
            if constexpr (TM) {
                Frag vacc[S::CT * S::NXT];
#pragma unroll
                for (int v = 0; v < S::CT * S::NXT; ++v)
                    vacc[v] = Frag{0.0, 0.0};
#pragma unroll
                for (int ks = 0; ks < W::KQ; ++ks) {
                    const int K = 4 * ks + (lane & 3);
                    double av[S::CT], bv[S::NXT];
#pragma unroll
                    for (int ti = 0; ti < S::CT; ++ti)
                        av[ti] = BA[K * W::PW + 8 * ti + rq];
#pragma unroll
                    for (int kt = 0; kt < S::NXT; ++kt) { // natural x column of this lane's B column
                        const int xc = 8 * (S::XT0 + kt) + rq - NU;
                        bv[kt] = (xc >= 0 && xc < NX) ? LQ[K * NX + (xc >= 0 && xc < NX ? xc : 0)] : 0.0;
                    }
#pragma unroll
                    for (int ti = 0; ti < S::CT; ++ti)
#pragma unroll
                        for (int kt = 0; kt < S::NXT; ++kt)
                            if (4 * ks + 3 >= 8 * (S::XT0 + kt) - NU) // L_Q upper part is zero
                                dmma(vacc[ti * S::NXT + kt], av[ti], bv[kt]);
                }
#pragma unroll
                for (int ti = 0; ti < S::CT; ++ti)
#pragma unroll
                    for (int kt = 0; kt < S::NXT; ++kt)
                        tm_st4(tmw + (uint32_t)((kt * S::TT + ti) * 4), vacc[ti * S::NXT + kt]);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            } else {
                Frag vacc[S::CT * W::NXC];
#pragma unroll
                for (int v = 0; v < S::CT * W::NXC; ++v)
                    vacc[v] = Frag{0.0, 0.0};
#pragma unroll
                for (int ks = 0; ks < W::KQ; ++ks) {
                    const int K = 4 * ks + (lane & 3);
                    double av[S::CT], bv[W::NXC];
#pragma unroll
                    for (int ti = 0; ti < S::CT; ++ti)
                        av[ti] = BA[K * W::PW + 8 * ti + rq];
#pragma unroll
                    for (int kt = 0; kt < W::NXC; ++kt) { // x-column of this lane's B column
                        const int vc = W::col_of(8 * kt + rq);
                        bv[kt] = vc >= 0 ? LQ[K * NX + (vc >= 0 ? vc : 0)] : 0.0; // rows >= nx: 0
                    }
#pragma unroll
                    for (int ti = 0; ti < S::CT; ++ti)
#pragma unroll
                        for (int kt = 0; kt < W::NXC; ++kt)
                            if (4 * ks + 3 >= 8 * kt) // L_Q upper part is zero
                                dmma(vacc[ti * W::NXC + kt], av[ti], bv[kt]);
                }
#pragma unroll
                for (int ti = 0; ti < S::CT; ++ti)
#pragma unroll
                    for (int kt = 0; kt < W::NXC; ++kt)
                        st_frag(Wsm + (ti * W::NXC + kt) * kTileElems, lane, vacc[ti * W::NXC + kt]);
            }
            __syncwarp();
            if (s + 2 < n) {
                if constexpr (W::PLAN_BA)
                    stage_BA_plan<NU, NX>(g, a.p, b, g.stage_of(c, s + 2), BA, fb, ctab);
                else
                    stage_BA<NU, NX>(g, a.p, b, g.stage_of(c, s + 2), BA, fb);
            }
            cp_commit();
        }
    }

    if (ph) ph[n * 8] = clock64();
    // -= LA LA' on the pure coupling tiles: the x columns of the last
    // stage's coupling rows (the terms the stage loop skipped)
#pragma unroll
    for (int kb = 0; kb < S::CT; ++kb)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int tj = S::CT; tj < RT_; ++tj)
#pragma unroll
                for (int ti = tj; ti < RT_; ++ti)
                    if (8 * kb + 7 >= NU) {
                        const Frag &li = P[S::T(ti, kb)], &lj = P[S::T(tj, kb)];
                        const double m = (h ? -li.b : -li.a);
                        dmma(P[S::T(ti, tj)], (8 * kb + cq + h >= NU) ? m : 0.0, h ? lj.b : lj.a);
                    }
    // trailing tiles (coupling x coupling = -Mfwd, rhs x coupling = -fwd)
#pragma unroll
    for (int u = 0; u < S::BT; ++u)
#pragma unroll
        for (int v = 0; v <= u; ++v)
            st_frag(a.trail + ((size_t)chain * g.NTT + S::T(u, v)) * kTileElems, lane,
                    P[S::T(S::CT + u, S::CT + v)]);
    unsigned long long my_fail =
        fail_piv >= 0 ? fail_key(kKindRiccati, c, fail_stage, fail_piv) : ~0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        my_fail = min(my_fail, __shfl_xor_sync(0xffffffffu, my_fail, o));
    if (lane == 0 && my_fail != ~0ull)
        atomicMin(a.fail + b, my_fail);
}

// ---- dispatch ----------------------------------------------------------------
namespace {
template <int NU, int NX, int WPB, int NY, bool TM = false>
bool launch_w(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    if (g.nu != NU || g.nx != NX)
        return false;
    if ((NY > 0) != (ra.p.aD != nullptr) || (NY > 0 && ra.p.ny != NY))
        return false;
    using W = WS<NU, NX, NY, TM>;
    const size_t smem = (size_t)WPB * W::SMEM * sizeof(double);
    static DeviceOnce once;
    once_per_device(once, [&] { return cudaFuncSetAttribute(riccati_warp_kernel<NU, NX, WPB, NY, TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    const int chains = ra.grid_chains();
    riccati_warp_kernel<NU, NX, WPB, NY, TM><<<(chains + WPB - 1) / WPB, 32 * WPB, smem, st>>>(ra);
    return true;
}
} // namespace

bool riccati_warp_fuses_aug(const Geo &g, int ny, const LaunchOpts &o) {
    return o.fused_aug && (o.panel == 0 || o.panel == 1) && g.nu == 8 && g.nx == 16 && ny == 24;
}

bool launch_riccati_warp(const Geo &g, cudaStream_t st, const RiccatiArgs &ra, const LaunchOpts &o) {
    if (ra.p.aD) // fused Newton-system augmentation (config 4 stage shape)
        return launch_w<8, 16, 1, 24>(g, st, ra);
    // W in tensor memory (12 chains per SM at config 1): opt-in
    // (CYQ_PANEL_WARP_TMEM) -- measured 1.52 vs 1.41 ms at config 1 (the
    // natural x-tile layout costs a 6th W W' k-slice and 168 registers
    // spill), see DESIGN.md §3.4
    if (o.panel == 5)
        return launch_w<10, 20, 4, 0, true>(g, st, ra);
    return launch_w<10, 20, 1, 0>(g, st, ra) || launch_w<8, 16, 1, 0>(g, st, ra) ||
           launch_w<4, 12, 1, 0>(g, st, ra) || launch_w<5, 10, 1, 0>(g, st, ra);
}

} // namespace cyqb
