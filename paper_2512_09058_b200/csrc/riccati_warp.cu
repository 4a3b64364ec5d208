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
// shuffles). Shared memory holds only what must be re-read in another
// layout: W = [V; ALQ; -wl] (operands of the next stage's W W' update),
// L_Q (the transposed B operand of V = BA' L_Q) and the cp.async staging
// buffers for the next stage's R, S, Q, B, A, r, q, f (issued one stage
// ahead; full-sector 16-byte copies when aligned).
#include "kkt_common.cuh"
#include "kernels.h"

#include "riccati_common.cuh"

#include <cstdlib>

namespace cyqb {

using namespace cyqb::ric;

template <int NU, int NX, int WPB, bool DIRECT, bool INV>
__global__ void __launch_bounds__(32 * WPB, DIRECT ? 12 / WPB : 1) riccati_warp_kernel(RiccatiArgs a) {
    using S = Shp<NU, NX>;
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int chain = blockIdx.x * WPB + wib;
    if (chain >= g.batch * g.P)
        return;
    const int b = chain / g.P, c = chain % g.P, n = g.n;
    const int rq = lane >> 2, cq = 2 * (lane & 3);

    constexpr int SMEM_DBL = DIRECT ? S::SMEM_DIRECT : S::SMEM_STAGED;
    double *base = sm + (size_t)wib * SMEM_DBL;
    double *tscr = base + SMEM_DBL - kTileElems; // 8x8 transpose scratch
    double *Wsm = base;                                   // TT x NXT tiles
    double *Lsm = Wsm + S::TT * S::NXT * kTileElems;      // NLQ tiles (x-x block of L)
    Stage<NU, NX> st;
    st.R = Lsm + S::NLQ * kTileElems;
    st.S = st.R + NU * NU;
    st.Q = st.S + NU * NX;
    st.r = st.Q + NX * NX;
    st.q = st.r + NU;
    st.B = st.R + S::HBp;
    st.A = st.B + NX * NU;
    st.f = st.A + NX * NX;
    double *ru0 = DIRECT ? st.R : st.B + S::BBp; // NU: S_0 x_init
    const bool implicit_rhs = (a.p.ru == nullptr);
    const double sgn = implicit_rhs ? -1.0 : 1.0;
    int fail_piv = -1, fail_stage = 0;

    // prologue: H_0, BA_0 and the x_init term of ru[0]
    {
        const int j0 = g.stage_of(c, 0);
        if (DIRECT) {
            point_H<NU, NX>(g, a.p, a.consts, b, j0, g.x_index_of(c, 0), st, lane);
            point_BA<NU, NX>(g, a.p, a.consts, b, j0, st, lane);
        } else {
            load_H<NU, NX>(g, a.p, b, j0, g.x_index_of(c, 0), st, lane);
            load_BA<NU, NX>(g, a.p, b, j0, st, lane);
        }
        cp_commit();
        if (implicit_rhs && c == 0 && lane < NU) {
            double s0 = 0;
            for (int k = 0; k < NX; ++k)
                s0 += __ldg(a.p.S + (size_t)b * g.N * NU * NX + lane * NX + k) *
                      __ldg(a.p.x_init + (size_t)b * NX + k);
            ru0[lane] = s0;
        }
        cp_wait<0>();
        __syncwarp();
    }

    Frag P[S::NT];
#pragma unroll
    for (int t = 0; t < S::NT; ++t)
        P[t] = Frag{0.0, 0.0};

    // optional phase timing (CYQ_PHASE_PROF): chain 0's lane 0 records
    // clock64 at the phase boundaries of every stage
    long long *ph = (a.phase && chain == 0 && lane == 0) ? a.phase : nullptr;
    for (int s = 0; s < n; ++s) {
        if (ph) ph[s * 8 + 0] = clock64();
        const int j = g.stage_of(c, s);
        const double *ru0p = (implicit_rhs && j == 0) ? ru0 : nullptr;
        if (s > 0) {
            cp_wait<1>(); // H_s has landed (the newest group may still fly)
            __syncwarp();
        }
        // ---- init pivot tiles, += W W' ------------------------------------
#pragma unroll
        for (int ti = 0; ti < S::TT; ++ti) {
#pragma unroll
            for (int tj = 0; tj <= ti && tj < S::CT; ++tj) {
                Frag &f = P[S::T(ti, tj)];
                const int r = 8 * ti + rq, col = 8 * tj + cq;
                f.a = pinit<NU, NX>(st, s == 0, j == 0, sgn, ru0p, ti, r, col);
                f.b = pinit<NU, NX>(st, s == 0, j == 0, sgn, ru0p, ti, r, col + 1);
            }
        }
        if (s > 0) {
            // k-slice outer, tiles inner: consecutive DMMAs hit different
            // accumulators (no dependent-DMMA stalls); each W fragment is
            // read from shared memory once per slice
#pragma unroll
            for (int kt = 0; kt < S::NXT; ++kt) {
                Frag w[S::TT];
#pragma unroll
                for (int i = 0; i < S::TT; ++i)
                    w[i] = ld_frag(Wsm + (i * S::NXT + kt) * kTileElems, lane);
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int ti = 0; ti < S::TT; ++ti)
#pragma unroll
                        for (int tj = 0; tj <= ti; ++tj)
                            dmma(P[S::T(ti, tj)], h ? w[ti].b : w[ti].a, h ? w[tj].b : w[tj].a);
            }
        }
        __syncwarp();
        // the H buffer is free: prefetch H_{s+1} (and BA_1 at s = 0)
        if (s + 1 < n) {
            if (DIRECT) {
                point_H<NU, NX>(g, a.p, a.consts, b, g.stage_of(c, s + 1), g.x_index_of(c, s + 1),
                                st, lane);
                if (s == 0)
                    point_BA<NU, NX>(g, a.p, a.consts, b, g.stage_of(c, 1), st, lane);
            } else {
                load_H<NU, NX>(g, a.p, b, g.stage_of(c, s + 1), g.x_index_of(c, s + 1), st, lane);
                if (s == 0)
                    load_BA<NU, NX>(g, a.p, b, g.stage_of(c, 1), st, lane);
            }
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
        // Step k of the diagonal tile and step k of every sub-diagonal tile of
        // block column kb are interleaved, so the independent sub-diagonal
        // work fills the latency of the pivot chain (broadcast, rsqrt) and
        // no per-column arrays stay live. Updates are unconditional FMAs with
        // zeroed multipliers instead of predicated branches.
        const int q2 = lane & 3; // this lane holds columns 2*q2, 2*q2 + 1
#pragma unroll
        for (int kb = 0; kb < S::CT; ++kb) {
            Frag &dg = P[S::T(kb, kb)];
            Frag idt{rq == cq ? 1.0 : 0.0, rq == cq + 1 ? 1.0 : 0.0};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                constexpr unsigned FULL = 0xffffffffu;
                const int src = k / 2;
                const double vk = (k & 1) ? dg.b : dg.a;
                double pv = __shfl_sync(FULL, vk, 4 * k + src);
                const double urk = __shfl_sync(FULL, vk, 4 * rq + src);
                const double uc0 = __shfl_sync(FULL, vk, 4 * cq + src);
                const double uc1 = __shfl_sync(FULL, vk, 4 * (cq + 1) + src);
                if (8 * kb + k < S::NUX) { // potrf pivot check (off the critical path)
                    const bool first = !(pv > dfloor && isfinite(pv)) && fail_piv < 0;
                    fail_piv = first ? 8 * kb + k : fail_piv;
                    fail_stage = first ? s : fail_stage;
                }
                const double iv = rsqrt_nr(pv);
                const double lc0 = (cq > k) ? uc0 * iv : 0.0;
                const double lc1 = (cq + 1 > k) ? uc1 * iv : 0.0;
                const double lrk = urk * iv;
                const double nv = (rq == k) ? pv * iv : lrk;
                if (k & 1)
                    dg.b = (q2 == src) ? nv : dg.b;
                else
                    dg.a = (q2 == src) ? nv : dg.a;
                dg.a -= lrk * lc0;
                dg.b -= lrk * lc1;
                if (!INV) {
#pragma unroll
                    for (int ti = kb + 1; ti < S::TT; ++ti) {
                        Frag &x = P[S::T(ti, kb)];
                        const double vq = (k & 1) ? x.b : x.a;
                        const double xrq = __shfl_sync(FULL, vq, 4 * rq + src) * iv;
                        if (k & 1)
                            x.b = (q2 == src) ? xrq : x.b;
                        else
                            x.a = (q2 == src) ? xrq : x.a;
                        x.a -= xrq * lc0;
                        x.b -= xrq * lc1;
                    }
                } else { // same step on one identity tile: ends as L_kk^{-T}
                    const double vq = (k & 1) ? idt.b : idt.a;
                    const double xrq = __shfl_sync(FULL, vq, 4 * rq + src) * iv;
                    if (k & 1)
                        idt.b = (q2 == src) ? xrq : idt.b;
                    else
                        idt.a = (q2 == src) ? xrq : idt.a;
                    idt.a -= xrq * lc0;
                    idt.b -= xrq * lc1;
                }
            }
            if (cq > rq) dg.a = 0.0;
            if (cq + 1 > rq) dg.b = 0.0;
            if (INV) {
                // L^{-1} = (L^{-T})' through a shared-memory transpose, then
                // every sub-diagonal tile at once: X <- X L^{-T} = X (L^{-1})'
                // (two DMMAs per tile instead of eight dependent pivot steps)
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
            }
            // trailing update C(ti,tj) -= L(ti,kb) L(tj,kb)': the next diagonal
            // tile first (its factorization can start early), then both k
            // slices over all tiles so consecutive DMMAs are independent
            if (kb + 1 < S::TT)
                tile_gemm_nt_sub(P[S::T(kb + 1, kb + 1)], P[S::T(kb + 1, kb)], P[S::T(kb + 1, kb)]);
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int tj = kb + 1; tj < S::TT; ++tj)
#pragma unroll
                    for (int ti = tj; ti < S::TT; ++ti)
                        if (!(ti == kb + 1 && tj == kb + 1)) {
                            const Frag &li = P[S::T(ti, kb)], &lj = P[S::T(tj, kb)];
                            dmma(P[S::T(ti, tj)], h ? -li.b : -li.a, h ? lj.b : lj.a);
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
            constexpr int RT = S::RHS / 8, RR = S::RHS % 8;
            if (rq == RR) {
                double *yv = a.y + ((size_t)chain * n + s) * S::NUX;
#pragma unroll
                for (int tj = 0; tj < S::CT; ++tj) {
                    const int col = 8 * tj + cq;
                    if (col < S::NUX) yv[col] = P[S::T(RT, tj)].a;
                    if (col + 1 < S::NUX) yv[col + 1] = P[S::T(RT, tj)].b;
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
                            acc += lv * (sgn * st.f[K - NU]);
                    }
                    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 8);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
                    constexpr int RT = S::RHS / 8, RR = S::RHS % 8;
                    const double xr = e ? P[S::T(RT, ct)].b : P[S::T(RT, ct)].a;
                    const double xp = __shfl_sync(0xffffffffu, xr, 4 * RR + (lane & 3));
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
            // W bottom rows: ALQ (x columns of the coupling rows), rhs row -wl
#pragma unroll
            for (int ti = S::CT; ti < S::TT; ++ti)
#pragma unroll
                for (int kt = 0; kt < S::NXT; ++kt) {
                    const int ct = S::XT0 + kt;
                    Frag w = P[S::T(ti, ct)];
                    const int r = 8 * ti + rq, c0 = 8 * ct + cq;
                    if (r == S::RHS) {
                        w.a = mw[kt][0];
                        w.b = mw[kt][1];
                    } else if (r > S::RHS) {
                        w.a = w.b = 0.0;
                    }
                    if (c0 < NU || c0 >= S::NUX) w.a = 0.0;
                    if (c0 + 1 < NU || c0 + 1 >= S::NUX) w.b = 0.0;
                    st_frag(Wsm + (ti * S::NXT + kt) * kTileElems, lane, w);
                }
            // L_Q tiles (x rows/cols, masked) -> Lsm for the transposed access
#pragma unroll
            for (int u = 0; u < S::NXT; ++u)
#pragma unroll
                for (int v = 0; v <= u; ++v) {
                    Frag w = P[S::T(S::XT0 + u, S::XT0 + v)];
                    const int K = 8 * (S::XT0 + u) + rq, C0 = 8 * (S::XT0 + v) + cq;
                    const bool rin = K >= NU && K < S::NUX;
                    if (!(rin && C0 >= NU && C0 < S::NUX && C0 <= K)) w.a = 0.0;
                    if (!(rin && C0 + 1 >= NU && C0 + 1 < S::NUX && C0 + 1 <= K)) w.b = 0.0;
                    st_frag(Lsm + S::T(u, v) * kTileElems, lane, w);
                }
            __syncwarp();
            if (ph) ph[s * 8 + 4] = clock64();
            // V = BA_{s+1}' L_Q : rows 0..nux-1 of W (DMMA), k-slice outer
            {
                Frag vacc[S::CT * S::NXT];
#pragma unroll
                for (int v = 0; v < S::CT * S::NXT; ++v)
                    vacc[v] = Frag{0.0, 0.0};
#pragma unroll
                for (int ks = 2 * S::XT0; ks < 2 * (S::XT1 + 1); ++ks) {
                    const int K = 4 * ks + (lane & 3);
                    const bool kin = K >= NU && K < S::NUX;
                    double av[S::CT], bv[S::NXT];
#pragma unroll
                    for (int ti = 0; ti < S::CT; ++ti) {
                        const int r = 8 * ti + rq;
                        av[ti] = (kin && r < S::NUX)
                                     ? (r < NU ? st.B[(K - NU) * NU + r] : st.A[(K - NU) * NX + (r - NU)])
                                     : 0.0;
                    }
#pragma unroll
                    for (int kt = 0; kt < S::NXT; ++kt) {
                        // B[kk][n] = L[K][8ct + n]: tile (K/8, ct) of Lsm
                        const int u = ks / 2 - S::XT0;
                        bv[kt] = (u >= kt) ? Lsm[S::T(u >= kt ? u : kt, kt) * kTileElems +
                                                 (4 * (ks & 1) + (lane & 3)) * 8 + (lane >> 2)]
                                           : 0.0;
                    }
#pragma unroll
                    for (int ti = 0; ti < S::CT; ++ti)
#pragma unroll
                        for (int kt = 0; kt < S::NXT; ++kt)
                            if (4 * ks + 3 >= 8 * (S::XT0 + kt)) // L_Q upper part is zero
                                dmma(vacc[ti * S::NXT + kt], av[ti], bv[kt]);
                }
#pragma unroll
                for (int v = 0; v < S::CT * S::NXT; ++v)
                    st_frag(Wsm + v * kTileElems, lane, vacc[v]);
            }
            __syncwarp();
            if (s + 2 < n) {
                if (DIRECT)
                    point_BA<NU, NX>(g, a.p, a.consts, b, g.stage_of(c, s + 2), st, lane);
                else
                    load_BA<NU, NX>(g, a.p, b, g.stage_of(c, s + 2), st, lane);
            }
            cp_commit();
        }
    }

    if (ph) ph[n * 8] = clock64();
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
template <int NU, int NX, int WPB, bool DIRECT, bool INV>
bool launch_wd(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    using S = Shp<NU, NX>;
    const size_t smem = (size_t)WPB * (DIRECT ? S::SMEM_DIRECT : S::SMEM_STAGED) * sizeof(double);
    static_assert(S::SMEM_STAGED % 2 == 0 && S::SMEM_DIRECT % 2 == 0, "16-byte aligned warps");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(riccati_warp_kernel<NU, NX, WPB, DIRECT, INV>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const int chains = g.batch * g.P;
    riccati_warp_kernel<NU, NX, WPB, DIRECT, INV><<<(chains + WPB - 1) / WPB, 32 * WPB, smem, st>>>(ra);
    return true;
}
template <int NU, int NX, int WPB> bool launch_w(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    if (g.nu != NU || g.nx != NX)
        return false;
    static const bool direct = getenv("CYQ_RICCATI_DIRECT") != nullptr;
    static const bool noinv = getenv("CYQ_RICCATI_NOINV") != nullptr;
    if (direct)
        return launch_wd<NU, NX, WPB, true, true>(g, st, ra);
    return noinv ? launch_wd<NU, NX, WPB, false, false>(g, st, ra)
                 : launch_wd<NU, NX, WPB, false, true>(g, st, ra);
}
} // namespace

bool launch_riccati_warp(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    if (getenv("CYQ_NO_WARP_KERNEL"))
        return false;
    static const int wpb = getenv("CYQ_RICCATI_WPB") ? atoi(getenv("CYQ_RICCATI_WPB")) : 1;
    if (wpb == 2)
        return launch_w<10, 20, 2>(g, st, ra) || launch_w<8, 16, 2>(g, st, ra) ||
               launch_w<4, 12, 2>(g, st, ra) || launch_w<5, 10, 2>(g, st, ra);
    return launch_w<10, 20, 1>(g, st, ra) || launch_w<8, 16, 1>(g, st, ra) ||
           launch_w<4, 12, 1>(g, st, ra) || launch_w<5, 10, 1>(g, st, ra);
}

} // namespace cyqb
