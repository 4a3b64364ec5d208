// Two-warp-per-chain stage-panel Riccati kernel, compile-time (nu, nx):
// the fast path for stage blocks up to nux = 32 (BASELINE configs 0, 1, 2,
// 4). Same algorithm and outputs as riccati_warp.cu / riccati.cu:
//   kkt_factor.cpp:125-158  modified Riccati recursion (LH, LB, Acl, LA)
//   kkt_factor.cpp:163-185  Mfwd = sum LB LB' + LA LA' (trailing block)
//   kkt_solve.cpp:72-134    forward substitution + coupling rows (rhs row)
//
// The panel's 8x8 tiles are split between the two warps of the CTA (tile t
// belongs to warp t % 2) and stay in the owner's registers for the whole
// stage (trailing coupling tiles: for the whole chain). Each pivot block
// column is published to shared memory once, after which the other warp
// reads it as DMMA operands; both warps factor the diagonal tile
// redundantly so the only cross-warp hand-offs are two 64-thread named
// barriers per block column. Half the registers per warp of the one-warp
// kernel -> twice the resident chains per SM, and each chain's DMMA work is
// shared by two SM sub-partitions.
#include "riccati_common.cuh"
#include "tiles.cuh"

#include <type_traits>

namespace cyqb {

using namespace cyqb::ric;

namespace {

template <int NU, int NX> struct C2 {
    using S = Shp<NU, NX>;
    // index of pivot tile (i, j < CT) in the published / stored layout
    __host__ __device__ static constexpr int PI(int i, int j) {
        return i < S::CT ? S::T(i, j) : S::CT * (S::CT + 1) / 2 + (i - S::CT) * S::CT + j;
    }
    static constexpr int OFF_V = S::NPT * kTileElems;
    static constexpr int OFF_H = OFF_V + S::CT * S::NXT * kTileElems;
    static constexpr int OFF_B = OFF_H + S::HBp;
    static constexpr int OFF_MW = OFF_B + S::BBp;
    static constexpr int OFF_RU0 = OFF_MW + ((NX + 1) & ~1);
    static constexpr int OFF_RED = OFF_RU0 + ((NU + 1) & ~1);
    static constexpr int SMEM = OFF_RED + 4;
};

__device__ __forceinline__ void bar2() { asm volatile("bar.sync 1, 64;\n" ::: "memory"); }

// compile-time loop: f(integral_constant<int, i>) for i in [B, E)
template <int B, int E, class F> __device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

template <int W, int NU, int NX>
__device__ __forceinline__ void cta2_body(const RiccatiArgs &a, double *sm, int chain) {
    using S = Shp<NU, NX>;
    using L = C2<NU, NX>;
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31, tid = threadIdx.x;
    const int b = chain / g.P, c = chain % g.P, n = g.n;
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    constexpr int RT = S::RHS / 8, RR = S::RHS % 8;

    double *Ps = sm;
    double *Vs = sm + L::OFF_V;
    Stage<NU, NX> st;
    st.R = sm + L::OFF_H;
    st.S = st.R + NU * NU;
    st.Q = st.S + NU * NX;
    st.r = st.Q + NX * NX;
    st.q = st.r + NU;
    st.B = sm + L::OFF_B;
    st.A = st.B + NX * NU;
    st.f = st.A + NX * NX;
    double *mwl = sm + L::OFF_MW, *ru0 = sm + L::OFF_RU0, *red = sm + L::OFF_RED;
    const bool implicit_rhs = (a.p.ru == nullptr);
    const double sgn = implicit_rhs ? -1.0 : 1.0;
    int fail_piv = -1, fail_stage = 0;

    {
        const int j0 = g.stage_of(c, 0);
        load_H<NU, NX, 64>(g, a.p, b, j0, g.x_index_of(c, 0), st, tid);
        load_BA<NU, NX, 64>(g, a.p, b, j0, st, tid);
        cp_commit();
        if (implicit_rhs && c == 0 && tid < NU) {
            double s0 = 0;
            for (int k = 0; k < NX; ++k)
                s0 += __ldg(a.p.S + (size_t)b * g.N * NU * NX + tid * NX + k) *
                      __ldg(a.p.x_init + (size_t)b * NX + k);
            ru0[tid] = s0;
        }
        cp_wait<0>();
        bar2();
    }

    Frag P[S::NT];
#pragma unroll
    for (int t = 0; t < S::NT; ++t)
        P[t] = Frag{0.0, 0.0};

    for (int s = 0; s < n; ++s) {
        const int j = g.stage_of(c, s);
        const double *ru0p = (implicit_rhs && j == 0) ? ru0 : nullptr;
        if (s > 0) {
            cp_wait<1>();
            bar2();
        }
        // ---- init own pivot tiles, += W W' -------------------------------
#pragma unroll
        for (int ti = 0; ti < S::TT; ++ti) {
#pragma unroll
            for (int tj = 0; tj <= ti; ++tj) {
                if (S::T(ti, tj) % 2 != W)
                    continue;
                Frag &f = P[S::T(ti, tj)];
                if (tj < S::CT) {
                    const int r = 8 * ti + rq, col = 8 * tj + cq;
                    f.a = pinit<NU, NX>(st, s == 0, j == 0, sgn, ru0p, ti, r, col);
                    f.b = pinit<NU, NX>(st, s == 0, j == 0, sgn, ru0p, ti, r, col + 1);
                }
                if (s > 0) {
#pragma unroll
                    for (int kt = 0; kt < S::NXT; ++kt) {
                        const int ct = S::XT0 + kt, c0 = 8 * ct + cq;
                        const bool m0 = c0 >= NU && c0 < S::NUX, m1 = c0 + 1 >= NU && c0 + 1 < S::NUX;
                        Frag w[2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int tt = h ? tj : ti;
                            if (tt < S::CT) {
                                w[h] = ld_frag(Vs + (tt * S::NXT + kt) * kTileElems, lane);
                            } else {
                                w[h] = ld_frag(Ps + L::PI(tt, ct) * kTileElems, lane);
                                const int r = 8 * tt + rq;
                                if (r == S::RHS) {
                                    w[h].a = m0 ? mwl[c0 - NU] : 0.0;
                                    w[h].b = m1 ? mwl[c0 + 1 - NU] : 0.0;
                                } else if (r > S::RHS) {
                                    w[h].a = w[h].b = 0.0;
                                }
                                if (!m0) w[h].a = 0.0;
                                if (!m1) w[h].b = 0.0;
                            }
                        }
                        tile_gemm_nt(f, w[0], w[1]);
                    }
                }
            }
        }
        // pivot floor (kernels.cpp:21-29): owners of top diagonal tiles
        {
            double m = 0.0;
#pragma unroll
            for (int kb = 0; kb < S::CT; ++kb) {
                if (S::T(kb, kb) % 2 != W)
                    continue;
                const Frag &d = P[S::T(kb, kb)];
                const double v = (rq & 1) ? d.b : d.a;
                if ((lane & 3) == rq / 2 && 8 * kb + rq < S::NUX)
                    m = fmax(m, fabs(v));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0)
                red[W] = m;
        }
        bar2(); // all W / staging reads done (Ps is about to be overwritten)
        if (S::T(0, 0) % 2 == W)
            st_frag(Ps + L::PI(0, 0) * kTileElems, lane, P[S::T(0, 0)]);
        if (s + 1 < n) {
            load_H<NU, NX, 64>(g, a.p, b, g.stage_of(c, s + 1), g.x_index_of(c, s + 1), st, tid);
            if (s == 0)
                load_BA<NU, NX, 64>(g, a.p, b, g.stage_of(c, 1), st, tid);
        }
        cp_commit();
        bar2(); // diag tile (0,0) published, red[] complete
        const double dfloor = 1e-14 * fmax(red[0], red[1]);

        // ---- blocked Cholesky of the pivot columns -----------------------
        const int q2 = lane & 3;
        static_for<0, S::CT>([&](auto kbc) {
            constexpr int kb = decltype(kbc)::value;
            constexpr unsigned FULL = 0xffffffffu;
            const bool own_d = S::T(kb, kb) % 2 == W;
            Frag dg = own_d ? P[S::T(kb, kb)] : ld_frag(Ps + L::PI(kb, kb) * kTileElems, lane);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int src = k / 2;
                const double vk = (k & 1) ? dg.b : dg.a;
                double pv = __shfl_sync(FULL, vk, 4 * k + src);
                const double urk = __shfl_sync(FULL, vk, 4 * rq + src);
                const double uc0 = __shfl_sync(FULL, vk, 4 * cq + src);
                const double uc1 = __shfl_sync(FULL, vk, 4 * (cq + 1) + src);
                if (8 * kb + k < S::NUX) {
                    const bool bad = !(pv > dfloor && isfinite(pv));
                    if (bad && fail_piv < 0) {
                        fail_piv = 8 * kb + k;
                        fail_stage = s;
                    }
                    pv = bad ? 1.0 : pv;
                }
                const double iv = rsqrt(pv);
                const double lc0 = (cq > k) ? uc0 * iv : 0.0;
                const double lc1 = (cq + 1 > k) ? uc1 * iv : 0.0;
                const double lrk = urk * iv;
                if (q2 == src) {
                    double &e = (k & 1) ? dg.b : dg.a;
                    e = (rq == k) ? pv * iv : lrk;
                }
                dg.a -= lrk * lc0;
                dg.b -= lrk * lc1;
#pragma unroll
                for (int ti = kb + 1; ti < S::TT; ++ti) {
                    if (S::T(ti, kb) % 2 != W)
                        continue;
                    Frag &x = P[S::T(ti, kb)];
                    const double vq = (k & 1) ? x.b : x.a;
                    const double xrq = __shfl_sync(FULL, vq, 4 * rq + src) * iv;
                    if (q2 == src) {
                        if (k & 1) x.b = xrq;
                        else x.a = xrq;
                    }
                    x.a -= xrq * lc0;
                    x.b -= xrq * lc1;
                }
            }
            if (cq > rq) dg.a = 0.0;
            if (cq + 1 > rq) dg.b = 0.0;
            if (own_d) {
                P[S::T(kb, kb)] = dg;
                st_frag(Ps + L::PI(kb, kb) * kTileElems, lane, dg);
            }
#pragma unroll
            for (int ti = kb + 1; ti < S::TT; ++ti)
                if (S::T(ti, kb) % 2 == W)
                    st_frag(Ps + L::PI(ti, kb) * kTileElems, lane, P[S::T(ti, kb)]);
            bar2(); // block column kb published
            // trailing update of own tiles: C(ti,tj) -= L(ti,kb) L(tj,kb)'
#define CYQ_LK(ti_)                                                                        \
    ((S::T((ti_), kb) % 2 == W) ? P[S::T((ti_), kb)]                                       \
                                : ld_frag(Ps + L::PI((ti_), kb) * kTileElems, lane))
            if (kb + 1 < S::CT && S::T(kb + 1, kb + 1) % 2 == W) {
                const Frag l = CYQ_LK(kb + 1);
                tile_gemm_nt_sub(P[S::T(kb + 1, kb + 1)], l, l);
                st_frag(Ps + L::PI(kb + 1, kb + 1) * kTileElems, lane, P[S::T(kb + 1, kb + 1)]);
            }
#pragma unroll
            for (int tj = kb + 1; tj < S::TT; ++tj) {
#pragma unroll
                for (int ti = tj; ti < S::TT; ++ti) {
                    if (S::T(ti, tj) % 2 != W)
                        continue;
                    if (ti == kb + 1 && tj == kb + 1 && kb + 1 < S::CT)
                        continue;
                    tile_gemm_nt_sub(P[S::T(ti, tj)], CYQ_LK(ti), CYQ_LK(tj));
                }
            }
            if (kb + 1 < S::CT)
                bar2(); // next diagonal tile published
#undef CYQ_LK
        });

        // ---- store own factor tiles and y_s' -----------------------------
        {
            double *dst = a.fac + ((size_t)chain * n + s) * S::NPT * kTileElems;
#pragma unroll
            for (int ti = 0; ti < S::TT; ++ti)
#pragma unroll
                for (int tj = 0; tj < S::CT; ++tj)
                    if (tj <= ti && S::T(ti, tj) % 2 == W)
                        st_frag(dst + L::PI(ti, tj) * kTileElems, lane, P[S::T(ti, tj)]);
            if (rq == RR) {
                double *yv = a.y + ((size_t)chain * n + s) * S::NUX;
#pragma unroll
                for (int tj = 0; tj < S::CT; ++tj) {
                    if (S::T(RT, tj) % 2 != W)
                        continue;
                    const int col = 8 * tj + cq;
                    if (col < S::NUX) yv[col] = P[S::T(RT, tj)].a;
                    if (col + 1 < S::NUX) yv[col + 1] = P[S::T(RT, tj)].b;
                }
            }
        }

        if (s + 1 < n) {
            // ---- W for stage s+1 ------------------------------------------
            if (s == 0) cp_wait<0>();
            else cp_wait<1>();
            bar2(); // BA_{s+1} landed (both warps' copies), Ps final
            if (W == 0) {
                // -wl_new = L_Q' fd + x'  (kkt_solve.cpp:85-90)
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
                            const Frag lt = ld_frag(Ps + L::PI(ti, ct) * kTileElems, lane);
                            const double lv = e ? lt.b : lt.a;
                            if (K >= NU && K < S::NUX && K >= C && C >= NU && C < S::NUX)
                                acc += lv * (sgn * st.f[K - NU]);
                        }
                        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
                        acc += __shfl_xor_sync(0xffffffffu, acc, 8);
                        acc += __shfl_xor_sync(0xffffffffu, acc, 16);
                        const double xp = Ps[L::PI(RT, ct) * kTileElems + RR * 8 + cq + e];
                        if (rq == 0 && C >= NU && C < S::NUX) {
                            mwl[C - NU] = acc + xp;
                            a.wl[((size_t)chain * n + s) * NX + (C - NU)] = -(acc + xp);
                        }
                    }
                }
            }
            // V = BA_{s+1}' L_Q (DMMA), tiles split between the warps
#pragma unroll
            for (int ti = 0; ti < S::CT; ++ti) {
#pragma unroll
                for (int kt = 0; kt < S::NXT; ++kt) {
                    if ((ti * S::NXT + kt) % 2 != (W ^ 1))
                        continue; // warp 1 takes the even tiles (warp 0 also does mw)
                    const int ct = S::XT0 + kt;
                    Frag f{0.0, 0.0};
                    const int r = 8 * ti + rq;
#pragma unroll
                    for (int ks = 2 * S::XT0; ks < 2 * (S::XT1 + 1); ++ks) {
                        if (4 * ks + 3 < 8 * ct)
                            continue;
                        const int K = 4 * ks + (lane & 3);
                        double av = 0.0;
                        if (K >= NU && K < S::NUX && r < S::NUX)
                            av = r < NU ? st.B[(K - NU) * NU + r] : st.A[(K - NU) * NX + (r - NU)];
                        const int Cb = 8 * ct + (lane >> 2);
                        double bv = 0.0;
                        if (K >= NU && K < S::NUX && Cb >= NU && Cb < S::NUX && K >= Cb)
                            bv = Ps[L::PI(K / 8, Cb / 8) * kTileElems + (K % 8) * 8 + Cb % 8];
                        dmma(f, av, bv);
                    }
                    st_frag(Vs + (ti * S::NXT + kt) * kTileElems, lane, f);
                }
            }
            bar2(); // mwl, V ready; BA buffer free
            if (s + 2 < n)
                load_BA<NU, NX, 64>(g, a.p, b, g.stage_of(c, s + 2), st, tid);
            cp_commit();
        }
    }

    // own trailing tiles (coupling x coupling = -Mfwd, rhs x coupling = -fwd)
#pragma unroll
    for (int u = 0; u < S::BT; ++u)
#pragma unroll
        for (int v = 0; v <= u; ++v)
            if (S::T(S::CT + u, S::CT + v) % 2 == W)
                st_frag(a.trail + ((size_t)chain * g.NTT + S::T(u, v)) * kTileElems, lane,
                        P[S::T(S::CT + u, S::CT + v)]);
    unsigned long long key = fail_piv >= 0 ? fail_key(kKindRiccati, c, fail_stage, fail_piv) : ~0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
    if (lane == 0 && key != ~0ull)
        atomicMin(a.fail + b, key);
}

} // namespace

template <int NU, int NX>
__global__ void __launch_bounds__(64) riccati_cta2_kernel(RiccatiArgs a) {
    extern __shared__ __align__(16) double sm[];
    if (threadIdx.x < 32)
        cta2_body<0, NU, NX>(a, sm, blockIdx.x);
    else
        cta2_body<1, NU, NX>(a, sm, blockIdx.x);
}

namespace {
template <int NU, int NX> bool launch_c2(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    if (g.nu != NU || g.nx != NX)
        return false;
    const size_t smem = (size_t)C2<NU, NX>::SMEM * sizeof(double);
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(riccati_cta2_kernel<NU, NX>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    riccati_cta2_kernel<NU, NX><<<g.batch * g.P, 64, smem, st>>>(ra);
    return true;
}
} // namespace

bool launch_riccati_cta2(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    return launch_c2<10, 20>(g, st, ra) || launch_c2<8, 16>(g, st, ra) ||
           launch_c2<4, 12>(g, st, ra) || launch_c2<5, 10>(g, st, ra);
}

} // namespace cyqb
