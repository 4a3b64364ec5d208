// Producer / consumer stage-panel Riccati kernel: TWO warps per partition
// column, specialised at compile time on (nu, nx) like riccati_warp.cu, same
// algorithm and outputs:
//   kkt_factor.cpp:125-158  modified Riccati recursion (LH, LB, Acl, LA)
//   kkt_factor.cpp:163-185  Mfwd = sum LB LB' + LA LA' (trailing block)
//   kkt_solve.cpp:72-134    forward substitution + coupling rows (rhs row)
//
// The extended panel is split by tile ROWS:
//  * producer warp P: the pivot block (tile rows 0 .. CT-1) -- the Cholesky
//    pivot chain, its sub-diagonal solves and trailing updates, V V', the
//    next stage's V = BA' L_Q and all cp.async staging;
//  * consumer warp C: the coupling + rhs rows (tile rows CT .. TT-1) -- W W'
//    for them, their column solves with the published L_kk^{-1}, their
//    trailing updates (including the chain-long -Mfwd / -fwd accumulators),
//    y, wl and the next stage's ALQ / -wl rows of W.
// Within a stage every dependence points from P to C (P never needs C's
// rows), so the pivot chain runs without waiting on the coupling-row DMMA
// work, which proceeds concurrently on another SM sub-partition, a column
// behind. Hand-offs are monotone stamps in shared memory (P publishes
// staged data / column kb / L_Q / V; C acknowledges consumption so P can
// reuse a buffer); every buffer has one writer.
#include "kkt_common.cuh"
#include "kernels.h"
#include "riccati_common.cuh"
#include "riccati_stage.cuh"

#include <cstdlib>

namespace cyqb {

using namespace cyqb::ric;

namespace {

template <int NU, int NX> struct PCS : PanelShape<NU, NX> {
    using B_ = PanelShape<NU, NX>;
    static constexpr int CT = B_::CT, BT = B_::BT, TT = B_::TT, NT = B_::NT, NXC = B_::NXC;
    static constexpr int NXR = B_::NXR, PW = B_::PW, NIMG = B_::NIMG;
    static constexpr int NP = CT * (CT + 1) / 2; // producer tiles (pivot block)
    static constexpr int NC = NT - NP;           // consumer tiles (coupling / rhs rows)
    static constexpr int NSUB = CT * (CT - 1) / 2; // published sub-diagonal pivot-block tiles
    // column buffer: sub-diagonal tile (ti, kb), kb < ti < CT -> slot, then CT L_kk^{-1}
    __host__ __device__ static constexpr int sub_slot(int ti, int kb) { return (ti - 1) * ti / 2 + kb; }
    // shared memory (doubles), all offsets even
    static constexpr int O_WV = 0;                              // CT x NXC tiles (V rows of W)
    static constexpr int O_WC = O_WV + CT * NXC * kTileElems;   // BT x NXC tiles (ALQ / -wl rows)
    static constexpr int O_LQ = O_WC + BT * NXC * kTileElems;   // NXR x NX
    static constexpr int O_IMG = O_LQ + NXR * NX;               // NIMG tiles
    static constexpr int O_IMR = O_IMG + NIMG * kTileElems;     // 2 x PW ([r; q] by stage parity)
    static constexpr int O_S = O_IMR + 2 * PW;                  // NU x NX
    static constexpr int O_BA = O_S + ((NU * NX + 1) & ~1);     // NXR x PW
    static constexpr int O_F = O_BA + NXR * PW;                 // 2 x NX (by stage parity)
    static constexpr int O_COL = O_F + 2 * ((NX + 1) & ~1);     // NSUB + CT tiles
    static constexpr int O_YX = O_COL + (NSUB + CT) * kTileElems; // NX
    static constexpr int O_RU0 = O_YX + ((NX + 1) & ~1);        // NU
    static constexpr int O_SCR = O_RU0 + ((NU + 1) & ~1);       // 64
    static constexpr int O_MB = O_SCR + kTileElems;             // mbarriers (8 bytes each)
    static constexpr int O_TAB = O_MB + 16;                     // staging copy plan (int16)
    static constexpr int SMEM = O_TAB + CopyPlan<NU, NX>::DOUBLES;
};

// Hand-off mbarriers (one arrival per phase, one phase per stage). P -> C:
// H_s staged, pivot column kb (kMbCol + kb), L_Q / f_{s+1}, V_{s+1}; C -> P:
// [r; q]_s read, V_s read, columns of stage s read, L_Q / f read. Every wait
// targets the next phase of its barrier; the acknowledgements keep either
// side from running two phases ahead (so parity waits are unambiguous).
enum : int { kMbH = 0, kMbLQ = 1, kMbV = 2, kMbCInit = 3, kMbCWW = 4, kMbCChol = 5, kMbCMW = 6, kMbCol = 7 };
// after the CT column barriers: P -> C "pivot-block image read" (C may stage
// H_{s+1} into it), and H_{s+1} landed (32 arrivals: one per consumer lane,
// each when that lane's copies complete -- cp.async.mbarrier.arrive.noinc)
template <int CT> struct MbX {
    static constexpr int kImgFree = kMbCol + CT, kHFill = kMbCol + CT + 1, kBAFill = kMbCol + CT + 2,
                         kCount = kMbCol + CT + 3;
};

} // namespace

template <int NU, int NX>
__global__ void __launch_bounds__(64, 6) riccati_pc_kernel(RiccatiArgs a) {
    using S = Shp<NU, NX>;
    using W = PCS<NU, NX>;
    constexpr int CT = W::CT, TT = W::TT, NXC = W::NXC;
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31, role = threadIdx.x >> 5; // 0 producer, 1 consumer
    griddep_launch();
    if ((int)blockIdx.x >= a.grid_chains())
        return;
    const int chain = a.chain_of(blockIdx.x);
    const int b = chain / g.P, c = chain % g.P, n = g.n;
    const int rq = lane >> 2, cq = 2 * (lane & 3), q2 = lane & 3;
    double *Wv = sm + W::O_WV, *Wc = sm + W::O_WC, *LQ = sm + W::O_LQ, *img = sm + W::O_IMG;
    double *imr = sm + W::O_IMR, *Sb = sm + W::O_S, *BA = sm + W::O_BA, *fbuf = sm + W::O_F;
    double *colb = sm + W::O_COL, *yx = sm + W::O_YX, *ru0 = sm + W::O_RU0, *tscr = sm + W::O_SCR;
    unsigned long long *mb = reinterpret_cast<unsigned long long *>(sm + W::O_MB);
    short *ctab = reinterpret_cast<short *>(sm + W::O_TAB);
    constexpr int FST = (NX + 1) & ~1; // f slot stride
    const bool implicit_rhs = (a.p.ru == nullptr);
    const double sgn = implicit_rhs ? -1.0 : 1.0;

    for (int i = threadIdx.x; i < W::SMEM; i += 64)
        sm[i] = 0.0;
    __syncthreads();
    static_assert(MbX<CT>::kCount <= 16, "mbarrier slots");
    if (role == 0)
        CopyPlan<NU, NX>::build(ctab, lane);
    if (threadIdx.x == 0) {
        for (int i = 0; i < MbX<CT>::kCount; ++i)
            mb_init(mb + i, (i == MbX<CT>::kHFill || i == MbX<CT>::kBAFill) ? 32 : 1);
    }
    if (role == 0 && lane < W::PW - W::NUX) { // unit padding diagonal of the image
        const int r = W::NUX + lane;
        img[S::T(r / 8, r / 8) * kTileElems + (r % 8) * 9] = 1.0;
    }
    if (role == 1 && implicit_rhs && c == 0 && lane < NU) { // S_0 x_init (ru[0] term)
        double s0 = 0;
        for (int k = 0; k < NX; ++k)
            s0 += __ldg(a.p.S + (size_t)b * g.N * NU * NX + lane * NX + k) *
                  __ldg(a.p.x_init + (size_t)b * NX + k);
        ru0[lane] = s0;
    }
    __syncthreads();

    if (role == 0) {
        // =============================== PRODUCER ===============================
        Frag P[W::NP];
        int fail_piv = -1, fail_stage = 0;
        {
            const int j0 = g.stage_of(c, 0);
            stage_H<NU, NX>(g, a.p, b, j0, g.x_index_of(c, 0), img, imr, Sb); // imr slot 0
            stage_BA<NU, NX>(g, a.p, b, j0, BA, fbuf);
            cp_commit();
        }
        long long *ph = (a.phase && chain == 0 && lane == 0) ? a.phase : nullptr;
        for (int s = 0; s < n; ++s) {
            const int j = g.stage_of(c, s);
            const bool j0 = j == 0;
            if (ph) ph[s * 16 + 0] = clock64();
            if (s == 0)
                cp_wait<0>(); // prologue: H_0, BA_0
            else
                mb_wait(mb + MbX<CT>::kHFill, (s - 1) & 1); // H_s staged by C has landed
            if (s > 0)
                mb_wait(mb + kMbCInit, (s - 1) & 1); // C has read [r; q]_{s-1}
            mb_signal(mb + kMbH, lane);
            if (ph) ph[s * 16 + 1] = clock64();
            // ---- init pivot block (image + S') and += V V' --------------------
#pragma unroll
            for (int ti = 0; ti < CT; ++ti)
#pragma unroll
                for (int tj = 0; tj <= ti; ++tj) {
                    Frag f = ld_frag(img + S::T(ti, tj) * kTileElems, lane);
                    if (8 * ti + 7 >= NU && 8 * tj < NU && !j0) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int r = 8 * ti + rq, col = 8 * tj + cq + h;
                            const bool isS = r >= NU && r < S::NUX && col < NU;
                            const double v = Sb[isS ? col * NX + (r - NU) : 0];
                            (h ? f.b : f.a) += isS ? v : 0.0;
                        }
                    }
                    P[S::T(ti, tj)] = f;
                }
            mb_signal(mb + MbX<CT>::kImgFree, lane); // image and S' read: C stages H_{s+1}
            if (s > 0) {
#pragma unroll
                for (int kt = 0; kt < NXC; ++kt) {
                    Frag w[CT];
#pragma unroll
                    for (int i = 0; i < CT; ++i)
                        w[i] = ld_frag(Wv + (i * NXC + kt) * kTileElems, lane);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (kt == W::NXF && W::HALF && h == 1)
                            continue;
#pragma unroll
                        for (int ti = 0; ti < CT; ++ti)
#pragma unroll
                            for (int tj = 0; tj <= ti; ++tj)
                                dmma(P[S::T(ti, tj)], h ? w[ti].b : w[ti].a, h ? w[tj].b : w[tj].a);
                    }
                }
            }
            if (ph) ph[s * 16 + 15] = clock64();
            // ---- pivot floor --------------------------------------------------
            double dmax = 0.0;
#pragma unroll
            for (int kb = 0; kb < CT; ++kb) {
                const Frag &d = P[S::T(kb, kb)];
                const double v = (rq & 1) ? d.b : d.a;
                if ((lane & 3) == rq / 2 && 8 * kb + rq < S::NUX)
                    dmax = fmax(dmax, fabs(v));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
            const double dfloor = 1e-14 * dmax;
            // ---- blocked Cholesky of the pivot block, column by column --------
            if (ph) ph[s * 16 + 2] = clock64();
            if (s > 0)
                mb_wait(mb + kMbCChol, (s - 1) & 1); // C is done with last stage's columns
            if (ph) ph[s * 16 + 3] = clock64();
#pragma unroll
            for (int kb = 0; kb < CT; ++kb) {
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
                    if (8 * kb + k < S::NUX) {
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
                st_frag(tscr, lane, idt);
                __syncwarp();
                const Frag linv{tscr[cq * 8 + rq], tscr[(cq + 1) * 8 + rq]};
                __syncwarp();
                st_frag(colb + (W::NSUB + kb) * kTileElems, lane, linv);
#pragma unroll
                for (int ti = kb + 1; ti < CT; ++ti) {
                    Frag r{0.0, 0.0};
                    tile_gemm_nt(r, P[S::T(ti, kb)], linv);
                    P[S::T(ti, kb)] = r;
                    st_frag(colb + W::sub_slot(ti, kb) * kTileElems, lane, r);
                }
                mb_signal(mb + kMbCol + kb, lane); // column kb of the pivot block
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int tj = kb + 1; tj < CT; ++tj)
#pragma unroll
                        for (int ti = tj; ti < CT; ++ti) {
                            const Frag &li = P[S::T(ti, kb)], &lj = P[S::T(tj, kb)];
                            dmma(P[S::T(ti, tj)], h ? -li.b : -li.a, h ? lj.b : lj.a);
                        }
            }
            if (ph) ph[s * 16 + 4] = clock64();
            // ---- store the pivot-block factor tiles -----------------------------
            {
                double *dst = a.fac + ((size_t)chain * n + s) * S::NPT * kTileElems;
#pragma unroll
                for (int t = 0; t < W::NP; ++t)
                    st_frag(dst + t * kTileElems, lane, P[t]);
            }
            // (H_{s+1} is staged by the consumer warp, off the pivot chain)
            if (s == 0 && n > 1) {
                stage_BA<NU, NX>(g, a.p, b, g.stage_of(c, 1), BA, fbuf + FST);
                cp_commit();
            }
            if (s + 1 < n) {
                // L_Q -> LQ once C has used the previous one
                if (s > 0)
                    mb_wait(mb + kMbCMW, (s - 1) & 1);
                {
                    const int lv = lane_v(), rql = lv >> 2, cql = 2 * (lv & 3);
#pragma unroll
                    for (int u = 0; u < S::NXT; ++u)
#pragma unroll
                        for (int v = 0; v <= u; ++v) {
                            const Frag w = P[S::T(S::XT0 + u, S::XT0 + v)];
                            const int K = 8 * (S::XT0 + u) + rql;
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int C = 8 * (S::XT0 + v) + cql + e;
                                if (K >= NU && K < S::NUX && C >= NU && C <= K)
                                    LQ[(K - NU) * NX + (C - NU)] = e ? w.b : w.a;
                            }
                        }
                }
                if (s == 0)
                    cp_wait<0>(); // BA_1, f_1 (the producer's own copies)
                else
                    mb_wait(mb + MbX<CT>::kBAFill, (s - 1) & 1); // BA_{s+1}, f_{s+1} staged by C
                mb_signal(mb + kMbLQ, lane);
                // V_{s+1} = BA' L_Q -> W rows 0..CT-1, once C has read V_s
                if (ph) ph[s * 16 + 5] = clock64();
                mb_wait(mb + kMbCWW, s & 1);
                if (ph) ph[s * 16 + 6] = clock64();
                {
                    Frag vacc[CT * NXC];
#pragma unroll
                    for (int v = 0; v < CT * NXC; ++v)
                        vacc[v] = Frag{0.0, 0.0};
#pragma unroll
                    for (int ks = 0; ks < W::KQ; ++ks) {
                        const int K = 4 * ks + (lane & 3);
                        double av[CT], bv[NXC];
#pragma unroll
                        for (int ti = 0; ti < CT; ++ti)
                            av[ti] = BA[K * W::PW + 8 * ti + rq];
#pragma unroll
                        for (int kt = 0; kt < NXC; ++kt) {
                            const int vc = W::col_of(8 * kt + rq);
                            bv[kt] = vc >= 0 ? LQ[K * NX + (vc >= 0 ? vc : 0)] : 0.0;
                        }
#pragma unroll
                        for (int ti = 0; ti < CT; ++ti)
#pragma unroll
                            for (int kt = 0; kt < NXC; ++kt)
                                if (4 * ks + 3 >= 8 * kt)
                                    dmma(vacc[ti * NXC + kt], av[ti], bv[kt]);
                    }
#pragma unroll
                    for (int v = 0; v < CT * NXC; ++v)
                        st_frag(Wv + v * kTileElems, lane, vacc[v]);
                }
                mb_signal(mb + kMbV, lane);
                if (ph) ph[s * 16 + 7] = clock64();
                __syncwarp();
            }
        }
        unsigned long long my_fail =
            fail_piv >= 0 ? fail_key(kKindRiccati, c, fail_stage, fail_piv) : ~0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            my_fail = min(my_fail, __shfl_xor_sync(0xffffffffu, my_fail, o));
        if (lane == 0 && my_fail != ~0ull)
            atomicMin(a.fail + b, my_fail);
    } else {
        // =============================== CONSUMER ===============================
        Frag Cf[W::NC]; // tile (ti, tj), ti >= CT at Cf[T(ti, tj) - NP]
#pragma unroll
        for (int t = 0; t < W::NC; ++t)
            Cf[t] = Frag{0.0, 0.0};
#define CFT(ti, tj) Cf[S::T(ti, tj) - W::NP]
        long long *ph = (a.phase && chain == 0 && lane == 0) ? a.phase : nullptr;
        for (int s = 0; s < n; ++s) {
            const int j = g.stage_of(c, s);
            const double *ru0p = (implicit_rhs && j == 0) ? ru0 : nullptr;
            if (ph) ph[s * 16 + 8] = clock64();
            mb_wait(mb + kMbH, s & 1);
            if (ph) ph[s * 16 + 9] = clock64();
            // ---- init coupling rows (BA_0 at s = 0) and the rhs row -------------
#pragma unroll
            for (int ti = CT; ti < TT; ++ti)
#pragma unroll
                for (int tj = 0; tj < CT; ++tj) {
                    Frag f{0.0, 0.0};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int rb = 8 * ti + rq - S::TOP, col = 8 * tj + cq + h;
                        double v = 0.0;
                        if (s == 0 && rb < NX && j < g.N) // BA_0 straight from global (A omitted at j = 0)
                            v = col < NU ? __ldg(a.p.B + ((size_t)b * g.N + j) * NX * NU + rb * NU + col)
                                         : ((j != 0 && col < S::NUX)
                                                ? __ldg(a.p.A + ((size_t)b * g.N + j) * NX * NX + rb * NX + (col - NU))
                                                : 0.0);
                        if (rb == NX)
                            v = sgn * imr[(s & 1) * W::PW + col] - ((ru0p && col < NU) ? ru0p[col] : 0.0);
                        (h ? f.b : f.a) = v;
                    }
                    CFT(ti, tj) = f;
                }
            mb_signal(mb + kMbCInit, lane);
            // ---- += W W' for my rows -----------------------------------------
            if (s > 0) {
                mb_wait(mb + kMbV, (s - 1) & 1);
                // V_s is computed: the BA buffer is free -- stage BA_{s+1} (and
                // f_{s+1} into the slot of f_{s-1}) for the producer's V_{s+1}
                if (s + 1 < n) {
                    stage_BA_plan<NU, NX>(g, a.p, b, g.stage_of(c, s + 1), BA, fbuf + ((s + 1) & 1) * FST, ctab);
                    __syncwarp();
                    __threadfence_block();
                    mb_arrive_on_copies(mb + MbX<CT>::kBAFill);
                }
#pragma unroll
                for (int kt = 0; kt < NXC; ++kt) {
                    Frag w[TT];
#pragma unroll
                    for (int i = 0; i < TT; ++i)
                        w[i] = i < CT ? ld_frag(Wv + (i * NXC + kt) * kTileElems, lane)
                                      : ld_frag(Wc + ((i - CT) * NXC + kt) * kTileElems, lane);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (kt == W::NXF && W::HALF && h == 1)
                            continue;
#pragma unroll
                        for (int ti = CT; ti < TT; ++ti)
#pragma unroll
                            for (int tj = 0; tj <= ti; ++tj)
                                dmma(CFT(ti, tj), h ? w[ti].b : w[ti].a, h ? w[tj].b : w[tj].a);
                    }
                }
            }
            mb_signal(mb + kMbCWW, lane);
            // ---- stage H_{s+1} for the producer ([r; q] into the parity slot
            // read at stage s-1), while the pivot chain runs -------------------
            if (s + 1 < n) {
                mb_wait(mb + MbX<CT>::kImgFree, s & 1);
                stage_H_plan<NU, NX>(g, a.p, b, g.stage_of(c, s + 1), g.x_index_of(c, s + 1), img,
                                     imr + ((s + 1) & 1) * W::PW, Sb, ctab);
                __syncwarp();
                __threadfence_block(); // identity / zero fills of padding stages
                mb_arrive_on_copies(mb + MbX<CT>::kHFill);
            }
            if (ph) ph[s * 16 + 10] = clock64();
            // ---- my rows of each pivot column --------------------------------
#pragma unroll
            for (int kb = 0; kb < CT; ++kb) {
                mb_wait(mb + kMbCol + kb, s & 1);
                const Frag linv = ld_frag(colb + (W::NSUB + kb) * kTileElems, lane);
#pragma unroll
                for (int ti = CT; ti < TT; ++ti) {
                    Frag r{0.0, 0.0};
                    tile_gemm_nt(r, CFT(ti, kb), linv);
                    CFT(ti, kb) = r;
                }
                // trailing: C(ti, tj) -= L(ti, kb) L(tj, kb)', tj > kb
#pragma unroll
                for (int tj = kb + 1; tj < TT; ++tj) {
                    const Frag lj = tj < CT ? ld_frag(colb + W::sub_slot(tj < CT ? tj : 1, kb) * kTileElems, lane)
                                            : CFT(tj < CT ? CT : tj, kb);
#pragma unroll
                    for (int ti = (tj > CT ? tj : CT); ti < TT; ++ti)
                        tile_gemm_nt_sub(CFT(ti, tj), CFT(ti, kb), lj);
                }
            }
            mb_signal(mb + kMbCChol, lane);
            if (ph) ph[s * 16 + 11] = clock64();
            // ---- store my factor tiles and y_s' -----------------------------
            {
                double *dst = a.fac + ((size_t)chain * n + s) * S::NPT * kTileElems;
#pragma unroll
                for (int ti = CT; ti < TT; ++ti)
#pragma unroll
                    for (int tj = 0; tj < CT; ++tj)
                        st_frag(dst + (W::NP + (ti - CT) * CT + tj) * kTileElems, lane, CFT(ti, tj));
                if (rq == W::RR) {
                    double *yv = a.y + ((size_t)chain * n + s) * S::NUX;
#pragma unroll
                    for (int tj = 0; tj < CT; ++tj) {
                        const int col = 8 * tj + cq;
                        const Frag f = CFT(W::RT, tj);
                        if (col < S::NUX) yv[col] = f.a;
                        if (col + 1 < S::NUX) yv[col + 1] = f.b;
                        if (col >= NU && col < S::NUX) yx[col - NU] = f.a;
                        if (col + 1 >= NU && col + 1 < S::NUX) yx[col + 1 - NU] = f.b;
                    }
                }
            }
            if (s + 1 < n) {
                // -wl_new = L_Q' (sgn f_{s+1}) + x'  (kkt_solve.cpp:85-90)
                if (ph) ph[s * 16 + 12] = clock64();
                mb_wait(mb + kMbLQ, s & 1);
                if (ph) ph[s * 16 + 13] = clock64();
                const double *fb = fbuf + ((s + 1) & 1) * FST;
                double mwl = 0.0;
                if (lane < NX) {
                    double acc = 0.0;
#pragma unroll 4
                    for (int k = lane; k < NX; ++k)
                        acc = fma(LQ[k * NX + lane], sgn * fb[k], acc);
                    mwl = acc + yx[lane];
                    a.wl[((size_t)chain * n + s) * NX + lane] = -mwl;
                }
                // W rows CT..TT-1: ALQ (x columns, compact positions) and -wl
                {
                    const int lv = lane_v(), rql = lv >> 2, cql = 2 * (lv & 3);
#pragma unroll
                    for (int ti = CT; ti < TT; ++ti)
#pragma unroll
                        for (int kt = 0; kt < S::NXT; ++kt) {
                            const int ct = S::XT0 + kt, r = 8 * ti + rql;
                            const Frag pf = CFT(ti, ct);
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int Cc = 8 * ct + cql + e;
                                if (Cc >= NU && Cc < S::NUX && r < S::RHS) {
                                    const int p = W::pos(Cc - NU);
                                    Wc[((ti - CT) * NXC + p / 8) * kTileElems + (r % 8) * 8 + p % 8] =
                                        e ? pf.b : pf.a;
                                }
                            }
                        }
                }
                if (lane < NX) { // the rhs row of W: -wl_new
                    const int p = W::pos(lane);
                    Wc[((W::RT - CT) * NXC + p / 8) * kTileElems + W::RR * 8 + p % 8] = mwl;
                }
                mb_signal(mb + kMbCMW, lane);
                if (ph) ph[s * 16 + 14] = clock64();
            }
        }
        // trailing tiles (coupling x coupling = -Mfwd, rhs x coupling = -fwd)
#pragma unroll
        for (int u = 0; u < S::BT; ++u)
#pragma unroll
            for (int v = 0; v <= u; ++v)
                st_frag(a.trail + ((size_t)chain * g.NTT + S::T(u, v)) * kTileElems, lane,
                        CFT(CT + u, CT + v));
#undef CFT
    }
}

namespace {
template <int NU, int NX> bool launch_p(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    if (g.nu != NU || g.nx != NX)
        return false;
    const size_t smem = (size_t)PCS<NU, NX>::SMEM * sizeof(double);
    static DeviceOnce once;
    once_per_device(once, [&] { return cudaFuncSetAttribute(riccati_pc_kernel<NU, NX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    riccati_pc_kernel<NU, NX><<<ra.grid_chains(), 64, smem, st>>>(ra);
    return true;
}
} // namespace

bool launch_riccati_pc(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    return launch_p<10, 20>(g, st, ra) || launch_p<8, 16>(g, st, ra) || launch_p<4, 12>(g, st, ra) ||
           launch_p<5, 10>(g, st, ra);
}

} // namespace cyqb
