// CTA-per-chain stage-panel Riccati kernel for LARGE stage blocks with
// tile-aligned dimensions (nu % 8 == 0, nx % 8 == 0; BASELINE config 3:
// nu = 32, nx = 64, nux = 96 -- the dense DMMA regime). Same algorithm and
// outputs as riccati_warp.cu / riccati.cu:
//   kkt_factor.cpp:125-158  modified Riccati recursion (LH, LB, Acl, LA)
//   kkt_factor.cpp:163-185  Mfwd = sum LB LB' + LA LA' (trailing block)
//   kkt_solve.cpp:72-134    forward substitution + coupling rows (rhs row)
//
// Execution model (one CTA of NW warps per partition column; the kernel
// comment has the details):
//  * the extended panel (TT x TT lower tiles, 231 at config 3) lives in the
//    registers of the BULK WARPS (1 .. NW-1) for the stage: every tile but the
//    pivot diagonal tiles (d, d) and the tiles left of them (d, d-1) is on a
//    per-warp LIST ordered by tile column descending, planned on the host
//    (launch_c) and kept packed in registers. At block column kb the tiles a
//    warp must update (tj > kb) are a PREFIX of its list, its own column-kb
//    tiles the slots right behind it: straight-line code entered at the right
//    slot, no predicated-off DMMA (they occupy the DMMA pipe like real ones),
//    no walk over the list, no indexed constant load (~100+ cycles each);
//  * blocked right-looking Cholesky with the serial chain DECOUPLED: the
//    PIVOT WARP (warp 0, on an SM sub-partition whose other warps hold only
//    tiles of the first block columns) solves (d, d-1) against L_{d-1}^{-1},
//    applies it to (d, d), factors (d, d) without a shuffle (the tile
//    replicated in every lane's registers) and publishes L_dd^{-1}; it only
//    arrives at the step barriers. A bulk warp, per block column: waits for
//    L_kk^{-1} (a release/acquire flag), solves its own column-kb tiles in
//    registers (X <- X L_kk^{-T}, two DMMAs) into column buffer kb % 3, one
//    CTA barrier, keeps its (d, d) / (d, d-1) up to date (handing them to the
//    pivot warp two steps before their turn) and applies column kb to its
//    list prefix (C -= L_i L_j', operands from the column buffer);
//  * shared memory holds W = [V; ALQ; -wl] (the next stage's W W' operand),
//    [B A] of the next stage (cp.async, one stage ahead), L_Q in x-space
//    (the B operand of V = BA' L_Q), three column buffers and the hand-off
//    slots; H_s is read straight from global memory (L2-prefetched one stage
//    ahead).
// Round-2 history at config 3 (256 x N=512): 32.4 ms (two barriers per block
// column, look-ahead by rotating owners, lists in constant memory) -> 24.5 ms;
// tools/trail_bench.cu and the CYQ_TRACE build (tools/phase_run.py) are the
// measurements behind each step.
#include "kkt_common.cuh"
#include "kernels.h"
#include "riccati_common.cuh"

#include <algorithm>
#include <vector>
#include <type_traits>
#include <cstdlib>

namespace cyqb {

using namespace cyqb::ric;

namespace {

// per-warp tile lists (host-built, launch_c): tile k of warp w is (ti, tj),
// tile columns non-increasing in k; count kb + 1 = number of the warp's tiles
// with tile column > kb (the update prefix at block column kb), count 0 =
// all its tiles.
// The kernel keeps both PACKED IN REGISTERS for the whole launch (c_lpk: three
// tiles per word, 5 bits each for ti and tj; c_cpk: sixteen 4-bit counts):
// an indexed constant load costs ~100 cycles, and the unrolled list walks
// issued one per tile -- predicated-off ones included -- on the critical
// path of every block column (the pick-up walk alone took ~1400 cycles of
// each ~3500-cycle column step).
constexpr int kMaxW = 16, kMaxL = 15, kMaxCT = 15, kLW = 5;
__constant__ unsigned c_lpk[kMaxW * kLW];
__constant__ unsigned long long c_cpk[kMaxW];
__constant__ unsigned c_ppk[kMaxW * 4]; // stored-factor tile index PI(ti, tj) of every list tile, a byte each

template <int NU, int NX, int NW> struct CS {
    static_assert(NU % 8 == 0 && NX % 8 == 0, "tile-aligned shapes only");
    static constexpr int NUX = NU + NX;
    static constexpr int CT = NUX / 8;            // pivot tile columns
    static constexpr int BT = (NX + 1 + 7) / 8;   // coupling + rhs tile rows
    static constexpr int TT = CT + BT;
    static constexpr int NT = TT * (TT + 1) / 2;
    // list tiles: all but the pivot diagonal tiles (d, d) and the tiles left
    // of them (d, d-1), which the pivot warp takes over (kernel comment)
    static constexpr int NL = NT - CT - (CT - 1);
    static_assert(NW % 4 == 0 && 3 * (NW / 4) >= CT && NW <= kMaxW && CT <= kMaxCT,
                  "one bulk warp (warp % 4 != 0) per pivot diagonal tile");
    static constexpr int TOP = 8 * CT, RHS = TOP + NX, RT = RHS / 8, RR = RHS % 8;
    static constexpr int XT0 = NU / 8, NXC = NX / 8; // x columns: tiles XT0 .. CT-1
    static constexpr int NPT = CT * (CT + 1) / 2 + BT * CT;
    static constexpr int MAXL = (NL + NW - 2) / (NW - 1); // tiles per warp; the pivot warp holds none
    // "pure" coupling tiles (rows and columns all coupling rows: tile rows
    // CT .. RT-1, tile row RT holds the rhs row): their ALQ_s ALQ_s' terms
    // cancel between stage s's trailing update and stage s+1's W W' (only
    // sum LB LB' + LA LA' stays in -Mfwd, kkt_factor.cpp:179-184). Every warp
    // holds NPS of them at list slots 0 .. NPS-1 in "skip mode": W W' and the
    // x-column (kb >= XT0) trailing updates of stages s < n-1 skip them
    // (compile-time loop starts: no predicated-off DMMAs)
    static constexpr int NPURE = (RT - CT) * (RT - CT + 1) / 2;
    static constexpr int NPS = NPURE / NW;
    static_assert(MAXL <= kMaxL && TT <= 32, "packed list: 15 tiles of 5 + 5 bits, 4-bit counts");
    // [B A] and L_Q row strides, padded by 8 doubles: the V = BA' L_Q
    // operand loads (4 rows x 8 columns per warp) then need the minimum two
    // shared-memory wavefronts instead of four
    static constexpr int PW = NUX + 8, LQS = NX + 8;
    // shared memory (doubles)
    static constexpr int O_W = 0;                                  // TT x NXC tiles
    static constexpr int O_COL = O_W + TT * NXC * kTileElems;      // 3 x TT tiles (by kb % 3)
    static constexpr int O_LINV = O_COL + 3 * TT * kTileElems;     // 2 tiles (by kb parity)
    static constexpr int O_BA = O_LINV + 2 * kTileElems;           // NX x PW
    static constexpr int O_LQ = O_BA + NX * PW;                    // NX x LQS (x-space L_Q)
    static constexpr int O_F = O_LQ + NX * LQS;                    // NX
    static constexpr int O_YX = O_F + NX;                          // NX (x part of y)
    static constexpr int O_MW = O_YX + NX;                         // NX (-wl_new)
    static constexpr int O_RU0 = O_MW + NX;                        // NU
    static constexpr int O_RED = O_RU0 + NU;                       // 32 (pivot floor)
    static constexpr int O_SCR = O_RED + 32;                       // 64 (transpose)
    static constexpr int O_SCR2 = O_SCR + kTileElems;              // 64 (L_kk out; upper part stays zero)
    static constexpr int O_DG = O_SCR2 + kTileElems;               // CT pivot diagonal tiles (hand-off)
    static constexpr int O_MB = O_DG + CT * kTileElems;            // 1 mbarrier ([B A] staging)
    static constexpr int O_LMB = O_MB + 2;                         // CT flags (L_kk^{-1} published), 32-bit
    static constexpr int O_HMB = O_LMB + (CT + 1) / 2;             // CT flags (tiles handed to the pivot warp)
    static constexpr int SMEM = O_HMB + (CT + 1) / 2 + 1;
    __host__ __device__ static constexpr int T(int i, int j) { return i * (i + 1) / 2 + j; }
    // stored-factor tile index of panel tile (i, j), j < CT
    __host__ __device__ static constexpr int PI(int i, int j) {
        return i < CT ? T(i, j) : CT * (CT + 1) / 2 + (i - CT) * CT + j;
    }
};

__device__ __forceinline__ void pf_lines(const double *p, int bytes, int tid, int nthr) {
    for (int o = tid * 128; o < bytes; o += nthr * 128)
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(reinterpret_cast<const char *>(p) + o));
}

// [B A]_j -> BA rows (A omitted for j = 0, zero for padding stages), f_j.
// TMA bulk copies (cp.async.bulk, one issuing thread, one copy per row into
// the padded row layout, completion counted in bytes on `mbar`); omitted /
// padding blocks zero-filled by all threads; per-thread cp.async when a
// source is not 16-byte aligned (then `mbar` gets a plain arrival and the
// waiter's cp.async.wait_group covers the copies). Every call is matched by
// one wait_BA.
template <int NU, int NX, int NW, bool TMA>
__device__ __forceinline__ void stage_BA_cta(const Geo &g, const ProbView &p, int b, int j, double *sm,
                                             int tid, unsigned long long *mbar) {
    using C = CS<NU, NX, NW>;
    constexpr int NTH = 32 * NW;
    const int N = g.N;
    double *ba = sm + C::O_BA;
    const bool in = j < N;
    const double *Bs = in ? p.B + ((size_t)b * N + j) * NX * NU : nullptr;
    const double *As = (in && j != 0) ? p.A + ((size_t)b * N + j) * NX * NX : nullptr;
    const double *fs = in ? (p.fd ? p.fd : p.f) + ((size_t)b * N + j) * NX : nullptr;
    const bool al = ((reinterpret_cast<uintptr_t>(Bs) | reinterpret_cast<uintptr_t>(As) |
                      reinterpret_cast<uintptr_t>(fs)) & 15) == 0 && (NU * 8) % 16 == 0 && (NX * 8) % 16 == 0;
    if (TMA && al) {
        // the last warp issues: one lane announces the bytes, then every
        // lane issues its share of the row copies
        if (tid >= NTH - 32) {
            const int l = tid - (NTH - 32);
            if (l == 0) {
                const unsigned bytes = (Bs ? NX * NU * 8 : 0) + (As ? NX * NX * 8 : 0) + (fs ? NX * 8 : 0);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)),
                             "r"(bytes)
                             : "memory");
            }
            __syncwarp();
            auto bulk = [&](double *dst, const double *src, unsigned nbytes) {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(dst)),
                             "l"(src), "r"(nbytes), "r"(smem_u32(mbar))
                             : "memory");
            };
            for (int r = l; Bs && r < NX; r += 32)
                bulk(ba + r * C::PW, Bs + r * NU, NU * 8);
            for (int r = l; As && r < NX; r += 32)
                bulk(ba + r * C::PW + NU, As + r * NX, NX * 8);
            if (fs && l == 0)
                bulk(sm + C::O_F, fs, NX * 8);
        }
        for (int e = tid; !Bs && e < NX * NU; e += NTH)
            ba[(e / NU) * C::PW + e % NU] = 0.0;
        for (int e = tid; !As && e < NX * NX; e += NTH)
            ba[(e / NX) * C::PW + NU + e % NX] = 0.0;
        for (int e = tid; !fs && e < NX; e += NTH)
            sm[C::O_F + e] = 0.0;
        return;
    }
    for (int e = 2 * tid; e < NX * NU; e += 2 * NTH) {
        double *d = ba + (e / NU) * C::PW + e % NU;
        if (Bs && al) {
            cp16(d, Bs + e);
        } else if (Bs) {
            cp8(d, Bs + e);
            cp8(d + 1, Bs + e + 1);
        } else
            d[0] = d[1] = 0.0;
    }
    for (int e = 2 * tid; e < NX * NX; e += 2 * NTH) {
        double *d = ba + (e / NX) * C::PW + NU + e % NX;
        if (As && al) {
            cp16(d, As + e);
        } else if (As) {
            cp8(d, As + e);
            cp8(d + 1, As + e + 1);
        } else
            d[0] = d[1] = 0.0;
    }
    for (int e = tid; e < NX; e += NTH) {
        if (fs)
            cp8(sm + C::O_F + e, fs + e);
        else
            sm[C::O_F + e] = 0.0;
    }
    cp_commit();
    if (tid == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}

// completion of the matching stage_BA_cta (phase `ph`, then advanced); the
// caller's __syncthreads makes the zero fills visible
__device__ __forceinline__ void wait_BA(unsigned long long *mbar, int &ph) {
    cp_wait<0>();
    mb_wait(mbar, ph & 1);
    ++ph;
}

// initial value of panel tile (ti, tj), tj < CT: H_s (top), [B A]_0 rows at
// s = 0 and the rhs row (bottom)
template <int NU, int NX, int NW>
__device__ __forceinline__ Frag init_tile(int ti, int tj, int rq, int cq, int s, double sgn,
                                          const double *Rg, const double *Sg, const double *Qg,
                                          const double *rg, const double *qg, const double *ru0p,
                                          const double *BA, bool aligned) {
    using C = CS<NU, NX, NW>;
    Frag f{0.0, 0.0};
    const int r = 8 * ti + rq, c0 = 8 * tj + cq;
    if (ti < C::CT) {
        if (r < NU && c0 < NU) { // R (full block; upper parts are don't-care)
            if (Rg && !aligned) {
                f = {__ldg(Rg + r * NU + c0), __ldg(Rg + r * NU + c0 + 1)};
            } else if (Rg) {
                const double2 v = __ldg(reinterpret_cast<const double2 *>(Rg + r * NU + c0));
                f = {v.x, v.y};
            } else
                f = {r == c0 ? 1.0 : 0.0, r == c0 + 1 ? 1.0 : 0.0};
        } else if (r >= NU && c0 >= NU) { // Q
            if (Qg && !aligned) {
                f = {__ldg(Qg + (r - NU) * NX + (c0 - NU)), __ldg(Qg + (r - NU) * NX + (c0 - NU) + 1)};
            } else if (Qg) {
                const double2 v = __ldg(reinterpret_cast<const double2 *>(Qg + (r - NU) * NX + (c0 - NU)));
                f = {v.x, v.y};
            } else
                f = {r == c0 ? 1.0 : 0.0, r == c0 + 1 ? 1.0 : 0.0};
        } else if (r >= NU && c0 < NU && Sg) { // S' (lower-left), transposed read
            f = {__ldg(Sg + c0 * NX + (r - NU)), __ldg(Sg + (c0 + 1) * NX + (r - NU))};
        }
    } else {
        const int rb = r - C::TOP;
        if (s == 0 && rb < NX)
            f = {BA[rb * C::PW + c0], BA[rb * C::PW + c0 + 1]};
        else if (rb == NX) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = c0 + h;
                double v = 0.0;
                if (col < NU)
                    v = (rg ? sgn * __ldg(rg + col) : 0.0) - (ru0p ? ru0p[col] : 0.0);
                else
                    v = qg ? sgn * __ldg(qg + col - NU) : 0.0;
                (h ? f.b : f.a) = v;
            }
        }
    }
    return f;
}

} // namespace

// Kernel layout: after the common set-up the CTA splits for good into the
// PIVOT WARP (warp 0) and the BULK WARPS (1 .. NW-1), two code paths with their
// own registers (the pivot path holds no panel tile, the bulk path none of the
// factorization's temporaries) that meet at named barriers:
//   1 + kb % 2  block column kb (bulk warps wait, the pivot warp only arrives)
//   3           stage top (W and BA_0 read, dgs[] written)
//   4           the CTA-wide phases after the column loop
// Warp 0 holds no list tile and runs the serial chain of the blocked Cholesky
// by itself -- solve (d, d-1) against L_{d-1}^{-1}, apply it to (d, d), factor
// (d, d), publish L_dd^{-1}. Its SM sub-partition (warps 0, 4, 8, ...) holds
// only tiles of the first block columns (host plan), so after the first steps
// no DMMA of another warp queues ahead of the chain's FP64 instructions. The
// bulk warps with warp % 4 != 0 each keep one pivot diagonal tile (dkb, dkb) in
// `dg` and the tile left of it (dkb, dkb-1) in `sd` up to date and hand both
// over through shared memory (flag hmb[dkb]) once column dkb-2 is applied.
template <int NU, int NX, int NW, bool TMA>
__global__ void __launch_bounds__(32 * NW, 1) riccati_cta_kernel(RiccatiArgs a) {
    using C = CS<NU, NX, NW>;
    constexpr int NTH = 32 * NW, MAXL = C::MAXL, CT = C::CT, TT = C::TT;
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int chain = a.chain_of(blockIdx.x);
    const int b = chain / g.P, c = chain % g.P, n = g.n, N = g.N;
    griddep_launch();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    double *Wsm = sm + C::O_W, *colb = sm + C::O_COL, *linvb = sm + C::O_LINV, *BA = sm + C::O_BA;
    double *LQ = sm + C::O_LQ, *fb = sm + C::O_F, *yx = sm + C::O_YX, *mw = sm + C::O_MW;
    double *ru0 = sm + C::O_RU0;
    double *tscr = sm + C::O_SCR, *tscr2 = sm + C::O_SCR2;
    const bool implicit_rhs = (a.p.ru == nullptr);
    const double sgn = implicit_rhs ? -1.0 : 1.0;
    for (int i = tid; i < C::SMEM; i += NTH)
        sm[i] = 0.0;
    unsigned long long *bamb = reinterpret_cast<unsigned long long *>(sm + C::O_MB);
    // hand-off flags (value s + 1 at stage s; zero-filled above)
    unsigned *lmb = reinterpret_cast<unsigned *>(sm + C::O_LMB);
    unsigned *hmb = reinterpret_cast<unsigned *>(sm + C::O_HMB);
    double *dgs = sm + C::O_DG;
    __syncthreads();
    if (tid == 0) {
        mb_init(bamb, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // prologue: BA_0, S_0 x_init (ru[0] term)
    {
        int ph0 = 0;
        const int j0 = g.stage_of(c, 0);
        stage_BA_cta<NU, NX, NW, TMA>(g, a.p, b, j0, sm, tid, bamb);
        if (implicit_rhs && c == 0)
            for (int i = tid; i < NU; i += NTH) {
                double s0 = 0;
                for (int k = 0; k < NX; ++k)
                    s0 += __ldg(a.p.S + (size_t)b * N * NU * NX + i * NX + k) *
                          __ldg(a.p.x_init + (size_t)b * NX + k);
                ru0[i] = s0;
            }
        wait_BA(bamb, ph0);
    }
    __syncthreads();

    // ---- pieces shared by the two paths ---------------------------------------
    struct StageIn {
        const double *Rg, *Sg, *Qg, *rg, *qg, *ru0p;
        bool aligned;
    };
    auto stage_in = [&](int s) {
        const int j = g.stage_of(c, s), xi = g.x_index_of(c, s);
        const bool j0 = j == 0, in = j < N, qin = xi <= N;
        StageIn r;
        r.Rg = in ? a.p.R + ((size_t)b * N + j) * NU * NU : nullptr;
        r.Sg = (in && !j0) ? a.p.S + ((size_t)b * N + j) * NU * NX : nullptr;
        r.Qg = qin ? a.p.Q + ((size_t)b * (N + 1) + xi) * NX * NX : nullptr;
        r.rg = in ? (a.p.ru ? a.p.ru : a.p.r) + ((size_t)b * N + j) * NU : nullptr;
        r.qg = qin ? (a.p.qx ? a.p.qx : a.p.q) + ((size_t)b * (N + 1) + xi) * NX : nullptr;
        r.ru0p = (implicit_rhs && j0) ? ru0 : nullptr;
        r.aligned = ((reinterpret_cast<uintptr_t>(a.p.R) | reinterpret_cast<uintptr_t>(a.p.Q)) & 15) == 0;
        return r;
    };
    auto tile0 = [&](int ti, int tj, int s, const StageIn &in) {
        return init_tile<NU, NX, NW>(ti, tj, rq, cq, s, sgn, in.Rg, in.Sg, in.Qg, in.rg, in.qg, in.ru0p, BA,
                                     in.aligned);
    };
    // prefetch H_{s+1} into L2
    auto prefetch_next = [&](int s) {
        if (s + 1 < n) {
            const int j1 = g.stage_of(c, s + 1), x1 = g.x_index_of(c, s + 1);
            if (j1 < N) {
                pf_lines(a.p.R + ((size_t)b * N + j1) * NU * NU, NU * NU * 8, tid, NTH);
                pf_lines(a.p.S + ((size_t)b * N + j1) * NU * NX, NU * NX * 8, tid, NTH);
            }
            if (x1 <= N)
                pf_lines(a.p.Q + ((size_t)b * (N + 1) + x1) * NX * NX, NX * NX * 8, tid, NTH);
        }
    };
    auto bar_wait = [](int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NTH) : "memory"); };
    auto bar_arrive = [](int id) {
        __threadfence_block();
        asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(NTH) : "memory");
    };
    // W of stage s+1 once the factor tiles of stage s are out (every warp):
    // -wl_new = L_Q' (sgn f) + x' (kkt_solve.cpp:85-90; 8 lanes per entry,
    // split k, shuffle-reduced), V = BA_{s+1}' L_Q -> W tile rows 0..CT-1
    // (DMMA, one tile per warp pass, two accumulators to halve the dependent
    // DMMA chain), the rhs row of W, [B A] of stage s+2 on its way
    auto next_W = [&](int s, int &baph, long long *ph) {
        wait_BA(bamb, baph); // BA_{s+1}, f_{s+1}
        bar_wait(4);
        if (ph) ph[s * 8 + 4] = clock64();
        for (int t0 = 4 * warp; t0 < NX; t0 += 4 * NW) {
            const int t = t0 + (lane >> 3), part = lane & 7;
            double q = 0.0, q1 = 0.0;
            if (t < NX) {
#pragma unroll
                for (int i = 0; i < NX / 8; i += 2) { // L_Q is lower triangular: rows k >= t
                    const int k0 = t + part + 8 * i, k1 = k0 + 8;
                    if (k0 < NX)
                        q = fma(LQ[k0 * C::LQS + t], fb[k0], q);
                    if (k1 < NX)
                        q1 = fma(LQ[k1 * C::LQS + t], fb[k1], q1);
                }
                q = sgn * (q + q1);
            }
            q += __shfl_xor_sync(0xffffffffu, q, 1);
            q += __shfl_xor_sync(0xffffffffu, q, 2);
            q += __shfl_xor_sync(0xffffffffu, q, 4);
            if (t < NX && part == 0) {
                q += yx[t];
                mw[t] = q;
                a.wl[((size_t)chain * n + s) * NX + t] = -q;
            }
        }
        if (ph) ph[s * 8 + 5] = clock64();
        // V tiles in pairs (ti, kt = P) + (ti, kt = NXC-1-P): L_Q is lower
        // triangular, so a pair is NXC + 1 k-tiles of work whatever P is, and
        // both tiles share the BA' operands. P is a compile-time case: every
        // operand is one 8-byte load at an immediate offset from two base
        // registers, four accumulator chains per pair.
        {
            constexpr int NP = (C::NXC + 1) / 2, NITEM = CT * NP;
            const double *pa0 = BA + (lane & 3) * C::PW + rq, *pb0 = LQ + (lane & 3) * C::LQS + rq;
            auto item = [&](auto PC, int ti) {
                constexpr int P = decltype(PC)::value, Q = C::NXC - 1 - P;
                const double *pa = pa0 + 8 * ti;
                Frag fa0{0.0, 0.0}, fa1{0.0, 0.0}, fb0{0.0, 0.0}, fb1{0.0, 0.0};
#pragma unroll
                for (int ks = 2 * P; ks < NX / 4; ++ks) {
                    const double av = pa[4 * ks * C::PW];
                    dmma((ks & 1) ? fa1 : fa0, av, pb0[4 * ks * C::LQS + 8 * P]);
                    if (Q != P && ks >= 2 * Q)
                        dmma((ks & 1) ? fb1 : fb0, av, pb0[4 * ks * C::LQS + 8 * Q]);
                }
                st_frag(Wsm + (ti * C::NXC + P) * kTileElems, lane, Frag{fa0.a + fa1.a, fa0.b + fa1.b});
                if (Q != P)
                    st_frag(Wsm + (ti * C::NXC + Q) * kTileElems, lane, Frag{fb0.a + fb1.a, fb0.b + fb1.b});
            };
            for (int v = warp; v < NITEM; v += NW) {
                const int ti = v % CT;
                switch (v / CT) {
                case 0: item(std::integral_constant<int, 0>{}, ti); break;
                case 1: if constexpr (NP > 1) item(std::integral_constant<int, (NP > 1 ? 1 : 0)>{}, ti); break;
                case 2: if constexpr (NP > 2) item(std::integral_constant<int, (NP > 2 ? 2 : 0)>{}, ti); break;
                case 3: if constexpr (NP > 3) item(std::integral_constant<int, (NP > 3 ? 3 : 0)>{}, ti); break;
                default: break;
                }
            }
            static_assert(NP <= 4, "V pair cases");
        }
        if (ph) ph[s * 8 + 6] = clock64();
        bar_wait(4); // mw ready, V written, BA / LQ reads done
        if (ph) ph[s * 8 + 7] = clock64();
        // rhs row of W: -wl in row RHS of tile row RT (other rows of that
        // tile row: coupling rows, stored by their owners)
        for (int t = tid; t < NX; t += NTH)
            Wsm[(C::RT * C::NXC + t / 8) * kTileElems + C::RR * 8 + t % 8] = mw[t];
        if (s + 2 < n)
            stage_BA_cta<NU, NX, NW, TMA>(g, a.p, b, g.stage_of(c, s + 2), sm, tid, bamb);
        bar_wait(4);
    };

    if (warp == 0) {
        // =====================================================================
        // PIVOT WARP
        // =====================================================================
        int baph = 1; // completed [B A] stagings (mbarrier phases)
        int fail_piv = -1, fail_stage = 0;
        Frag dg{0.0, 0.0};
#ifdef CYQ_TRACE
        // pivot-warp event clocks: a.phase[6144 + d * 8 + e] (stage CYQ_TRACE, chain 0)
        long long *ptrc = (a.phase && chain == 0 && tid == 0) ? a.phase + 6144 : nullptr;
#define PTRC(d, e) do { if (ptrc && s == CYQ_TRACE) ptrc[(d) * 8 + (e)] = clock64(); } while (0)
#else
#define PTRC(d, e) do { } while (0)
#endif
        // Factors the diagonal tile dg (L_kk, upper zeroed) and publishes
        // L_kk^{-1} -> linv[kb & 1], WITHOUT a shuffle: the tile goes through
        // shared memory into EVERY lane's registers (lower triangle, 36
        // doubles), every lane runs the same right-looking Cholesky on it, then
        // the lanes of row-quad rq back-substitute row rq of L^{-1} (x L = e_rq')
        // and pick their C-layout fragment of it. The shuffle version's ~14
        // SHFL per pivot queue behind the bulk warps' shared-memory traffic
        // (1.4k cycles in a quiet SM, 1.8k in this kernel); this one is the
        // rsqrt -> mul -> fma chain and ~200 FP64 instructions on an idle pipe.
        // L_kk leaves through tscr2 (stores of the same value by every lane).
        auto factor_diag = [&](int kb, double dfloor, int s, unsigned *flag) {
            st_frag(tscr, lane, dg);
            __syncwarp();
            double L[8][8], iv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j <= i; j += 2) {
                    const double2 v = *reinterpret_cast<const double2 *>(tscr + 8 * i + j);
                    L[i][j] = v.x;
                    if (j + 1 <= i)
                        L[i][j + 1] = v.y;
                }
            // column rq of X = L^{-1} rides along, one row behind the pivots:
            // x[i] = 0 (i < rq), iv[rq] (i = rq), else -iv[i] sum_{k < i} L[i][k]
            // x[k] (row i of L is final after pivot i-1) -- the same code in
            // every lane; only x[7] is left after the last pivot
            double x[8];
            double *xo = linvb + (kb & 1) * kTileElems + rq;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double pv = L[k][k];
                const bool first = !(pv > dfloor && isfinite(pv)) && fail_piv < 0;
                fail_piv = first ? 8 * kb + k : fail_piv;
                fail_stage = first ? s : fail_stage;
                iv[k] = rsqrt_nr(pv);
                if (k + 1 < 8) { // the next pivot first
                    L[k + 1][k] *= iv[k];
                    L[k + 1][k + 1] = fma(-L[k + 1][k], L[k + 1][k], L[k + 1][k + 1]);
                }
                L[k][k] = pv * iv[k];
#pragma unroll
                for (int i = k + 2; i < 8; ++i)
                    L[i][k] *= iv[k];
#pragma unroll
                for (int j = k + 1; j < 8; ++j)
#pragma unroll
                    for (int i = j; i < 8; ++i)
                        if (!(i == k + 1 && j == k + 1))
                            L[i][j] = fma(-L[i][k], L[j][k], L[i][j]);
                {
                    double t = 0.0;
#pragma unroll
                    for (int m = 0; m < k; ++m)
                        t = fma(L[k][m], x[m], t);
                    x[k] = k < rq ? 0.0 : (k == rq ? iv[k] : -iv[k] * t);
                    xo[8 * k] = x[k]; // X(k, rq): the four lanes of a quad store the same value
                }
            }
            PTRC(kb, 3);
            PTRC(kb, 4);
            flag_set(flag, s + 1, lane); // L_kk^{-1} is out: the bulk warps go on
            // L_kk -> tscr2 (row-major lower triangle; the upper part was
            // zero-filled at the start and is never written) -> dg
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j <= i; j += 2) {
                    if (j + 1 <= i)
                        *reinterpret_cast<double2 *>(tscr2 + 8 * i + j) = make_double2(L[i][j], L[i][j + 1]);
                    else
                        tscr2[8 * i + j] = L[i][j];
                }
            __syncwarp();
            dg = ld_frag(tscr2, lane);
        };
        // Block column d: the tiles (d, d-1) and (d, d) arrive from their
        // owner (hmb[d]; updates of the block columns < d-1 applied); L(d, d-1)
        // = X L_{d-1}^{-T} goes to column buffer (d-1) % 3 (every warp's
        // operand at step d-1) before the arrival at that step's barrier (ids
        // 1 + kb % 2: the arrival for step kb follows the completion of step
        // kb-2's barrier -- the hand-over waited for -- not of step kb-1's), to
        // the stored factor and to the x-space L_Q; then (d, d) -= L L',
        // factor, publish L_dd^{-1} (lmb[d]), store L_dd
        auto pivot_step = [&](int d, double dfloor, int s) {
            PTRC(d, 0);
            double *fdst = a.fac + ((size_t)chain * n + s) * C::NPT * kTileElems;
            if (d > 0)
                flag_wait(hmb + d, s + 1);
            dg = ld_frag(dgs + d * kTileElems, lane);
            if (d > 0) {
                double *slot = colb + (((d - 1) % 3) * TT + d) * kTileElems;
                const Frag x = ld_frag(slot, lane);
                const Frag linv = ld_frag(linvb + ((d - 1) & 1) * kTileElems, lane);
                Frag li{0.0, 0.0};
                tile_gemm_nt(li, x, linv);
                st_frag(slot, lane, li);
                bar_arrive(1 + ((d - 1) & 1));
                tile_gemm_nt_sub(dg, li, li);
                st_frag(fdst + C::PI(d, d - 1) * kTileElems, lane, li);
                if (d - 1 >= C::XT0) {
                    const int r = 8 * d + rq - NU, c0 = 8 * (d - 1) + cq - NU;
                    LQ[r * C::LQS + c0] = li.a;
                    LQ[r * C::LQS + c0 + 1] = li.b;
                }
            }
            PTRC(d, 1);
            factor_diag(d, dfloor, s, lmb + d);
            PTRC(d, 5);
            st_frag(fdst + C::PI(d, d) * kTileElems, lane, dg);
            if (d >= C::XT0) {
                const int r = 8 * d + rq - NU, c0 = 8 * d + cq - NU;
                LQ[r * C::LQS + c0] = dg.a;
                LQ[r * C::LQS + c0 + 1] = dg.b;
            }
        };
        for (int s = 0; s < n; ++s) {
            const StageIn in = stage_in(s);
            // every pivot diagonal tile H_s + W W' (two at a time: the 16 DMMAs
            // of a tile are one dependent chain) -> dgs[]; the pivot floor
            // 1e-14 max |diag| (kernels.cpp:21-29)
            double vmax = 0.0;
#pragma unroll 1
            for (int d = 0; d < CT; d += 2) {
                const int d1 = d + 1 < CT ? d + 1 : d;
                Frag t0 = tile0(d, d, s, in), t1 = tile0(d1, d1, s, in);
                if (s > 0) {
#pragma unroll
                    for (int kt = 0; kt < C::NXC; ++kt) {
                        const Frag w0 = ld_frag(Wsm + (d * C::NXC + kt) * kTileElems, lane);
                        const Frag w1 = ld_frag(Wsm + (d1 * C::NXC + kt) * kTileElems, lane);
                        dmma(t0, w0.a, w0.a);
                        dmma(t1, w1.a, w1.a);
                        dmma(t0, w0.b, w0.b);
                        dmma(t1, w1.b, w1.b);
                    }
                }
                const double v0 = (rq & 1) ? t0.b : t0.a, v1 = (rq & 1) ? t1.b : t1.a;
                vmax = fmax(vmax, ((lane & 3) == rq / 2) ? fmax(fabs(v0), fabs(v1)) : 0.0);
                st_frag(dgs + d * kTileElems, lane, t0);
                st_frag(dgs + d1 * kTileElems, lane, t1);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
            const double dfloor = 1e-14 * vmax;
            prefetch_next(s);
            // stage top: only an arrival for s > 0 (block column 0 starts while
            // the bulk warps finish W W'); at s = 0 the [B A] copy below
            // overwrites BA_0, still being read
            if (s > 0)
                bar_arrive(3);
            else
                bar_wait(3);
            if (s == 0 && n > 1)
                stage_BA_cta<NU, NX, NW, TMA>(g, a.p, b, g.stage_of(c, 1), sm, tid, bamb);
#pragma unroll 1
            for (int d = 0; d < CT; ++d)
                pivot_step(d, dfloor, s);
            bar_arrive(1 + ((CT - 1) & 1)); // barrier of the last block column
            if (s + 1 < n)
                next_W(s, baph, nullptr);
        }
        unsigned long long my_fail = fail_piv >= 0 ? fail_key(kKindRiccati, c, fail_stage, fail_piv) : ~0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            my_fail = min(my_fail, __shfl_xor_sync(0xffffffffu, my_fail, o));
        if (lane == 0 && my_fail != ~0ull)
            atomicMin(a.fail + b, my_fail);
#undef PTRC
        return;
    }

    // =========================================================================
    // BULK WARPS
    // =========================================================================
    int baph = 1;
    const int dkb = (warp & 3) ? (warp >> 2) * 3 + (warp & 3) - 1 : -1;
    const bool diag_owner = dkb >= 0 && dkb < CT;
    // my list tiles: opk[k] = byte offsets of the (ti, tj) slots in a column
    // buffer, ti in the low half (compile-time k everywhere: plain registers).
    // The packed words pass through an empty asm so that the compiler keeps
    // them in registers: it otherwise re-reads the constant bank, ~100+
    // cycles per indexed load, at the top of every block-column step
    unsigned lpk[kLW];
#pragma unroll
    for (int i = 0; i < kLW; ++i) {
        lpk[i] = c_lpk[warp * kLW + i];
        asm volatile("" : "+r"(lpk[i]));
    }
    unsigned opk[MAXL];
#pragma unroll
    for (int k = 0; k < MAXL; ++k) {
        const unsigned e = (lpk[k / 3] >> (10 * (k % 3))) & 1023u;
        opk[k] = ((e & 31u) << 9) | ((e >> 5) << 25);
    }
    unsigned long long cpk = c_cpk[warp];
    asm volatile("" : "+l"(cpk));
    unsigned ppk[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        ppk[i] = c_ppk[warp * 4 + i];
        asm volatile("" : "+r"(ppk[i]));
    }
#define PIK(k) ((ppk[(k) / 4] >> (8 * ((k) % 4))) & 255u)
    const int mycnt = (int)(cpk & 15u);
#define LTI(k) ((int)((opk[k] >> 9) & 31u))
#define LTJ(k) ((int)(opk[k] >> 25))
#define CNT(kb) ((int)((cpk >> (4 * (kb))) & 15u))
    Frag acc[MAXL];
#pragma unroll
    for (int k = 0; k < MAXL; ++k)
        acc[k] = Frag{0.0, 0.0};
    Frag dg{0.0, 0.0}, sd{0.0, 0.0};
    long long *ph = (a.phase && chain == 0 && tid == 32) ? a.phase : nullptr; // a bulk warp's view
#ifdef CYQ_TRACE
    // per-warp event clocks of the column loop at stage CYQ_TRACE (chain 0):
    // a.phase[4096 + ((kb * NW + warp) * 8 + e)]
    long long *trc = (a.phase && chain == 0 && lane == 0) ? a.phase + 4096 : nullptr;
#define TRC(e) do { if (trc && s == CYQ_TRACE) trc[(kb * NW + warp) * 8 + (e)] = clock64(); } while (0)
#else
#define TRC(e) do { } while (0)
#endif
    for (int s = 0; s < n; ++s) {
        if (ph) ph[s * 8 + 0] = clock64();
        const StageIn in = stage_in(s);
        // ---- init (H_s from global, coupling rows BA_0 at s = 0, rhs row) and
        // += W W' (s > 0): first the tile left of my diagonal tile (the owner
        // of (1, 0) hands it over at once: block column 0 updates nothing of
        // it), then my list tiles. The tiles the pivot warp takes over go
        // through shared memory: (dkb, dkb-1) into its slot of column buffer
        // (dkb-1) % 3, (dkb, dkb) back into dgs[]
        auto hand_over = [&]() {
            if (dkb >= 2)
                st_frag(dgs + dkb * kTileElems, lane, dg);
            st_frag(colb + (((dkb - 1) % 3) * TT + dkb) * kTileElems, lane, sd);
            flag_set(hmb + dkb, s + 1, lane);
        };
        if (diag_owner && dkb > 0) {
            sd = tile0(dkb, dkb - 1, s, in);
            if (s > 0) {
#pragma unroll
                for (int kt = 0; kt < C::NXC; ++kt) {
                    const Frag wi = ld_frag(Wsm + (dkb * C::NXC + kt) * kTileElems, lane);
                    const Frag wj = ld_frag(Wsm + ((dkb - 1) * C::NXC + kt) * kTileElems, lane);
                    tile_gemm_nt(sd, wi, wj);
                }
            }
            if (dkb == 1)
                hand_over();
        }
#pragma unroll
        for (int k = 0; k < MAXL; ++k) {
            if (k >= mycnt)
                break;
            const int ti = LTI(k), tj = LTJ(k);
            if (tj < CT)
                acc[k] = tile0(ti, tj, s, in);
        }
        if (s > 0) {
#pragma unroll
            for (int k = C::NPS; k < MAXL; ++k) { // skip-mode pure tiles: no W W'
                if (k >= mycnt)
                    break;
                const int ti = LTI(k), tj = LTJ(k);
#pragma unroll
                for (int kt = 0; kt < C::NXC; ++kt) {
                    const Frag wi = ld_frag(Wsm + (ti * C::NXC + kt) * kTileElems, lane);
                    const Frag wj = ld_frag(Wsm + (tj * C::NXC + kt) * kTileElems, lane);
                    tile_gemm_nt(acc[k], wi, wj);
                }
            }
        }
        prefetch_next(s);
        if (ph) ph[s * 8 + 1] = clock64();
        bar_wait(3); // W and BA_0 reads done, dgs[] written
        if (s == 0 && n > 1)
            stage_BA_cta<NU, NX, NW, TMA>(g, a.p, b, g.stage_of(c, 1), sm, tid, bamb);
        if (diag_owner && dkb >= 2)
            dg = ld_frag(dgs + dkb * kTileElems, lane);

        // ---- blocked Cholesky, the pivot chain decoupled --------------------
        // Per block column kb a bulk warp waits for L_kk^{-1} (lmb[kb]),
        // solves its own (complete) column-kb tiles in registers (X <- X
        // L_kk^{-T}, two DMMAs) into column buffer kb % 3, passes the step's
        // barrier, brings its (dkb, dkb) / (dkb, dkb-1) up to date (handing
        // them over at kb = dkb - 2) and applies column kb to its list prefix.
        // The pivot warp meanwhile runs block column kb + 1. Buffer kb % 3 is
        // next written at step kb + 3: by the owners' hand-over during the
        // trailing updates of step kb + 1, i.e. after the barrier of step kb +
        // 1, which every warp reaches with its reads of step kb done.
        // (per-step values carried along instead of recomputed: the chain of
        // dependent integer instructions at the loop top was ~150 cycles)
        unsigned long long cw = cpk;
        int cb = 0;
#pragma unroll 1
        for (int kb = 0; kb < CT; ++kb) {
            const int par = kb & 1;
            double *col = colb + cb * TT * kTileElems;
            cb = cb == 2 ? 0 : cb + 1;
            TRC(0);
            const int hi = (int)((unsigned)cw & 15u);
            cw >>= 4;
            const int cnt = (int)((unsigned)cw & 15u);
            const unsigned colS = smem_u32(col) + 16 * lane;
            auto lds = [](unsigned a) {
                Frag f;
                asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(f.a), "=d"(f.b) : "r"(a) : "memory");
                return f;
            };
            auto sts = [](unsigned a, const Frag &f) {
                asm volatile("st.shared.v2.f64 [%0], {%1,%2};" ::"r"(a), "d"(f.a), "d"(f.b) : "memory");
            };
            // (A) my column-kb tiles: list positions [cnt, hi), straight-line
            // code entered at slot cnt through a compare tree (a walk over
            // the unrolled list costs issue slots for every slot it skips, a
            // switch becomes a jump table: an indexed constant load per step)
            // a solved tile of the x columns also feeds stage s+1: L_Q (x block of
            // the pivot tiles) -> LQ (x-space, row-major), ALQ rows (coupling rows)
            // -> W tile rows >= CT (both next read after this stage's block columns)
            auto fill_next = [&](unsigned o, const Frag &r) {
                const int ti = (int)((o >> 9) & 31u), tj = (int)(o >> 25);
                if (s + 1 < n && tj >= C::XT0) {
                    if (ti < CT) {
                        const int rr = 8 * ti + rq - NU, c0 = 8 * tj + cq - NU;
                        LQ[rr * C::LQS + c0] = r.a;
                        LQ[rr * C::LQS + c0 + 1] = r.b;
                    } else
                        st_frag(Wsm + (ti * C::NXC + (tj - C::XT0)) * kTileElems, lane, r);
                }
            };
            if (hi > cnt) {
                double *fdst = a.fac + ((size_t)chain * n + s) * C::NPT * kTileElems;
                flag_wait(lmb + kb, s + 1);
                TRC(5);
                const Frag linv = ld_frag(linvb + par * kTileElems, lane);
                TRC(7);
#define SOLVE_AT(K)                                                                                    \
    SV_##K : if constexpr (K < MAXL) {                                                                 \
        if (K >= hi)                                                                                   \
            goto SV_END;                                                                               \
        constexpr int T = K < MAXL ? K : 0;                                                            \
        Frag r{0.0, 0.0};                                                                              \
        tile_gemm_nt(r, acc[T], linv);                                                                 \
        acc[T] = r;                                                                                    \
        sts(colS + (opk[T] & 0xffffu), r);                                                             \
        st_frag(fdst + PIK(T) * kTileElems, lane, r);                                                  \
        fill_next(opk[T], r);                                                                          \
    }
                if (cnt < 8) {
                    if (cnt < 4) {
                        if (cnt < 2) {
                            if (cnt == 0)
                                goto SV_0;
                            goto SV_1;
                        }
                        if (cnt == 2)
                            goto SV_2;
                        goto SV_3;
                    }
                    if (cnt < 6) {
                        if (cnt == 4)
                            goto SV_4;
                        goto SV_5;
                    }
                    if (cnt == 6)
                        goto SV_6;
                    goto SV_7;
                }
                if (cnt < 12) {
                    if (cnt < 10) {
                        if (cnt == 8)
                            goto SV_8;
                        goto SV_9;
                    }
                    if (cnt == 10)
                        goto SV_10;
                    goto SV_11;
                }
                if (cnt < 13)
                    goto SV_12;
                if (cnt < 14)
                    goto SV_13;
                goto SV_14;
                SOLVE_AT(0) SOLVE_AT(1) SOLVE_AT(2) SOLVE_AT(3) SOLVE_AT(4) SOLVE_AT(5) SOLVE_AT(6) SOLVE_AT(7)
                SOLVE_AT(8) SOLVE_AT(9) SOLVE_AT(10) SOLVE_AT(11) SOLVE_AT(12) SOLVE_AT(13) SOLVE_AT(14)
            SV_END:;
#undef SOLVE_AT
            }
            TRC(1);
            bar_wait(1 + par); // column kb solved (the pivot warp's tile (kb+1, kb) included)
            TRC(2);
            // (B) the diagonal-tile owners apply column kb to (dkb, dkb) and
            // (dkb, dkb-1); the owner of block column kb+2's hands them over
            if (diag_owner && dkb > kb + 1) {
                const Frag li = ld_frag(col + dkb * kTileElems, lane);
                const Frag lj = ld_frag(col + (dkb - 1) * kTileElems, lane);
                tile_gemm_nt_sub(dg, li, li);
                tile_gemm_nt_sub(sd, li, lj);
                if (dkb == kb + 2)
                    hand_over();
            }
            TRC(3);
            // trailing update of my prefix: C(ti, tj) -= L(ti, kb) L(tj, kb)',
            // tiles cnt-1 .. 0 (.. NPS when the ALQ ALQ' terms cancel on the
            // pure tiles)
            {
                const bool skip = kb >= C::XT0 && s + 1 < n;
#define UPD_CASE(K)                                                                                    \
    case K:                                                                                            \
        if constexpr (K <= MAXL && K >= 1) {                                                           \
            if (K == C::NPS && skip)                                                                   \
                break;                                                                                 \
            constexpr int T = (K >= 1 && K <= MAXL) ? K - 1 : 0;                                       \
            const Frag li = lds(colS + (opk[T] & 0xffffu)), lj = lds(colS + (opk[T] >> 16));           \
            tile_gemm_nt_sub(acc[T], li, lj);                                                          \
        }
                switch ((skip && cnt <= C::NPS) ? 0 : cnt) {
                    UPD_CASE(15) UPD_CASE(14) UPD_CASE(13) UPD_CASE(12) UPD_CASE(11) UPD_CASE(10) UPD_CASE(9)
                    UPD_CASE(8) UPD_CASE(7) UPD_CASE(6) UPD_CASE(5) UPD_CASE(4) UPD_CASE(3) UPD_CASE(2)
                    UPD_CASE(1)
                default: break;
                }
#undef UPD_CASE
            }
            TRC(4);
        }
        if (ph) ph[s * 8 + 2] = clock64();

        // ---- y_s' (the factor tiles and the x-column tiles stage s+1 needs went
        // out as they were solved)
        {
#pragma unroll
            for (int k = 0; k < MAXL; ++k) {
                if (k >= mycnt)
                    break;
                const int ti = LTI(k), tj = LTJ(k);
                if (tj < CT && ti == C::RT && rq == C::RR) {
                    double *yv = a.y + ((size_t)chain * n + s) * C::NUX;
                    yv[8 * tj + cq] = acc[k].a;
                    yv[8 * tj + cq + 1] = acc[k].b;
                    if (tj >= C::XT0) {
                        yx[8 * tj + cq - NU] = acc[k].a;
                        yx[8 * tj + cq + 1 - NU] = acc[k].b;
                    }
                }
            }
        }
        if (ph) ph[s * 8 + 3] = clock64();

        if (s + 1 < n) {
            // ---- W for stage s+1 (L_Q and the ALQ rows went out as they were solved)
            next_W(s, baph, ph);
        }
    }

    if (ph) ph[n * 8] = clock64();
    // trailing tiles (coupling x coupling = -Mfwd, rhs x coupling = -fwd)
#pragma unroll
    for (int k = 0; k < MAXL; ++k) {
        if (k >= mycnt)
            break;
        const int ti = LTI(k), tj = LTJ(k);
        if (tj >= CT)
            st_frag(a.trail + ((size_t)chain * g.NTT + C::T(ti - CT, tj - CT)) * kTileElems, lane,
                    acc[k]);
    }
#undef LTI
#undef LTJ
#undef CNT
#undef PIK
#undef TRC
}

namespace {
constexpr int kPL = 32; // plan-time list stride

// Host tile plan of the CTA panel: h[w * kPL + k] = (ti << 8 | tj) of warp
// w's list slot k, nown[w] its tile count, cnt[w * (kMaxCT + 1) + kb] the
// number of its tiles with tile column >= kb ... see the comment inside.
// Returns false if the plan does not place every list tile once within MAXL
// slots per warp in tile-column-descending order (tests/test_cta_plan.py
// checks the rest through cyqb_debug_cta_plan).
template <class C, int NW> bool plan_tiles(unsigned short *h, unsigned char *cnt, int *nown) {
    std::fill(h, h + kMaxW * kPL, (unsigned short)0);
    std::fill(cnt, cnt + kMaxW * (kMaxCT + 1), (unsigned char)0);
    std::fill(nown, nown + kMaxW, 0);
    {
        // tile plan. The skip-mode pure tiles go first (NPS per warp at slots
        // 0 .. NPS-1; they take trailing updates only from the u columns, kb <
        // XT0); the pivot warp (0) holds no tile. The other warps of its SM
        // sub-partition (w % 4 == 0) then fill up with the tiles of the first
        // block columns -- column 0 (never updated) first -- so that
        // sub-partition issues no DMMA after the first steps and the pivot
        // chain's FP64 instructions are not queued behind any. Every
        // other tile goes, in tile-column-descending order, to the bulk warp
        // that minimises the modelled time sum_kb max(DMMA issue per bulk
        // sub-partition). Lists stay in tile-column-descending order.
        double load[kMaxW][kMaxCT] = {};
        const double kUpd = 2 * 16.0; // cycles: one tile update
        auto quiet = [&](int w) { return w % 4 == 0; };
        auto cost = [&]() {
            double t = 0;
            for (int kb = 0; kb < C::CT; ++kb) {
                double sp[4] = {};
                for (int w = 0; w < NW; ++w)
                    sp[w % 4] += load[w][kb];
                t += std::max(std::max(sp[1], sp[2]), sp[3]);
            }
            return t;
        };
        bool placed[64][64] = {};
        auto give = [&](int w, int ti, int tj, int upd_cols) {
            for (int kb = 0; kb < upd_cols; ++kb)
                load[w][kb] += kUpd;
            h[w * kPL + nown[w]++] = (unsigned short)((ti << 8) | tj);
            placed[ti][tj] = true;
        };
        {
            int w = 0; // the pivot warp (0) holds no tile
            for (int tj = C::RT - 1; tj >= C::CT && C::NPS > 0; --tj)
                for (int ti = C::RT - 1; ti >= tj; --ti) {
                    if (w >= (NW - 1) * C::NPS)
                        break;
                    give(1 + w % (NW - 1), ti, tj, C::XT0);
                    ++w;
                }
        }
        {
            // quiet sub-partition: the pivot warp fills up with column-0
            // tiles, the others take block columns 0, 1, 2, ... round-robin
            // until their slots are full
            std::vector<int> quiet_part[kMaxW];
            int room[kMaxW] = {};
            for (int w = 4; w < NW; w += 4)
                room[w] = C::MAXL - nown[w];
            int w = 4 % NW;
            for (int tj = 0; tj < C::CT; ++tj)
                for (int ti = tj + 2; ti < C::TT; ++ti) { // (tj+1, tj) is the pivot warp's
                    int q = -1;
                    if (tj == 0 && room[0] > 0)
                        q = 0;
                    else
                        for (int t = 0; t < NW / 4 && q < 0; ++t, w = (w + 4) % NW)
                            if (w != 0 && room[w] > 0)
                                q = w;
                    if (q < 0)
                        continue;
                    if (q != 0)
                        w = (q + 4) % NW;
                    quiet_part[q].push_back((ti << 8) | tj);
                    placed[ti][tj] = true;
                    --room[q];
                }
            // column-descending order inside each list
            for (int q = 0; q < NW; q += 4) {
                std::stable_sort(quiet_part[q].begin(), quiet_part[q].end(),
                                 [](int x, int y) { return (x & 255) > (y & 255); });
                for (int e : quiet_part[q]) {
                    placed[e >> 8][e & 255] = false;
                    give(q, e >> 8, e & 255, std::min(e & 255, C::CT));
                }
            }
        }
        for (int tj = C::TT - 1; tj >= 0; --tj)
            for (int ti = C::TT - 1; ti >= tj; --ti) {
                if ((ti == tj && tj < C::CT) || (ti == tj + 1 && ti < C::CT) || placed[ti][tj])
                    continue;
                int best = -1;
                double bc = 0;
                for (int w = 0; w < NW; ++w) {
                    if (quiet(w) || nown[w] >= C::MAXL)
                        continue;
                    for (int kb = 0; kb < std::min(tj, C::CT); ++kb)
                        load[w][kb] += kUpd;
                    const double cw = cost() + 1e-3 * nown[w];
                    for (int kb = 0; kb < std::min(tj, C::CT); ++kb)
                        load[w][kb] -= kUpd;
                    if (best < 0 || cw < bc)
                        best = w, bc = cw;
                }
                if (best < 0) { // bulk warps full: a quiet warp (not the pivot warp) takes it
                    for (int w = 4; w < NW && best < 0; w += 4)
                        if (nown[w] < C::MAXL)
                            best = w;
                    if (best < 0)
                        return false;
                    // keep its list in column-descending order: insert before lower columns
                    int pos = nown[best];
                    while (pos > C::NPS && (h[best * kPL + pos - 1] & 255) < tj) {
                        h[best * kPL + pos] = h[best * kPL + pos - 1];
                        --pos;
                    }
                    h[best * kPL + pos] = (unsigned short)((ti << 8) | tj);
                    ++nown[best];
                    placed[ti][tj] = true;
                    for (int kb = 0; kb < std::min(tj, C::CT); ++kb)
                        load[best][kb] += kUpd;
                    continue;
                }
                give(best, ti, tj, std::min(tj, C::CT));
            }
        // the plan must place every list tile once, within MAXL slots per
        // warp, tile columns non-increasing from slot NPS on
        {
            int seen = 0;
            for (int w = 0; w < NW; ++w) {
                if (nown[w] > C::MAXL)
                    return false;
                for (int k = 0; k < nown[w]; ++k) {
                    ++seen;
                    if (k > C::NPS && (h[w * kPL + k] & 255) > (h[w * kPL + k - 1] & 255))
                        return false;
                }
            }
            if (seen != C::NL)
                return false;
        }
        for (int w = 0; w < NW; ++w) {
            cnt[w * (kMaxCT + 1)] = (unsigned char)nown[w];
            for (int kb = 0; kb < C::CT; ++kb) {
                int m = 0;
                for (int k = 0; k < nown[w]; ++k)
                    m += (h[w * kPL + k] & 255) > kb;
                cnt[w * (kMaxCT + 1) + kb + 1] = (unsigned char)m;
            }
        }
    }
    return true;
}

template <int NU, int NX, int NW, bool TMA> bool launch_c(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    if (g.nu != NU || g.nx != NX)
        return false;
    using C = CS<NU, NX, NW>;
    const size_t smem = (size_t)C::SMEM * sizeof(double);
    static DeviceOnce once;
    once_per_device(once, [&]() -> cudaError_t {
        const cudaError_t e0 = cudaFuncSetAttribute(riccati_cta_kernel<NU, NX, NW, TMA>,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e0 != cudaSuccess)
            return e0;
        unsigned short h[kMaxW * kPL];
        unsigned char cnt[kMaxW * (kMaxCT + 1)];
        int nown[kMaxW];
        if (!plan_tiles<C, NW>(h, cnt, nown))
            return cudaErrorInvalidValue;
        unsigned lpk[kMaxW * kLW] = {};
        unsigned long long cpk[kMaxW] = {};
        for (int w = 0; w < NW; ++w) {
            for (int k = 0; k < nown[w]; ++k) {
                const unsigned ti = h[w * kPL + k] >> 8, tj = h[w * kPL + k] & 255;
                lpk[w * kLW + k / 3] |= (ti | (tj << 5)) << (10 * (k % 3));
            }
            for (int kb = 0; kb < 16; ++kb) // counts past CT repeat the last one (nothing to publish)
                cpk[w] |= (unsigned long long)cnt[w * (kMaxCT + 1) + std::min(kb, C::CT)] << (4 * kb);
        }
        unsigned ppk[kMaxW * 4] = {};
        static_assert(C::NPT <= 256 && kMaxL <= 16, "stored-tile indices packed as bytes");
        for (int w = 0; w < NW; ++w)
            for (int k = 0; k < nown[w]; ++k) {
                const int ti = h[w * kPL + k] >> 8, tj = h[w * kPL + k] & 255;
                if (tj < C::CT)
                    ppk[w * 4 + k / 4] |= (unsigned)C::PI(ti, tj) << (8 * (k % 4));
            }
        cudaError_t e1 = cudaMemcpyToSymbol(c_lpk, lpk, sizeof lpk);
        if (e1 == cudaSuccess)
            e1 = cudaMemcpyToSymbol(c_ppk, ppk, sizeof ppk);
        return e1 != cudaSuccess ? e1 : cudaMemcpyToSymbol(c_cpk, cpk, sizeof cpk);
    });
    riccati_cta_kernel<NU, NX, NW, TMA><<<ra.grid_chains(), 32 * NW, smem, st>>>(ra);
    return true;
}
} // namespace

// tma: stage [B A] with TMA bulk copies instead of cp.async (opt-in,
// CYQ_PANEL_CTA_TMA: measured 35.2 vs 32.3 ms at config 3)
bool launch_riccati_cta(const Geo &g, cudaStream_t st, const RiccatiArgs &ra, bool tma) {
    // 16 warps per chain CTA: 13 / 14 / 20 / 24 warps measured 38.6 / 36.3
    // / 37.9 / 38.9 ms vs 32.3 ms at config 3
    return tma ? launch_c<32, 64, 16, true>(g, st, ra) : launch_c<32, 64, 16, false>(g, st, ra);
}

} // namespace cyqb

// Not part of the C ABI (include/cyqlone_b200.h): the config-3 tile plan for
// tests/test_cta_plan.py -- lists[16 * 32] = (ti << 8 | tj), counts[16 * 16],
// nown[16], dims[6] = {TT, CT, RT, MAXL, NPS, NW}. Returns 0 if the plan is valid.
extern "C" int cyqb_debug_cta_plan(unsigned short *lists, unsigned char *counts, int *nown, int *dims) {
    using C = cyqb::CS<32, 64, 16>;
    dims[0] = C::TT, dims[1] = C::CT, dims[2] = C::RT, dims[3] = C::MAXL, dims[4] = C::NPS, dims[5] = 16;
    return cyqb::plan_tiles<C, 16>(lists, counts, nown) ? 0 : 1;
}
