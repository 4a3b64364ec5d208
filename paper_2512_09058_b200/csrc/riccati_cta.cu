// CTA-per-chain stage-panel Riccati kernel for LARGE stage blocks with
// tile-aligned dimensions (nu % 8 == 0, nx % 8 == 0; BASELINE config 3:
// nu = 32, nx = 64, nux = 96 -- the dense DMMA regime). Same algorithm and
// outputs as riccati_warp.cu / riccati.cu:
//   kkt_factor.cpp:125-158  modified Riccati recursion (LH, LB, Acl, LA)
//   kkt_factor.cpp:163-185  Mfwd = sum LB LB' + LA LA' (trailing block)
//   kkt_solve.cpp:72-134    forward substitution + coupling rows (rhs row)
//
// Execution model (one CTA of NW warps per partition column):
//  * the extended panel (TT x TT lower tiles, 231 at config 3) is owned
//    tile-by-tile by the warps (tile t -> warp t % NW) and lives in their
//    registers for the stage (coupling x coupling tiles for the chain);
//  * blocked Cholesky, per pivot block column kb: the owner of (kb, kb)
//    factors it with an identity tile carried through the pivot steps
//    (L_kk^{-1} for free) and publishes L_kk^{-1}; the owners of the
//    sub-diagonal tiles solve them by two DMMAs and publish the column;
//    every owner applies C -= L_i L_j' to its trailing tiles. The owner of
//    (kb+1, kb+1) updates and factors it FIRST (look-ahead), so the next
//    pivot chain overlaps this column's trailing DMMAs; the column buffer
//    is double-buffered by kb parity -> two __syncthreads per block column;
//  * shared memory holds W = [V; ALQ; -wl] (the next stage's W W' operand),
//    [B A] of the next stage (cp.async, one stage ahead), L_Q in x-space
//    (the B operand of V = BA' L_Q) and the column buffers; H_s is read
//    straight from global memory (L2-prefetched one stage ahead).
#include "kkt_common.cuh"
#include "kernels.h"
#include "riccati_common.cuh"

#include <cstdlib>

namespace cyqb {

using namespace cyqb::ric;

namespace {

// (ti << 8 | tj) of lower-triangular tile t = ti (ti + 1) / 2 + tj
__constant__ unsigned short c_tij[1024];

template <int NU, int NX, int NW> struct CS {
    static_assert(NU % 8 == 0 && NX % 8 == 0, "tile-aligned shapes only");
    static constexpr int NUX = NU + NX;
    static constexpr int CT = NUX / 8;            // pivot tile columns
    static constexpr int BT = (NX + 1 + 7) / 8;   // coupling + rhs tile rows
    static constexpr int TT = CT + BT;
    static constexpr int NT = TT * (TT + 1) / 2;
    static constexpr int TOP = 8 * CT, RHS = TOP + NX, RT = RHS / 8, RR = RHS % 8;
    static constexpr int XT0 = NU / 8, NXC = NX / 8; // x columns: tiles XT0 .. CT-1
    static constexpr int NPT = CT * (CT + 1) / 2 + BT * CT;
    static constexpr int MAXT = (NT + NW - 1) / NW;
    static constexpr int PW = NUX;                 // [B A] row length
    // shared memory (doubles)
    static constexpr int O_W = 0;                                  // TT x NXC tiles
    static constexpr int O_COL = O_W + TT * NXC * kTileElems;      // 2 x TT tiles
    static constexpr int O_LINV = O_COL + 2 * TT * kTileElems;     // 2 tiles (by kb parity)
    static constexpr int O_BA = O_LINV + 2 * kTileElems;           // NX x PW
    static constexpr int O_LQ = O_BA + NX * PW;                    // NX x NX (x-space L_Q)
    static constexpr int O_F = O_LQ + NX * NX;                     // NX
    static constexpr int O_YX = O_F + NX;                          // NX (x part of y)
    static constexpr int O_MW = O_YX + NX;                         // NX (-wl_new)
    static constexpr int O_RU0 = O_MW + NX;                        // NU
    static constexpr int O_RED = O_RU0 + NU;                       // 32 (pivot floor)
    static constexpr int O_SCR = O_RED + 32;                       // 2 x 64 (transpose, by parity)
    static constexpr int SMEM = O_SCR + 2 * kTileElems;
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

// [B A]_j -> BA rows (A omitted for j = 0, zero for padding stages), f_j
template <int NU, int NX, int NW>
__device__ __forceinline__ void stage_BA_cta(const Geo &g, const ProbView &p, int b, int j, double *sm,
                                             int tid) {
    using C = CS<NU, NX, NW>;
    constexpr int NTH = 32 * NW;
    const int N = g.N;
    double *ba = sm + C::O_BA;
    const bool in = j < N;
    const double *Bs = in ? p.B + ((size_t)b * N + j) * NX * NU : nullptr;
    const double *As = (in && j != 0) ? p.A + ((size_t)b * N + j) * NX * NX : nullptr;
    const bool al = ((reinterpret_cast<uintptr_t>(Bs) | reinterpret_cast<uintptr_t>(As)) & 15) == 0;
    for (int e = 2 * tid; e < NX * NU; e += 2 * NTH) {
        double *d = ba + (e / NU) * C::PW + e % NU;
        if (Bs && al)
            cp16(d, Bs + e);
        else if (Bs) {
            cp8(d, Bs + e);
            cp8(d + 1, Bs + e + 1);
        } else
            d[0] = d[1] = 0.0;
    }
    for (int e = 2 * tid; e < NX * NX; e += 2 * NTH) {
        double *d = ba + (e / NX) * C::PW + NU + e % NX;
        if (As && al)
            cp16(d, As + e);
        else if (As) {
            cp8(d, As + e);
            cp8(d + 1, As + e + 1);
        } else
            d[0] = d[1] = 0.0;
    }
    const double *fs = (p.fd ? p.fd : p.f);
    for (int e = tid; e < NX; e += NTH) {
        if (in)
            cp8(sm + C::O_F + e, fs + ((size_t)b * N + j) * NX + e);
        else
            sm[C::O_F + e] = 0.0;
    }
}

} // namespace

template <int NU, int NX, int NW>
__global__ void __launch_bounds__(32 * NW, 1) riccati_cta_kernel(RiccatiArgs a) {
    using C = CS<NU, NX, NW>;
    constexpr int NTH = 32 * NW, MAXT = C::MAXT, CT = C::CT, TT = C::TT, NT = C::NT;
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int chain = blockIdx.x;
    const int b = chain / g.P, c = chain % g.P, n = g.n, N = g.N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rq = lane >> 2, cq = 2 * (lane & 3), q2 = lane & 3;
    double *Wsm = sm + C::O_W, *colb = sm + C::O_COL, *linvb = sm + C::O_LINV, *BA = sm + C::O_BA;
    double *LQ = sm + C::O_LQ, *fb = sm + C::O_F, *yx = sm + C::O_YX, *mw = sm + C::O_MW;
    double *ru0 = sm + C::O_RU0;
    unsigned long long *red = reinterpret_cast<unsigned long long *>(sm + C::O_RED);
    double *tscr = sm + C::O_SCR;
    const bool implicit_rhs = (a.p.ru == nullptr);
    const double sgn = implicit_rhs ? -1.0 : 1.0;
    int fail_piv = -1, fail_stage = 0;

    // my tiles: t = warp + k NW -> (ti, tj) from the constant-memory table
    // of the triangular enumeration (warp-uniform loads, no index registers)
#define mtt(k) (warp + (k) * NW)
#define mt(k) (mtt(k) < NT ? (int)c_tij[mtt(k)] : -1)
#define mti(k) (mtt(k) < NT ? (int)(c_tij[mtt(k)] >> 8) : -1)
#define mtj(k) (mtt(k) < NT ? (int)(c_tij[mtt(k)] & 255) : -1)
    for (int i = tid; i < C::SMEM; i += NTH)
        sm[i] = 0.0;
    __syncthreads();
    // prologue: BA_0, S_0 x_init (ru[0] term)
    {
        const int j0 = g.stage_of(c, 0);
        stage_BA_cta<NU, NX, NW>(g, a.p, b, j0, sm, tid);
        cp_commit();
        if (implicit_rhs && c == 0)
            for (int i = tid; i < NU; i += NTH) {
                double s0 = 0;
                for (int k = 0; k < NX; ++k)
                    s0 += __ldg(a.p.S + (size_t)b * N * NU * NX + i * NX + k) *
                          __ldg(a.p.x_init + (size_t)b * NX + k);
                ru0[i] = s0;
            }
        cp_wait<0>();
    }
    __syncthreads();

    Frag acc[MAXT];
#pragma unroll
    for (int k = 0; k < MAXT; ++k)
        acc[k] = Frag{0.0, 0.0};

    for (int s = 0; s < n; ++s) {
        const int j = g.stage_of(c, s), xi = g.x_index_of(c, s);
        const bool j0 = j == 0, in = j < N, qin = xi <= N;
        const double *Rg = in ? a.p.R + ((size_t)b * N + j) * NU * NU : nullptr;
        const double *Sg = (in && !j0) ? a.p.S + ((size_t)b * N + j) * NU * NX : nullptr;
        const double *Qg = qin ? a.p.Q + ((size_t)b * (N + 1) + xi) * NX * NX : nullptr;
        const double *rg = in ? (a.p.ru ? a.p.ru : a.p.r) + ((size_t)b * N + j) * NU : nullptr;
        const double *qg = qin ? (a.p.qx ? a.p.qx : a.p.q) + ((size_t)b * (N + 1) + xi) * NX : nullptr;
        const double *ru0p = (implicit_rhs && j0) ? ru0 : nullptr;
        const bool aligned = ((reinterpret_cast<uintptr_t>(a.p.R) | reinterpret_cast<uintptr_t>(a.p.Q)) & 15) == 0;
        // ---- init (H_s from global, coupling rows BA_0 at s = 0, rhs row) ---
#pragma unroll
        for (int k = 0; k < MAXT; ++k) {
            const int ti = mti(k), tj = mtj(k);
            if (ti < 0 || tj >= CT)
                continue;
            Frag f{0.0, 0.0};
            const int r = 8 * ti + rq, c0 = 8 * tj + cq;
            if (ti < CT) {
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
                        const double2 v =
                            __ldg(reinterpret_cast<const double2 *>(Qg + (r - NU) * NX + (c0 - NU)));
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
            acc[k] = f;
        }
        // ---- += W W' (s > 0) --------------------------------------------
        if (s > 0) {
#pragma unroll
            for (int k = 0; k < MAXT; ++k) {
                const int ti = mti(k), tj = mtj(k);
                if (ti < 0)
                    continue;
#pragma unroll
                for (int kt = 0; kt < C::NXC; ++kt) {
                    const Frag wi = ld_frag(Wsm + (ti * C::NXC + kt) * kTileElems, lane);
                    const Frag wj = ld_frag(Wsm + (tj * C::NXC + kt) * kTileElems, lane);
                    tile_gemm_nt(acc[k], wi, wj);
                }
            }
        }
        // prefetch H_{s+1} into L2; BA_1 at s = 0 (BA_0 has been read)
        if (s + 1 < n) {
            const int j1 = g.stage_of(c, s + 1), x1 = g.x_index_of(c, s + 1);
            if (j1 < N) {
                pf_lines(a.p.R + ((size_t)b * N + j1) * NU * NU, NU * NU * 8, tid, NTH);
                pf_lines(a.p.S + ((size_t)b * N + j1) * NU * NX, NU * NX * 8, tid, NTH);
            }
            if (x1 <= N)
                pf_lines(a.p.Q + ((size_t)b * (N + 1) + x1) * NX * NX, NX * NX * 8, tid, NTH);
        }
        __syncthreads(); // W and BA_0 reads done
        if (s == 0 && n > 1)
            stage_BA_cta<NU, NX, NW>(g, a.p, b, g.stage_of(c, 1), sm, tid);
        cp_commit();
        // ---- pivot floor: max |diag| (kernels.cpp:21-29) ---------------------
#pragma unroll
        for (int k = 0; k < MAXT; ++k)
            if (mti(k) >= 0 && mti(k) == mtj(k) && mti(k) < CT && (lane & 3) == rq / 2) {
                const double v = (rq & 1) ? acc[k].b : acc[k].a;
                atomicMax(red + (lane & 31), (unsigned long long)__double_as_longlong(fabs(v)));
            }
        __syncthreads();
        double dm = __longlong_as_double((long long)red[lane]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
        const double dfloor = 1e-14 * dm;

        // ---- blocked Cholesky with look-ahead ----------------------------
        // factor_diag: the owner's (kb, kb) tile -> L_kk (upper zeroed) and
        // L_kk^{-1} -> linv[kb & 1], L_kk -> column buffer slot kb.
        // factor_diag: the diagonal tile (kb, kb), handed over in the column
        // buffer slot kb by its owner, is factored in place there (L_kk, upper
        // zeroed) and L_kk^{-1} goes to linv[kb & 1]; one code copy, no
        // register-array indexing (the owner reloads L_kk into its register
        // tile in the next sub-diagonal phase)
        auto factor_diag = [&](int kb) {
            if (C::T(kb, kb) % NW != warp)
                return;
            double *slot = colb + ((kb & 1) * TT + kb) * kTileElems;
            Frag dg = ld_frag(slot, lane);
            Frag idt{rq == cq ? 1.0 : 0.0, rq == cq + 1 ? 1.0 : 0.0};
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int src = kk / 2;
                const double vk = (kk & 1) ? dg.b : dg.a;
                const double pv = __shfl_sync(0xffffffffu, vk, 4 * kk + src);
                const double urk = __shfl_sync(0xffffffffu, vk, 4 * rq + src);
                const double uc0 = __shfl_sync(0xffffffffu, vk, 4 * cq + src);
                const double uc1 = __shfl_sync(0xffffffffu, vk, 4 * (cq + 1) + src);
                const bool first = !(pv > dfloor && isfinite(pv)) && fail_piv < 0;
                fail_piv = first ? 8 * kb + kk : fail_piv;
                fail_stage = first ? s : fail_stage;
                const double iv = rsqrt_nr(pv);
                const double lc0 = (cq > kk) ? uc0 * iv : 0.0;
                const double lc1 = (cq + 1 > kk) ? uc1 * iv : 0.0;
                const double lrk = urk * iv;
                const double nv = (rq == kk) ? pv * iv : lrk;
                if (kk & 1)
                    dg.b = (q2 == src) ? nv : dg.b;
                else
                    dg.a = (q2 == src) ? nv : dg.a;
                dg.a -= lrk * lc0;
                dg.b -= lrk * lc1;
                const double vq = (kk & 1) ? idt.b : idt.a;
                const double xrq = __shfl_sync(0xffffffffu, vq, 4 * rq + src) * iv;
                if (kk & 1)
                    idt.b = (q2 == src) ? xrq : idt.b;
                else
                    idt.a = (q2 == src) ? xrq : idt.a;
                idt.a -= xrq * lc0;
                idt.b -= xrq * lc1;
            }
            if (cq > rq) dg.a = 0.0;
            if (cq + 1 > rq) dg.b = 0.0;
            st_frag(slot, lane, dg);
            double *ts = tscr + (kb & 1) * kTileElems;
            st_frag(ts, lane, idt); // L^{-1} = (L^{-T})'
            __syncwarp();
            st_frag(linvb + (kb & 1) * kTileElems, lane, Frag{ts[cq * 8 + rq], ts[(cq + 1) * 8 + rq]});
            __syncwarp();
        };
        // the owner of (0, 0) hands it over
#pragma unroll
        for (int k = 0; k < MAXT; ++k)
            if (mt(k) == 0)
                st_frag(colb, lane, acc[k]);
        __syncwarp();
        factor_diag(0);
        __syncthreads();
#pragma unroll 1
        for (int kb = 0; kb < CT; ++kb) {
            const int par = kb & 1;
            double *col = colb + par * TT * kTileElems;
            // sub-diagonal tiles of column kb: X <- X L_kk^{-T} = X (L_kk^{-1})';
            // the owner of (kb, kb) takes L_kk back into its register tile
            {
                const Frag linv = ld_frag(linvb + par * kTileElems, lane);
#pragma unroll
                for (int k = 0; k < MAXT; ++k)
                    if (mt(k) == ((kb << 8) | kb))
                        acc[k] = ld_frag(col + kb * kTileElems, lane);
#pragma unroll
                for (int k = 0; k < MAXT; ++k)
                    if (mtj(k) == kb && mti(k) > kb) {
                        Frag r{0.0, 0.0};
                        tile_gemm_nt(r, acc[k], linv);
                        acc[k] = r;
                        st_frag(col + mti(k) * kTileElems, lane, r);
                    }
            }
            __syncthreads(); // column kb published
            // look-ahead: (kb+1, kb+1) first, then factor it
            if (kb + 1 < CT) {
                const int pk = ((kb + 1) << 8) | (kb + 1);
#pragma unroll
                for (int k = 0; k < MAXT; ++k)
                    if (mt(k) == pk) {
                        const Frag li = ld_frag(col + (kb + 1) * kTileElems, lane);
                        tile_gemm_nt_sub(acc[k], li, li);
                        st_frag(colb + (((kb + 1) & 1) * TT + kb + 1) * kTileElems, lane, acc[k]);
                    }
                __syncwarp();
                factor_diag(kb + 1);
            }
            // trailing update of my other tiles: C(ti, tj) -= L(ti, kb) L(tj, kb)'
#pragma unroll
            for (int k = 0; k < MAXT; ++k) {
                const int ti = mti(k), tj = mtj(k);
                if (tj > kb && !(ti == kb + 1 && tj == kb + 1 && kb + 1 < CT)) {
                    const Frag li = ld_frag(col + ti * kTileElems, lane);
                    const Frag lj = ld_frag(col + tj * kTileElems, lane);
                    tile_gemm_nt_sub(acc[k], li, lj);
                }
            }
            __syncthreads(); // column kb consumed, L_{kb+1} / linv published
        }
        if (tid < 32)
            red[tid] = 0ull;

        // ---- store the factor tiles and y_s' ---------------------------------
        {
            double *dst = a.fac + ((size_t)chain * n + s) * C::NPT * kTileElems;
#pragma unroll
            for (int k = 0; k < MAXT; ++k) {
                const int ti = mti(k), tj = mtj(k);
                if (ti >= 0 && tj < CT) {
                    st_frag(dst + C::PI(ti, tj) * kTileElems, lane, acc[k]);
                    if (ti == C::RT && rq == C::RR) {
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
        }

        if (s + 1 < n) {
            // ---- W for stage s+1 -------------------------------------------
            // L_Q (x block of the pivot tiles) -> LQ (x-space, row-major)
#pragma unroll
            for (int k = 0; k < MAXT; ++k) {
                const int ti = mti(k), tj = mtj(k);
                if (ti >= C::XT0 && ti < CT && tj >= C::XT0) {
                    const int r = 8 * ti + rq - NU, c0 = 8 * tj + cq - NU;
                    LQ[r * NX + c0] = acc[k].a;
                    LQ[r * NX + c0 + 1] = acc[k].b;
                }
                // ALQ rows (coupling rows, x columns) -> W tile rows >= CT
                if (ti >= CT && tj >= C::XT0 && tj < CT)
                    st_frag(Wsm + (ti * C::NXC + (tj - C::XT0)) * kTileElems, lane, acc[k]);
            }
            cp_wait<0>(); // BA_{s+1}, f_{s+1}
            __syncthreads();
            // -wl_new = L_Q' (sgn f) + x'   (kkt_solve.cpp:85-90)
            for (int t = tid; t < NX; t += NTH) {
                double q = 0.0;
                for (int k = t; k < NX; ++k)
                    q += LQ[k * NX + t] * (sgn * fb[k]);
                q += yx[t];
                mw[t] = q;
                a.wl[((size_t)chain * n + s) * NX + t] = -q;
            }
            // V = BA_{s+1}' L_Q -> W tile rows 0..CT-1 (DMMA, one tile per warp pass)
            for (int v = warp; v < CT * C::NXC; v += NW) {
                const int ti = v / C::NXC, kt = v % C::NXC;
                Frag f{0.0, 0.0};
                for (int ks = 2 * kt; ks < NX / 4; ++ks) { // L_Q upper part is zero
                    const int K = 4 * ks + (lane & 3);
                    const double av = BA[K * C::PW + 8 * ti + rq];
                    const double bv = LQ[K * NX + 8 * kt + rq];
                    dmma(f, av, bv);
                }
                st_frag(Wsm + (ti * C::NXC + kt) * kTileElems, lane, f);
            }
            __syncthreads(); // mw ready, V written, BA / LQ reads done
            // rhs row of W: -wl in row RHS of tile row RT (other rows of
            // that tile row: coupling rows, already stored above)
            for (int t = tid; t < NX; t += NTH)
                Wsm[(C::RT * C::NXC + t / 8) * kTileElems + C::RR * 8 + t % 8] = mw[t];
            if (s + 2 < n)
                stage_BA_cta<NU, NX, NW>(g, a.p, b, g.stage_of(c, s + 2), sm, tid);
            cp_commit();
            __syncthreads();
        }
    }

    // trailing tiles (coupling x coupling = -Mfwd, rhs x coupling = -fwd)
#pragma unroll
    for (int k = 0; k < MAXT; ++k) {
        const int ti = mti(k), tj = mtj(k);
        if (tj >= CT)
            st_frag(a.trail + ((size_t)chain * g.NTT + C::T(ti - CT, tj - CT)) * kTileElems, lane,
                    acc[k]);
    }
    unsigned long long my_fail =
        fail_piv >= 0 ? fail_key(kKindRiccati, c, fail_stage, fail_piv) : ~0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        my_fail = min(my_fail, __shfl_xor_sync(0xffffffffu, my_fail, o));
    if (lane == 0 && my_fail != ~0ull)
        atomicMin(a.fail + b, my_fail);
#undef mti
#undef mtj
#undef mt
#undef mtt
}

namespace {
template <int NU, int NX, int NW> bool launch_c(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    if (g.nu != NU || g.nx != NX)
        return false;
    using C = CS<NU, NX, NW>;
    const size_t smem = (size_t)C::SMEM * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(riccati_cta_kernel<NU, NX, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        unsigned short h[1024];
        for (int t = 0, ti = 0; t < 1024; ++t) {
            while ((ti + 1) * (ti + 2) / 2 <= t)
                ++ti;
            h[t] = (unsigned short)((ti << 8) | (t - ti * (ti + 1) / 2));
        }
        cudaMemcpyToSymbol(c_tij, h, sizeof h);
        attr = true;
    }
    riccati_cta_kernel<NU, NX, NW><<<g.batch * g.P, 32 * NW, smem, st>>>(ra);
    return true;
}
} // namespace

bool launch_riccati_cta(const Geo &g, cudaStream_t st, const RiccatiArgs &ra) {
    if (getenv("CYQ_NO_CTA_KERNEL"))
        return false;
    return launch_c<32, 64, 16>(g, st, ra);
}

} // namespace cyqb
