// Back substitution for large tile-aligned stage blocks (nu % 8 == 0,
// nx % 8 == 0; BASELINE config 3: nu = 32, nx = 64). Same algorithm and
// outputs as backsub.cu / backsub_warp.cu (kkt_solve.cpp:185-307):
//   y_s   = [u'; x']_s - [LB ALQ]_s' lam_f
//   s = n-1:  x_s += L_Q^{-1} lam_b                      (T' lam_b)
//   s < n-1:  w  = -wl_s - ALQ_s' lam_f,  t = w - L_Q' (BA_{s+1} z_{s+1}),
//             lam^{j(s+1)} = -L_Q t,   x_s -= t
//   z_s   = LH_s^{-T} y_s
// One warp per chain with NO shared-memory staging of the factor: every
// stored 8x8 tile is read straight from global memory as one coalesced
// 512-byte fragment load, all the loads of a phase are independent of each
// other, and the warp keeps only vectors in shared memory (~5 KB), so 16+
// chains per SM hide the latency and the kernel streams the factor at HBM
// rate (the generic kernel staged 150 KB of tiles per warp: one warp / SM).
// Triangular solves go block by block; the diagonal 8x8 solves use
// reciprocal pivots and shuffles.
#include "kernels.h"
#include "tiles.cuh"

#include <cstdlib>

namespace cyqb {

namespace {

template <int NU, int NX> struct BT {
    static constexpr int NUX = NU + NX, CT = NUX / 8, XT = NX / 8, XT0 = NU / 8;
    static constexpr int NPT = CT * (CT + 1) / 2 + ((NX + 1 + 7) / 8) * CT;
    static constexpr int TOP = 8 * CT;
    // per-warp shared vectors (doubles)
    static constexpr int O_LF = 0, O_LB = NX, O_Y = 2 * NX, O_Z = 2 * NX + NUX;
    static constexpr int O_W = 2 * NX + 2 * NUX, O_ZN = O_W + NX, O_T = O_ZN + NX;
    static constexpr int O_V = O_T + NX, O_SCR = O_V + NUX;
    static constexpr int PER_WARP = O_SCR + 64;
    __device__ static int tile(int i, int j) {
        return i < CT ? i * (i + 1) / 2 + j : CT * (CT + 1) / 2 + (i - CT) * CT + j;
    }
};

// out[8 j + c] (+)= sum_i M(i, j)[r][c] v[8 i + r] over tile rows i in [i0, i1)
// for tile columns j in [j0, j1): transposed matvec of stored tiles
template <int NU, int NX>
__device__ __forceinline__ void tmv_t(const double *tiles, int i0, int i1, int j0, int j1, const double *v,
                                      double *out, double sgn, bool acc, bool lower, int lane) {
    using B = BT<NU, NX>;
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    constexpr int MI = 8; // tile rows per batch: all loads of a batch in flight at once
    for (int j = j0; j < j1; ++j) {
        double a0 = 0.0, a1 = 0.0;
        for (int ib = i0; ib < i1; ib += MI) {
            Frag f[MI];
#pragma unroll
            for (int u = 0; u < MI; ++u) {
                const int i = ib + u;
                const bool on = i < i1 && !(lower && i < j);
                f[u] = on ? ld_frag_g(tiles + B::tile(i, j) * kTileElems, lane) : Frag{0.0, 0.0};
            }
#pragma unroll
            for (int u = 0; u < MI; ++u) {
                const int i = ib + u;
                const double vi = i < i1 ? v[8 * (i - i0) + rq] : 0.0;
                a0 = fma(f[u].a, vi, a0);
                a1 = fma(f[u].b, vi, a1);
            }
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        }
        if (rq == 0) {
            double *o0 = out + 8 * (j - j0) + cq;
            o0[0] = (acc ? o0[0] : 0.0) + sgn * a0;
            o0[1] = (acc ? o0[1] : 0.0) + sgn * a1;
        }
    }
}

// out[8 i + r] (+)= sum_j M(i, j)[r][c] v[8 j + c] (lower: j <= i)
template <int NU, int NX>
__device__ __forceinline__ void tmv(const double *tiles, int i0, int i1, int j0, int j1, const double *v,
                                    double *out, double sgn, bool acc, bool lower, int lane) {
    using B = BT<NU, NX>;
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    for (int i = i0; i < i1; ++i) {
        double s = 0.0;
#pragma unroll 4
        for (int j = j0; j < j1; ++j) {
            if (lower && j > i)
                continue;
            const Frag f = ld_frag_g(tiles + B::tile(i, j) * kTileElems, lane);
            s = fma(f.a, v[8 * (j - j0) + cq], s);
            s = fma(f.b, v[8 * (j - j0) + cq + 1], s);
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if ((lane & 3) == 0) {
            double *o0 = out + 8 * (i - i0) + rq;
            *o0 = (acc ? *o0 : 0.0) + sgn * s;
        }
    }
}

// Solve L x = r (forward, TR = false) or L' x = r (backward, TR = true) for
// one lower-triangular 8x8 tile L (global), r / x: 8 entries in shared
// memory (in place). Lane k < 8 holds r_k.
template <bool TR>
__device__ __forceinline__ void tile_solve(const double *L, double *r, double *scr, int lane) {
    __syncwarp();
    st_frag(scr, lane, ld_frag_g(L, lane));
    __syncwarp();
    const int k = lane & 7;
    double rk = r[k];
    const double ik = tiles::rcp_nr(scr[k * 9]);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int p = TR ? 7 - s : s;
        const double xp = __shfl_sync(0xffffffffu, rk, p) * __shfl_sync(0xffffffffu, ik, p);
        if (k == p)
            rk = xp;
        // forward: r_k -= L[k][p] x_p (k > p); backward: r_k -= L[p][k] x_p (k < p)
        const bool upd = TR ? (k < p) : (k > p);
        if (upd)
            rk -= (TR ? scr[p * 8 + k] : scr[k * 8 + p]) * xp;
    }
    __syncwarp();
    if (lane < 8)
        r[k] = rk;
    __syncwarp();
}

} // namespace

template <int NU, int NX, int WPB>
#ifdef CYQ_BT_MINB
__global__ void __launch_bounds__(32 * WPB, CYQ_BT_MINB) backsub_tile_kernel(BacksubArgs a) {
#else
__global__ void __launch_bounds__(32 * WPB) backsub_tile_kernel(BacksubArgs a) {
#endif
    using B = BT<NU, NX>;
    constexpr int NUX = B::NUX, CT = B::CT, XT = B::XT, XT0 = B::XT0;
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const size_t chain = (size_t)blockIdx.x * WPB + wib;
    griddep_wait(); // the Schur kernel's multipliers
    if (chain >= (size_t)g.batch * g.P)
        return;
    const int b = (int)(chain / g.P), c = (int)(chain % g.P), n = g.n, N = g.N;
    double *base = sm + (size_t)wib * B::PER_WARP;
    double *lf = base + B::O_LF, *lb = base + B::O_LB, *Y = base + B::O_Y, *z = base + B::O_Z;
    double *w = base + B::O_W, *zn = base + B::O_ZN, *t = base + B::O_T, *v = base + B::O_V;
    double *scr = base + B::O_SCR;
    for (int k = lane; k < NX; k += 32) {
        lf[k] = a.lamc[((size_t)b * g.P + c) * NX + k];
        lb[k] = a.lamc[((size_t)b * g.P + (c - 1 + g.P) % g.P) * NX + k];
    }
    __syncwarp();
    for (int s = n - 1; s >= 0; --s) {
        const double *tiles = a.fac + (chain * n + s) * B::NPT * kTileElems;
        const int j = g.stage_of(c, s), xi = g.x_index_of(c, s);
        // y -= [LB ALQ]' lam_f  (coupling tile rows CT .. CT+XT-1)
        tmv_t<NU, NX>(tiles, CT, CT + XT, 0, CT, lf, v, 1.0, false, false, lane);
        __syncwarp();
        const double *yv = a.y + (chain * n + s) * NUX;
        for (int k = lane; k < NUX; k += 32) {
            Y[k] = __ldg(yv + k) - v[k];
            if (k >= NU && s + 1 < n)
                w[k - NU] = -__ldg(a.wl + (chain * n + s) * NX + (k - NU)) - v[k];
        }
        __syncwarp();
        if (s == n - 1) {
            // x += L_Q^{-1} lam_b: blocked forward solve with L_Q
            for (int k = lane; k < NX; k += 32)
                t[k] = lb[k];
            __syncwarp();
            for (int kb = 0; kb < XT; ++kb) {
                tile_solve<false>(tiles + B::tile(XT0 + kb, XT0 + kb) * kTileElems, t + 8 * kb, scr, lane);
                if (kb + 1 < XT) // t_i -= L(i, kb) t_kb, i > kb
                    tmv<NU, NX>(tiles, XT0 + kb + 1, XT0 + XT, XT0 + kb, XT0 + kb + 1, t + 8 * kb,
                                t + 8 * (kb + 1), -1.0, true, false, lane);
                __syncwarp();
            }
            for (int k = lane; k < NX; k += 32)
                Y[NU + k] += t[k];
        } else {
            const int j1 = g.stage_of(c, s + 1);
            // zn = BA_{s+1} z_{s+1}: coalesced row reads (lane = column pair
            // of A / column of B), 32 row partials per lane, then a butterfly
            // reduce-scatter leaves row r of the batch in lane r
            const bool in = j1 < N;
            const double *Bg = a.p.B + ((size_t)b * N + j1) * NX * NU;
            const double *Ag = a.p.A + ((size_t)b * N + j1) * NX * NX;
            static_assert(NX % 16 == 0 && NX <= 64 && NU <= 32, "zn layout");
            const double za0 = z[NU + 2 * lane], za1 = z[NU + 2 * lane + 1];
            const double zb = lane < NU ? z[lane] : 0.0;
            // 16 rows per pass (16 partials per lane: 64 registers, no
            // spills): a 4-step butterfly leaves row r0 + (lane & 15) in
            // lanes l and l ^ 16 (each half of the columns), one more xor
            // adds the halves
#pragma unroll
            for (int r0 = 0; r0 < NX; r0 += 16) {
                double pr[16];
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    double acc = 0.0;
                    if (in) {
                        if (j1 != 0 && 2 * lane < NX) {
                            const double2 av = __ldg(reinterpret_cast<const double2 *>(Ag + (r0 + r) * NX) + lane);
                            acc = fma(av.x, za0, av.y * za1);
                        }
                        if (lane < NU)
                            acc = fma(__ldg(Bg + (r0 + r) * NU + lane), zb, acc);
                    }
                    pr[r] = acc;
                }
                // reduce-scatter: after step h, lane keeps the rows whose bit
                // h matches its own
#pragma unroll
                for (int h = 8; h >= 1; h >>= 1) {
#pragma unroll
                    for (int r = 0; r < h; ++r) {
                        const bool up = (lane & h) != 0;
                        const double send = up ? pr[r] : pr[r + h];
                        const double keep = up ? pr[r + h] : pr[r];
                        pr[r] = keep + __shfl_xor_sync(0xffffffffu, send, h);
                    }
                }
                const double row = pr[0] + __shfl_xor_sync(0xffffffffu, pr[0], 16);
                if (lane < 16)
                    zn[r0 + lane] = row;
            }
            __syncwarp();
            // t = w - L_Q' zn
            tmv_t<NU, NX>(tiles, XT0, CT, XT0, CT, zn, t, 1.0, false, true, lane);
            __syncwarp();
            for (int k = lane; k < NX; k += 32)
                t[k] = w[k] - t[k];
            __syncwarp();
            // lam^{j(s+1)} = -L_Q t ; x -= t
            tmv<NU, NX>(tiles, XT0, CT, XT0, CT, t, v, -1.0, false, true, lane);
            __syncwarp();
            for (int k = lane; k < NX; k += 32) {
                if (j1 < N)
                    a.sol.lam[((size_t)b * N + j1) * NX + k] = v[k];
                Y[NU + k] -= t[k];
            }
        }
        __syncwarp();
        // z = LH^{-T} Y, block rows from the bottom: z_kb = L_kk^{-T} Y_kb,
        // then Y_j -= L(kb, j)' z_kb for j < kb
        for (int kb = CT - 1; kb >= 0; --kb) {
            tile_solve<true>(tiles + B::tile(kb, kb) * kTileElems, Y + 8 * kb, scr, lane);
            if (kb > 0)
                tmv_t<NU, NX>(tiles, kb, kb + 1, 0, kb, Y + 8 * kb, Y, -1.0, true, false, lane);
            __syncwarp();
        }
        for (int k = lane; k < NUX; k += 32) {
            const double val = Y[k];
            z[k] = val;
            if (k < NU) {
                if (j < N)
                    a.sol.u[((size_t)b * N + j) * NU + k] = val;
            } else if (xi <= N) {
                a.sol.x[((size_t)b * (N + 1) + xi) * NX + (k - NU)] = val;
            }
        }
        __syncwarp();
    }
    if (c == 0)
        for (int k = lane; k < NX; k += 32)
            a.sol.x[(size_t)b * (N + 1) * NX + k] = __ldg(a.p.x_init + (size_t)b * NX + k);
}

namespace {
template <int NU, int NX> bool launch_bt(const Geo &g, cudaStream_t st, const BacksubArgs &ba) {
    if (g.nu != NU || g.nx != NX)
        return false;
    constexpr int WPB = 4;
    const size_t smem = (size_t)WPB * BT<NU, NX>::PER_WARP * sizeof(double);
    const int chains = g.batch * g.P;
    launch_pdl(backsub_tile_kernel<NU, NX, WPB>, dim3((chains + WPB - 1) / WPB), dim3(32 * WPB), smem, st, 1, ba);
    return true;
}
} // namespace

bool launch_backsub_tile(const Geo &g, cudaStream_t st, const BacksubArgs &ba) {
    return launch_bt<32, 64>(g, st, ba);
}

} // namespace cyqb
