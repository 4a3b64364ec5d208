// Schur-complement assembly + cyclic-reduction factorization of the coupling
// system on register-resident FP64 DMMA tiles (compile-time nx; one CTA per
// OCP instance, one warp per independent block operation). The fast path
// for nx <= 24; other shapes use the scalar kernel in schur_cr.cu. Both
// write the same per-instance workspace (SchurLayout, dense row-major
// blocks), so the CR solve and everything downstream is shared.
//
// Restates:
//   kkt_factor.cpp:163-178    T = L_Q^{-T}, Mbwd = T T', W = T LA'
//   kkt_factor.cpp:194-212    assemble_schur (diag[c] = Mfwd_c + Mbwd_{c+1},
//                             subdiag[c-1] = -W_c')
//   block_tridiag.cpp:126-171 cr_level: L = chol(M_k), U = K_{k-1}' L^{-T},
//                             Y = K_k L^{-T}; M' = M - U U' - Y_prev Y_prev',
//                             K' = -Y U'
//   block_tridiag.cpp:173-197 cr_factor_base
// Each odd-block elimination is one panel [M_k; K_{k-1}'; K_k] factored by
// the shared tile Cholesky (tiles.cuh); the even-block updates are DMMA
// rank products of the warp's U / Y tiles, written as contributions and
// summed by the CTA (fixed order: bit-reproducible).
#include "kernels.h"
#include "tiles.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace cyqb {

using tiles::T;

namespace {


// dense row-major n x n block <-> register tiles (XT x XT), padding: `pad`
// on the diagonal, zero elsewhere
template <int NX, int XT>
__device__ __forceinline__ Frag load_tile(const double *blk, int ti, int tj, int lane, bool lower,
                                          double pad, bool trans = false) {
    const int r = 8 * ti + (lane >> 2), c0 = 8 * tj + 2 * (lane & 3);
    Frag f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int c = c0 + h;
        double v;
        if (r < NX && c < NX)
            v = (lower && c > r) ? 0.0 : (trans ? blk[c * NX + r] : blk[r * NX + c]);
        else
            v = (r == c) ? pad : 0.0;
        (h ? f.b : f.a) = v;
    }
    return f;
}
template <int NX>
__device__ __forceinline__ void store_tile(double *blk, int ti, int tj, int lane, Frag f,
                                           bool lower_only = false, double scale = 1.0) {
    const int r = 8 * ti + (lane >> 2), c0 = 8 * tj + 2 * (lane & 3);
    if (r < NX) {
        if (c0 < NX && !(lower_only && c0 > r)) blk[r * NX + c0] = scale * f.a;
        if (c0 + 1 < NX && !(lower_only && c0 + 1 > r)) blk[r * NX + c0 + 1] = scale * f.b;
    }
}

__device__ __forceinline__ int stored_tile_t(const Geo &g, int ti, int tj) {
    return ti < g.CT ? tri_index(ti, tj) : g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
}
__device__ __forceinline__ double fac_at_t(const Geo &g, const double *st, int r, int col) {
    return st[stored_tile_t(g, r / 8, col / 8) * kTileElems + (r % 8) * 8 + col % 8];
}

// Per-level launch structure: every kernel maps one warp to one independent
// block operation across ALL instances of the batch (phase-1 columns, then the
// odd-block eliminations of one CR level), so the GPU's warp slots are filled
// by the whole batch instead of one instance's shrinking level. The even-block
// assembly (M' = M - U U' - Y_prev Y_prev') is folded into the next level's
// loads.
constexpr int kWPB = 4; // warps per CTA

struct WarpTask {
    int b, i; // instance, block index
};
__device__ __forceinline__ bool warp_task(int count_per_inst, int batch, WarpTask &t) {
    const int w = blockIdx.x * kWPB + (threadIdx.x >> 5);
    if (w >= count_per_inst * batch)
        return false;
    t.b = w / count_per_inst;
    t.i = w % count_per_inst;
    return true;
}

// level-l reduced system block M_l[i] (tile (ti, tj)), assembled on the fly:
//   l = 0: Mfwd_i + Mbwd_{i+1}            (assemble_schur, kkt_factor.cpp:194-212)
//   l > 0: M'_{l-1}[i] - Y_{i-1} Y_{i-1}'  (cr_level even update)
template <int NX, int XT>
__device__ __forceinline__ Frag m_tile(const double *ws, const SchurLayout &Lo, int P, int l, int i,
                                       int ti, int tj, int lane, bool lower) {
    constexpr int nn = NX * NX;
    Frag f, g2{0.0, 0.0};
    if (l == 0) {
        f = load_tile<NX, XT>(ws + Lo.D + i * nn, ti, tj, lane, lower, 1.0);
        g2 = load_tile<NX, XT>(ws + Lo.Mb + ((i + 1) % P) * nn, ti, tj, lane, lower, 0.0);
        f.a += g2.a;
        f.b += g2.b;
    } else {
        f = load_tile<NX, XT>(ws + Lo.level(l - 1, P, NX, 3) + i * nn, ti, tj, lane, lower, 1.0);
        if (i > 0) {
            g2 = load_tile<NX, XT>(ws + Lo.level(l - 1, P, NX, 5) + (i - 1) * nn, ti, tj, lane,
                                   lower, 0.0);
            f.a -= g2.a;
            f.b -= g2.b;
        }
    }
    return f;
}
template <int NX> __device__ __forceinline__ const double *k_blk(const double *ws, const SchurLayout &Lo,
                                                                int P, int l, int i) {
    return (l == 0 ? ws + Lo.K : ws + Lo.level(l - 1, P, NX, 4)) + i * NX * NX;
}

template <int NX> __global__ void __launch_bounds__(32 * kWPB) schur_p1_kernel(SchurArgs a) {
    constexpr int XT = (NX + 7) / 8, NL = XT * (XT + 1) / 2, nn = NX * NX;
    const Geo &g = a.g;
    WarpTask tk;
    if (!warp_task(g.P, g.batch, tk))
        return;
    const int b = tk.b, c = tk.i, lane = threadIdx.x & 31;
    const int P = g.P, nu = g.nu, n = g.n, top = 8 * g.CT;
    const SchurLayout Lo = SchurLayout::make(P, NX);
    double *ws = a.schur + (size_t)b * Lo.total;
    double *D = ws + Lo.D, *K = ws + Lo.K, *Mb = ws + Lo.Mb, *Zg = ws + Lo.Z;
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    const size_t chain = (size_t)b * P + c;
    const double *st = a.fac + (chain * n + (n - 1)) * g.NPT * kTileElems;
    Frag Lq[NL], X[XT * XT];
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            Frag f;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = 8 * i + rq, k = 8 * j + cq + h;
                const double v = (r < NX && k < NX) ? (k <= r ? fac_at_t(g, st, nu + r, nu + k) : 0.0)
                                                    : (r == k ? 1.0 : 0.0);
                (h ? f.b : f.a) = v;
            }
            Lq[T(i, j)] = f;
        }
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j < XT; ++j) {
            const int r = 8 * i + rq, k = 8 * j + cq;
            X[i * XT + j] = Frag{r == k ? 1.0 : 0.0, r == k + 1 ? 1.0 : 0.0};
        }
    tiles::trsm_rows<XT, XT>(X, Lq, lane); // X = I L_Q^{-T} = T (rows)
    double *Zc = Zg + c * nn;              // Z = T' (bwd_neg = Z' x' in the solve)
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j < XT; ++j) {
            const Frag f = X[i * XT + j];
            const int r = 8 * i + rq, k0 = 8 * j + cq;
            if (r < NX) {
                if (k0 < NX) Zc[k0 * NX + r] = f.a;
                if (k0 + 1 < NX) Zc[(k0 + 1) * NX + r] = f.b;
            }
        }
    // Mbwd = T T' (kkt_factor.cpp:174)
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            Frag acc{0.0, 0.0};
#pragma unroll
            for (int kt = 0; kt < XT; ++kt)
                tile_gemm_nt(acc, X[i * XT + kt], X[j * XT + kt]);
            store_tile<NX>(Mb + c * nn, i, j, lane, acc);
            if (i != j) {
                const int r = 8 * i + rq, k0 = 8 * j + cq;
                if (r < NX) {
                    if (k0 < NX) Mb[c * nn + k0 * NX + r] = acc.a;
                    if (k0 + 1 < NX) Mb[c * nn + (k0 + 1) * NX + r] = acc.b;
                }
            }
        }
    if (c > 0) { // subdiag[c-1] = -W_c' = -LA T'  (kkt_factor.cpp:203-209)
        Frag LA[XT * XT];
#pragma unroll
        for (int i = 0; i < XT; ++i)
#pragma unroll
            for (int j = 0; j < XT; ++j) {
                Frag f;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = 8 * i + rq, k = 8 * j + cq + h;
                    (h ? f.b : f.a) = (r < NX && k < NX) ? fac_at_t(g, st, top + r, nu + k) : 0.0;
                }
                LA[i * XT + j] = f;
            }
#pragma unroll
        for (int i = 0; i < XT; ++i)
#pragma unroll
            for (int j = 0; j < XT; ++j) {
                Frag acc{0.0, 0.0};
#pragma unroll
                for (int kt = 0; kt < XT; ++kt)
                    tile_gemm_nt_sub(acc, LA[i * XT + kt], X[j * XT + kt]);
                store_tile<NX>(K + (c - 1) * nn, i, j, lane, acc);
            }
    } else {
        for (int e = lane; e < nn; e += 32)
            K[(P - 1) * nn + e] = 0.0;
    }
    // raw diag[c] = Mfwd_c = -(trailing coupling block); Mbwd_{c+1} is added
    // when the level-0 eliminations load it
    const double *tr = a.trail + chain * g.NTT * kTileElems;
    for (int e = lane; e < nn; e += 32) {
        const int i = e / NX, jj = e % NX;
        const int r = max(i, jj), cc = min(i, jj);
        D[c * nn + e] = -tr[tri_index(r / 8, cc / 8) * kTileElems + (r % 8) * 8 + cc % 8];
    }
}

// One odd-block elimination of CR level l (block_tridiag.cpp:126-171) per warp.
template <int NX> __global__ void __launch_bounds__(32 * kWPB) schur_elim_kernel(SchurArgs a, int l) {
    constexpr int XT = (NX + 7) / 8, NL = XT * (XT + 1) / 2, nn = NX * NX;
    const Geo &g = a.g;
    const int P = g.P, s = P >> l, half = s / 2;
    WarpTask tk;
    if (!warp_task(half, g.batch, tk))
        return;
    const int b = tk.b, mm = tk.i, k = 2 * mm + 1, lane = threadIdx.x & 31;
    const SchurLayout Lo = SchurLayout::make(P, NX);
    double *ws = a.schur + (size_t)b * Lo.total;
    double *Ll = ws + Lo.level(l, P, NX, 0), *Ul = ws + Lo.level(l, P, NX, 1);
    double *Yl = ws + Lo.level(l, P, NX, 2), *M2 = ws + Lo.level(l, P, NX, 3);
    double *K2 = ws + Lo.level(l, P, NX, 4), *CY = ws + Lo.level(l, P, NX, 5);
    Frag Dg[NL], R[2 * XT * XT];
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j)
            Dg[T(i, j)] = m_tile<NX, XT>(ws, Lo, P, l, k, i, j, lane, true);
    const bool has_y = k < s - 1;
    const double *Kp = k_blk<NX>(ws, Lo, P, l, k - 1), *Kk = k_blk<NX>(ws, Lo, P, l, k);
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j < XT; ++j) {
            R[i * XT + j] = load_tile<NX, XT>(Kp, i, j, lane, false, 0.0, true); // K_{k-1}'
            R[(XT + i) * XT + j] = has_y ? load_tile<NX, XT>(Kk, i, j, lane, false, 0.0)
                                         : Frag{0.0, 0.0};
        }
    const double dfloor = 1e-14 * tiles::diag_absmax<XT>(Dg, NX, lane);
    int pf = -1;
    tiles::panel_cholesky<XT, XT>(Dg, NX, dfloor, lane, pf);
    tiles::trsm_rows<2 * XT, XT>(R, Dg, lane); // U = K_{k-1}' L^{-T}, Y = K_k L^{-T}
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j < XT; ++j) {
            store_tile<NX>(Ll + mm * nn, i, j, lane, j <= i ? Dg[T(i, j)] : Frag{0.0, 0.0});
            store_tile<NX>(Ul + mm * nn, i, j, lane, R[i * XT + j]);
            store_tile<NX>(Yl + mm * nn, i, j, lane, R[(XT + i) * XT + j]);
        }
    // M'_{mm} = M[2mm] - U U' (the Y_{mm-1} term is subtracted by the next
    // level's loads), CY[mm] = Y Y', K'_{mm} = -Y U'
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j < XT; ++j) {
            Frag uu{0.0, 0.0}, yy{0.0, 0.0}, yu{0.0, 0.0};
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int kt = 0; kt < XT; ++kt) {
                    const Frag &ui = R[i * XT + kt], &uj = R[j * XT + kt];
                    const Frag &yi = R[(XT + i) * XT + kt], &yj = R[(XT + j) * XT + kt];
                    dmma(uu, h ? ui.b : ui.a, h ? uj.b : uj.a);
                    dmma(yy, h ? yi.b : yi.a, h ? yj.b : yj.a);
                    dmma(yu, h ? -yi.b : -yi.a, h ? uj.b : uj.a);
                }
            Frag m = m_tile<NX, XT>(ws, Lo, P, l, 2 * mm, i, j, lane, false);
            m.a -= uu.a;
            m.b -= uu.b;
            store_tile<NX>(M2 + mm * nn, i, j, lane, m);
            store_tile<NX>(CY + mm * nn, i, j, lane, yy);
            store_tile<NX>(K2 + mm * nn, i, j, lane, (mm < half - 1) ? yu : Frag{0.0, 0.0});
        }
    unsigned long long key = pf >= 0 ? fail_key(kKindCR, l, k, pf) : ~0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
    if (lane == 0 && key != ~0ull)
        atomicMin(a.fail + b, key);
}

// cr_factor_base (block_tridiag.cpp:173-197), one warp per instance.
template <int NX> __global__ void __launch_bounds__(32 * kWPB) schur_base_kernel(SchurArgs a) {
    constexpr int XT = (NX + 7) / 8, NL = XT * (XT + 1) / 2;
    const Geo &g = a.g;
    WarpTask tk;
    if (!warp_task(1, g.batch, tk))
        return;
    const int b = tk.b, lane = threadIdx.x & 31, P = g.P;
    const SchurLayout Lo = SchurLayout::make(P, NX);
    double *ws = a.schur + (size_t)b * Lo.total;
    Frag Dg[NL];
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j)
            Dg[T(i, j)] = m_tile<NX, XT>(ws, Lo, P, Lo.levels, 0, i, j, lane, true);
    const double dfloor = 1e-14 * tiles::diag_absmax<XT>(Dg, NX, lane);
    int pf = -1;
    tiles::panel_cholesky<XT, XT>(Dg, NX, dfloor, lane, pf);
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j < XT; ++j)
            store_tile<NX>(ws + Lo.Lbase, i, j, lane, j <= i ? Dg[T(i, j)] : Frag{0.0, 0.0});
    if (lane == 0 && pf >= 0)
        atomicMin(a.fail + b, fail_key(kKindCR, Lo.levels, 0, pf));
}

template <int NX> bool launch_st(const Geo &g, cudaStream_t st, const SchurArgs &sa) {
    if (g.nx != NX)
        return false;
    auto grid = [&](int per) { return (g.batch * per + kWPB - 1) / kWPB; };
    schur_p1_kernel<NX><<<grid(g.P), 32 * kWPB, 0, st>>>(sa);
    const int levels = SchurLayout::make(g.P, NX).levels;
    for (int l = 0, s = g.P; l < levels; ++l, s /= 2)
        schur_elim_kernel<NX><<<grid(s / 2), 32 * kWPB, 0, st>>>(sa, l);
    schur_base_kernel<NX><<<grid(1), 32 * kWPB, 0, st>>>(sa);
    return true;
}

} // namespace

// Tile-based CR factorization (phase 1 + 2 of schur_cr_kernel); the caller
// then runs schur_cr_kernel with do_factor = 0 for the rhs and CR solve.
bool launch_schur_tiles(const Geo &g, cudaStream_t st, const SchurArgs &sa) {
    return launch_st<20>(g, st, sa) || launch_st<16>(g, st, sa) || launch_st<12>(g, st, sa) ||
           launch_st<10>(g, st, sa);
}

} // namespace cyqb
