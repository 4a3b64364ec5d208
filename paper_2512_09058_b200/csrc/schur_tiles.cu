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

constexpr int kSchurTileWarps = 8;

__device__ __forceinline__ void barc() { __syncthreads(); }

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

template <int NX> __global__ void __launch_bounds__(32 * kSchurTileWarps) schur_tile_kernel(SchurArgs a) {
    constexpr int XT = (NX + 7) / 8, NL = XT * (XT + 1) / 2;
    const Geo &g = a.g;
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NW = blockDim.x >> 5;
    const int P = g.P, nu = g.nu, n = g.n, top = 8 * g.CT;
    constexpr int nn = NX * NX;
    const SchurLayout Lo = SchurLayout::make(P, NX);
    double *ws = a.schur + (size_t)b * Lo.total;
    double *D = ws + Lo.D, *K = ws + Lo.K, *Mb = ws + Lo.Mb, *Zg = ws + Lo.Z;
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    unsigned long long my_fail = ~0ull;

    // ---- phase 1: T = L_Q^{-T} per column; Mbwd = T T', -W' = -LA T' ------
    for (int c = warp; c < P; c += NW) {
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
        // Z = T' = L_Q^{-1} kept for the solve-only path (bwd_neg = Z' x')
        double *Zc = Zg + c * nn;
#pragma unroll
        for (int i = 0; i < XT; ++i)
#pragma unroll
            for (int j = 0; j < XT; ++j) {
                // store T transposed: Z(r, k) = T(k, r)
                const Frag f = X[i * XT + j];
                const int r = 8 * i + rq, k0 = 8 * j + cq;
                if (r < NX) {
                    if (k0 < NX) Zc[k0 * NX + r] = f.a;
                    if (k0 + 1 < NX) Zc[(k0 + 1) * NX + r] = f.b;
                }
            }
        // Mbwd = T T' (dense, symmetric)
#pragma unroll
        for (int i = 0; i < XT; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) {
                Frag acc{0.0, 0.0};
#pragma unroll
                for (int kt = 0; kt < XT; ++kt)
                    tile_gemm_nt(acc, X[i * XT + kt], X[j * XT + kt]);
                store_tile<NX>(Mb + c * nn, i, j, lane, acc);
                if (i != j) { // mirror
                    const int r = 8 * i + rq, k0 = 8 * j + cq;
                    if (r < NX) {
                        if (k0 < NX) Mb[c * nn + k0 * NX + r] = acc.a;
                        if (k0 + 1 < NX) Mb[c * nn + (k0 + 1) * NX + r] = acc.b;
                    }
                }
            }
        // subdiag[c-1] = -W_c' = -LA T'
        if (c > 0) {
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
        // diag[c] = Mfwd_c = -(trailing coupling block)
        const double *tr = a.trail + chain * g.NTT * kTileElems;
        for (int e = lane; e < nn; e += 32) {
            const int i = e / NX, jj = e % NX;
            const int r = max(i, jj), cc = min(i, jj);
            D[c * nn + e] = -tr[tri_index(r / 8, cc / 8) * kTileElems + (r % 8) * 8 + cc % 8];
        }
    }
    barc();
    for (int e = threadIdx.x; e < P * nn; e += blockDim.x) {
        const int c = e / nn;
        D[e] += Mb[((c + 1) % P) * nn + (e % nn)];
    }
    barc();

    // ---- phase 2: cyclic reduction factor ---------------------------------
    int s = P;
    for (int l = 0; l < Lo.levels; ++l, s /= 2) {
        const int half = s / 2;
        const double *Ml = l == 0 ? D : ws + Lo.level(l - 1, P, NX, 3);
        const double *Kl = l == 0 ? K : ws + Lo.level(l - 1, P, NX, 4);
        double *Ll = ws + Lo.level(l, P, NX, 0), *Ul = ws + Lo.level(l, P, NX, 1);
        double *Yl = ws + Lo.level(l, P, NX, 2), *M2 = ws + Lo.level(l, P, NX, 3);
        double *K2 = ws + Lo.level(l, P, NX, 4);
        // contributions go to the next level's M2 (U U'), K2 (-Y U') and a
        // Y Y' scratch in the (not yet used) Lbase..rhs gap: use Mb[] (free)
        double *CY = Mb;
        for (int mm = warp; mm < half; mm += NW) {
            const int k = 2 * mm + 1;
            Frag Dg[NL], R[2 * XT * XT];
#pragma unroll
            for (int i = 0; i < XT; ++i)
#pragma unroll
                for (int j = 0; j <= i; ++j)
                    Dg[T(i, j)] = load_tile<NX, XT>(Ml + k * nn, i, j, lane, true, 1.0);
            const bool has_y = k < s - 1;
#pragma unroll
            for (int i = 0; i < XT; ++i)
#pragma unroll
                for (int j = 0; j < XT; ++j) {
                    R[i * XT + j] = load_tile<NX, XT>(Kl + (k - 1) * nn, i, j, lane, false, 0.0, true);
                    R[(XT + i) * XT + j] = has_y ? load_tile<NX, XT>(Kl + k * nn, i, j, lane, false, 0.0)
                                                 : Frag{0.0, 0.0};
                }
            const double dfloor = 1e-14 * tiles::diag_absmax<XT>(Dg, NX, lane);
            int pf = -1;
            tiles::panel_cholesky<XT, XT>(Dg, NX, dfloor, lane, pf);
            if (pf >= 0)
                my_fail = min(my_fail, fail_key(kKindCR, l, k, pf));
            tiles::trsm_rows<2 * XT, XT>(R, Dg, lane);
#pragma unroll
            for (int i = 0; i < XT; ++i)
#pragma unroll
                for (int j = 0; j < XT; ++j) {
                    if (j <= i)
                        store_tile<NX>(Ll + mm * nn, i, j, lane, Dg[T(i, j)]);
                    else
                        store_tile<NX>(Ll + mm * nn, i, j, lane, Frag{0.0, 0.0});
                    store_tile<NX>(Ul + mm * nn, i, j, lane, R[i * XT + j]);
                    store_tile<NX>(Yl + mm * nn, i, j, lane, R[(XT + i) * XT + j]);
                }
            // contributions: M2[mm] <- M[2mm] - U U' (Y Y' of block mm-1 added
            // below), CY[mm] = Y Y', K2[mm] = -Y U'
#pragma unroll
            for (int i = 0; i < XT; ++i)
#pragma unroll
                for (int j = 0; j < XT; ++j) {
                    Frag uu{0.0, 0.0}, yy{0.0, 0.0}, yu{0.0, 0.0};
#pragma unroll
                    for (int kt = 0; kt < XT; ++kt) {
                        tile_gemm_nt(uu, R[i * XT + kt], R[j * XT + kt]);
                        tile_gemm_nt(yy, R[(XT + i) * XT + kt], R[(XT + j) * XT + kt]);
                        tile_gemm_nt_sub(yu, R[(XT + i) * XT + kt], R[j * XT + kt]);
                    }
                    Frag m = load_tile<NX, XT>(Ml + 2 * mm * nn, i, j, lane, false, 0.0);
                    m.a -= uu.a;
                    m.b -= uu.b;
                    store_tile<NX>(M2 + mm * nn, i, j, lane, m);
                    store_tile<NX>(CY + mm * nn, i, j, lane, yy);
                    store_tile<NX>(K2 + mm * nn, i, j, lane,
                                   (mm < half - 1) ? yu : Frag{0.0, 0.0});
                }
        }
        barc();
        for (int e = threadIdx.x; e < half * nn; e += blockDim.x) {
            const int mm = e / nn;
            if (mm > 0)
                M2[e] -= CY[e - nn];
        }
        barc();
    }
    if (warp == 0) {
        const double *Mlast = Lo.levels == 0 ? D : ws + Lo.level(Lo.levels - 1, P, NX, 3);
        Frag Dg[NL];
#pragma unroll
        for (int i = 0; i < XT; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j)
                Dg[T(i, j)] = load_tile<NX, XT>(Mlast, i, j, lane, true, 1.0);
        const double dfloor = 1e-14 * tiles::diag_absmax<XT>(Dg, NX, lane);
        int pf = -1;
        tiles::panel_cholesky<XT, XT>(Dg, NX, dfloor, lane, pf);
        if (pf >= 0)
            my_fail = min(my_fail, fail_key(kKindCR, Lo.levels, 0, pf));
#pragma unroll
        for (int i = 0; i < XT; ++i)
#pragma unroll
            for (int j = 0; j < XT; ++j)
                store_tile<NX>(ws + Lo.Lbase, i, j, lane, j <= i ? Dg[T(i, j)] : Frag{0.0, 0.0});
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        my_fail = min(my_fail, __shfl_xor_sync(0xffffffffu, my_fail, o));
    if (lane == 0 && my_fail != ~0ull)
        atomicMin(a.fail + b, my_fail);
}

template <int NX> bool launch_st(const Geo &g, cudaStream_t st, const SchurArgs &sa) {
    if (g.nx != NX)
        return false;
    schur_tile_kernel<NX><<<g.batch, 32 * std::max(1, std::min(kSchurTileWarps, g.P / 2)), 0, st>>>(sa);
    return true;
}

} // namespace

// Tile-based CR factorization (phase 1 + 2 of schur_cr_kernel); the caller
// then runs schur_cr_kernel with do_factor = 0 for the rhs and CR solve.
bool launch_schur_tiles(const Geo &g, cudaStream_t st, const SchurArgs &sa) {
    if (getenv("CYQ_NO_SCHUR_TILES"))
        return false;
    return launch_st<20>(g, st, sa) || launch_st<16>(g, st, sa) || launch_st<12>(g, st, sa) ||
           launch_st<10>(g, st, sa);
}

} // namespace cyqb
