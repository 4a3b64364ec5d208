// CTA-cooperative FP64 tile linear algebra on memory-resident blocks
// (XT x XT grids of 8x8 C-fragment tiles, tile (i, j) at blk + (i XT + j) 64,
// global or shared memory). Every routine is called by all NW warps of the
// CTA; output tiles are spread over the warps, every rank-8 step is two
// DMMAs (mma.sync m8n8k4 f64), and transposed operands are read as
// transposed tiles (two 8-byte loads per lane) -- no transpose passes.
// Used for the large-nx Schur complement / cyclic reduction (schur_big.cu),
// where one block op is 64 x 64 (config 3).
//
// Restates the batla kernels the reference's cr_level / factor phases use
// (kernels.cpp:32-58 potrf, :95-119 trsm, :158-220 syrk / gemm, :246-271
// trtri) for whole blocks instead of per lane.
#pragma once

#include "kkt_common.cuh"
#include "tiles.cuh"

namespace cyqb {
namespace ctat {

__device__ __forceinline__ Frag ldt(const double *tile, int lane) { // transposed tile
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    return {tile[cq * 8 + rq], tile[(cq + 1) * 8 + rq]};
}

// k-range modes of cta_gemm (which k-tiles can be nonzero)
enum : int { kAll = 0, kLeJ = 1, kGeMaxIJ = 2, kGeJ = 3 };

// C(i, j) = [Cin(i, j)] + sgn * sum_k opA(i, k) opB(j, k)'
//   opA(i, k) = TA ? A(k, i)' : A(i, k);  opB(j, k) = TB ? B(k, j)' : B(j, k)
// over the output tiles (i, j), j <= i only when LOWER; Cin may alias C.
template <int XT, int NW, bool TA, bool TB, int KM, bool LOWER>
__device__ __forceinline__ void cta_gemm(double *C, const double *Cin, double sgn, const double *A,
                                         const double *B, int warp, int lane) {
    constexpr int NO = LOWER ? XT * (XT + 1) / 2 : XT * XT;
    for (int o = warp; o < NO; o += NW) {
        int i, j;
        if (LOWER) {
            i = 0;
            while ((i + 1) * (i + 2) / 2 <= o)
                ++i;
            j = o - i * (i + 1) / 2;
        } else {
            i = o / XT;
            j = o % XT;
        }
        const int klo = KM == kGeMaxIJ ? (i > j ? i : j) : (KM == kGeJ ? j : 0);
        const int khi = KM == kLeJ ? j + 1 : XT;
        Frag acc = Cin ? ld_frag(Cin + (i * XT + j) * kTileElems, lane) : Frag{0.0, 0.0};
#pragma unroll
        for (int k = 0; k < XT; ++k) {
            if (k < klo || k >= khi)
                continue;
            const Frag a = TA ? ldt(A + (k * XT + i) * kTileElems, lane) : ld_frag(A + (i * XT + k) * kTileElems, lane);
            const Frag b = TB ? ldt(B + (k * XT + j) * kTileElems, lane) : ld_frag(B + (j * XT + k) * kTileElems, lane);
            dmma(acc, sgn * a.a, b.a);
            dmma(acc, sgn * a.b, b.b);
        }
        st_frag(C + (i * XT + j) * kTileElems, lane, acc);
    }
}

// In-place blocked lower Cholesky of the block M (lower tiles used; potrf
// semantics of kernels.cpp:32-58 with the pivot floor 1e-14 max|diag|) and
// its inverse Li = L^{-1} (lower tiles). The diagonal tile is factored by
// warp 0 with an identity tile carried through the pivot steps (L_kk^{-1}
// for free); sub-diagonal tiles are solved by DMMA against L_kk^{-1}; the
// off-diagonal inverse tiles follow row by row:
//   S'    = sum_{k=j}^{i-1} Li(k, j)' L(i, k)'
//   Li_ij = -Li_ii S''
// `scr` = 64 doubles of shared memory (transpose). Returns the first failing
// pivot (block-local index) in fail (warp 0 only; -1 if none).
template <int XT, int NW>
__device__ void cta_potrf_inv(double *M, double *Li, double *scr, int npiv, int warp, int lane,
                              int tid, int &fail) {
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    // pivot floor: max |diag| (every warp computes it; XT * 8 loads)
    double dmax = 0.0;
    for (int d = lane; d < 8 * XT; d += 32)
        if (d < npiv)
            dmax = fmax(dmax, fabs(M[((d / 8) * XT + d / 8) * kTileElems + (d % 8) * 9]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    const double dfloor = 1e-14 * dmax;
    for (int kb = 0; kb < XT; ++kb) {
        if (warp == 0) {
            Frag dg[1] = {ld_frag(M + (kb * XT + kb) * kTileElems, lane)};
            Frag zd[1], ld[1];
            int f = -1;
            tiles::chol_inv<1, 1>(dg, zd, ld, npiv - 8 * kb, dfloor, lane, f, scr);
            if (f >= 0 && fail < 0)
                fail = 8 * kb + f;
            st_frag(M + (kb * XT + kb) * kTileElems, lane, dg[0]);
            st_frag(Li + (kb * XT + kb) * kTileElems, lane, ld[0]);
        }
        __syncthreads();
        const Frag ldk = ld_frag(Li + (kb * XT + kb) * kTileElems, lane);
        for (int ti = kb + 1 + warp; ti < XT; ti += NW) { // X <- X L_kk^{-T}
            Frag r{0.0, 0.0};
            tile_gemm_nt(r, ld_frag(M + (ti * XT + kb) * kTileElems, lane), ldk);
            st_frag(M + (ti * XT + kb) * kTileElems, lane, r);
        }
        __syncthreads();
        // trailing update of the lower tiles kb < tj <= ti
        const int m = XT - kb - 1, nt = m * (m + 1) / 2;
        for (int o = warp; o < nt; o += NW) {
            int a = 0;
            while ((a + 1) * (a + 2) / 2 <= o)
                ++a;
            const int ti = kb + 1 + a, tj = kb + 1 + (o - a * (a + 1) / 2);
            Frag c = ld_frag(M + (ti * XT + tj) * kTileElems, lane);
            tile_gemm_nt_sub(c, ld_frag(M + (ti * XT + kb) * kTileElems, lane),
                             ld_frag(M + (tj * XT + kb) * kTileElems, lane));
            st_frag(M + (ti * XT + tj) * kTileElems, lane, c);
        }
        __syncthreads();
    }
    (void)tid;
    (void)rq;
    (void)cq;
    // off-diagonal tiles of L^{-1}, row by row
    for (int i = 1; i < XT; ++i) {
        for (int j = warp; j < i; j += NW) {
            Frag st{0.0, 0.0};
            for (int k = j; k < i; ++k)
                tile_gemm_nt(st, ldt(Li + (k * XT + j) * kTileElems, lane),
                             ld_frag(M + (i * XT + k) * kTileElems, lane));
            Frag li{0.0, 0.0};
            tile_gemm_nt_sub(li, ld_frag(Li + (i * XT + i) * kTileElems, lane), st);
            st_frag(Li + (i * XT + j) * kTileElems, lane, li);
        }
        __syncthreads();
    }
}

// Diagonal-tile inverses of an already factored lower L (memory): Li(k, k)
// = L_kk^{-1} for every k (warps take tiles), then the off-diagonal tiles
// of Li = L^{-1} as in cta_potrf_inv.
template <int XT, int NW>
__device__ void cta_trtri(const double *L, double *Li, double *scr, int warp, int lane) {
    for (int k = warp; k < XT; k += NW) {
        Frag lk[1] = {ld_frag(L + (k * XT + k) * kTileElems, lane)};
        Frag zd[1], ld[1];
        tiles::diag_inverses<1, 1>(lk, zd, ld, lane, scr + warp * kTileElems);
        st_frag(Li + (k * XT + k) * kTileElems, lane, ld[0]);
    }
    __syncthreads();
    for (int i = 1; i < XT; ++i) {
        for (int j = warp; j < i; j += NW) {
            Frag st{0.0, 0.0};
            for (int k = j; k < i; ++k)
                tile_gemm_nt(st, ldt(Li + (k * XT + j) * kTileElems, lane),
                             ld_frag(L + (i * XT + k) * kTileElems, lane));
            Frag li{0.0, 0.0};
            tile_gemm_nt_sub(li, ld_frag(Li + (i * XT + i) * kTileElems, lane), st);
            st_frag(Li + (i * XT + j) * kTileElems, lane, li);
        }
        __syncthreads();
    }
}

// y = op(M) v for a vector in shared memory (8 XT entries), M in memory;
// LOWER: only tiles j <= i of M are read (others are zero). Output written
// to y (shared, may not alias v); all warps participate (tile rows spread).
template <int XT, int NW, bool TRANS, bool LOWER>
__device__ __forceinline__ void cta_matvec(const double *M, const double *v, double *y, double sgn,
                                           bool accumulate, int warp, int lane) {
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    for (int r = warp; r < XT; r += NW) { // output tile row r (entries 8 r .. 8 r + 7)
        if (!TRANS) {
            double acc = 0.0;
            for (int j = 0; j < XT; ++j) {
                if (LOWER && j > r)
                    continue;
                const Frag f = ld_frag(M + (r * XT + j) * kTileElems, lane);
                acc = fma(f.a, v[8 * j + cq], acc);
                acc = fma(f.b, v[8 * j + cq + 1], acc);
            }
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            if ((lane & 3) == 0)
                y[8 * r + rq] = (accumulate ? y[8 * r + rq] : 0.0) + sgn * acc;
        } else { // y[8 r + c] = sum_i M(i, r)[.., c] v[i]
            double a0 = 0.0, a1 = 0.0;
            for (int i = 0; i < XT; ++i) {
                if (LOWER && r > i)
                    continue;
                const Frag f = ld_frag(M + (i * XT + r) * kTileElems, lane);
                const double vi = v[8 * i + rq];
                a0 = fma(f.a, vi, a0);
                a1 = fma(f.b, vi, a1);
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                a0 += __shfl_xor_sync(0xffffffffu, a0, o);
                a1 += __shfl_xor_sync(0xffffffffu, a1, o);
            }
            if (rq == 0) {
                y[8 * r + cq] = (accumulate ? y[8 * r + cq] : 0.0) + sgn * a0;
                y[8 * r + cq + 1] = (accumulate ? y[8 * r + cq + 1] : 0.0) + sgn * a1;
            }
        }
    }
}

} // namespace ctat
} // namespace cyqb
