// Register-resident 8x8 FP64 tile algorithms for one warp (compile-time
// tile shapes). A "panel" is a lower-trapezoidal set of C-fragment tiles
// P[T(i, j)], j <= i, rows 0..TT-1; its first CT tile columns are pivots.
//
// The blocked Cholesky restates batla::potrf + trsm(right_lower_trans) +
// syrk (kernels.cpp:32-58, 95-119, 158-168) for a stacked panel: the
// diagonal 8x8 tiles are factored with warp shuffles (one rsqrt per pivot),
// the rows below are solved in the same pivot steps, and the trailing
// updates are DMMA rank-8 products of register tiles.
#pragma once

#include "kkt_common.cuh"

namespace cyqb {
namespace tiles {

__host__ __device__ constexpr int T(int i, int j) { return i * (i + 1) / 2 + j; }

constexpr unsigned kFull = 0xffffffffu;

// Blocked Cholesky of the first CT tile columns of a TT-row panel.
// Pivots with global column index >= npiv are padding (unit, unchecked).
// On a pivot failure (potrf semantics: !(p > dfloor) or non-finite) the
// first failing global pivot index is stored in `fail` and the pivot is
// replaced by 1 so the sweep completes.
template <int TT, int CT, int NT>
__device__ __forceinline__ void panel_cholesky(Frag (&P)[NT], int npiv, double dfloor, int lane,
                                               int &fail) {
    const int rq = lane >> 2, cq = 2 * (lane & 3), q2 = lane & 3;
#pragma unroll
    for (int kb = 0; kb < CT; ++kb) {
        Frag &dg = P[T(kb, kb)];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int src = k / 2;
            const double vk = (k & 1) ? dg.b : dg.a;
            double pv = __shfl_sync(kFull, vk, 4 * k + src);
            const double urk = __shfl_sync(kFull, vk, 4 * rq + src);
            const double uc0 = __shfl_sync(kFull, vk, 4 * cq + src);
            const double uc1 = __shfl_sync(kFull, vk, 4 * (cq + 1) + src);
            if (8 * kb + k < npiv) {
                const bool bad = !(pv > dfloor && isfinite(pv));
                fail = (bad && fail < 0) ? 8 * kb + k : fail;
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
#pragma unroll
            for (int ti = kb + 1; ti < TT; ++ti) {
                Frag &x = P[T(ti, kb)];
                const double vq = (k & 1) ? x.b : x.a;
                const double xrq = __shfl_sync(kFull, vq, 4 * rq + src) * iv;
                if (k & 1)
                    x.b = (q2 == src) ? xrq : x.b;
                else
                    x.a = (q2 == src) ? xrq : x.a;
                x.a -= xrq * lc0;
                x.b -= xrq * lc1;
            }
        }
        if (cq > rq) dg.a = 0.0;
        if (cq + 1 > rq) dg.b = 0.0;
        if (kb + 1 < TT)
            tile_gemm_nt_sub(P[T(kb + 1, kb + 1)], P[T(kb + 1, kb)], P[T(kb + 1, kb)]);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int tj = kb + 1; tj < TT; ++tj)
#pragma unroll
                for (int ti = tj; ti < TT; ++ti)
                    if (!(ti == kb + 1 && tj == kb + 1)) {
                        const Frag &li = P[T(ti, kb)], &lj = P[T(tj, kb)];
                        dmma(P[T(ti, tj)], h ? -li.b : -li.a, h ? lj.b : lj.a);
                    }
    }
}

// Rows X (RT x CT tiles, X[i * CT + j]) <- X L^{-T} for a factored lower
// L (CT x CT tiles, L[T(i, j)]): TrsmMode::right_lower_trans
// (kernels.cpp:107-119) in the tile layout.
template <int RT, int CT, int NL>
__device__ __forceinline__ void trsm_rows(Frag (&X)[RT * CT], const Frag (&L)[NL], int lane) {
    const int rq = lane >> 2, cq = 2 * (lane & 3), q2 = lane & 3;
#pragma unroll
    for (int kb = 0; kb < CT; ++kb) {
        const Frag &dg = L[T(kb, kb)];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int src = k / 2;
            const double vk = (k & 1) ? dg.b : dg.a;
            const double dkk = __shfl_sync(kFull, vk, 4 * k + src);
            const double uc0 = __shfl_sync(kFull, vk, 4 * cq + src);
            const double uc1 = __shfl_sync(kFull, vk, 4 * (cq + 1) + src);
            const double iv = 1.0 / dkk;
            const double lc0 = (cq > k) ? uc0 : 0.0;
            const double lc1 = (cq + 1 > k) ? uc1 : 0.0;
#pragma unroll
            for (int ti = 0; ti < RT; ++ti) {
                Frag &x = X[ti * CT + kb];
                const double vq = (k & 1) ? x.b : x.a;
                const double xrq = __shfl_sync(kFull, vq, 4 * rq + src) * iv;
                if (q2 == src) {
                    if (k & 1) x.b = xrq;
                    else x.a = xrq;
                }
                x.a -= xrq * lc0;
                x.b -= xrq * lc1;
            }
        }
#pragma unroll
        for (int tj = kb + 1; tj < CT; ++tj)
#pragma unroll
            for (int ti = 0; ti < RT; ++ti)
                tile_gemm_nt_sub(X[ti * CT + tj], X[ti * CT + kb], L[T(tj, kb)]);
    }
}

// 1/a: MUFU.RCP64H seed + two Newton steps (full double precision for the
// positive finite pivots it is used on; no division slow path).
__device__ __forceinline__ double rcp_nr(double a) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a, y, 1.0);
    y = fma(y, e, y);
    e = fma(-a, y, 1.0);
    return fma(y, e, y);
}

// 8x8 transpose of a C-fragment tile through a 64-double shared scratch
__device__ __forceinline__ Frag tile_transpose(Frag x, double *scr, int lane) {
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    __syncwarp();
    st_frag(scr, lane, x);
    __syncwarp();
    Frag t{scr[cq * 8 + rq], scr[(cq + 1) * 8 + rq]};
    __syncwarp();
    return t;
}

// Lower Cholesky of an XT x XT tile block (lower tiles L[T(i, j)]) that also
// yields the inverses of its diagonal tiles: the identity tile carried
// through the same 8 pivot steps ends as Zd = L_kk^{-T}, Ld = L_kk^{-1} is
// its transpose. The sub-diagonal tiles are then solved by two DMMAs each
// (X L_kk^{-T} = X Ld') instead of eight dependent pivot updates.
// potrf semantics as panel_cholesky (kernels.cpp:32-58).
template <int XT, int NL>
__device__ __forceinline__ void chol_inv(Frag (&L)[NL], Frag (&Zd)[XT], Frag (&Ld)[XT], int npiv,
                                         double dfloor, int lane, int &fail, double *scr) {
    const int rq = lane >> 2, cq = 2 * (lane & 3), q2 = lane & 3;
#pragma unroll
    for (int kb = 0; kb < XT; ++kb) {
        Frag &dg = L[T(kb, kb)];
        Frag idt{rq == cq ? 1.0 : 0.0, rq == cq + 1 ? 1.0 : 0.0};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int src = k / 2;
            const double vk = (k & 1) ? dg.b : dg.a;
            double pv = __shfl_sync(kFull, vk, 4 * k + src);
            const double urk = __shfl_sync(kFull, vk, 4 * rq + src);
            const double uc0 = __shfl_sync(kFull, vk, 4 * cq + src);
            const double uc1 = __shfl_sync(kFull, vk, 4 * (cq + 1) + src);
            const double ik = (k & 1) ? idt.b : idt.a;
            const double irk = __shfl_sync(kFull, ik, 4 * rq + src);
            if (8 * kb + k < npiv) {
                const bool bad = !(pv > dfloor && isfinite(pv));
                fail = (bad && fail < 0) ? 8 * kb + k : fail;
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
            const double xrq = irk * iv;
            if (k & 1)
                idt.b = (q2 == src) ? xrq : idt.b;
            else
                idt.a = (q2 == src) ? xrq : idt.a;
            idt.a -= xrq * lc0;
            idt.b -= xrq * lc1;
        }
        if (cq > rq) dg.a = 0.0;
        if (cq + 1 > rq) dg.b = 0.0;
        Zd[kb] = idt;
        Ld[kb] = tile_transpose(idt, scr, lane);
#pragma unroll
        for (int ti = kb + 1; ti < XT; ++ti) {
            Frag r{0.0, 0.0};
            tile_gemm_nt(r, L[T(ti, kb)], Ld[kb]);
            L[T(ti, kb)] = r;
        }
        if (kb + 1 < XT)
            tile_gemm_nt_sub(L[T(kb + 1, kb + 1)], L[T(kb + 1, kb)], L[T(kb + 1, kb)]);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int tj = kb + 1; tj < XT; ++tj)
#pragma unroll
                for (int ti = tj; ti < XT; ++ti)
                    if (!(ti == kb + 1 && tj == kb + 1)) {
                        const Frag &li = L[T(ti, kb)], &lj = L[T(tj, kb)];
                        dmma(L[T(ti, tj)], h ? -li.b : -li.a, h ? lj.b : lj.a);
                    }
    }
}

// Diagonal-tile inverses of an already factored lower L (trtri on the
// diagonal tiles, kernels.cpp:246-271): the XT identity sweeps run
// interleaved (independent), Zd = L_kk^{-T}, Ld = L_kk^{-1}.
template <int XT, int NL>
__device__ __forceinline__ void diag_inverses(const Frag (&L)[NL], Frag (&Zd)[XT], Frag (&Ld)[XT],
                                              int lane, double *scr) {
    const int rq = lane >> 2, cq = 2 * (lane & 3), q2 = lane & 3;
#pragma unroll
    for (int kb = 0; kb < XT; ++kb)
        Zd[kb] = Frag{rq == cq ? 1.0 : 0.0, rq == cq + 1 ? 1.0 : 0.0};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int src = k / 2;
#pragma unroll
        for (int kb = 0; kb < XT; ++kb) {
            const Frag &dg = L[T(kb, kb)];
            Frag &idt = Zd[kb];
            const double vk = (k & 1) ? dg.b : dg.a;
            const double pv = __shfl_sync(kFull, vk, 4 * k + src);
            const double uc0 = __shfl_sync(kFull, vk, 4 * cq + src);
            const double uc1 = __shfl_sync(kFull, vk, 4 * (cq + 1) + src);
            const double ik = (k & 1) ? idt.b : idt.a;
            const double xrq = __shfl_sync(kFull, ik, 4 * rq + src) * rcp_nr(pv);
            const double lc0 = (cq > k) ? uc0 : 0.0;
            const double lc1 = (cq + 1 > k) ? uc1 : 0.0;
            if (k & 1)
                idt.b = (q2 == src) ? xrq : idt.b;
            else
                idt.a = (q2 == src) ? xrq : idt.a;
            idt.a -= xrq * lc0;
            idt.b -= xrq * lc1;
        }
    }
#pragma unroll
    for (int kb = 0; kb < XT; ++kb)
        Ld[kb] = tile_transpose(Zd[kb], scr + kb * kTileElems, lane);
}

// Blocked inverse of a factored lower L from its diagonal-tile inverses,
// NT-form DMMA products only (C += A B'):
//   St    = sum_{k=j}^{i-1} Z_jk L_ik'     (= (sum_k L_ik Li_kj)')
//   Li_ij = -Ld_i St'                      (L^{-1}, lower, row tiles)
//   Z_ji  = -St Ld_i'                      (L^{-T}, upper, row tiles)
// Z is XT x XT (i * XT + j); Li lower tiles T(i, j).
template <int XT, int NL>
__device__ __forceinline__ void blocked_inverse(const Frag (&L)[NL], const Frag (&Zd)[XT],
                                                const Frag (&Ld)[XT], Frag (&Li)[NL],
                                                Frag (&Z)[XT * XT]) {
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
        for (int j = 0; j < XT; ++j)
            if (i > j)
                Z[i * XT + j] = Frag{0.0, 0.0};
#pragma unroll
    for (int i = 0; i < XT; ++i) {
        Li[T(i, i)] = Ld[i];
        Z[i * XT + i] = Zd[i];
    }
#pragma unroll
    for (int i = 1; i < XT; ++i)
#pragma unroll
        for (int j = i - 1; j >= 0; --j) {
            Frag st{0.0, 0.0};
#pragma unroll
            for (int k = j; k < i; ++k)
                tile_gemm_nt(st, Z[j * XT + k], L[T(i, k)]);
            Frag li{0.0, 0.0}, z{0.0, 0.0};
            tile_gemm_nt_sub(li, Ld[i], st);
            tile_gemm_nt_sub(z, st, Ld[i]);
            Li[T(i, j)] = li;
            Z[j * XT + i] = z;
        }
}

// max |diag| over the first npiv diagonal entries of the CT diagonal tiles
template <int CT, int NT>
__device__ __forceinline__ double diag_absmax(const Frag (&P)[NT], int npiv, int lane) {
    const int rq = lane >> 2;
    double m = 0.0;
#pragma unroll
    for (int kb = 0; kb < CT; ++kb) {
        const Frag &d = P[T(kb, kb)];
        const double v = (rq & 1) ? d.b : d.a;
        if ((lane & 3) == rq / 2 && 8 * kb + rq < npiv)
            m = fmax(m, fabs(v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        m = fmax(m, __shfl_xor_sync(kFull, m, o));
    return m;
}

} // namespace tiles
} // namespace cyqb
