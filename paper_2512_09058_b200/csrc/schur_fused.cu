// Schur complement + cyclic reduction, factor and solve, fused into ONE
// kernel per batch: one CTA per OCP instance, NW warps taking the
// independent block operations of each phase, __syncthreads between the
// phases/levels. All per-instance blocks are 8x8-tile-ordered (C-fragment
// order, XT x XT tiles per nx x nx block) so every load/store is a coalesced
// 512-byte tile, and the whole instance's working set stays hot in L2 for
// the few microseconds the CTA lives (the per-level batch-wide kernels in
// schur_tiles.cu stream it through HBM instead).
//
// Restates:
//   kkt_factor.cpp:163-178    T = L_Q^{-T}, Mbwd = T T', W = T LA'
//   kkt_factor.cpp:194-212    assemble_schur: diag[c] = Mfwd_c + Mbwd_{c+1},
//                             subdiag[c-1] = -W_c' = -LA_c T_c'
//   block_tridiag.cpp:126-171 cr_level: L = chol(M_k), U = K_{k-1}' L^{-T},
//                             Y = K_k L^{-T}, M' = M - U U' - Y_prev Y_prev',
//                             K' = -Y U'
//   block_tridiag.cpp:173-197 cr_factor_base
//   kkt_solve.cpp:137-182     Schur rhs b_i = fd[n i] - fwd_i + bwd_neg_{i+1}
//   block_tridiag.cpp:252-333 CRFactor::forward / backward, then negate
//
// B200 reformulation: each elimination forms Linv = L^{-1} once -- the
// Cholesky carries an identity tile through its pivot steps (diagonal-tile
// inverses for free), the off-diagonal inverse tiles are NT-form DMMA
// products (tiles::blocked_inverse) -- so U, Y are DMMA products (U = K_{k-1}' Linv', Y = K_k Linv') instead of
// two dependent triangular solves, and the CR solve is matrix-vector
// products only (L^{-1} v = Linv v, L^{-T} v = Linv' v): no sequential
// trsv on the solve path. K_{k-1}' is read as transposed tiles directly from
// the tile-ordered workspace (two 8-byte loads per lane per tile).
#include "kernels.h"
#include "tiles.cuh"

#include <cooperative_groups.h>

#include <cstdlib>

namespace cyqb {

using tiles::T;

namespace {

template <int NX> struct SF {
    static constexpr int XT = (NX + 7) / 8;
    static constexpr int NL = XT * (XT + 1) / 2; // tiles of a lower block
    static constexpr int NF = XT * XT;           // tiles of a full block
    static constexpr int XP = 8 * XT;            // padded vector length
};

__device__ __forceinline__ int fidx(int XT, int i, int j) { return i * XT + j; }

// transposed 8x8 tile load from the tile-ordered workspace: returns the
// C-fragment of tile' (lane holds X'[rq][cq], X'[rq][cq+1] = X[cq][rq], X[cq+1][rq])
__device__ __forceinline__ Frag ld_frag_t(const double *tile, int lane) {
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    return {tile[cq * 8 + rq], tile[(cq + 1) * 8 + rq]};
}

// workspace loads: ld.global.cg (L2) when the blocks are rewritten by other
// SMs (the cluster variant), ld.global.ca (L1 + L2) when one CTA owns the
// instance -- the CTA's own global stores invalidate its L1 lines, and the
// __syncthreads between phases orders them (config 0 Schur: 25 -> 21 us)
template <bool L1> __device__ __forceinline__ Frag ldw(const double *tile, int lane) {
    const double2 v = L1 ? __ldca(reinterpret_cast<const double2 *>(tile) + lane)
                         : __ldcg(reinterpret_cast<const double2 *>(tile) + lane);
    return {v.x, v.y};
}
template <bool L1> __device__ __forceinline__ Frag ldw_t(const double *tile, int lane) {
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    if (L1)
        return {__ldca(tile + cq * 8 + rq), __ldca(tile + (cq + 1) * 8 + rq)};
    return {__ldcg(tile + cq * 8 + rq), __ldcg(tile + (cq + 1) * 8 + rq)};
}

__device__ __forceinline__ Frag fadd(Frag x, Frag y) { return {x.a + y.a, x.b + y.b}; }
__device__ __forceinline__ Frag fsub(Frag x, Frag y) { return {x.a - y.a, x.b - y.b}; }

__device__ __forceinline__ double fac_elem(const Geo &g, const double *st, int r, int col) {
    const int ti = r / 8, tj = col / 8;
    const int t = ti < g.CT ? tri_index(ti, tj) : g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
    return __ldg(st + t * kTileElems + (r % 8) * 8 + col % 8);
}

// y = M v (FULL: XT x XT tiles; else lower tiles T(i, j)); v: XP doubles in
// shared memory; out[i] = row 8 i + rq, valid in every lane of the quad
template <int XT, bool FULL, bool L1>
__device__ __forceinline__ void matvec(const double *M, const double *v, double (&out)[XT], int lane) {
    const int cq = 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < XT; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < XT; ++j) {
            if (!FULL && j > i)
                continue;
            const Frag f = ldw<L1>(M + (FULL ? fidx(XT, i, j) : T(i, j)) * kTileElems, lane);
            acc = fma(f.a, v[8 * j + cq], acc);
            acc = fma(f.b, v[8 * j + cq + 1], acc);
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        out[i] = acc;
    }
}
// y = M' v; out[j][h] = entry 8 j + cq + h, valid in every lane with that cq
template <int XT, bool FULL, bool L1>
__device__ __forceinline__ void matvec_t(const double *M, const double *v, double (&out)[XT][2],
                                         int lane) {
    const int rq = lane >> 2;
#pragma unroll
    for (int j = 0; j < XT; ++j) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int i = 0; i < XT; ++i) {
            if (!FULL && j > i)
                continue;
            const Frag f = ldw<L1>(M + (FULL ? fidx(XT, i, j) : T(i, j)) * kTileElems, lane);
            const double vi = v[8 * i + rq];
            a0 = fma(f.a, vi, a0);
            a1 = fma(f.b, vi, a1);
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        }
        out[j][0] = a0;
        out[j][1] = a1;
    }
}


// tile slot of block tile (i, j) for the three storage modes
enum : int { kFull = 0, kLower = 1, kUpper = 2 };
template <int XT, int MODE> __device__ __forceinline__ constexpr bool tile_present(int i, int j) {
    return MODE == kFull || (MODE == kLower ? j <= i : j >= i);
}
template <int XT, int MODE> __device__ __forceinline__ constexpr int tile_slot(int i, int j) {
    return MODE == kFull ? i * XT + j : (MODE == kLower ? T(i, j) : T(j, i));
}

// y = M v with M in registers (same conventions as matvec)
template <int XT, int MODE, int N>
__device__ __forceinline__ void matvec_r(const Frag (&M)[N], const double *v, double (&out)[XT],
                                         int lane) {
    const int cq = 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < XT; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < XT; ++j) {
            if (!tile_present<XT, MODE>(i, j))
                continue;
            const Frag f = M[tile_slot<XT, MODE>(i, j)];
            acc = fma(f.a, v[8 * j + cq], acc);
            acc = fma(f.b, v[8 * j + cq + 1], acc);
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        out[i] = acc;
    }
}
// y = M v with M upper triangular stored as tiles T(j, i) (memory)
template <int XT, bool L1>
__device__ __forceinline__ void matvec_upper(const double *M, const double *v, double (&out)[XT],
                                             int lane) {
    const int cq = 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < XT; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = i; j < XT; ++j) {
            const Frag f = ldw<L1>(M + T(j, i) * kTileElems, lane);
            acc = fma(f.a, v[8 * j + cq], acc);
            acc = fma(f.b, v[8 * j + cq + 1], acc);
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        out[i] = acc;
    }
}

} // namespace

// Per-instance workspace of the fused path, in 8x8 tiles (64 doubles):
//   Tt[P]   upper   T_c = L_Q(last stage)^{-T} per column, tile (i, j) at
//                   slot T(j, i)                             (persistent)
//   Li[P-1] lower   L^{-1} of every odd-block elimination    (persistent)
//   U[P-1], Y[P-1]  full                                      (persistent)
//   Lb      lower   L_base^{-1}                               (persistent)
//   D[P], Mb[P]     lower: Mfwd_c, Mbwd_c                     (scratch)
//   K[P]    full    level-0 subdiagonal                       (scratch)
// Li/U/Y of level l (half = P >> (l+1) blocks) start at block P - (P >> l).
// The CR levels run in place in D / K: at level l, block i is
//   M_i = D[i << l] - D[(i << l) - 2^(l-1)]  (l > 0, i > 0; the CY term)
//   M_i = D[i] + Mb[(i + 1) % P]             (l = 0)
//   K_i = K[i << l]
// and elimination mm writes M' -> D[2mm << l], CY -> D[(2mm+1) << l],
// K' -> K[2mm << l]: every slot is read and rewritten by one warp only.
//   PCR tail (g.tail = T > 1 blocks, FactorOptions::tail = pcr):
//   PLi[(lgT+1) T] lower, PU[lgT T], PY[lgT T] full   (persistent)
//   PM[2 T] lower, PK[2 T] full                        (scratch, by level parity)
// The CR levels then stop at crl = levels - lgT (T blocks left) and the
// base factorization is replaced by the PCR levels.
struct SFLayout {
    long long Tt, Li, U, Y, Lb, D, Mb, K, PLi, PU, PY, PM, PK, total; // doubles
    int XT, NL, NF, XP, levels, T, lgT, crl;
    __host__ __device__ static SFLayout make(int P, int nx, int tail = 1) {
        SFLayout s;
        s.XT = (nx + 7) / 8;
        s.NL = s.XT * (s.XT + 1) / 2;
        s.NF = s.XT * s.XT;
        s.XP = 8 * s.XT;
        int lg = 0;
        while ((1 << lg) < P)
            ++lg;
        s.levels = lg;
        const long long tl = 64LL * s.NL, tf = 64LL * s.NF;
        long long o = 0;
        s.Tt = o; o += P * tl;
        s.Li = o; o += (P - 1) * tl;
        s.U = o; o += (P - 1) * tf;
        s.Y = o; o += (P - 1) * tf;
        s.Lb = o; o += tl;
        s.D = o; o += P * tl;
        s.Mb = o; o += P * tl;
        s.K = o; o += P * tf;
        s.T = tail > 1 ? tail : 1;
        s.lgT = 0;
        while ((1 << s.lgT) < s.T)
            ++s.lgT;
        s.crl = s.levels - s.lgT;
        s.PLi = o; o += (s.T > 1 ? (s.lgT + 1) * s.T : 0) * tl;
        s.PU = o; o += (long long)s.lgT * s.T * tf;
        s.PY = o; o += (long long)s.lgT * s.T * tf;
        s.PM = o; o += (s.T > 1 ? 2 * s.T : 0) * tl;
        s.PK = o; o += (s.T > 1 ? 2 * s.T : 0) * tf;
        s.total = o;
        return s;
    }
};

size_t schur_fused_doubles(const Geo &g) { return (size_t)SFLayout::make(g.P, g.nx, g.tail).total; }

bool schur_fused_blocks(const Geo &g, SchurBlocks &out) {
    const SFLayout L = SFLayout::make(g.P, g.nx, g.tail);
    out = SchurBlocks{L.Tt, L.Li, L.U, L.Y, L.Lb, L.Mb, L.total, false, false, L.crl};
    return true;
}

namespace {

template <int XP> __host__ __device__ constexpr size_t sf_smem_doubles(int NW, int NF, int P) {
    return (size_t)NW * NF * kTileElems + 2 * (size_t)P * XP;
}

// CL > 1: one thread-block CLUSTER per instance (a single long horizon,
// config 2): the tasks of every phase / CR level are spread over the CL * NW
// warps of the cluster, phases are separated by cluster barriers (release /
// acquire: the global workspace writes of one CTA are visible to the
// others), and the solve vectors live in rank 0's shared memory, reached
// through distributed shared memory.
template <int NX, int NW, int CL>
__global__ void __launch_bounds__(32 * NW, NW <= 4 ? 16 / NW : 1) schur_fused_kernel(SchurArgs a) {
    using F = SF<NX>;
    constexpr int XT = F::XT, NL = F::NL, NF = F::NF, XP = F::XP;
    constexpr bool L1 = CL == 1;
    constexpr long long TL = 64LL * NL, TF = 64LL * NF;
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    namespace cg = cooperative_groups;
    const int crank = CL > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int b = blockIdx.x / CL, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int vwarp = crank * NW + warp, vtid = crank * 32 * NW + threadIdx.x;
    griddep_launch();
    griddep_wait(); // the stage panel's factor tiles
    constexpr int VNW = CL * NW, VNTH = CL * 32 * NW;
    auto csync = [&]() {
        if (CL > 1)
            cg::this_cluster().sync();
        else
            __syncthreads();
    };
    const int rq = lane >> 2, cq = 2 * (lane & 3), q2 = lane & 3;
    const int P = g.P, nu = g.nu, n = g.n, top = 8 * g.CT;
    const SFLayout Lo = SFLayout::make(P, NX, g.tail);
    double *ws = a.schur + (size_t)b * Lo.total;
    double *scr = sm + (size_t)warp * NF * kTileElems; // per-warp transpose scratch
    // solve vectors: xs (P x XP) and bwd_neg (P x XP), the latter dead once
    // the Schur rhs is assembled and reused for the even-block contributions
    // U x_k | Y x_k of the CR levels; in a cluster xs lives in rank 0's and
    // bwd_neg in rank 1's shared memory (DSMEM)
    double *vecs = sm + (size_t)NW * NF * kTileElems;
    double *xs = vecs, *bns = vecs + (size_t)P * XP;
    if (CL > 1) {
        xs = cg::this_cluster().map_shared_rank(vecs, 0);
        bns = cg::this_cluster().map_shared_rank(vecs, 1);
    }
    double *cu = bns;                                  // P/2 x XP each
    double *cy = cu + (size_t)(P / 2) * XP;
    double *D = ws + Lo.D, *Mb = ws + Lo.Mb, *K = ws + Lo.K;
    unsigned long long my_fail = ~0ull;
    const bool fwd_fused = a.do_factor && a.do_solve; // CR forward inside the factor levels
    long long *ph = (a.phase && b == 0 && crank == 0 && threadIdx.x == 0) ? a.phase : nullptr;
    int php = 0;
    if (ph) ph[php++] = clock64();

    // ---- phase 1: per-column T, Mbwd, K, Mfwd and bwd_neg ----------------
    // (kkt_factor.cpp:163-178, 194-212; kkt_solve.cpp:128-131)
    for (int c = vwarp; c < P; c += VNW) {
        const size_t chain = (size_t)b * P + c;
        const double *yv = a.y + (chain * n + (n - 1)) * g.nux + nu;
        if (a.do_factor) {
            const double *st = a.fac + (chain * n + (n - 1)) * g.NPT * kTileElems;
            const double *tr = a.trail + chain * g.NTT * kTileElems;
            Frag Lq[NL];
            double *Dc = D + c * TL;
#pragma unroll
            for (int i = 0; i < XT; ++i)
#pragma unroll
                for (int j = 0; j <= i; ++j) {
                    Frag dm;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int r = 8 * i + rq, k = 8 * j + cq + h;
                        const bool in = r < NX && k < NX;
                        (h ? Lq[T(i, j)].b : Lq[T(i, j)].a) =
                            in ? (k <= r ? fac_elem(g, st, nu + r, nu + k) : 0.0) : (r == k ? 1.0 : 0.0);
                        // Mfwd_c = -(trailing coupling block), unit padding diagonal
                        const int rr = r > k ? r : k, kk = r > k ? k : r;
                        (h ? dm.b : dm.a) =
                            in ? -__ldg(tr + tri_index(rr / 8, kk / 8) * kTileElems + (rr % 8) * 8 + kk % 8)
                               : (r == k ? 1.0 : 0.0);
                    }
                    st_frag(Dc + T(i, j) * kTileElems, lane, dm);
                }
            double yx[XT][2];
            if (a.do_solve)
#pragma unroll
                for (int j = 0; j < XT; ++j) {
                    const int k = 8 * j + cq;
                    yx[j][0] = k < NX ? __ldg(yv + k) : 0.0;
                    yx[j][1] = k + 1 < NX ? __ldg(yv + k + 1) : 0.0;
                }
            Frag X[NF]; // T = L_Q^{-T} (rows): diagonal-tile inverses + blocked DMMA inverse
            {
                Frag Zd[XT], Ld[XT], Li[NL];
                tiles::diag_inverses<XT, NL>(Lq, Zd, Ld, lane, scr);
                tiles::blocked_inverse<XT, NL>(Lq, Zd, Ld, Li, X);
            }
            // persistent T: read again only by kkt::solve on a kept factor --
            // a factor + solve call works on transient scratch
            if (!a.do_solve) {
                double *Tc = ws + Lo.Tt + c * TL;
#pragma unroll
                for (int i = 0; i < XT; ++i)
#pragma unroll
                    for (int j = i; j < XT; ++j)
                        st_frag(Tc + T(j, i) * kTileElems, lane, X[i * XT + j]);
            }
            // Mbwd = T T' (kkt_factor.cpp:174), lower tiles
            double *Mbc = Mb + c * TL;
#pragma unroll
            for (int i = 0; i < XT; ++i)
#pragma unroll
                for (int j = 0; j <= i; ++j) {
                    Frag acc{0.0, 0.0};
#pragma unroll
                    for (int t = i; t < XT; ++t) // T upper: X[i][t] = 0 for t < i
                        tile_gemm_nt(acc, X[i * XT + t], X[j * XT + t]);
                    st_frag(Mbc + T(i, j) * kTileElems, lane, acc);
                }
            // subdiag[c-1] = -W_c' = -LA T' (kkt_factor.cpp:203-209); K[P-1] = 0
            double *Kc = K + (size_t)((c + P - 1) % P) * TF;
#pragma unroll
            for (int i = 0; i < XT; ++i) {
                Frag la[XT];
#pragma unroll
                for (int t = 0; t < XT; ++t)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int r = 8 * i + rq, k = 8 * t + cq + h;
                        (h ? la[t].b : la[t].a) =
                            (c > 0 && r < NX && k < NX) ? fac_elem(g, st, top + r, nu + k) : 0.0;
                    }
#pragma unroll
                for (int j = 0; j < XT; ++j) {
                    Frag acc{0.0, 0.0};
#pragma unroll
                    for (int t = j; t < XT; ++t)
                        tile_gemm_nt_sub(acc, la[t], X[j * XT + t]);
                    st_frag(Kc + (i * XT + j) * kTileElems, lane, acc);
                }
            }
            if (a.do_solve) { // bwd_neg_c = T x'_{n-1}
#pragma unroll
                for (int i = 0; i < XT; ++i) {
                    double acc = 0.0;
#pragma unroll
                    for (int j = i; j < XT; ++j) {
                        acc = fma(X[i * XT + j].a, yx[j][0], acc);
                        acc = fma(X[i * XT + j].b, yx[j][1], acc);
                    }
                    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                    if (q2 == 0)
                        bns[c * XP + 8 * i + rq] = acc;
                }
            }
        } else if (a.do_solve) { // solve only: bwd_neg_c from the stored T
            if (lane < XP)
                scr[lane] = lane < NX ? __ldg(yv + lane) : 0.0;
            __syncwarp();
            double o[XT];
            matvec_upper<XT, L1>(ws + Lo.Tt + c * TL, scr, o, lane);
#pragma unroll
            for (int i = 0; i < XT; ++i)
                if (q2 == 0)
                    bns[c * XP + 8 * i + rq] = o[i];
            __syncwarp();
        }
    }
    csync();
    if (ph) ph[php++] = clock64();

    // ---- Schur rhs b_i = fd[n i] - fwd_i + bwd_neg_{(i+1) % P} -----------
    // (kkt_solve.cpp:137-160); fd[0] of EqRhs::of_problem carries -A_0 x_init
    if (a.do_solve) {
        ProbAcc pa{a.p, g, b};
        for (int e = vtid; e < P * XP; e += VNTH) {
            const int i = e / XP, k = e % XP;
            double v = 0.0;
            if (k < NX) {
                const int jst = n * i;
                v = pa.fd(jst, k);
                if (jst == 0 && a.p.fd == nullptr) {
                    double ax = 0.0;
#pragma unroll
                    for (int m = 0; m < NX; ++m)
                        ax = fma(pa.A(0, k, m), __ldg(a.p.x_init + (size_t)b * NX + m), ax);
                    v -= ax;
                }
                const double *tr = a.trail + ((size_t)b * P + i) * g.NTT * kTileElems;
                v += __ldg(tr + tri_index(NX / 8, k / 8) * kTileElems + (NX % 8) * 8 + k % 8);
                v += bns[((i + 1) % P) * XP + k];
            }
            xs[e] = v;
        }
        csync();
    }

    // M_i of the level-l reduced system (see SFLayout)
    auto m_at = [&](int l, int i, int ti, int tj) -> Frag {
        if (l == 0)
            return fadd(ldw<L1>(D + i * TL + T(ti, tj) * kTileElems, lane),
                        ldw<L1>(Mb + ((i + 1) % P) * TL + T(ti, tj) * kTileElems, lane));
        Frag f = ldw<L1>(D + (i << l) * TL + T(ti, tj) * kTileElems, lane);
        if (i > 0)
            f = fsub(f, ldw<L1>(D + ((i << l) - (1 << (l - 1))) * TL + T(ti, tj) * kTileElems, lane));
        return f;
    };
    const int Tb = Lo.T, Lc = Lo.crl; // PCR tail blocks, CR levels before it
    double *bt = cu;                  // PCR: L^{-1} x per tail block (T x XP, dead cu / cy)

    // ---- phase 2: CR levels (block_tridiag.cpp:126-238), in place ---------
    // With a right-hand side at hand the CR forward sweep
    // (block_tridiag.cpp:252-296) runs inside the levels on the register
    // tiles: x_k <- L^{-1} x_k, then U x_k / Y x_k go to the even blocks.
    if (a.do_factor) {
        for (int l = 0, s = P; l < Lc; ++l, s >>= 1) {
            const int half = s / 2;
            const long long out0 = P - (P >> l);
            auto m_tile = [&](int i, int ti, int tj) -> Frag { return m_at(l, i, ti, tj); };
            for (int mm = vwarp; mm < half; mm += VNW) {
                const int k = 2 * mm + 1;
                const bool has_y = k < s - 1;
                const double *Kp = K + ((k - 1) << l) * TF, *Kk = K + (k << l) * TF;
                Frag Lt[NL];
#pragma unroll
                for (int i = 0; i < XT; ++i)
#pragma unroll
                    for (int j = 0; j <= i; ++j)
                        Lt[T(i, j)] = m_tile(k, i, j);
                const double dfloor = 1e-14 * tiles::diag_absmax<XT>(Lt, NX, lane);
                int pf = -1;
                Frag Li[NL];
                {
                    Frag Zd[XT], Ld[XT], Z[NF];
                    tiles::chol_inv<XT, NL>(Lt, Zd, Ld, NX, dfloor, lane, pf, scr);
                    tiles::blocked_inverse<XT, NL>(Lt, Zd, Ld, Li, Z);
                }
                if (pf >= 0)
                    my_fail = min(my_fail, fail_key(kKindCR, l, k, pf));
                double *Lio = ws + Lo.Li + (out0 + mm) * TL;
#pragma unroll
                for (int t = 0; t < NL; ++t)
                    st_frag(Lio + t * kTileElems, lane, Li[t]);
                double *xk = xs + (size_t)(k << l) * XP;
                if (fwd_fused) { // x_k <- L^{-1} x_k
                    double o[XT];
                    matvec_r<XT, kLower>(Li, xk, o, lane);
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < XT; ++i)
                        if (q2 == 0)
                            xk[8 * i + rq] = o[i];
                    __syncwarp();
                }
                // U = K_{k-1}' Linv', Y = K_k Linv' (Y = 0 at the last slot)
                Frag U[NF], Y[NF];
#pragma unroll
                for (int i = 0; i < XT; ++i) {
                    Frag kp[XT], kk[XT];
#pragma unroll
                    for (int t = 0; t < XT; ++t) {
                        kp[t] = ldw_t<L1>(Kp + fidx(XT, t, i) * kTileElems, lane); // (K_{k-1}')(i, t)
                        kk[t] = has_y ? ldw<L1>(Kk + fidx(XT, i, t) * kTileElems, lane) : Frag{0.0, 0.0};
                    }
#pragma unroll
                    for (int j = 0; j < XT; ++j) {
                        Frag u{0.0, 0.0}, y{0.0, 0.0};
#pragma unroll
                        for (int t = 0; t <= j; ++t) {
                            tile_gemm_nt(u, kp[t], Li[T(j, t)]);
                            tile_gemm_nt(y, kk[t], Li[T(j, t)]);
                        }
                        U[i * XT + j] = u;
                        Y[i * XT + j] = y;
                    }
                }
                double *Uo = ws + Lo.U + (out0 + mm) * TF, *Yo = ws + Lo.Y + (out0 + mm) * TF;
#pragma unroll
                for (int t = 0; t < NF; ++t) {
                    st_frag(Uo + t * kTileElems, lane, U[t]);
                    st_frag(Yo + t * kTileElems, lane, Y[t]);
                }
                if (fwd_fused) { // contributions U x_k -> x_{2mm}, Y x_k -> x_{2mm+2}
                    double ou[XT], oy[XT];
                    matvec_r<XT, kFull>(U, xk, ou, lane);
                    matvec_r<XT, kFull>(Y, xk, oy, lane);
#pragma unroll
                    for (int i = 0; i < XT; ++i)
                        if (q2 == 0) {
                            cu[mm * XP + 8 * i + rq] = ou[i];
                            cy[mm * XP + 8 * i + rq] = oy[i];
                        }
                }
                // M' = M_{2mm} - U U' -> D[2mm << l] (the Y_{mm-1} term is
                // subtracted by the next level's loads), CY = Y Y' ->
                // D[(2mm+1) << l], K' = -Y U' -> K[2mm << l]
                double *M2o = D + ((2 * mm) << l) * TL, *CYo = D + (k << l) * TL;
                double *K2o = K + ((2 * mm) << l) * TF;
                const bool last = mm == half - 1;
#pragma unroll
                for (int i = 0; i < XT; ++i)
#pragma unroll
                    for (int j = 0; j < XT; ++j) {
                        Frag uu{0.0, 0.0}, yy{0.0, 0.0}, yu{0.0, 0.0};
#pragma unroll
                        for (int t = 0; t < XT; ++t) {
                            if (j <= i) {
                                tile_gemm_nt(uu, U[i * XT + t], U[j * XT + t]);
                                tile_gemm_nt(yy, Y[i * XT + t], Y[j * XT + t]);
                            }
                            if (!last)
                                tile_gemm_nt_sub(yu, Y[i * XT + t], U[j * XT + t]);
                        }
                        if (j <= i) {
                            st_frag(M2o + T(i, j) * kTileElems, lane, fsub(m_tile(2 * mm, i, j), uu));
                            st_frag(CYo + T(i, j) * kTileElems, lane, yy);
                        }
                        st_frag(K2o + fidx(XT, i, j) * kTileElems, lane, yu);
                    }
            }
            csync();
            if (fwd_fused) { // x_{2mm} -= U_mm x_{2mm+1} + Y_{mm-1} x_{2mm-1}
                for (int e = vtid; e < half * XP; e += VNTH) {
                    const int mm = e / XP, r = e % XP;
                    double d = cu[e];
                    if (mm > 0)
                        d += cy[e - XP];
                    xs[(size_t)((2 * mm) << l) * XP + r] -= d;
                }
                csync();
            }
            if (ph) ph[php++] = clock64();
        }
        if (Tb == 1) {
            // ---- cr_factor_base (block_tridiag.cpp:173-197) --------------------
            if (vwarp == 0) {
                Frag Lt[NL];
#pragma unroll
                for (int i = 0; i < XT; ++i)
#pragma unroll
                    for (int j = 0; j <= i; ++j)
                        Lt[T(i, j)] = Lo.levels == 0
                                          ? fadd(ldw<L1>(D + T(i, j) * kTileElems, lane),
                                                 ldw<L1>(Mb + T(i, j) * kTileElems, lane))
                                          : ldw<L1>(D + T(i, j) * kTileElems, lane);
                const double dfloor = 1e-14 * tiles::diag_absmax<XT>(Lt, NX, lane);
                int pf = -1;
                Frag Li[NL];
                {
                    Frag Zd[XT], Ld[XT], Z[NF];
                    tiles::chol_inv<XT, NL>(Lt, Zd, Ld, NX, dfloor, lane, pf, scr);
                    tiles::blocked_inverse<XT, NL>(Lt, Zd, Ld, Li, Z);
                }
                if (pf >= 0)
                    my_fail = min(my_fail, fail_key(kKindCR, Lo.levels, 0, pf));
#pragma unroll
                for (int t = 0; t < NL; ++t)
                    st_frag(ws + Lo.Lb + t * kTileElems, lane, Li[t]);
                if (fwd_fused) { // base solve x_0 <- L_b^{-T} L_b^{-1} x_0
                    double o[XT], o2[XT][2];
                    matvec_r<XT, kLower>(Li, xs, o, lane);
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < XT; ++i)
                        if (q2 == 0)
                            xs[8 * i + rq] = o[i];
                    __syncwarp();
                    matvec_t<XT, false, L1>(ws + Lo.Lb, xs, o2, lane);
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < XT; ++j)
                        if (rq == 0) {
                            xs[8 * j + cq] = o2[j][0];
                            xs[8 * j + cq + 1] = o2[j][1];
                        }
                }
            }
        } else {
            // ---- PCR tail (block_tridiag.cpp:364-486, pcr_factor) on the T
            // blocks left at level Lc: every level works on all T blocks;
            // level pl (stride st = 2^pl) forms L_k^{-1}, Y_k = K_k L_k^{-T},
            // U_k = K_{k-st}' L_k^{-T}, then M'_k = M_k - Y_{k-st} Y_{k-st}' -
            // U_{k+st} U_{k+st}', K'_k = -Y_{k+st} U_{k+st}' (the wrapped
            // couplings of the non-circular tail are zero and skipped); the
            // last level factors every block. With a rhs the resolve
            // (PCRFactor::resolve) runs inside the levels.
            auto pm = [&](int pl, int k, int ti, int tj) -> Frag {
                return pl == 0 ? m_at(Lc, k, ti, tj)
                               : ldw<L1>(ws + Lo.PM + ((pl - 1) & 1) * Tb * TL + k * TL + T(ti, tj) * kTileElems,
                                     lane);
            };
            auto pk = [&](int pl, int k) -> const double * {
                return pl == 0 ? K + (size_t)(k << Lc) * TF : ws + Lo.PK + ((pl - 1) & 1) * Tb * TF + k * TF;
            };
            for (int pl = 0; pl <= Lo.lgT; ++pl) {
                const int st = 1 << pl;
                const bool fin = pl == Lo.lgT;
                for (int k = vwarp; k < Tb; k += VNW) {
                    Frag Lt[NL];
#pragma unroll
                    for (int i = 0; i < XT; ++i)
#pragma unroll
                        for (int j = 0; j <= i; ++j)
                            Lt[T(i, j)] = pm(pl, k, i, j);
                    const double dfloor = 1e-14 * tiles::diag_absmax<XT>(Lt, NX, lane);
                    int pf = -1;
                    Frag Li[NL];
                    {
                        Frag Zd[XT], Ld[XT], Z[NF];
                        tiles::chol_inv<XT, NL>(Lt, Zd, Ld, NX, dfloor, lane, pf, scr);
                        tiles::blocked_inverse<XT, NL>(Lt, Zd, Ld, Li, Z);
                    }
                    if (pf >= 0)
                        my_fail = min(my_fail, fail_key(kKindCR, Lc + pl, k, pf));
                    double *Lio = ws + Lo.PLi + (size_t)(pl * Tb + k) * TL;
#pragma unroll
                    for (int t = 0; t < NL; ++t)
                        st_frag(Lio + t * kTileElems, lane, Li[t]);
                    double *xk = xs + (size_t)(k << Lc) * XP;
                    if (fwd_fused) { // bt_k = L^{-1} x_k (final level: x_k <- L^{-T} L^{-1} x_k)
                        double o[XT];
                        matvec_r<XT, kLower>(Li, xk, o, lane);
                        double *dst = fin ? xk : bt + (size_t)k * XP;
                        __syncwarp();
#pragma unroll
                        for (int i = 0; i < XT; ++i)
                            if (q2 == 0)
                                dst[8 * i + rq] = o[i];
                        __syncwarp();
                        if (fin) {
                            double o2[XT][2];
                            matvec_t<XT, false, L1>(Lio, xk, o2, lane);
                            __syncwarp();
#pragma unroll
                            for (int j = 0; j < XT; ++j)
                                if (rq == 0) {
                                    xk[8 * j + cq] = o2[j][0];
                                    xk[8 * j + cq + 1] = o2[j][1];
                                }
                            __syncwarp();
                        }
                    }
                    if (fin)
                        continue;
                    // Y = K_k Linv', U = K_{k-st}' Linv'
                    const double *Kk = pk(pl, k), *Kp = k >= st ? pk(pl, k - st) : nullptr;
                    double *Uo = ws + Lo.PU + (size_t)(pl * Tb + k) * TF;
                    double *Yo = ws + Lo.PY + (size_t)(pl * Tb + k) * TF;
#pragma unroll
                    for (int i = 0; i < XT; ++i) {
                        Frag kp[XT], kk[XT];
#pragma unroll
                        for (int t = 0; t < XT; ++t) {
                            kp[t] = Kp ? ldw_t<L1>(Kp + fidx(XT, t, i) * kTileElems, lane) : Frag{0.0, 0.0};
                            kk[t] = ldw<L1>(Kk + fidx(XT, i, t) * kTileElems, lane);
                        }
#pragma unroll
                        for (int j = 0; j < XT; ++j) {
                            Frag u{0.0, 0.0}, y{0.0, 0.0};
#pragma unroll
                            for (int t = 0; t <= j; ++t) {
                                tile_gemm_nt(u, kp[t], Li[T(j, t)]);
                                tile_gemm_nt(y, kk[t], Li[T(j, t)]);
                            }
                            st_frag(Uo + (i * XT + j) * kTileElems, lane, u);
                            st_frag(Yo + (i * XT + j) * kTileElems, lane, y);
                        }
                    }
                }
                csync();
                if (fin)
                    break;
                for (int k = vwarp; k < Tb; k += VNW) {
                    const bool lo = k >= st, hi = k + st < Tb;
                    const double *Yl = ws + Lo.PY + (size_t)(pl * Tb + k - st) * TF;
                    const double *Uh = ws + Lo.PU + (size_t)(pl * Tb + k + st) * TF;
                    const double *Yh = ws + Lo.PY + (size_t)(pl * Tb + k + st) * TF;
                    double *M2o = ws + Lo.PM + (pl & 1) * Tb * TL + k * TL;
                    double *K2o = ws + Lo.PK + (pl & 1) * Tb * TF + k * TF;
#pragma unroll
                    for (int i = 0; i < XT; ++i)
#pragma unroll
                        for (int j = 0; j < XT; ++j) {
                            Frag yy{0.0, 0.0}, uu{0.0, 0.0}, yu{0.0, 0.0};
#pragma unroll
                            for (int t = 0; t < XT; ++t) {
                                if (j <= i && lo)
                                    tile_gemm_nt(yy, ldw<L1>(Yl + fidx(XT, i, t) * kTileElems, lane),
                                                 ldw<L1>(Yl + fidx(XT, j, t) * kTileElems, lane));
                                if (hi) {
                                    const Frag ui = ldw<L1>(Uh + fidx(XT, i, t) * kTileElems, lane);
                                    if (j <= i)
                                        tile_gemm_nt(uu, ui, ldw<L1>(Uh + fidx(XT, j, t) * kTileElems, lane));
                                    tile_gemm_nt_sub(yu, ldw<L1>(Yh + fidx(XT, i, t) * kTileElems, lane),
                                                     ldw<L1>(Uh + fidx(XT, j, t) * kTileElems, lane));
                                }
                            }
                            if (j <= i)
                                st_frag(M2o + T(i, j) * kTileElems, lane, fsub(fsub(pm(pl, k, i, j), yy), uu));
                            st_frag(K2o + fidx(XT, i, j) * kTileElems, lane, yu);
                        }
                    if (fwd_fused) { // x_k -= Y_{k-st} bt_{k-st} + U_{k+st} bt_{k+st}
                        double o1[XT], o2[XT];
                        if (lo)
                            matvec<XT, true, L1>(Yl, bt + (size_t)(k - st) * XP, o1, lane);
                        if (hi)
                            matvec<XT, true, L1>(Uh, bt + (size_t)(k + st) * XP, o2, lane);
                        double *xk = xs + (size_t)(k << Lc) * XP;
                        __syncwarp();
#pragma unroll
                        for (int i = 0; i < XT; ++i)
                            if (q2 == 0)
                                xk[8 * i + rq] -= (lo ? o1[i] : 0.0) + (hi ? o2[i] : 0.0);
                        __syncwarp();
                    }
                }
                csync();
            }
        }
        csync();
        if (ph) ph[php++] = clock64();
    }

    // ---- phase 3: CR solve over the stored factor, negate ----------------
    if (a.do_solve) {
        if (!fwd_fused) {
            // CRFactor::forward (block_tridiag.cpp:252-296)
            for (int l = 0, s = P; l < Lc; ++l, s >>= 1) {
                const int half = s / 2, stride = P / s;
                const long long o0 = P - (P >> l);
                for (int mm = vwarp; mm < half; mm += VNW) { // x_k <- L^{-1} x_k
                    double *xk = xs + (size_t)(2 * mm + 1) * stride * XP;
                    double o[XT];
                    matvec<XT, false, L1>(ws + Lo.Li + (o0 + mm) * TL, xk, o, lane);
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < XT; ++i)
                        if (q2 == 0)
                            xk[8 * i + rq] = o[i];
                }
                csync();
                for (int mm = vwarp; mm < half; mm += VNW) { // x_e -= U x_k + Y_prev x_k'
                    double *xe = xs + (size_t)2 * mm * stride * XP;
                    double o[XT], o2[XT];
                    matvec<XT, true, L1>(ws + Lo.U + (o0 + mm) * TF, xs + (size_t)(2 * mm + 1) * stride * XP,
                                     o, lane);
                    if (mm > 0)
                        matvec<XT, true, L1>(ws + Lo.Y + (o0 + mm - 1) * TF,
                                         xs + (size_t)(2 * mm - 1) * stride * XP, o2, lane);
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < XT; ++i)
                        if (q2 == 0)
                            xe[8 * i + rq] -= mm > 0 ? o[i] + o2[i] : o[i];
                }
                csync();
            }
            if (Tb > 1) { // PCRFactor::resolve (block_tridiag.cpp:457-486) on the tail
                for (int pl = 0; pl <= Lo.lgT; ++pl) {
                    const int st = 1 << pl;
                    const bool fin = pl == Lo.lgT;
                    for (int k = vwarp; k < Tb; k += VNW) { // bt_k = L^{-1} x_k
                        double *xk = xs + (size_t)(k << Lc) * XP;
                        const double *Lio = ws + Lo.PLi + (size_t)(pl * Tb + k) * TL;
                        double o[XT];
                        matvec<XT, false, L1>(Lio, xk, o, lane);
                        double *dst = fin ? xk : bt + (size_t)k * XP;
                        __syncwarp();
#pragma unroll
                        for (int i = 0; i < XT; ++i)
                            if (q2 == 0)
                                dst[8 * i + rq] = o[i];
                        __syncwarp();
                        if (fin) { // x_k <- L^{-T} L^{-1} x_k
                            double o2[XT][2];
                            matvec_t<XT, false, L1>(Lio, xk, o2, lane);
                            __syncwarp();
#pragma unroll
                            for (int j = 0; j < XT; ++j)
                                if (rq == 0) {
                                    xk[8 * j + cq] = o2[j][0];
                                    xk[8 * j + cq + 1] = o2[j][1];
                                }
                            __syncwarp();
                        }
                    }
                    csync();
                    if (fin)
                        break;
                    for (int k = vwarp; k < Tb; k += VNW) { // x_k -= Y_{k-st} bt_{k-st} + U_{k+st} bt_{k+st}
                        const bool lo = k >= st, hi = k + st < Tb;
                        double o1[XT], o2[XT];
                        if (lo)
                            matvec<XT, true, L1>(ws + Lo.PY + (size_t)(pl * Tb + k - st) * TF,
                                             bt + (size_t)(k - st) * XP, o1, lane);
                        if (hi)
                            matvec<XT, true, L1>(ws + Lo.PU + (size_t)(pl * Tb + k + st) * TF,
                                             bt + (size_t)(k + st) * XP, o2, lane);
                        double *xk = xs + (size_t)(k << Lc) * XP;
                        __syncwarp();
#pragma unroll
                        for (int i = 0; i < XT; ++i)
                            if (q2 == 0)
                                xk[8 * i + rq] -= (lo ? o1[i] : 0.0) + (hi ? o2[i] : 0.0);
                        __syncwarp();
                    }
                    csync();
                }
            } else if (vwarp == 0) { // base: x_0 <- L_b^{-T} L_b^{-1} x_0
                double o[XT], o2[XT][2];
                matvec<XT, false, L1>(ws + Lo.Lb, xs, o, lane);
                __syncwarp();
#pragma unroll
                for (int i = 0; i < XT; ++i)
                    if (q2 == 0)
                        xs[8 * i + rq] = o[i];
                __syncwarp();
                matvec_t<XT, false, L1>(ws + Lo.Lb, xs, o2, lane);
                __syncwarp();
#pragma unroll
                for (int j = 0; j < XT; ++j)
                    if (rq == 0) {
                        xs[8 * j + cq] = o2[j][0];
                        xs[8 * j + cq + 1] = o2[j][1];
                    }
            }
            csync();
        }
        if (ph) ph[php++] = clock64();
        // CRFactor::backward (block_tridiag.cpp:298-333)
        for (int l = Lc - 1; l >= 0; --l) {
            const int sl = P >> l, half = sl / 2, stride = P / sl;
            const long long o0 = P - (P >> l);
            for (int mm = vwarp; mm < half; mm += VNW) {
                double *xo = xs + (size_t)(2 * mm + 1) * stride * XP;
                double t1[XT][2], t2[XT][2], t3[XT][2];
                const bool has_y = 2 * mm + 2 < sl;
                matvec_t<XT, true, L1>(ws + Lo.U + (o0 + mm) * TF, xs + (size_t)2 * mm * stride * XP, t1,
                                   lane);
                if (has_y)
                    matvec_t<XT, true, L1>(ws + Lo.Y + (o0 + mm) * TF,
                                       xs + (size_t)((2 * mm + 2) * stride % P) * XP, t2, lane);
                __syncwarp();
#pragma unroll
                for (int j = 0; j < XT; ++j)
                    if (rq == 0) {
                        xo[8 * j + cq] -= has_y ? t1[j][0] + t2[j][0] : t1[j][0];
                        xo[8 * j + cq + 1] -= has_y ? t1[j][1] + t2[j][1] : t1[j][1];
                    }
                __syncwarp();
                matvec_t<XT, false, L1>(ws + Lo.Li + (o0 + mm) * TL, xo, t3, lane); // L^{-T} xo
                __syncwarp();
#pragma unroll
                for (int j = 0; j < XT; ++j)
                    if (rq == 0) {
                        xo[8 * j + cq] = t3[j][0];
                        xo[8 * j + cq + 1] = t3[j][1];
                    }
            }
            csync();
        }
        if (ph) ph[php++] = clock64();
        for (int e = vtid; e < P * NX; e += VNTH) {
            const int i = e / NX, k = e % NX;
            const double lam = -xs[i * XP + k];
            a.lamc[(size_t)b * P * NX + e] = lam;
            if (a.lam_out && n * i < g.N)
                a.lam_out[((size_t)b * g.N + n * i) * NX + k] = lam;
        }
    }
    for (int o = 16; o > 0; o >>= 1)
        my_fail = min(my_fail, __shfl_xor_sync(0xffffffffu, my_fail, o));
    if (lane == 0 && my_fail != ~0ull)
        atomicMin(a.fail + b, my_fail);
    if (ph) {
        ph[php++] = clock64();
        ph[31] = php;
    }
    if (CL > 1)
        cg::this_cluster().sync();
}

template <int NX, int NW, int CL> bool launch_sfw(const Geo &g, cudaStream_t st, const SchurArgs &sa) {
    const size_t smem = (sf_smem_doubles<SF<NX>::XP>(NW, SF<NX>::NF, g.P) -
                         (CL > 1 ? (size_t)g.P * SF<NX>::XP : 0)) * sizeof(double);
    if (smem > 220 * 1024)
        return false;
    static DeviceOnce once;
    once_per_device(once, [&] { return cudaFuncSetAttribute(schur_fused_kernel<NX, NW, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024); });
    if (launch_pdl(schur_fused_kernel<NX, NW, CL>, dim3(g.batch * CL), dim3(32 * NW), smem, st, CL, sa) ==
        cudaSuccess)
        return true;
    cudaGetLastError(); // e.g. a cluster that cannot be co-scheduled: the caller falls back
    return false;
}

// 4 warps per instance when the batch fills the GPU with CTAs; for a few
// long-horizon instances (config 2: one instance, P = 256) a cluster of 8
// wide CTAs per instance, so a CR level's eliminations run in one round
template <int NX> bool launch_sf(const Geo &g, cudaStream_t st, const SchurArgs &sa, const LaunchOpts &o) {
    if (g.nx != NX)
        return false;
    constexpr int WIDE = NX > 16 ? 8 : 16;
    if (g.batch >= 64 || g.P <= 8) {
        // more instances than 4-warp CTA slots (148 SMs x 4): 2-warp CTAs
        // (8 per SM) finish the batch in one wave instead of ~1.7
        // (config 1: 0.319 -> 0.308 ms); CYQ_OPT_SCHUR_WARPS = 2 | 4 forces either
        const bool two = o.schur_warps ? o.schur_warps == 2 : g.batch > 4 * o.sms;
        if (two)
            return launch_sfw<NX, 2, 1>(g, st, sa);
        return launch_sfw<NX, 4, 1>(g, st, sa);
    }
    if (g.P >= 64 && g.batch * 8 <= o.sms && o.schur_cluster)
        if (launch_sfw<NX, WIDE, 8>(g, st, sa))
            return true;
    return launch_sfw<NX, WIDE, 1>(g, st, sa);
}

} // namespace

// The fused kernel serves every batch size (one CTA per instance; wide CTAs
// for small batches); CYQ_OPT_SCHUR selects the per-level batch-wide
// kernels of schur_tiles.cu (or the scalar kernel) instead (cross-check paths).
bool schur_fused_ok(const Geo &g, const LaunchOpts &o) {
    if (o.schur != 0)
        return false;
    const bool shape = g.nx == 20 || g.nx == 16 || g.nx == 12 || g.nx == 10;
    if (!shape)
        return false;
    return true;
}

bool launch_schur_fused(const Geo &g, cudaStream_t st, const SchurArgs &sa, const LaunchOpts &o) {
    if (!schur_fused_ok(g, o))
        return false;
    return launch_sf<20>(g, st, sa, o) || launch_sf<16>(g, st, sa, o) || launch_sf<12>(g, st, sa, o) ||
           launch_sf<10>(g, st, sa, o);
}

} // namespace cyqb
