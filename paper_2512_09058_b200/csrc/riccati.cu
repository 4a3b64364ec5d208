// Stage-panel Riccati factorization + fused forward substitution (one CTA per
// partition column), FP64 DMMA tiles in shared memory.
//
// Restates, per column c of instance b:
//   kkt_factor.cpp:125-158  modified Riccati recursion (LH, LB, Acl, LA)
//   kkt_factor.cpp:163-185  Schur contribution Mfwd = sum LB LB' + LA LA'
//   kkt_solve.cpp:72-134    forward substitution + coupling rows (fwd)
// as one symmetric elimination of the extended stage panel (kkt_common.cuh).
// Mbwd / W (T = L_Q^{-T}, kkt_factor.cpp:168-178) and bwd_neg are formed by
// the Schur kernel from the stored last-stage blocks.
#include "kkt_common.cuh"
#include "kernels.h"

namespace cyqb {

namespace {

// Initial value of panel entry (r, col) at stage position s (before W W').
__device__ double panel_init(const Geo &g, const ProbAcc &pa, int s, int j,
                             int xi, int r, int col, bool x0_terms,
                             const double *ru0_adj) {
    const int nu = g.nu, nux = g.nux, top = 8 * g.CT;
    if (r < top) { // top block: H_s (lower), identity padding
        if (r >= nux || col >= nux)
            return r == col ? 1.0 : 0.0;
        if (col > r)
            return 0.0;
        if (r < nu)
            return pa.R(j, r, col);
        if (col < nu)
            return j != 0 ? pa.S(j, col, r - nu) : 0.0; // S' block
        return pa.Q(xi, r - nu, col - nu);
    }
    const int rb = r - top;
    if (rb < g.nx) { // coupling rows: hatBA_0 = [B A] at s = 0
        if (s != 0 || col >= nux)
            return 0.0;
        if (col < nu)
            return pa.B(j, rb, col);
        return j != 0 ? pa.A(j, rb, col - nu) : 0.0;
    }
    if (rb == g.nx) { // rhs row: [ru_j ; qx_xi]
        if (col < nu) {
            double v = pa.ru(j, col);
            if (x0_terms && j == 0)
                v -= ru0_adj[col];
            return v;
        }
        if (col < nux)
            return pa.qx(xi, col - nu);
    }
    return 0.0;
}

} // namespace

__global__ void __launch_bounds__(256)
riccati_panel_kernel(RiccatiArgs a) {
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int chain = blockIdx.x;
    const int b = chain / g.P, c = chain % g.P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NW = blockDim.x >> 5;
    const int TT = g.TT, CT = g.CT, NXT = g.NXT, XT0 = g.XT0;
    const int NT = TT * (TT + 1) / 2;
    const int nu = g.nu, nx = g.nx, nux = g.nux, top = 8 * CT;
    const int rq = lane >> 2, cq = 2 * (lane & 3);

    double *pan = sm;                       // NT tiles
    double *W = pan + NT * kTileElems;      // TT x NXT tiles
    double *vec = W + TT * NXT * kTileElems; // scratch vectors
    double *wl_old = vec;                   // nx
    double *mwl = vec + 32 * ((nx + 31) / 32); // nx: -wl_new
    double *ru0 = mwl + 32 * ((nx + 31) / 32); // nu: S_0 x_init
    double *red = ru0 + 32 * ((nu + 31) / 32); // reduction scratch (32)

    ProbAcc pa{a.p, g, b};
    const bool x0_terms = (a.p.ru == nullptr);
    unsigned long long my_fail = ~0ull;

    // S_0 x_init for ru[0] (EqRhs::of_problem, ocp.cpp:171), column 0 only
    if (x0_terms && c == 0) {
        for (int i = threadIdx.x; i < nu; i += blockDim.x) {
            double s0 = 0;
            for (int k = 0; k < nx; ++k)
                s0 += pa.S(0, i, k) * __ldg(a.p.x_init + (size_t)b * nx + k);
            ru0[i] = s0;
        }
    }
    // trailing tiles start at zero
    for (int i = threadIdx.x; i < NT * kTileElems; i += blockDim.x)
        pan[i] = 0.0;
    __syncthreads();

    for (int s = 0; s < g.n; ++s) {
        const int j = g.stage_of(c, s), xi = g.x_index_of(c, s);
        // (1)+(2): initialise pivot tiles, then all tiles += W W'
        for (int t = warp; t < NT; t += NW) {
            int ti = 0;
            while (tri_index(ti + 1, 0) <= t)
                ++ti;
            const int tj = t - tri_index(ti, 0);
            double *tile = pan + t * kTileElems;
            Frag f;
            if (tj < CT) {
                const int r = 8 * ti + rq, col = 8 * tj + cq;
                f.a = panel_init(g, pa, s, j, xi, r, col, x0_terms, ru0);
                f.b = panel_init(g, pa, s, j, xi, r, col + 1, x0_terms, ru0);
            } else {
                f = ld_frag(tile, lane);
            }
            if (s > 0) {
                for (int kt = 0; kt < NXT; ++kt)
                    tile_gemm_nt(f, ld_frag(W + (ti * NXT + kt) * kTileElems, lane),
                                 ld_frag(W + (tj * NXT + kt) * kTileElems, lane));
            }
            st_frag(tile, lane, f);
        }
        __syncthreads();
        // potrf pivot floor: max |diag| of H_s + V V' (kernels.cpp:21-29)
        if (warp == 0) {
            double m = 0;
            for (int d = lane; d < nux; d += 32) {
                const int t = tri_index(d / 8, d / 8);
                m = fmax(m, fabs(pan[t * kTileElems + (d % 8) * 9]));
            }
            for (int o = 16; o > 0; o >>= 1)
                m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0)
                red[0] = m;
        }
        __syncthreads();
        const double dfloor = 1e-14 * red[0];

        // (3) blocked Cholesky of the pivot columns
        for (int kb = 0; kb < CT; ++kb) {
            // every warp factors the diagonal tile redundantly (registers)
            Frag dg = ld_frag(pan + tri_index(kb, kb) * kTileElems, lane);
            double inv[8], lc0[8], lc1[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int src = 4 * k + k / 2;
                double pv = __shfl_sync(0xffffffffu, (k & 1) ? dg.b : dg.a, src);
                const int kcol = 8 * kb + k;
                if (kcol < nux && !(pv > dfloor && isfinite(pv))) {
                    my_fail = min(my_fail, fail_key(kKindRiccati, c, s, kcol));
                    pv = 1.0; // keep going; the status reports the failure
                }
                const double d = sqrt(pv);
                const double iv = 1.0 / d;
                inv[k] = iv;
                if ((lane & 3) == k / 2) {
                    double &e = (k & 1) ? dg.b : dg.a;
                    if (rq == k)
                        e = d;
                    else if (rq > k)
                        e *= iv;
                }
                const double vk = (k & 1) ? dg.b : dg.a;
                const double lrk = __shfl_sync(0xffffffffu, vk, 4 * rq + k / 2);
                lc0[k] = __shfl_sync(0xffffffffu, vk, 4 * cq + k / 2);
                lc1[k] = __shfl_sync(0xffffffffu, vk, 4 * (cq + 1) + k / 2);
                if (cq > k && rq >= cq)
                    dg.a -= lrk * lc0[k];
                if (cq + 1 > k && rq >= cq + 1)
                    dg.b -= lrk * lc1[k];
            }
            if (warp == 0) {
                Frag o = dg;
                if (cq > rq) o.a = 0.0;
                if (cq + 1 > rq) o.b = 0.0;
                st_frag(pan + tri_index(kb, kb) * kTileElems, lane, o);
            }
            // sub-diagonal tiles: X <- X L^{-T}
            for (int ti = kb + 1 + warp; ti < TT; ti += NW) {
                double *tile = pan + tri_index(ti, kb) * kTileElems;
                Frag x = ld_frag(tile, lane);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if ((lane & 3) == k / 2) {
                        if (k & 1) x.b *= inv[k];
                        else x.a *= inv[k];
                    }
                    const double vk = (k & 1) ? x.b : x.a;
                    const double xrk = __shfl_sync(0xffffffffu, vk, 4 * rq + k / 2);
                    if (cq > k) x.a -= xrk * lc0[k];
                    if (cq + 1 > k) x.b -= xrk * lc1[k];
                }
                st_frag(tile, lane, x);
            }
            __syncthreads();
            // trailing update: C(ti,tj) -= L(ti,kb) L(tj,kb)'
            const int m = TT - kb - 1;
            const int nupd = m * (m + 1) / 2;
            for (int u = warp; u < nupd; u += NW) {
                int ui = 0;
                while ((ui + 1) * (ui + 2) / 2 <= u)
                    ++ui;
                const int uj = u - ui * (ui + 1) / 2;
                const int ti = kb + 1 + ui, tj = kb + 1 + uj;
                double *tile = pan + tri_index(ti, tj) * kTileElems;
                Frag cf = ld_frag(tile, lane);
                tile_gemm_nt_sub(cf, ld_frag(pan + tri_index(ti, kb) * kTileElems, lane),
                                 ld_frag(pan + tri_index(tj, kb) * kTileElems, lane));
                st_frag(tile, lane, cf);
            }
            __syncthreads();
        }

        // (4) store the pivot tiles (the factor) and the forward-sweep y_s
        {
            double *dst = a.fac + ((size_t)chain * g.n + s) * g.NPT * kTileElems;
            const int ntop = CT * (CT + 1) / 2;
            const int n2 = g.NPT * kTileElems / 2;
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int t = (2 * i) / kTileElems, off = (2 * i) % kTileElems;
                int src;
                if (t < ntop) {
                    src = t;
                } else {
                    const int bi = (t - ntop) / CT, bj = (t - ntop) % CT;
                    src = tri_index(CT + bi, bj);
                }
                reinterpret_cast<double2 *>(dst)[i] =
                    reinterpret_cast<const double2 *>(pan + src * kTileElems + off)[0];
            }
            double *yv = a.y + ((size_t)chain * g.n + s) * nux;
            const int rr = top + nx;
            for (int k = threadIdx.x; k < nux; k += blockDim.x)
                yv[k] = pan[tri_index(rr / 8, k / 8) * kTileElems + (rr % 8) * 8 + k % 8];
        }

        if (s + 1 < g.n) {
            // (5) W for stage s+1: wl_new = -L_Q' wl_old - x'  (kkt_solve.cpp:85-90)
            const int j1 = g.stage_of(c, s + 1);
            for (int k = threadIdx.x; k < nx; k += blockDim.x)
                wl_old[k] = pa.fd(j1, k);
            __syncthreads();
            for (int t = threadIdx.x; t < nx; t += blockDim.x) {
                double q = 0;
                const int C = nu + t;
                for (int k = t; k < nx; ++k) {
                    const int K = nu + k;
                    q += pan[tri_index(K / 8, C / 8) * kTileElems + (K % 8) * 8 + C % 8] *
                         wl_old[k];
                }
                const int rr = top + nx;
                const double xp = pan[tri_index(rr / 8, C / 8) * kTileElems + (rr % 8) * 8 + C % 8];
                mwl[t] = q + xp;
                a.wl[((size_t)chain * g.n + s) * nx + t] = -(q + xp);
            }
            __syncthreads();
            // W tiles: top rows V = BA_{s+1}' L_Q (DMMA), bottom rows ALQ, -wl
            const int nwt = TT * NXT;
            for (int t = warp; t < nwt; t += NW) {
                const int ti = t / NXT, kt = t % NXT;
                const int ct = XT0 + kt;
                Frag f{0.0, 0.0};
                if (ti < CT) {
                    const int r = 8 * ti + rq; // A operand row
                    for (int ks = 2 * XT0; ks < 2 * (XT0 + NXT); ++ks) {
                        if (4 * ks + 3 < 8 * ct)
                            continue; // L_Q upper part is zero
                        const int Ka = 4 * ks + (lane & 3);
                        double av = 0.0;
                        if (Ka >= nu && Ka < nux && r < nux) {
                            const int k = Ka - nu;
                            av = r < nu ? pa.B(j1, k, r)
                                        : (j1 != 0 ? pa.A(j1, k, r - nu) : 0.0);
                        }
                        const int Kb = 4 * ks + (lane & 3), Cb = 8 * ct + (lane >> 2);
                        double bv = 0.0;
                        if (Kb >= nu && Kb < nux && Cb >= nu && Cb < nux && Kb >= Cb)
                            bv = pan[tri_index(Kb / 8, Cb / 8) * kTileElems + (Kb % 8) * 8 + Cb % 8];
                        dmma(f, av, bv);
                    }
                } else {
                    f = ld_frag(pan + tri_index(ti, ct) * kTileElems, lane);
                    const int rb = 8 * ti + rq - top;
                    if (rb == nx) {
                        const int c0 = 8 * ct + cq;
                        f.a = (c0 >= nu && c0 < nux) ? mwl[c0 - nu] : 0.0;
                        f.b = (c0 + 1 >= nu && c0 + 1 < nux) ? mwl[c0 + 1 - nu] : 0.0;
                    } else if (rb > nx) {
                        f.a = f.b = 0.0;
                    }
                    const int c0 = 8 * ct + cq;
                    if (c0 < nu || c0 >= nux) f.a = 0.0;
                    if (c0 + 1 < nu || c0 + 1 >= nux) f.b = 0.0;
                }
                st_frag(W + t * kTileElems, lane, f);
            }
            __syncthreads();
        }
    }

    // trailing tiles: coupling x coupling = -Mfwd, rhs x coupling = -fwd
    {
        double *dst = a.trail + (size_t)chain * g.NTT * kTileElems;
        const int t0 = tri_index(CT, CT);
        for (int u = 0, t = 0; u < g.BT; ++u) {
            for (int v = 0; v <= u; ++v, ++t) {
                const double *src = pan + (tri_index(CT + u, 0) + CT + v) * kTileElems;
                for (int i = threadIdx.x; i < kTileElems; i += blockDim.x)
                    dst[t * kTileElems + i] = src[i];
            }
        }
        (void)t0;
    }
    // first failure of this column (reduced over the warp, one atomic)
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(0xffffffffu, my_fail, o);
        my_fail = min(my_fail, other);
    }
    if (lane == 0 && my_fail != ~0ull)
        atomicMin(a.fail + b, my_fail);
}

} // namespace cyqb
