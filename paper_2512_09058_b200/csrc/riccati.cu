// Stage-panel Riccati factorization + fused forward substitution (one CTA per
// partition column), FP64 DMMA tiles, register-resident accumulators.
//
// Restates, per column c of instance b:
//   kkt_factor.cpp:125-158  modified Riccati recursion (LH, LB, Acl, LA)
//   kkt_factor.cpp:163-185  Schur contribution Mfwd = sum LB LB' + LA LA'
//   kkt_solve.cpp:72-134    forward substitution + coupling rows (fwd)
// as one symmetric elimination of the extended stage panel (kkt_common.cuh).
// Mbwd / W (T = L_Q^{-T}, kkt_factor.cpp:168-178) and bwd_neg are formed by
// the Schur kernel from the stored last-stage blocks.
//
// Execution model (per CTA = one chain, NW warps):
//  * every 8x8 panel tile has a fixed owner warp (t % NW) that keeps it in
//    registers (MAXT tiles per warp) for the whole stage -- trailing
//    (coupling) tiles for the whole chain; rank-8 updates are two DMMAs on
//    register accumulators, operands published through shared memory;
//  * stage data (R, S, Q, B, A and the rhs vectors) is staged into shared
//    memory with cp.async one stage ahead, so HBM latency is off the
//    critical path and global reads are full-sector;
//  * pivots use one rsqrt per column (no divisions on the critical path).
#include "kkt_common.cuh"
#include "kernels.h"

namespace cyqb {

namespace {

__device__ __forceinline__ void cp8(double *dst, const double *src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// copies `cnt` doubles (async), or fills identity / zero when src == nullptr
__device__ __forceinline__ void stage_copy(double *dst, const double *src, int cnt, int diag_n,
                                           int tid, int nthr) {
    if (src) {
        for (int i = tid; i < cnt; i += nthr)
            cp8(dst + i, src + i);
    } else {
        for (int i = tid; i < cnt; i += nthr)
            dst[i] = (diag_n > 0 && i / diag_n == i % diag_n) ? 1.0 : 0.0;
    }
}

struct Bufs {
    // H buffer: R (nu x nu) | S (nu x nx) | Q (nx x nx) | r (nu) | q (nx)
    double *R, *S, *Q, *r, *q;
    // BA buffer: B (nx x nu) | A (nx x nx) | f (nx)
    double *B, *A, *f;
};

// Direct mode (panels too large to also stage the stage data in shared
// memory): point the buffers at the global matrices instead, with identity /
// zero constants for padding stages.
__device__ void point_H(const Geo &g, const ProbView &p, const double *cst, int b, int j, int xi,
                        Bufs &bf) {
    const int nu = g.nu, nx = g.nx, N = g.N;
    const double *eye_nu = cst, *eye_nx = cst + nu * nu, *zero = eye_nx + nx * nx;
    const bool in = j < N;
    bf.R = const_cast<double *>(in ? p.R + ((size_t)b * N + j) * nu * nu : eye_nu);
    bf.S = const_cast<double *>(in ? p.S + ((size_t)b * N + j) * nu * nx : zero);
    bf.Q = const_cast<double *>(xi <= N ? p.Q + ((size_t)b * (N + 1) + xi) * nx * nx : eye_nx);
    bf.r = const_cast<double *>(in ? (p.ru ? p.ru : p.r) + ((size_t)b * N + j) * nu : zero);
    bf.q = const_cast<double *>(xi <= N ? (p.qx ? p.qx : p.q) + ((size_t)b * (N + 1) + xi) * nx : zero);
}
__device__ void point_BA(const Geo &g, const ProbView &p, const double *cst, int b, int j,
                         Bufs &bf) {
    const int nu = g.nu, nx = g.nx, N = g.N;
    const double *zero = cst + nu * nu + nx * nx;
    const bool in = j < N;
    bf.B = const_cast<double *>(in ? p.B + ((size_t)b * N + j) * nx * nu : zero);
    bf.A = const_cast<double *>((in && j != 0) ? p.A + ((size_t)b * N + j) * nx * nx : zero);
    bf.f = const_cast<double *>(in ? (p.fd ? p.fd : p.f) + ((size_t)b * N + j) * nx : zero);
}

// Issue the (async) loads of H_j (R_j, S_j, Q_xi, r_j, q_xi).
__device__ void load_H(const Geo &g, const ProbView &p, int b, int j, int xi, Bufs &bf,
                       int tid, int nthr, const double *cst) {
    if (cst) {
        point_H(g, p, cst, b, j, xi, bf);
        return;
    }
    const int nu = g.nu, nx = g.nx, N = g.N;
    const bool in = j < N;
    stage_copy(bf.R, in ? p.R + ((size_t)b * N + j) * nu * nu : nullptr, nu * nu, nu, tid, nthr);
    stage_copy(bf.S, in ? p.S + ((size_t)b * N + j) * nu * nx : nullptr, nu * nx, 0, tid, nthr);
    stage_copy(bf.Q, xi <= N ? p.Q + ((size_t)b * (N + 1) + xi) * nx * nx : nullptr, nx * nx,
               nx, tid, nthr);
    const double *rs = p.ru ? p.ru : p.r;
    const double *qs = p.qx ? p.qx : p.q;
    stage_copy(bf.r, in ? rs + ((size_t)b * N + j) * nu : nullptr, nu, 0, tid, nthr);
    stage_copy(bf.q, xi <= N ? qs + ((size_t)b * (N + 1) + xi) * nx : nullptr, nx, 0, tid, nthr);
}

// Issue the (async) loads of BA_j = [B_j A_j] and f_j (fd).
__device__ void load_BA(const Geo &g, const ProbView &p, int b, int j, Bufs &bf, int tid,
                        int nthr, const double *cst) {
    if (cst) {
        point_BA(g, p, cst, b, j, bf);
        return;
    }
    const int nu = g.nu, nx = g.nx, N = g.N;
    const bool in = j < N;
    stage_copy(bf.B, in ? p.B + ((size_t)b * N + j) * nx * nu : nullptr, nx * nu, 0, tid, nthr);
    stage_copy(bf.A, (in && j != 0) ? p.A + ((size_t)b * N + j) * nx * nx : nullptr, nx * nx, 0,
               tid, nthr);
    const double *fs = p.fd ? p.fd : p.f;
    stage_copy(bf.f, in ? fs + ((size_t)b * N + j) * nx : nullptr, nx, 0, tid, nthr);
}

// Initial value of panel entry (r, col) of a pivot tile (before W W').
__device__ __forceinline__ double panel_init(const Geo &g, const Bufs &bf, int s, int j,
                                             double sgn, const double *ru0, int r, int col) {
    const int nu = g.nu, nux = g.nux, top = 8 * g.CT;
    if (r < top) { // top block: H_s (lower), identity padding
        if (r >= nux || col >= nux)
            return r == col ? 1.0 : 0.0;
        if (col > r)
            return 0.0;
        if (r < nu)
            return bf.R[r * nu + col];
        if (col < nu)
            return j != 0 ? bf.S[col * g.nx + (r - nu)] : 0.0; // S' block
        return bf.Q[(r - nu) * g.nx + (col - nu)];
    }
    const int rb = r - top;
    if (rb < g.nx) { // coupling rows: hatBA_0 = [B A] at s = 0
        if (s != 0 || col >= nux)
            return 0.0;
        return col < nu ? bf.B[rb * nu + col] : bf.A[rb * g.nx + (col - nu)];
    }
    if (rb == g.nx) { // rhs row: [ru_j ; qx_xi]
        if (col < nu)
            return sgn * bf.r[col] - (ru0 ? ru0[col] : 0.0);
        if (col < nux)
            return sgn * bf.q[col - nu];
    }
    return 0.0;
}

} // namespace

template <int MAXT>
__global__ void __launch_bounds__(MAXT == 32 ? 256 : 128, (MAXT <= 8 ? 4 : 1))
riccati_panel_kernel_t(RiccatiArgs a) {
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int chain = a.chain_of(blockIdx.x);
    const int b = chain / g.P, c = chain % g.P;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NW = blockDim.x >> 5, NTH = blockDim.x;
    const int TT = g.TT, CT = g.CT, NXT = g.NXT, XT0 = g.XT0;
    const int NT = TT * (TT + 1) / 2;
    const int nu = g.nu, nx = g.nx, nux = g.nux, top = 8 * CT, n = g.n;
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    const int rhs_tile = (top + nx) / 8, rhs_r = (top + nx) % 8;

    // ---- shared memory carve-up --------------------------------------
    double *pan = sm;                              // NT tiles
    double *Vs = pan + NT * kTileElems;            // CT x NXT tiles
    const double *cst = a.staged ? nullptr : a.consts;
    double *hb = Vs + CT * NXT * kTileElems;
    const int stg = a.staged ? (nu * nu + nu * nx + nx * nx + nu + nx + nx * nu + nx * nx + nx) : 0;
    Bufs bf;
    bf.R = hb;
    bf.S = bf.R + nu * nu;
    bf.Q = bf.S + nu * nx;
    bf.r = bf.Q + nx * nx;
    bf.q = bf.r + nu;
    bf.B = bf.q + nx;
    bf.A = bf.B + nx * nu;
    bf.f = bf.A + nx * nx;
    double *mwl = hb + stg;        // nx: -wl_new (the rhs row of W)
    double *ru0 = mwl + nx;        // nu: S_0 x_init
    double *red = ru0 + nu;        // 32
    unsigned char *tab = reinterpret_cast<unsigned char *>(red + 32); // 2*NT

    const bool implicit_rhs = (a.p.ru == nullptr);
    const double sgn = implicit_rhs ? -1.0 : 1.0; // EqRhs::of_problem negation
    unsigned long long my_fail = ~0ull;

    for (int t = tid; t < NT; t += NTH) {
        int ti = 0;
        while (tri_index(ti + 1, 0) <= t)
            ++ti;
        tab[2 * t] = (unsigned char)ti;
        tab[2 * t + 1] = (unsigned char)(t - tri_index(ti, 0));
    }
    // prologue: stage 0 data (H_0, BA_0), S_0 x_init for the ru[0] term
    {
        const int j0 = g.stage_of(c, 0), x0i = g.x_index_of(c, 0);
        load_H(g, a.p, b, j0, x0i, bf, tid, NTH, cst);
        load_BA(g, a.p, b, j0, bf, tid, NTH, cst);
        cp_commit();
        if (implicit_rhs && c == 0) {
            for (int i = tid; i < nu; i += NTH) {
                double s0 = 0;
                for (int k = 0; k < nx; ++k)
                    s0 += __ldg(a.p.S + (size_t)b * g.N * nu * nx + i * nx + k) *
                          __ldg(a.p.x_init + (size_t)b * nx + k);
                ru0[i] = s0;
            }
        }
        if (tid < 32)
            reinterpret_cast<unsigned long long *>(red)[tid] = 0ull;
        cp_wait_all();
    }
    __syncthreads();

    // register-resident tiles owned by this warp: t = warp + k * NW
    Frag acc[MAXT];
#pragma unroll
    for (int k = 0; k < MAXT; ++k)
        acc[k] = Frag{0.0, 0.0};

    for (int s = 0; s < n; ++s) {
        const int j = g.stage_of(c, s);
        const double *ru0p = (implicit_rhs && j == 0) ? ru0 : nullptr;
        // ---- S1: init pivot tiles, then += W W' (all into registers) ---
#pragma unroll
        for (int k = 0; k < MAXT; ++k) {
            const int t = warp + k * NW;
            if (t < NT) {
                const int ti = tab[2 * t], tj = tab[2 * t + 1];
                Frag f = acc[k];
                if (tj < CT) {
                    const int r = 8 * ti + rq, col = 8 * tj + cq;
                    f.a = panel_init(g, bf, s, j, sgn, ru0p, r, col);
                    f.b = panel_init(g, bf, s, j, sgn, ru0p, r, col + 1);
                }
                if (s > 0) {
                    for (int kt = 0; kt < NXT; ++kt) {
                        Frag wi, wj;
                        const int ct = XT0 + kt, c0 = 8 * ct + cq;
                        const bool m0 = c0 >= nu && c0 < nux, m1 = c0 + 1 >= nu && c0 + 1 < nux;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int tt = h ? tj : ti;
                            Frag w;
                            if (tt < CT) {
                                w = ld_frag(Vs + (tt * NXT + kt) * kTileElems, lane);
                            } else {
                                w = ld_frag(pan + tri_index(tt, ct) * kTileElems, lane);
                                if (tt == rhs_tile && rq == rhs_r) {
                                    w.a = m0 ? mwl[c0 - nu] : 0.0;
                                    w.b = m1 ? mwl[c0 + 1 - nu] : 0.0;
                                }
                                if (!m0) w.a = 0.0;
                                if (!m1) w.b = 0.0;
                            }
                            if (h) wj = w; else wi = w;
                        }
                        tile_gemm_nt(f, wi, wj);
                    }
                }
                acc[k] = f;
            }
        }
        __syncthreads(); // all reads of W / staging done
        // prefetch the next stage's H (H buffer is free now); BA_1 at s = 0
        if (s + 1 < n)
            load_H(g, a.p, b, g.stage_of(c, s + 1), g.x_index_of(c, s + 1), bf, tid, NTH, cst);
        if (s == 0 && n > 1)
            load_BA(g, a.p, b, g.stage_of(c, 1), bf, tid, NTH, cst);
        cp_commit();
        // publish block column 0
#pragma unroll
        for (int k = 0; k < MAXT; ++k) {
            const int t = warp + k * NW;
            if (t < NT && tab[2 * t + 1] == 0)
                st_frag(pan + t * kTileElems, lane, acc[k]);
        }
        __syncthreads();
        // pivot floor: max |diag| of H_s + V V' over the nux real pivots
        // (kernels.cpp:21-29); owners of the top diagonal tiles publish
        // |diag| through atomicMax on the (non-negative) bit patterns
#pragma unroll
        for (int k = 0; k < MAXT; ++k) {
            const int t = warp + k * NW;
            if (t < NT && tab[2 * t] == tab[2 * t + 1] && tab[2 * t] < CT &&
                (lane & 3) == rq / 2) {
                const double v = (rq & 1) ? acc[k].b : acc[k].a;
                const int d = 8 * tab[2 * t] + rq;
                if (d < nux)
                    atomicMax(reinterpret_cast<unsigned long long *>(red) + (d & 31),
                              (unsigned long long)__double_as_longlong(fabs(v)));
            }
        }
        __syncthreads();
        double dmax = __longlong_as_double(
            (long long)reinterpret_cast<const unsigned long long *>(red)[lane]);
        for (int o = 16; o > 0; o >>= 1)
            dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        const double dfloor = 1e-14 * dmax;

        // ---- S2: blocked Cholesky of the pivot columns -----------------
        for (int kb = 0; kb < CT; ++kb) {
            // every warp factors the diagonal tile redundantly
            Frag dg = ld_frag(pan + tri_index(kb, kb) * kTileElems, lane);
            double inv[8], lc0[8], lc1[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double vk_un = (k & 1) ? dg.b : dg.a; // column k, unscaled
                double pv = __shfl_sync(0xffffffffu, vk_un, 4 * k + k / 2);
                // broadcast the unscaled column while the rsqrt is in flight
                const double urk = __shfl_sync(0xffffffffu, vk_un, 4 * rq + k / 2);
                const double uc0 = __shfl_sync(0xffffffffu, vk_un, 4 * cq + k / 2);
                const double uc1 = __shfl_sync(0xffffffffu, vk_un, 4 * (cq + 1) + k / 2);
                const int kcol = 8 * kb + k;
                if (kcol < nux && !(pv > dfloor && isfinite(pv))) {
                    my_fail = min(my_fail, fail_key(kKindRiccati, c, s, kcol));
                    pv = 1.0;
                }
                const double iv = rsqrt(pv);
                inv[k] = iv;
                lc0[k] = uc0 * iv;
                lc1[k] = uc1 * iv;
                const double lrk = urk * iv;
                if ((lane & 3) == k / 2) {
                    double &e = (k & 1) ? dg.b : dg.a;
                    if (rq == k)
                        e = pv * iv;
                    else if (rq > k)
                        e = lrk;
                }
                if (cq > k && rq >= cq)
                    dg.a -= lrk * lc0[k];
                if (cq + 1 > k && rq >= cq + 1)
                    dg.b -= lrk * lc1[k];
            }
            // owner of (kb,kb) keeps L in registers (zero upper part)
            // and sub-diagonal tiles: X <- X L^{-T}; publish both
#pragma unroll
            for (int k = 0; k < MAXT; ++k) {
                const int t = warp + k * NW;
                if (t < NT && tab[2 * t + 1] == kb) {
                    const int ti = tab[2 * t];
                    Frag x = acc[k];
                    if (ti == kb) {
                        x = dg;
                        if (cq > rq) x.a = 0.0;
                        if (cq + 1 > rq) x.b = 0.0;
                    } else {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const double vq = (q & 1) ? x.b : x.a;
                            const double xrq = __shfl_sync(0xffffffffu, vq, 4 * rq + q / 2) * inv[q];
                            if ((lane & 3) == q / 2) {
                                if (q & 1) x.b = xrq;
                                else x.a = xrq;
                            }
                            if (cq > q) x.a -= xrq * lc0[q];
                            if (cq + 1 > q) x.b -= xrq * lc1[q];
                        }
                    }
                    acc[k] = x;
                    st_frag(pan + t * kTileElems, lane, x);
                }
            }
            __syncthreads();
            // trailing update of own tiles: C(ti,tj) -= L(ti,kb) L(tj,kb)'
#pragma unroll
            for (int k = 0; k < MAXT; ++k) {
                const int t = warp + k * NW;
                if (t < NT) {
                    const int ti = tab[2 * t], tj = tab[2 * t + 1];
                    if (tj > kb) {
                        tile_gemm_nt_sub(acc[k], ld_frag(pan + tri_index(ti, kb) * kTileElems, lane),
                                         ld_frag(pan + tri_index(tj, kb) * kTileElems, lane));
                        if (tj == kb + 1 && tj < CT)
                            st_frag(pan + t * kTileElems, lane, acc[k]); // next block column
                    }
                }
            }
            __syncthreads();
        }
        // re-arm the dmax scratch for the next stage
        if (tid < 32)
            reinterpret_cast<unsigned long long *>(red)[tid] = 0ull;

        // ---- S3: store the pivot tiles (the factor) and y_s' ------------
        {
            double *dst = a.fac + ((size_t)chain * n + s) * g.NPT * kTileElems;
            const int ntop = CT * (CT + 1) / 2;
            const int n2 = g.NPT * kTileElems / 2;
            for (int i = tid; i < n2; i += NTH) {
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
            double *yv = a.y + ((size_t)chain * n + s) * nux;
            for (int k = tid; k < nux; k += NTH)
                yv[k] = pan[tri_index(rhs_tile, k / 8) * kTileElems + rhs_r * 8 + k % 8];
        }

        if (s + 1 < n) {
            // ---- S4: W for stage s+1 --------------------------------------
            cp_wait_all(); // BA_{s+1} (and H_{s+1}) have landed
            __syncthreads();
            // -wl_new = L_Q' fd + x'   (kkt_solve.cpp:85-90)
            for (int t = tid; t < nx; t += NTH) {
                double q = 0;
                const int C = nu + t;
                for (int k = t; k < nx; ++k) {
                    const int K = nu + k;
                    q += pan[tri_index(K / 8, C / 8) * kTileElems + (K % 8) * 8 + C % 8] *
                         (sgn * bf.f[k]);
                }
                const double xp = pan[tri_index(rhs_tile, C / 8) * kTileElems + rhs_r * 8 + C % 8];
                mwl[t] = q + xp;
                a.wl[((size_t)chain * n + s) * nx + t] = -(q + xp);
            }
            // V = BA_{s+1}' L_Q (DMMA; A from the BA buffer, B from the panel)
            const int nvt = CT * NXT;
            for (int v = warp; v < nvt; v += NW) {
                const int ti = v / NXT, kt = v % NXT, ct = XT0 + kt;
                Frag f{0.0, 0.0};
                const int r = 8 * ti + rq;
                for (int ks = 2 * XT0; ks < 2 * (XT0 + NXT); ++ks) {
                    if (4 * ks + 3 < 8 * ct)
                        continue; // L_Q upper part is zero
                    const int K = 4 * ks + (lane & 3);
                    double av = 0.0;
                    if (K >= nu && K < nux && r < nux) {
                        const int kk = K - nu;
                        av = r < nu ? bf.B[kk * nu + r] : bf.A[kk * nx + (r - nu)];
                    }
                    const int Cb = 8 * ct + (lane >> 2);
                    double bv = 0.0;
                    if (K >= nu && K < nux && Cb >= nu && Cb < nux && K >= Cb)
                        bv = pan[tri_index(K / 8, Cb / 8) * kTileElems + (K % 8) * 8 + Cb % 8];
                    dmma(f, av, bv);
                }
                st_frag(Vs + v * kTileElems, lane, f);
            }
            __syncthreads();
            if (s + 2 < n) {
                load_BA(g, a.p, b, g.stage_of(c, s + 2), bf, tid, NTH, cst);
                cp_commit();
            }
        }
    }

    // trailing tiles (coupling x coupling = -Mfwd, rhs x coupling = -fwd)
#pragma unroll
    for (int k = 0; k < MAXT; ++k) {
        const int t = warp + k * NW;
        if (t < NT) {
            const int ti = tab[2 * t], tj = tab[2 * t + 1];
            if (tj >= CT) {
                const int u = ti - CT, v = tj - CT;
                st_frag(a.trail + ((size_t)chain * g.NTT + tri_index(u, v)) * kTileElems, lane,
                        acc[k]);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1)
        my_fail = min(my_fail, __shfl_xor_sync(0xffffffffu, my_fail, o));
    if (lane == 0 && my_fail != ~0ull)
        atomicMin(a.fail + b, my_fail);
}

template __global__ void riccati_panel_kernel_t<4>(RiccatiArgs);
template __global__ void riccati_panel_kernel_t<8>(RiccatiArgs);
template __global__ void riccati_panel_kernel_t<16>(RiccatiArgs);
template __global__ void riccati_panel_kernel_t<32>(RiccatiArgs);

size_t riccati_smem_bytes(const Geo &g, bool staged) {
    const int nt = g.TT * (g.TT + 1) / 2;
    size_t dbl = (size_t)(nt + g.CT * g.NXT) * kTileElems + g.nx + g.nu + 32;
    if (staged)
        dbl += (size_t)g.nu * g.nu + g.nu * g.nx + g.nx * g.nx + g.nu + g.nx +
               (size_t)g.nx * g.nu + g.nx * g.nx + g.nx;
    return dbl * sizeof(double) + 2 * nt + 64;
}
bool riccati_staged(const Geo &g) { return riccati_smem_bytes(g, true) <= 200 * 1024; }
size_t riccati_smem_bytes(const Geo &g) { return riccati_smem_bytes(g, riccati_staged(g)); }
size_t riccati_consts_doubles(const Geo &g) {
    return (size_t)g.nu * g.nu + (size_t)g.nx * g.nx +
           (size_t)g.nx * (g.nx > g.nu ? g.nx : g.nu) + g.nx + g.nu;
}

} // namespace cyqb
