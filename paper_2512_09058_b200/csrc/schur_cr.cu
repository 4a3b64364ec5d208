// Schur-complement assembly + cyclic-reduction factor/solve of the coupling
// system, one CTA per OCP instance (warps take independent blocks).
//
// Restates:
//   kkt_factor.cpp:163-178   T = L_Q^{-T}, Mbwd = T T', W = T LA'
//   kkt_factor.cpp:194-212   assemble_schur (diag, subdiag)
//   block_tridiag.cpp:126-238 cr_level / cr_factor / cr_factor_base (non-circular)
//   kkt_solve.cpp:137-182     Schur rhs, CRFactor::forward/backward, negate
//   block_tridiag.cpp:252-333 CRFactor::forward / backward
// Blocks live in a per-instance global workspace (L2-resident); all block
// kernels are warp-cooperative and deterministic (fixed reduction order).
#include "kernels.h"

namespace cyqb {

namespace {

// ---- warp-level dense kernels on row-major n x n blocks (ld = n) --------

// In-place lower Cholesky; potrf semantics of kernels.cpp:32-58 (relative
// pivot floor 1e-14 * max|diag| of the input). Returns failing pivot or -1.
__device__ int w_potrf(double *A, int n, int lane) {
    double dmax = 0;
    for (int d = 0; d < n; ++d)
        dmax = fmax(dmax, fabs(A[d * n + d]));
    int fail = -1;
    for (int k = 0; k < n; ++k) {
        __syncwarp();
        double pv = A[k * n + k];
        if (!(pv > 1e-14 * dmax && isfinite(pv))) {
            if (fail < 0) fail = k;
            pv = 1.0;
        }
        const double d = sqrt(pv), inv = 1.0 / d;
        __syncwarp();
        if (lane == 0)
            A[k * n + k] = d;
        for (int i = k + 1 + lane; i < n; i += 32)
            A[i * n + k] *= inv;
        __syncwarp();
        for (int i = k + 1 + lane; i < n; i += 32) {
            const double lik = A[i * n + k];
            for (int j = k + 1; j <= i; ++j)
                A[i * n + j] -= lik * A[j * n + k];
        }
    }
    __syncwarp();
    // zero the strict upper triangle: the factor is lower triangular
    for (int i = lane; i < n; i += 32)
        for (int j = i + 1; j < n; ++j)
            A[i * n + j] = 0.0;
    __syncwarp();
    return fail;
}

// B (m x n) <- B L^{-T}   (TrsmMode::right_lower_trans), rows per lane.
__device__ void w_trsm_rlt(double *B, int m, int n, const double *L, int lane) {
    for (int r = lane; r < m; r += 32) {
        double *br = B + r * n;
        for (int c = 0; c < n; ++c) {
            double x = br[c];
            for (int k = 0; k < c; ++k)
                x -= br[k] * L[c * n + k];
            br[c] = x / L[c * n + c];
        }
    }
    __syncwarp();
}

// C (lower) -= A A'
__device__ void w_syrk_sub(double *C, const double *A, int n, int lane) {
    for (int i = lane; i < n; i += 32)
        for (int j = 0; j <= i; ++j) {
            double s = 0;
            for (int k = 0; k < n; ++k)
                s += A[i * n + k] * A[j * n + k];
            C[i * n + j] -= s;
        }
    __syncwarp();
}

// x <- L^{-1} x (lower, column-oriented); x shared in global/smem
__device__ void w_trsv_l(const double *L, double *x, int n, int lane) {
    for (int k = 0; k < n; ++k) {
        __syncwarp();
        const double xk = x[k] / L[k * n + k];
        __syncwarp();
        if (lane == 0)
            x[k] = xk;
        for (int i = k + 1 + lane; i < n; i += 32)
            x[i] -= L[i * n + k] * xk;
    }
    __syncwarp();
}

// x <- L^{-T} x
__device__ void w_trsv_lt(const double *L, double *x, int n, int lane) {
    for (int k = n - 1; k >= 0; --k) {
        __syncwarp();
        const double xk = x[k] / L[k * n + k];
        __syncwarp();
        if (lane == 0)
            x[k] = xk;
        for (int i = lane; i < k; i += 32)
            x[i] -= L[k * n + i] * xk;
    }
    __syncwarp();
}

// y -= op(A) x
__device__ void w_gemv_sub(const double *A, bool trans, const double *x,
                           double *y, int n, int lane) {
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
        double s = 0;
        for (int k = 0; k < n; ++k)
            s += (trans ? A[k * n + i] : A[i * n + k]) * x[k];
        y[i] -= s;
    }
    __syncwarp();
}

__device__ __forceinline__ int stored_tile(const Geo &g, int ti, int tj) {
    return ti < g.CT ? tri_index(ti, tj) : g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
}
// entry (r, col) of the stored pivot tiles of one stage
__device__ __forceinline__ double fac_at(const Geo &g, const double *st, int r, int col) {
    return st[stored_tile(g, r / 8, col / 8) * kTileElems + (r % 8) * 8 + col % 8];
}

} // namespace

__global__ void __launch_bounds__(256) schur_cr_kernel(SchurArgs a) {
    const Geo &g = a.g;
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NW = blockDim.x >> 5;
    const int P = g.P, nx = g.nx, nu = g.nu, n = g.n;
    const long long nn = (long long)nx * nx;
    const SchurLayout L = SchurLayout::make(P, nx);
    double *ws = a.schur + (size_t)b * L.total;
    double *D = ws + L.D, *K = ws + L.K, *Mb = ws + L.Mb, *Z = ws + L.Z;
    double *bn = ws + L.bn, *rhs = ws + L.rhs;
    const int top = 8 * g.CT;
    unsigned long long my_fail = ~0ull;

    if (a.do_factor || a.do_solve) {
        // ---- phase 1: per-column Schur contributions ----------------------
        for (int c = warp; c < P; c += NW) {
            const size_t chain = (size_t)b * P + c;
            const double *st = a.fac + (chain * n + (n - 1)) * g.NPT * kTileElems;
            double *Zc = Z + c * nn;
            // Z = L_Q^{-1} (column per lane), L_Q = LH_{n-1}[nu:, nu:]
            for (int jc = lane; jc < nx; jc += 32) {
                for (int i = 0; i < jc; ++i)
                    Zc[i * nx + jc] = 0.0;
                Zc[jc * nx + jc] = 1.0 / fac_at(g, st, nu + jc, nu + jc);
                for (int i = jc + 1; i < nx; ++i) {
                    double s = 0;
                    for (int k = jc; k < i; ++k)
                        s += fac_at(g, st, nu + i, nu + k) * Zc[k * nx + jc];
                    Zc[i * nx + jc] = -s / fac_at(g, st, nu + i, nu + i);
                }
            }
            __syncwarp();
            if (a.do_factor) {
                // Mbwd = T T' = Z' Z ; K[c-1] = -W' = -(LA Z) ; D[c] = Mfwd_c
                const double *tr = a.trail + chain * g.NTT * kTileElems;
                for (int i = lane; i < nx; i += 32) {
                    for (int jj = 0; jj < nx; ++jj) {
                        double s = 0;
                        for (int k = max(i, jj); k < nx; ++k)
                            s += Zc[k * nx + i] * Zc[k * nx + jj];
                        Mb[c * nn + i * nx + jj] = s;
                        // -Mfwd lives in the trailing coupling block (lower)
                        const int r = max(i, jj), cc = min(i, jj);
                        const int u = r / 8, v = cc / 8;
                        D[c * nn + i * nx + jj] =
                            -tr[tri_index(u, v) * kTileElems + (r % 8) * 8 + cc % 8];
                        if (c > 0) {
                            double w = 0;
                            for (int k = jj; k < nx; ++k)
                                w += fac_at(g, st, top + i, nu + k) * Zc[k * nx + jj];
                            K[(c - 1) * nn + i * nx + jj] = -w;
                        }
                    }
                }
                if (c == P - 1)
                    for (int i = lane; i < nn; i += 32)
                        K[(P - 1) * nn + i] = 0.0;
            }
            if (a.do_solve) {
                // bwd_neg_c = T x'_{n-1} = Z' x'
                const double *yv = a.y + (chain * n + (n - 1)) * g.nux;
                for (int i = lane; i < nx; i += 32) {
                    double s = 0;
                    for (int k = i; k < nx; ++k)
                        s += Zc[k * nx + i] * yv[nu + k];
                    bn[c * nx + i] = s;
                }
            }
        }
        __syncthreads();
        // ---- phase 1b: diag += Mbwd of the next column; Schur rhs --------
        if (a.do_factor)
            for (long long e = threadIdx.x; e < (long long)P * nn; e += blockDim.x) {
                const int c = (int)(e / nn);
                D[e] += Mb[((c + 1) % P) * nn + (e % nn)];
            }
        if (a.do_solve) {
            ProbAcc pa{a.p, g, b};
            for (int e = threadIdx.x; e < P * nx; e += blockDim.x) {
                const int i = e / nx, k = e % nx;
                const int jst = n * i;
                double v = pa.fd(jst, k);
                if (jst == 0 && a.p.fd == nullptr) // fd[0] -= A_0 x_init
                    for (int m = 0; m < nx; ++m)
                        v -= pa.A(0, k, m) * __ldg(a.p.x_init + (size_t)b * nx + m);
                const size_t chain = (size_t)b * P + i;
                const double *tr = a.trail + chain * g.NTT * kTileElems;
                const int rr = nx; // rhs row inside the trailing block
                // trailing (rhs, coupling k) = -fwd_i[k]
                v += tr[tri_index(rr / 8, k / 8) * kTileElems + (rr % 8) * 8 + k % 8];
                v += bn[((i + 1) % P) * nx + k];
                rhs[e] = v;
            }
        }
        __syncthreads();
    }

    // ---- phase 2: cyclic reduction factor (block_tridiag.cpp:126-238) ----
    if (a.do_factor) {
        int s = P;
        for (int l = 0; l < L.levels; ++l, s /= 2) {
            const int half = s / 2;
            const double *Ml = l == 0 ? D : ws + L.level(l - 1, P, nx, 3);
            const double *Kl = l == 0 ? K : ws + L.level(l - 1, P, nx, 4);
            double *Ll = ws + L.level(l, P, nx, 0), *Ul = ws + L.level(l, P, nx, 1);
            double *Yl = ws + L.level(l, P, nx, 2), *M2 = ws + L.level(l, P, nx, 3);
            double *K2 = ws + L.level(l, P, nx, 4);
            for (int mm = warp; mm < half; mm += NW) {
                const int k = 2 * mm + 1;
                double *Lm = Ll + mm * nn, *Um = Ul + mm * nn, *Ym = Yl + mm * nn;
                for (int e = lane; e < nn; e += 32) {
                    const int r = e / nx, cc = e % nx;
                    Lm[e] = r >= cc ? Ml[k * nn + e] : 0.0;
                    Um[e] = Kl[(k - 1) * nn + cc * nx + r];
                    Ym[e] = k < s - 1 ? Kl[k * nn + e] : 0.0;
                }
                __syncwarp();
                const int pf = w_potrf(Lm, nx, lane);
                if (pf >= 0)
                    my_fail = min(my_fail, fail_key(kKindCR, l, k, pf));
                w_trsm_rlt(Um, nx, nx, Lm, lane);
                if (k < s - 1)
                    w_trsm_rlt(Ym, nx, nx, Lm, lane);
            }
            __syncthreads();
            for (int mm = warp; mm < half; mm += NW) {
                double *Md = M2 + mm * nn, *Kd = K2 + mm * nn;
                for (int e = lane; e < nn; e += 32)
                    Md[e] = Ml[2 * mm * nn + e];
                __syncwarp();
                w_syrk_sub(Md, Ul + mm * nn, nx, lane);
                if (mm > 0)
                    w_syrk_sub(Md, Yl + (mm - 1) * nn, nx, lane);
                for (int e = lane; e < nn; e += 32) {
                    const int r = e / nx, cc = e % nx;
                    double v = 0;
                    if (mm < half - 1)
                        for (int q = 0; q < nx; ++q)
                            v -= Yl[mm * nn + r * nx + q] * Ul[mm * nn + cc * nx + q];
                    Kd[e] = v;
                }
            }
            __syncthreads();
        }
        if (warp == 0) {
            const double *Mlast = L.levels == 0 ? D : ws + L.level(L.levels - 1, P, nx, 3);
            double *Lb = ws + L.Lbase;
            for (int e = lane; e < nn; e += 32) {
                const int r = e / nx, cc = e % nx;
                Lb[e] = r >= cc ? Mlast[e] : 0.0;
            }
            __syncwarp();
            const int pf = w_potrf(Lb, nx, lane);
            if (pf >= 0)
                my_fail = min(my_fail, fail_key(kKindCR, L.levels, 0, pf));
        }
        __syncthreads();
    }

    // ---- phase 3: CR solve (block_tridiag.cpp:252-333), negate ----------
    if (a.do_solve) {
        double *x = rhs;
        int s = P;
        for (int l = 0; l < L.levels; ++l, s /= 2) {
            const int half = s / 2, stride = P / s;
            const double *Ll = ws + L.level(l, P, nx, 0), *Ul = ws + L.level(l, P, nx, 1);
            const double *Yl = ws + L.level(l, P, nx, 2);
            for (int mm = warp; mm < half; mm += NW)
                w_trsv_l(Ll + mm * nn, x + (2 * mm + 1) * stride * nx, nx, lane);
            __syncthreads();
            for (int mm = warp; mm < half; mm += NW) {
                double *ye = x + 2 * mm * stride * nx;
                w_gemv_sub(Ul + mm * nn, false, x + (2 * mm + 1) * stride * nx, ye, nx, lane);
                if (mm > 0)
                    w_gemv_sub(Yl + (mm - 1) * nn, false,
                               x + ((2 * (mm - 1) + 1) * stride % P) * nx, ye, nx, lane);
            }
            __syncthreads();
        }
        if (warp == 0) {
            w_trsv_l(ws + L.Lbase, x, nx, lane);
            w_trsv_lt(ws + L.Lbase, x, nx, lane);
        }
        __syncthreads();
        s = P >> L.levels;
        for (int l = L.levels - 1; l >= 0; --l, s *= 2) {
            const int sl = 2 * s, half = sl / 2, stride = P / sl;
            const double *Ll = ws + L.level(l, P, nx, 0), *Ul = ws + L.level(l, P, nx, 1);
            const double *Yl = ws + L.level(l, P, nx, 2);
            for (int mm = warp; mm < half; mm += NW) {
                double *xo = x + (2 * mm + 1) * stride * nx;
                w_gemv_sub(Ul + mm * nn, true, x + 2 * mm * stride * nx, xo, nx, lane);
                if (2 * mm + 2 < sl)
                    w_gemv_sub(Yl + mm * nn, true, x + ((2 * mm + 2) * stride % P) * nx, xo, nx,
                               lane);
                w_trsv_lt(Ll + mm * nn, xo, nx, lane);
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < P * nx; e += blockDim.x) {
            const double lam = -x[e];
            a.lamc[(size_t)b * P * nx + e] = lam;
            const int i = e / nx, k = e % nx;
            if (a.lam_out && n * i < g.N)
                a.lam_out[((size_t)b * g.N + n * i) * nx + k] = lam;
        }
    }
    for (int o = 16; o > 0; o >>= 1)
        my_fail = min(my_fail, __shfl_xor_sync(0xffffffffu, my_fail, o));
    if (lane == 0 && my_fail != ~0ull)
        atomicMin(a.fail + b, my_fail);
}

} // namespace cyqb
