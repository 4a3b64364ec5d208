// Schur-complement assembly + cyclic-reduction factor/solve of the coupling
// system, one CTA per OCP instance (warps take independent blocks).
//
// Restates:
//   kkt_factor.cpp:163-178    T = L_Q^{-T}, Mbwd = T T', W = T LA'
//   kkt_factor.cpp:194-212    assemble_schur (diag, subdiag)
//   block_tridiag.cpp:126-238 cr_level / cr_factor / cr_factor_base (non-circular)
//   kkt_solve.cpp:137-182     Schur rhs, CRFactor::forward/backward, negate
//   block_tridiag.cpp:252-333 CRFactor::forward / backward
// The level arrays live in a per-instance global workspace (L2-resident);
// every block operation stages its operands in per-warp shared-memory
// scratch (row stride nx|1 to avoid bank conflicts) and runs warp-wide.
// Fixed reduction orders: results are bit-reproducible.
#include "kernels.h"

#include <algorithm>

namespace cyqb {

namespace {

__host__ __device__ __forceinline__ int stride_of(int n) { return n | 1; }

// copy an n x n block global (ld n) -> scratch (ld s); lower only if `lower`
__device__ void w_load(double *dst, int s, const double *src, int n, bool lower, bool trans,
                       int lane) {
    for (int e = lane; e < n * n; e += 32) {
        const int r = e / n, c = e % n;
        const double v = trans ? src[c * n + r] : src[e];
        dst[r * s + c] = (!lower || c <= r) ? v : 0.0;
    }
    __syncwarp();
}
__device__ void w_store(double *dst, const double *src, int s, int n, double scale, int lane) {
    __syncwarp();
    for (int e = lane; e < n * n; e += 32)
        dst[e] = scale * src[(e / n) * s + e % n];
}

// In-place lower Cholesky (potrf semantics of kernels.cpp:32-58: relative
// pivot floor 1e-14 * max|diag| of the input). Returns failing pivot or -1.
__device__ int w_potrf(double *A, int s, int n, int lane) {
    double dmax = 0;
    for (int d = 0; d < n; ++d)
        dmax = fmax(dmax, fabs(A[d * s + d]));
    int fail = -1;
    for (int k = 0; k < n; ++k) {
        __syncwarp();
        double pv = A[k * s + k];
        if (!(pv > 1e-14 * dmax && isfinite(pv))) {
            if (fail < 0) fail = k;
            pv = 1.0;
        }
        const double iv = rsqrt(pv);
        __syncwarp();
        if (lane == 0)
            A[k * s + k] = pv * iv;
        for (int i = k + 1 + lane; i < n; i += 32)
            A[i * s + k] *= iv;
        __syncwarp();
        for (int e = lane; e < (n - k - 1) * (n - k - 1); e += 32) {
            const int i = k + 1 + e / (n - k - 1), j = k + 1 + e % (n - k - 1);
            if (j <= i)
                A[i * s + j] -= A[i * s + k] * A[j * s + k];
        }
    }
    __syncwarp();
    return fail;
}

// B (m x n) <- B L^{-T}  (TrsmMode::right_lower_trans), a row per lane
__device__ void w_trsm_rlt(double *B, int sb, int m, int n, const double *L, int sl, int lane) {
    for (int r = lane; r < m; r += 32) {
        double *br = B + r * sb;
        for (int c = 0; c < n; ++c) {
            double x = br[c];
            for (int k = 0; k < c; ++k)
                x -= br[k] * L[c * sl + k];
            br[c] = x / L[c * sl + c];
        }
    }
    __syncwarp();
}

// C (lower) -= A A'   (all n x n elements spread over lanes)
__device__ void w_syrk_sub(double *C, int sc, const double *A, int sa, int n, int lane) {
    for (int e = lane; e < n * n; e += 32) {
        const int i = e / n, j = e % n;
        if (j > i)
            continue;
        double acc = 0;
        for (int k = 0; k < n; ++k)
            acc += A[i * sa + k] * A[j * sa + k];
        C[i * sc + j] -= acc;
    }
    __syncwarp();
}

// x <- L^{-1} x / L^{-T} x  (global or shared vectors; column-oriented)
__device__ void w_trsv(const double *L, int sl, double *x, int n, bool trans, int lane) {
    for (int kk = 0; kk < n; ++kk) {
        const int k = trans ? n - 1 - kk : kk;
        __syncwarp();
        const double xk = x[k] / L[k * sl + k];
        __syncwarp();
        if (lane == 0)
            x[k] = xk;
        if (!trans) {
            for (int i = k + 1 + lane; i < n; i += 32)
                x[i] -= L[i * sl + k] * xk;
        } else {
            for (int i = lane; i < k; i += 32)
                x[i] -= L[k * sl + i] * xk;
        }
    }
    __syncwarp();
}

// y -= op(A) x   (A in scratch with row stride sa)
__device__ void w_gemv_sub(const double *A, int sa, bool trans, const double *x, double *y,
                           int n, int lane) {
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
        double acc = 0;
        for (int k = 0; k < n; ++k)
            acc += (trans ? A[k * sa + i] : A[i * sa + k]) * x[k];
        y[i] -= acc;
    }
    __syncwarp();
}

__device__ __forceinline__ int stored_tile(const Geo &g, int ti, int tj) {
    return ti < g.CT ? tri_index(ti, tj) : g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
}
__device__ __forceinline__ double fac_at(const Geo &g, const double *st, int r, int col) {
    return st[stored_tile(g, r / 8, col / 8) * kTileElems + (r % 8) * 8 + col % 8];
}

} // namespace

size_t schur_smem_bytes(const Geo &g) { return schur_smem_for(g, schur_warps(g)); }
size_t schur_smem_for(const Geo &g, int nw) {
    const int s = stride_of(g.nx);
    return ((size_t)nw * 4 * g.nx * s + (size_t)g.P * g.nx) * sizeof(double);
}
// solve-only launches (factor done by the tile kernels): a few warps per
// instance, several instances per SM
int schur_warps_solve(const Geo &g) {
    const int w = schur_warps(g);
    return w < 4 ? w : 4;
}

int schur_warps(const Geo &g) {
    const size_t per = 4 * (size_t)g.nx * stride_of(g.nx) * sizeof(double);
    const size_t xbytes = (size_t)g.P * g.nx * sizeof(double);
    int nw = (int)std::min<size_t>(8, (200 * 1024 - std::min<size_t>(xbytes, 100 * 1024)) / per);
    nw = nw < 1 ? 1 : nw;
    const int want = g.P / 2 > 1 ? g.P / 2 : 1;
    return nw < want ? nw : want;
}

__global__ void __launch_bounds__(256) schur_cr_kernel(SchurArgs a) {
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NW = blockDim.x >> 5;
    const int P = g.P, nx = g.nx, nu = g.nu, n = g.n;
    const int ss = stride_of(nx);
    const long long nn = (long long)nx * nx;
    const SchurLayout L = SchurLayout::make(P, nx);
    double *ws = a.schur + (size_t)b * L.total;
    double *D = ws + L.D, *K = ws + L.K, *Mb = ws + L.Mb, *Zg = ws + L.Z;
    double *bn = ws + L.bn, *rhs = ws + L.rhs;
    const int top = 8 * g.CT;
    double *S0 = sm + (size_t)warp * 4 * nx * ss, *S1 = S0 + nx * ss, *S2 = S1 + nx * ss,
           *S3 = S2 + nx * ss;
    double *xs = sm + (size_t)NW * 4 * nx * ss; // P * nx (CR solve vector)
    unsigned long long my_fail = ~0ull;

    // ---- phase 1: per-column T-contributions (Z = L_Q^{-1} = T') --------
    for (int c = warp; c < P; c += NW) {
        const size_t chain = (size_t)b * P + c;
        const double *st = a.fac + (chain * n + (n - 1)) * g.NPT * kTileElems;
        double *Zc = Zg + c * nn;
        if (a.do_factor) {
            // L_Q of the last stage position -> S0, LA -> S1
            for (int e = lane; e < nx * nx; e += 32) {
                const int r = e / nx, k = e % nx;
                S0[r * ss + k] = k <= r ? fac_at(g, st, nu + r, nu + k) : 0.0;
                S1[r * ss + k] = fac_at(g, st, top + r, nu + k);
            }
            __syncwarp();
            // Z = L_Q^{-1}: column per lane (trtri, kernels.cpp:246-271)
            for (int jc = lane; jc < nx; jc += 32) {
                for (int i = 0; i < jc; ++i)
                    S2[i * ss + jc] = 0.0;
                S2[jc * ss + jc] = 1.0 / S0[jc * ss + jc];
                for (int i = jc + 1; i < nx; ++i) {
                    double acc = 0;
                    for (int k = jc; k < i; ++k)
                        acc += S0[i * ss + k] * S2[k * ss + jc];
                    S2[i * ss + jc] = -acc / S0[i * ss + i];
                }
            }
            __syncwarp();
            w_store(Zc, S2, ss, nx, 1.0, lane);
            // Mbwd = Z' Z ; K[c-1] = -(LA Z) ; D[c] = Mfwd_c (from -Mfwd trail)
            const double *tr = a.trail + chain * g.NTT * kTileElems;
            for (int e = lane; e < nx * nx; e += 32) {
                const int i = e / nx, jj = e % nx;
                double m = 0;
                for (int k = max(i, jj); k < nx; ++k)
                    m += S2[k * ss + i] * S2[k * ss + jj];
                Mb[c * nn + e] = m;
                const int r = max(i, jj), cc = min(i, jj);
                D[c * nn + e] = -tr[tri_index(r / 8, cc / 8) * kTileElems + (r % 8) * 8 + cc % 8];
                if (c > 0) {
                    double w = 0;
                    for (int k = jj; k < nx; ++k)
                        w += S1[i * ss + k] * S2[k * ss + jj];
                    K[(c - 1) * nn + e] = -w;
                }
            }
            if (c == P - 1)
                for (int e = lane; e < nn; e += 32)
                    K[(P - 1) * nn + e] = 0.0;
        }
        if (a.do_solve) {
            // bwd_neg_c = T x'_{n-1} = Z' x'
            if (!a.do_factor)
                w_load(S2, ss, Zc, nx, false, false, lane);
            const double *yv = a.y + (chain * n + (n - 1)) * g.nux;
            for (int k = lane; k < nx; k += 32)
                S3[k] = yv[nu + k];
            __syncwarp();
            for (int i = lane; i < nx; i += 32) {
                double acc = 0;
                for (int k = i; k < nx; ++k)
                    acc += S2[k * ss + i] * S3[k];
                bn[c * nx + i] = acc;
            }
        }
        __syncwarp();
    }
    __syncthreads();
    // ---- phase 1b: diag += Mbwd of the next column; Schur rhs -----------
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
            const int rr = nx; // rhs row inside the trailing block: -fwd_i
            v += tr[tri_index(rr / 8, k / 8) * kTileElems + (rr % 8) * 8 + k % 8];
            v += bn[((i + 1) % P) * nx + k];
            rhs[e] = v;
        }
    }
    __syncthreads();

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
                w_load(S0, ss, Ml + k * nn, nx, true, false, lane);
                w_load(S1, ss, Kl + (k - 1) * nn, nx, false, true, lane); // U = K_{k-1}'
                const int pf = w_potrf(S0, ss, nx, lane);
                if (pf >= 0)
                    my_fail = min(my_fail, fail_key(kKindCR, l, k, pf));
                w_trsm_rlt(S1, ss, nx, nx, S0, ss, lane);
                w_store(Ll + mm * nn, S0, ss, nx, 1.0, lane);
                w_store(Ul + mm * nn, S1, ss, nx, 1.0, lane);
                if (k < s - 1) {
                    w_load(S2, ss, Kl + k * nn, nx, false, false, lane);
                    w_trsm_rlt(S2, ss, nx, nx, S0, ss, lane);
                    w_store(Yl + mm * nn, S2, ss, nx, 1.0, lane);
                } else {
                    for (int e = lane; e < nn; e += 32)
                        Yl[mm * nn + e] = 0.0;
                }
            }
            __syncthreads();
            for (int mm = warp; mm < half; mm += NW) {
                w_load(S0, ss, Ml + 2 * mm * nn, nx, true, false, lane);
                w_load(S1, ss, Ul + mm * nn, nx, false, false, lane);
                w_syrk_sub(S0, ss, S1, ss, nx, lane);
                if (mm > 0) {
                    w_load(S2, ss, Yl + (mm - 1) * nn, nx, false, false, lane);
                    w_syrk_sub(S0, ss, S2, ss, nx, lane);
                }
                w_store(M2 + mm * nn, S0, ss, nx, 1.0, lane);
                if (mm < half - 1) { // K' = -Y U'
                    w_load(S3, ss, Yl + mm * nn, nx, false, false, lane);
                    for (int e = lane; e < nn; e += 32) {
                        const int r = e / nx, cc = e % nx;
                        double acc = 0;
                        for (int q = 0; q < nx; ++q)
                            acc += S3[r * ss + q] * S1[cc * ss + q];
                        K2[mm * nn + e] = -acc;
                    }
                } else {
                    for (int e = lane; e < nn; e += 32)
                        K2[mm * nn + e] = 0.0;
                }
                __syncwarp();
            }
            __syncthreads();
        }
        if (warp == 0) {
            const double *Mlast = L.levels == 0 ? D : ws + L.level(L.levels - 1, P, nx, 3);
            w_load(S0, ss, Mlast, nx, true, false, lane);
            const int pf = w_potrf(S0, ss, nx, lane);
            if (pf >= 0)
                my_fail = min(my_fail, fail_key(kKindCR, L.levels, 0, pf));
            w_store(ws + L.Lbase, S0, ss, nx, 1.0, lane);
        }
        __syncthreads();
    }

    // ---- phase 3: CR solve (block_tridiag.cpp:252-333), negate ----------
    // x lives in shared memory; every block is staged into the warp's
    // scratch with coalesced loads before its sequential trsv / gemv.
    if (a.do_solve) {
        double *x = xs;
        for (int e = threadIdx.x; e < P * nx; e += blockDim.x)
            x[e] = rhs[e];
        __syncthreads();
        int s = P;
        for (int l = 0; l < L.levels; ++l, s /= 2) {
            const int half = s / 2, stride = P / s;
            const double *Ll = ws + L.level(l, P, nx, 0), *Ul = ws + L.level(l, P, nx, 1);
            const double *Yl = ws + L.level(l, P, nx, 2);
            for (int mm = warp; mm < half; mm += NW) {
                w_load(S0, ss, Ll + mm * nn, nx, false, false, lane);
                w_trsv(S0, ss, x + (2 * mm + 1) * stride * nx, nx, false, lane);
            }
            __syncthreads();
            for (int mm = warp; mm < half; mm += NW) {
                double *ye = x + 2 * mm * stride * nx;
                w_load(S1, ss, Ul + mm * nn, nx, false, false, lane);
                w_gemv_sub(S1, ss, false, x + (2 * mm + 1) * stride * nx, ye, nx, lane);
                if (mm > 0) {
                    w_load(S2, ss, Yl + (mm - 1) * nn, nx, false, false, lane);
                    w_gemv_sub(S2, ss, false, x + ((2 * (mm - 1) + 1) * stride % P) * nx, ye,
                               nx, lane);
                }
            }
            __syncthreads();
        }
        if (warp == 0) {
            w_load(S0, ss, ws + L.Lbase, nx, false, false, lane);
            w_trsv(S0, ss, x, nx, false, lane);
            w_trsv(S0, ss, x, nx, true, lane);
        }
        __syncthreads();
        s = P >> L.levels;
        for (int l = L.levels - 1; l >= 0; --l, s *= 2) {
            const int sl = 2 * s, half = sl / 2, stride = P / sl;
            const double *Ll = ws + L.level(l, P, nx, 0), *Ul = ws + L.level(l, P, nx, 1);
            const double *Yl = ws + L.level(l, P, nx, 2);
            for (int mm = warp; mm < half; mm += NW) {
                double *xo = x + (2 * mm + 1) * stride * nx;
                w_load(S1, ss, Ul + mm * nn, nx, false, false, lane);
                w_gemv_sub(S1, ss, true, x + 2 * mm * stride * nx, xo, nx, lane);
                if (2 * mm + 2 < sl) {
                    w_load(S2, ss, Yl + mm * nn, nx, false, false, lane);
                    w_gemv_sub(S2, ss, true, x + ((2 * mm + 2) * stride % P) * nx, xo, nx, lane);
                }
                w_load(S0, ss, Ll + mm * nn, nx, false, false, lane);
                w_trsv(S0, ss, xo, nx, true, lane);
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
