// Back substitution through the block columns (one CTA per partition column)
// and gather into the stage-major EqSolution layout.
//
// Restates kkt_solve.cpp:185-307 (pass 1 "y = D w - LA' lam" and the
// bottom-up L' solve, fused into one reverse sweep over the stage positions
// since pass 1 only touches the stage it visits):
//   y_s   = [u'; x']_s - [LB ALQ]_s' lam_f
//   s = n-1:  x_s += L_Q^{-1} lam_b                      (T' lam_b)
//   s < n-1:  w  = -wl_s - ALQ_s' lam_f
//             t  = w - L_Q' (BA_{s+1} z_{s+1})
//             lam^{j(s+1)} = -L_Q t,   x_s -= t            (L_Q^{-1} L_Q = I)
//   z_s   = LH_s^{-T} y_s
// The stage's stored pivot tiles are staged in shared memory (coalesced
// 16-byte loads); the triangular sweeps run on warp 0, the mat-vecs on all
// threads.
#include "kernels.h"

namespace cyqb {

namespace {
__device__ __forceinline__ int stored_tile_b(const Geo &g, int ti, int tj) {
    return ti < g.CT ? tri_index(ti, tj) : g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
}
} // namespace

__global__ void __launch_bounds__(256) backsub_kernel(BacksubArgs a) {
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int chain = blockIdx.x;
    const int b = chain / g.P, c = chain % g.P;
    const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nu = g.nu, nx = g.nx, nux = g.nux, n = g.n, top = 8 * g.CT;
    const int vpad = 32 * ((nux + 31) / 32);

    double *tiles = sm;                         // NPT tiles
    double *Y = tiles + g.NPT * kTileElems;     // nux
    double *z = Y + vpad;                        // nux (z_{s+1}, then z_s)
    double *lf = z + vpad;                       // nx
    double *lb = lf + vpad;                      // nx
    double *w = lb + vpad;                       // nx
    double *zn = w + vpad;                       // nx
    double *t1 = zn + vpad;                      // nx
    double *idg = t1 + vpad;                     // nux: 1 / diag(LH)

    auto P = [&](int r, int col) -> double {
        return tiles[stored_tile_b(g, r / 8, col / 8) * kTileElems + (r % 8) * 8 + col % 8];
    };
    ProbAcc pa{a.p, g, b};
    const int cb = (c - 1 + g.P) % g.P;
    for (int k = tid; k < nx; k += NT) {
        lf[k] = a.lamc[((size_t)b * g.P + c) * nx + k];
        lb[k] = a.lamc[((size_t)b * g.P + cb) * nx + k];
    }

    for (int s = n - 1; s >= 0; --s) {
        const int j = g.stage_of(c, s), xi = g.x_index_of(c, s);
        __syncthreads();
        {
            const double2 *src = reinterpret_cast<const double2 *>(
                a.fac + ((size_t)chain * n + s) * g.NPT * kTileElems);
            double2 *dst = reinterpret_cast<double2 *>(tiles);
            for (int i = tid; i < g.NPT * kTileElems / 2; i += NT)
                dst[i] = __ldg(src + i);
            const double *yv = a.y + ((size_t)chain * n + s) * nux;
            for (int k = tid; k < nux; k += NT)
                Y[k] = __ldg(yv + k);
        }
        __syncthreads();
        // y -= [LB ALQ]' lam_f ; reciprocal diagonal of LH
        for (int k = tid; k < nux; k += NT) {
            double gk = 0;
            for (int q = 0; q < nx; ++q)
                gk += P(top + q, k) * lf[q];
            Y[k] -= gk;
            if (k >= nu && s + 1 < n)
                w[k - nu] = -__ldg(a.wl + ((size_t)chain * n + s) * nx + (k - nu)) - gk;
            idg[k] = 1.0 / P(k, k);
        }
        __syncthreads();
        if (s == n - 1) {
            // x += L_Q^{-1} lam_b  (T' lam_b, kkt_solve.cpp:218-223)
            if (warp == 0) {
                for (int k = lane; k < nx; k += 32)
                    t1[k] = lb[k];
                for (int k = 0; k < nx; ++k) {
                    __syncwarp();
                    const double xk = t1[k] * idg[nu + k];
                    __syncwarp();
                    if (lane == 0)
                        t1[k] = xk;
                    for (int i = k + 1 + lane; i < nx; i += 32)
                        t1[i] -= P(nu + i, nu + k) * xk;
                }
                __syncwarp();
                for (int k = lane; k < nx; k += 32)
                    Y[nu + k] += t1[k];
            }
        } else {
            const int j1 = g.stage_of(c, s + 1);
            // zn = BA_{s+1} z_{s+1}
            for (int i = tid; i < nx; i += NT) {
                double v = 0;
                for (int k = 0; k < nu; ++k)
                    v += pa.B(j1, i, k) * z[k];
                if (j1 != 0)
                    for (int k = 0; k < nx; ++k)
                        v += pa.A(j1, i, k) * z[nu + k];
                zn[i] = v;
            }
            __syncthreads();
            // t = w - L_Q' zn
            for (int i = tid; i < nx; i += NT) {
                double v = w[i];
                for (int k = i; k < nx; ++k)
                    v -= P(nu + k, nu + i) * zn[k];
                t1[i] = v;
            }
            __syncthreads();
            // lam^{j(s+1)} = -L_Q t ; x -= t
            for (int i = tid; i < nx; i += NT) {
                double v = 0;
                for (int k = 0; k <= i; ++k)
                    v -= P(nu + i, nu + k) * t1[k];
                if (j1 < g.N)
                    a.sol.lam[((size_t)b * g.N + j1) * nx + i] = v;
                Y[nu + i] -= t1[i];
            }
        }
        __syncthreads();
        // z = LH^{-T} Y (back substitution over the top block)
        if (warp == 0) {
            for (int r = nux - 1; r >= 0; --r) {
                __syncwarp();
                const double zr = Y[r] * idg[r];
                __syncwarp();
                if (lane == 0)
                    Y[r] = zr;
                for (int k = lane; k < r; k += 32)
                    Y[k] -= P(r, k) * zr;
            }
        }
        __syncthreads();
        for (int k = tid; k < nux; k += NT) {
            const double v = Y[k];
            z[k] = v;
            if (k < nu) {
                if (j < g.N)
                    a.sol.u[((size_t)b * g.N + j) * nu + k] = v;
            } else if (xi <= g.N) {
                a.sol.x[((size_t)b * (g.N + 1) + xi) * nx + (k - nu)] = v;
            }
        }
    }
    if (c == 0)
        for (int k = tid; k < nx; k += NT)
            a.sol.x[(size_t)b * (g.N + 1) * nx + k] = __ldg(a.p.x_init + (size_t)b * nx + k);
}

} // namespace cyqb
