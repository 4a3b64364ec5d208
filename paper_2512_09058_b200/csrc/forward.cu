// Forward substitution over a stored factor, for kkt::solve with a new
// right-hand side (kkt_solve.cpp:41-134): one warp per partition column.
//
// The fused factor kernels produce the forward sweep of EqRhs::of_problem as
// the rhs row of the stage panel; for any other rhs this kernel replays that
// row against the stored pivot tiles:
//   b_s    = [ru_j; qx_xi] - BA_s' (L_Q(s-1) wl_{s-1})      (s > 0)
//   y_s    = LH_s^{-1} b_s
//   wl_s   = -L_Q(s)' fd_{j(s+1)} - y_x                     (s < n-1)
//   fwd    = sum_s [LB ALQ]_s y_s + sum_{s<n-1} ALQ_s wl_s
// writing y, wl and -fwd (into the rhs row of the trailing tiles, where the
// Schur solve reads it), exactly what the fused kernels leave behind.
#include "kernels.h"

namespace cyqb {

namespace {
__device__ __forceinline__ int fw_tile(const Geo &g, int ti, int tj) {
    return ti < g.CT ? tri_index(ti, tj) : g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
}
} // namespace

__host__ __device__ size_t forward_smem_per_warp(const Geo &g) {
    const int vp = 2 * ((g.nux + 1) / 2), xp = 2 * ((g.nx + 1) / 2);
    return ((size_t)g.NPT * kTileElems + 2 * vp + 3 * xp) * sizeof(double);
}

__global__ void __launch_bounds__(64) forward_kernel(BacksubArgs a, double *y_out, double *wl_out,
                                                     double *trail) {
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const size_t chain = (size_t)blockIdx.x * wpb + wib;
    if (chain >= (size_t)g.batch * g.P)
        return;
    const int b = (int)(chain / g.P), c = (int)(chain % g.P);
    const int nu = g.nu, nx = g.nx, nux = g.nux, n = g.n, top = 8 * g.CT;
    const int vp = 2 * ((nux + 1) / 2), xp = 2 * ((nx + 1) / 2);
    double *tiles = sm + (size_t)wib * (forward_smem_per_warp(g) / sizeof(double));
    double *bv = tiles + g.NPT * kTileElems; // nux: b_s, then y_s
    double *tq = bv + vp;                     // nux scratch
    double *wl = tq + vp;                     // nx: wl_{s-1}, then wl_s
    double *tv = wl + xp;                     // nx: L_Q(s-1) wl_{s-1}
    double *fw = tv + xp;                     // nx: fwd accumulator
    ProbAcc pa{a.p, g, b};
    auto Pt = [&](int r, int col) -> double {
        return tiles[fw_tile(g, r / 8, col / 8) * kTileElems + (r % 8) * 8 + col % 8];
    };
    for (int i = lane; i < nx; i += 32)
        fw[i] = 0.0;
    for (int s = 0; s < n; ++s) {
        const int j = g.stage_of(c, s), xi = g.x_index_of(c, s);
        // b_s = [ru_j; qx_xi] - BA_s' t  (t = L_Q(s-1) wl_{s-1} from the previous stage)
        for (int k = lane; k < nux; k += 32) {
            double v = k < nu ? pa.ru(j, k) : pa.qx(xi, k - nu);
            if (s > 0)
                for (int i = 0; i < nx; ++i) {
                    const double ba = k < nu ? pa.B(j, i, k) : (j != 0 ? pa.A(j, i, k - nu) : 0.0);
                    v -= ba * tv[i];
                }
            tq[k] = v;
        }
        __syncwarp();
        // this stage's stored pivot tiles
        {
            const double2 *src = reinterpret_cast<const double2 *>(
                a.fac + (chain * n + s) * g.NPT * kTileElems);
            double2 *dst = reinterpret_cast<double2 *>(tiles);
            for (int i = lane; i < g.NPT * kTileElems / 2; i += 32)
                dst[i] = __ldg(src + i);
        }
        __syncwarp();
        // y = LH^{-1} b  (forward substitution, column oriented)
        for (int k = 0; k < nux; ++k) {
            const double yk = tq[k] / Pt(k, k);
            __syncwarp();
            if (lane == 0)
                tq[k] = yk;
            for (int i = k + 1 + lane; i < nux; i += 32)
                tq[i] -= Pt(i, k) * yk;
            __syncwarp();
        }
        for (int k = lane; k < nux; k += 32)
            y_out[(chain * n + s) * nux + k] = tq[k];
        // fwd += [LB ALQ] y
        for (int i = lane; i < nx; i += 32) {
            double v = 0.0;
            for (int k = 0; k < nux; ++k)
                v += Pt(top + i, k) * tq[k];
            fw[i] += v;
        }
        __syncwarp();
        if (s + 1 < n) {
            const int j1 = g.stage_of(c, s + 1);
            // wl_s = -L_Q' fd_{j1} - y_x ; fwd += ALQ wl_s ; t = L_Q wl_s
            for (int i = lane; i < nx; i += 32) {
                double v = 0.0;
                for (int k = i; k < nx; ++k)
                    v += Pt(nu + k, nu + i) * pa.fd(j1, k);
                wl[i] = -v - tq[nu + i];
                wl_out[(chain * n + s) * nx + i] = wl[i];
            }
            __syncwarp();
            for (int i = lane; i < nx; i += 32) {
                double v = 0.0, t = 0.0;
                for (int k = 0; k < nx; ++k) {
                    v += Pt(top + i, nu + k) * wl[k];
                    if (k <= i)
                        t += Pt(nu + i, nu + k) * wl[k];
                }
                fw[i] += v;
                tv[i] = t;
            }
            __syncwarp();
        }
    }
    // -fwd into the rhs row (row nx) of the trailing block
    double *tr = trail + chain * g.NTT * kTileElems;
    for (int i = lane; i < nx; i += 32)
        tr[tri_index(nx / 8, i / 8) * kTileElems + (nx % 8) * 8 + i % 8] = -fw[i];
}

} // namespace cyqb
