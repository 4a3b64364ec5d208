// Back substitution through the block columns (one warp per partition
// column) and gather into the stage-major EqSolution layout.
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
// Memory-bound: each stage reads its stored pivot tiles (LH, LB, ALQ), y_s,
// wl_s and BA_{s+1} once. They are staged with cp.async into a per-warp
// double buffer one stage ahead (16-byte granules), so the HBM stream
// overlaps the sequential triangular sweeps of the previous stage.
#include "kernels.h"

namespace cyqb {

namespace {

__device__ __forceinline__ void bs_cp8(double *dst, const double *src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void bs_cp16(double *dst, const double *src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void bs_copy(double *dst, const double *src, int cnt, int lane) {
    if (!src) {
        for (int i = lane; i < cnt; i += 32)
            dst[i] = 0.0;
        return;
    }
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        for (int i = 2 * lane; i + 1 < cnt; i += 64)
            bs_cp16(dst + i, src + i);
        if ((cnt & 1) && lane == 0)
            bs_cp8(dst + cnt - 1, src + cnt - 1);
    } else {
        for (int i = lane; i < cnt; i += 32)
            bs_cp8(dst + i, src + i);
    }
}

struct BsBuf {
    double *tiles, *y, *wl, *B, *A;
};

__host__ __device__ inline int bs_buf_doubles(const Geo &g) {
    const int v = (g.NPT * kTileElems + g.nux + g.nx + g.nx * g.nu + g.nx * g.nx);
    return (v + 1) & ~1;
}
__host__ __device__ inline int bs_vec_doubles(const Geo &g) {
    const int vp = 2 * ((g.nux + 1) / 2), xp = 2 * ((g.nx + 1) / 2);
    return 3 * vp + 5 * xp;
}

__device__ BsBuf bs_carve(double *base, const Geo &g) {
    BsBuf b;
    b.tiles = base;
    b.y = b.tiles + g.NPT * kTileElems;
    b.wl = b.y + g.nux;
    b.B = b.wl + g.nx;
    b.A = b.B + g.nx * g.nu;
    return b;
}

// stage s data: pivot tiles, y_s, wl_s (s < n-1) and BA_{s+1}
__device__ void bs_issue(const BacksubArgs &a, const BsBuf &bf, size_t chain, int b, int c,
                         int s, int lane) {
    const Geo &g = a.g;
    const int n = g.n, nx = g.nx, nu = g.nu, N = g.N;
    bs_copy(bf.tiles, a.fac + (chain * n + s) * g.NPT * kTileElems, g.NPT * kTileElems, lane);
    bs_copy(bf.y, a.y + (chain * n + s) * g.nux, g.nux, lane);
    if (s + 1 < n) {
        bs_copy(bf.wl, a.wl + (chain * n + s) * nx, nx, lane);
        const int j1 = g.stage_of(c, s + 1);
        const bool in = j1 < N;
        bs_copy(bf.B, in ? a.p.B + ((size_t)b * N + j1) * nx * nu : nullptr, nx * nu, lane);
        bs_copy(bf.A, (in && j1 != 0) ? a.p.A + ((size_t)b * N + j1) * nx * nx : nullptr,
                nx * nx, lane);
    }
    asm volatile("cp.async.commit_group;\n");
}

__device__ __forceinline__ int bs_stored_tile(const Geo &g, int ti, int tj) {
    return ti < g.CT ? tri_index(ti, tj) : g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
}

} // namespace

__host__ __device__ size_t backsub_smem_per_warp(const Geo &g, int nbuf) {
    return ((size_t)nbuf * bs_buf_doubles(g) + bs_vec_doubles(g)) * sizeof(double);
}
// single buffer + high occupancy (many warps alternate load / compute)
__host__ __device__ int backsub_nbuf(const Geo &) { return 1; }
int backsub_wpb(const Geo &g) {
    int w = BACKSUB_WPB;
    while (w > 1 && (size_t)w * backsub_smem_per_warp(g, backsub_nbuf(g)) > 200 * 1024)
        w /= 2;
    return w;
}
size_t backsub_smem_bytes(const Geo &g) {
    return (size_t)backsub_wpb(g) * backsub_smem_per_warp(g, backsub_nbuf(g));
}

__global__ void __launch_bounds__(32 * BACKSUB_WPB, 4) backsub_kernel(BacksubArgs a) {
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const size_t chain = (size_t)blockIdx.x * (blockDim.x >> 5) + wib;
    if (chain >= (size_t)g.batch * g.P)
        return;
    const int b = (int)(chain / g.P), c = (int)(chain % g.P);
    const int nu = g.nu, nx = g.nx, nux = g.nux, n = g.n, top = 8 * g.CT;
    const int nbuf = backsub_nbuf(g);
    double *wbase = sm + (size_t)wib * (backsub_smem_per_warp(g, nbuf) / sizeof(double));
    BsBuf buf[2];
    buf[0] = bs_carve(wbase, g);
    buf[1] = bs_carve(wbase + (nbuf > 1 ? bs_buf_doubles(g) : 0), g);
    double *vec = wbase + nbuf * bs_buf_doubles(g);
    const int vp = 2 * ((nux + 1) / 2), xp = 2 * ((nx + 1) / 2);
    double *Y = vec, *z = Y + vp, *idg = z + vp;
    double *lf = idg + vp, *lb = lf + xp, *w = lb + xp, *zn = w + xp, *t1 = zn + xp;

    for (int k = lane; k < nx; k += 32) {
        lf[k] = a.lamc[((size_t)b * g.P + c) * nx + k];
        lb[k] = a.lamc[((size_t)b * g.P + (c - 1 + g.P) % g.P) * nx + k];
    }
    bs_issue(a, buf[0], chain, b, c, n - 1, lane);

    for (int s = n - 1; s >= 0; --s) {
        const BsBuf &bf = buf[nbuf > 1 ? (s & 1) ^ ((n - 1) & 1) : 0];
        if (nbuf > 1 && s > 0) { // prefetch stage s-1 into the other buffer
            bs_issue(a, buf[((s - 1) & 1) ^ ((n - 1) & 1)], chain, b, c, s - 1, lane);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncwarp();
        const int j = g.stage_of(c, s), xi = g.x_index_of(c, s);
        auto P = [&](int r, int col) -> double {
            return bf.tiles[bs_stored_tile(g, r / 8, col / 8) * kTileElems + (r % 8) * 8 + col % 8];
        };
        // y -= [LB ALQ]' lam_f ; 1 / diag(LH)
        for (int k = lane; k < nux; k += 32) {
            double gk = 0;
            for (int q = 0; q < nx; ++q)
                gk += P(top + q, k) * lf[q];
            Y[k] = bf.y[k] - gk;
            if (k >= nu && s + 1 < n)
                w[k - nu] = -bf.wl[k - nu] - gk;
            idg[k] = 1.0 / P(k, k);
        }
        __syncwarp();
        if (s == n - 1) {
            // x += L_Q^{-1} lam_b  (T' lam_b, kkt_solve.cpp:218-223)
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
        } else {
            const int j1 = g.stage_of(c, s + 1);
            // zn = BA_{s+1} z_{s+1}
            for (int i = lane; i < nx; i += 32) {
                double v = 0;
                for (int k = 0; k < nu; ++k)
                    v += bf.B[i * nu + k] * z[k];
                for (int k = 0; k < nx; ++k)
                    v += bf.A[i * nx + k] * z[nu + k];
                zn[i] = v;
            }
            __syncwarp();
            // t = w - L_Q' zn
            for (int i = lane; i < nx; i += 32) {
                double v = w[i];
                for (int k = i; k < nx; ++k)
                    v -= P(nu + k, nu + i) * zn[k];
                t1[i] = v;
            }
            __syncwarp();
            // lam^{j(s+1)} = -L_Q t ; x -= t
            for (int i = lane; i < nx; i += 32) {
                double v = 0;
                for (int k = 0; k <= i; ++k)
                    v -= P(nu + i, nu + k) * t1[k];
                if (j1 < g.N)
                    a.sol.lam[((size_t)b * g.N + j1) * nx + i] = v;
                Y[nu + i] -= t1[i];
            }
        }
        // z = LH^{-T} Y (back substitution over the top block)
        for (int r = nux - 1; r >= 0; --r) {
            __syncwarp();
            const double zr = Y[r] * idg[r];
            __syncwarp();
            if (lane == 0)
                Y[r] = zr;
            for (int k = lane; k < r; k += 32)
                Y[k] -= P(r, k) * zr;
        }
        __syncwarp();
        for (int k = lane; k < nux; k += 32) {
            const double v = Y[k];
            z[k] = v;
            if (k < nu) {
                if (j < g.N)
                    a.sol.u[((size_t)b * g.N + j) * nu + k] = v;
            } else if (xi <= g.N) {
                a.sol.x[((size_t)b * (g.N + 1) + xi) * nx + (k - nu)] = v;
            }
        }
        __syncwarp();
        if (nbuf == 1 && s > 0)
            bs_issue(a, buf[0], chain, b, c, s - 1, lane);
    }
    if (c == 0)
        for (int k = lane; k < nx; k += 32)
            a.sol.x[(size_t)b * (g.N + 1) * nx + k] = __ldg(a.p.x_init + (size_t)b * nx + k);
}

} // namespace cyqb
