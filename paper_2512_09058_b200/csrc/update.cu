// Low-rank factorization update of the stage panels:
// kkt::update's column path (kkt_update.cpp:79-213, update_column) on the
// GPU factor, with the hyperbolic Householder / Givens rotation sweeps of
// batla::hyh_transform / hyh_apply (kernels.cpp:360-453).
//
// One warp per updated partition column (chain), the stages in factor order
// s = 0 .. n-1. The factor tiles of a stage (LH = [L_R; L_S L_Q], coupling
// rows [LB ALQ]) are unpacked into the warp's shared memory,
// rotated, and written back in place:
//   * new update columns of stage j = stage_of(c, s): sqrt|dsigma_i| x
//     [D_j(i, :)' ; C_j(i, :)' ; 0] (sign of dsigma_i), the terminal rows
//     C_term at j = 0 (kkt_update.cpp:95-134);
//   * rotations (k outer, pivot p inner) of [L_R; L_S; LB] against
//     [Yu; Yx; Yl] -- hyperbolic for negative signs (breakdown when
//     u^2 - v^2 <= 0), Givens otherwise, the annihilated entries set to 0;
//   * s < n-1: Acl += Yl S Yx' (Acl = ALQ L_Q' unpacked from the stored
//     ALQ = Acl L_Q^{-T}), Yu, Yx <- [B A]_{s+1}' Yx, rotations of L_Q
//     against Yx, ALQ <- Acl L_Q^{-T} (kkt_update.cpp:140-171);
//   * s = n-1: rotations of L_Q against Yx, the same rotations applied to
//     (LA, Xi_F = Yl), then -Mfwd += Xi_F S Xi_F' in the trailing tiles
//     (kkt_update.cpp:172-211, 455-460; sc_Mbwd, sc_W and T follow from the
//     updated L_Q and LA when the Schur kernel re-runs).
// A breakdown flags the column for refactorization (kkt_update.cpp:430-434).
#include "kernels.h"

namespace cyqb {

namespace {

struct Lay { // shared-memory layout of one warp (doubles)
    int nux, nx, nu, cap;
    int LH, CP, AC, YU, YX, YL, T1, T2, RC, total;
    __host__ __device__ Lay(int nx_, int nu_, int cap_) : nux(nx_ + nu_), nx(nx_), nu(nu_), cap(cap_ > 0 ? cap_ : 1) {
        LH = 0;                   // nux x nux (row-major; lower part used)
        CP = LH + nux * nux;      // nx x nux  coupling rows [LB ALQ]
        AC = CP + nx * nux;       // nx x nx   Acl
        YU = AC + nx * nx;        // nu x cap
        YX = YU + nu * cap;       // nx x cap
        YL = YX + nx * cap;       // nx x cap
        T1 = YL + nx * cap;       // nu x cap  (B' Yx)
        T2 = T1 + nu * cap;       // nx x cap  (A' Yx)
        RC = T2 + nx * cap;       // rotation record: 2 x nx x cap (cc, ss) + kind
        total = RC + 3 * nx * cap + cap;
    }
};

// element (r, k) of the stored pivot tiles of one stage
__device__ __forceinline__ double *tile_el(const Geo &g, double *st, int r, int k) {
    const int ti = r / 8, tj = k / 8;
    const int t = ti < g.CT ? tri_index(ti, tj) : g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
    return st + (size_t)t * kTileElems + (r % 8) * 8 + k % 8;
}

// One rotation sweep: pivots p < np of F (rows r >= p; F(r, p) at F[r * fs + p])
// against the m columns of G (G(r, k) at G[r * gs + k]), both stacked over
// `rows` rows given by the row maps. Records (cc, ss, kind) when rec != null.
// Returns false on a hyperbolic breakdown.
template <class FR, class GR>
__device__ bool hyh_sweep(FR fref, GR gref, int rows, int np, int m, const int *sign, int lane, double *rec,
                          int rec_stride) {
    for (int k = 0; k < m; ++k) {
        const bool hyper = sign[k] < 0; // df = +I: hyperbolic iff the column's sign is -1
        for (int p = 0; p < np; ++p) {
            __syncwarp();
            const double u = *fref(p, p), v = *gref(p, k);
            double cc, ss;
            if (hyper) {
                const double rho2 = u * u - v * v;
                if (!(rho2 > 0.0) || !isfinite(rho2))
                    return false;
                const double rho = sqrt(rho2);
                cc = u / rho;
                ss = v / rho;
            } else {
                const double rho = hypot(u, v);
                if (rho == 0.0) {
                    cc = 1.0;
                    ss = 0.0;
                } else {
                    cc = u / rho;
                    ss = v / rho;
                }
            }
            if (rec && lane == 0) {
                rec[(size_t)k * rec_stride + p] = cc;
                rec[(size_t)k * rec_stride + p + rec_stride * m] = ss;
            }
            __syncwarp();
            if (cc == 1.0 && ss == 0.0)
                continue;
            for (int r = p + lane; r < rows; r += 32) {
                double *fp = fref(r, p), *gp = gref(r, k);
                const double fu = *fp, gv = *gp;
                if (hyper) {
                    *fp = cc * fu - ss * gv;
                    *gp = -ss * fu + cc * gv;
                } else {
                    *fp = cc * fu + ss * gv;
                    *gp = -ss * fu + cc * gv;
                }
            }
        }
    }
    __syncwarp();
    // the annihilated entries are exact zeros by construction (kernels.cpp:445-449)
    for (int e = lane; e < np * m; e += 32)
        *gref(e / m, e % m) = 0.0;
    __syncwarp();
    return true;
}

__global__ void __launch_bounds__(32) update_columns_kernel(UpdateArgs a) {
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31;
    if ((int)blockIdx.x >= a.n)
        return;
    const int chain = a.chains[blockIdx.x];
    const int b = chain / g.P, c = chain % g.P, n = g.n, N = g.N, nx = g.nx, nu = g.nu, nux = g.nux;
    const int ny = a.ny, nyt = a.ny_term;
    const Lay L(nx, nu, a.cap);
    double *LH = sm + L.LH, *CP = sm + L.CP, *AC = sm + L.AC, *YU = sm + L.YU, *YX = sm + L.YX, *YL = sm + L.YL;
    double *T1 = sm + L.T1, *T2 = sm + L.T2, *RC = sm + L.RC;
    int *sg = reinterpret_cast<int *>(sm + L.RC + 3 * nx * L.cap);
    const int cs = L.cap;
    int m = 0;
    for (int s = 0; s < n; ++s) {
        const int j = g.stage_of(c, s);
        double *st = a.fac + ((size_t)chain * n + s) * g.NPT * kTileElems;
        // ---- new update columns of stage j ----------------------------------
        const int m0 = m;
        if (j < N) {
            const double *dsj = a.ds + ((size_t)b * N + j) * ny;
            for (int i = 0; i < ny; ++i) {
                const double dv = __ldg(dsj + i);
                if (dv == 0.0)
                    continue;
                if (m >= cs) { // more columns than planned: refactor instead
                    if (lane == 0)
                        a.breakdown[blockIdx.x] = 1;
                    return;
                }
                const double sq = sqrt(fabs(dv));
                for (int r = lane; r < nu; r += 32)
                    YU[r * cs + m] = __ldg(a.D + (((size_t)b * N + j) * ny + i) * nu + r) * sq;
                for (int r = lane; r < nx; r += 32) {
                    YX[r * cs + m] = j == 0 ? 0.0 : __ldg(a.C + (((size_t)b * N + j) * ny + i) * nx + r) * sq;
                    YL[r * cs + m] = 0.0;
                }
                if (lane == 0)
                    sg[m] = dv > 0.0 ? 1 : -1;
                ++m;
            }
        }
        if (j == 0) { // terminal rows act on the x part of the u^0 stage
            for (int i = 0; i < nyt; ++i) {
                const double dv = __ldg(a.ds_term + (size_t)b * nyt + i);
                if (dv == 0.0)
                    continue;
                if (m >= cs) {
                    if (lane == 0)
                        a.breakdown[blockIdx.x] = 1;
                    return;
                }
                const double sq = sqrt(fabs(dv));
                for (int r = lane; r < nu; r += 32)
                    YU[r * cs + m] = 0.0;
                for (int r = lane; r < nx; r += 32) {
                    YX[r * cs + m] = __ldg(a.C_term + ((size_t)b * nyt + i) * nx + r) * sq;
                    YL[r * cs + m] = 0.0;
                }
                if (lane == 0)
                    sg[m] = dv > 0.0 ? 1 : -1;
                ++m;
            }
        }
        (void)m0;
        if (m == 0)
            continue; // nothing to carry yet: this stage's factor is unchanged
        // ---- unpack the stage (LH lower, coupling rows [LB ALQ]) -------------
        for (int e = lane; e < nux * nux; e += 32) {
            const int r = e / nux, k = e % nux;
            LH[e] = k <= r ? *tile_el(g, st, r, k) : 0.0;
        }
        const int top = 8 * g.CT;
        for (int e = lane; e < nx * nux; e += 32)
            CP[e] = *tile_el(g, st, top + e / nux, e % nux);
        __syncwarp();
        const bool last = s + 1 == n;
        if (!last) { // Acl = ALQ L_Q' (rows of ALQ: CP[:, nu:], L_Q = LH[nu:, nu:])
            for (int e = lane; e < nx * nx; e += 32) {
                const int r = e / nx, k = e % nx;
                double v = 0.0;
                for (int q = 0; q <= k; ++q)
                    v = fma(CP[r * nux + nu + q], LH[(nu + k) * nux + nu + q], v);
                AC[e] = v;
            }
            __syncwarp();
        }
        // ---- [L_R; L_S; LB] against [Yu; Yx; Yl], pivots 0 .. nu-1 -----------
        auto f1 = [&](int r, int p) -> double * {
            return r < nux ? LH + r * nux + p : CP + (r - nux) * nux + p;
        };
        auto g1 = [&](int r, int k) -> double * {
            return r < nu ? YU + r * cs + k : (r < nux ? YX + (r - nu) * cs + k : YL + (r - nux) * cs + k);
        };
        bool ok = hyh_sweep(f1, g1, nux + nx, nu, m, sg, lane, nullptr, 0);
        if (ok && !last) {
            // Acl += Yl S Yx' (kkt_update.cpp:144-154)
            for (int e = lane; e < nx * nx; e += 32) {
                const int r = e / nx, q = e % nx;
                double v = AC[e];
                for (int k = 0; k < m; ++k)
                    v += (double)sg[k] * YL[r * cs + k] * YX[q * cs + k];
                AC[e] = v;
            }
            // [Yu; Yx] <- BAt_{s+1} Yx = [B' ; A']_{j2} Yx (A omitted at j2 = 0,
            // zero for padding stages)
            const int j2 = g.stage_of(c, s + 1);
            const double *Bj = j2 < N ? a.p.B + ((size_t)b * N + j2) * nx * nu : nullptr;
            const double *Aj = (j2 < N && j2 != 0) ? a.p.A + ((size_t)b * N + j2) * nx * nx : nullptr;
            for (int e = lane; e < nu * m; e += 32) {
                const int r = e / m, k = e % m;
                double v = 0.0;
                if (Bj)
                    for (int q = 0; q < nx; ++q)
                        v = fma(__ldg(Bj + q * nu + r), YX[q * cs + k], v);
                T1[r * cs + k] = v;
            }
            for (int e = lane; e < nx * m; e += 32) {
                const int r = e / m, k = e % m;
                double v = 0.0;
                if (Aj)
                    for (int q = 0; q < nx; ++q)
                        v = fma(__ldg(Aj + q * nx + r), YX[q * cs + k], v);
                T2[r * cs + k] = v;
            }
            __syncwarp();
            // L_Q against Yx, pivots 0 .. nx-1
            auto fq = [&](int r, int p) -> double * { return LH + (nu + r) * nux + nu + p; };
            auto gq = [&](int r, int k) -> double * { return YX + r * cs + k; };
            ok = hyh_sweep(fq, gq, nx, nx, m, sg, lane, nullptr, 0);
            if (ok) {
                for (int e = lane; e < nu * m; e += 32)
                    YU[(e / m) * cs + e % m] = T1[(e / m) * cs + e % m];
                for (int e = lane; e < nx * m; e += 32)
                    YX[(e / m) * cs + e % m] = T2[(e / m) * cs + e % m];
                // ALQ <- Acl L_Q^{-T}: X L_Q' = Acl, row by row
                for (int r = lane; r < nx; r += 32)
                    for (int k = 0; k < nx; ++k) {
                        double v = AC[r * nx + k];
                        for (int q = 0; q < k; ++q)
                            v -= CP[r * nux + nu + q] * LH[(nu + k) * nux + nu + q];
                        CP[r * nux + nu + k] = v / LH[(nu + k) * nux + nu + k];
                    }
            }
        } else if (ok) {
            // last stage: L_Q against Yx, keeping the rotations, then the same
            // rotations on (LA, Xi_F = Yl) (hyh_apply)
            auto fq = [&](int r, int p) -> double * { return LH + (nu + r) * nux + nu + p; };
            auto gq = [&](int r, int k) -> double * { return YX + r * cs + k; };
            ok = hyh_sweep(fq, gq, nx, nx, m, sg, lane, RC, nx);
            if (ok) {
                for (int k = 0; k < m; ++k)
                    for (int p = 0; p < nx; ++p) {
                        __syncwarp();
                        const double cc = RC[(size_t)k * nx + p], ss = RC[(size_t)k * nx + p + nx * m];
                        if (cc == 1.0 && ss == 0.0)
                            continue;
                        const bool hyper = sg[k] < 0;
                        for (int r = lane; r < nx; r += 32) {
                            double *fp = CP + r * nux + nu + p, *gp = YL + r * cs + k;
                            const double fu = *fp, gv = *gp;
                            *fp = hyper ? cc * fu - ss * gv : cc * fu + ss * gv;
                            *gp = -ss * fu + cc * gv;
                        }
                    }
                __syncwarp();
                // -Mfwd += Xi_F S Xi_F' (lower elements of the trailing tiles)
                double *tr = a.trail + (size_t)chain * g.NTT * kTileElems;
                for (int e = lane; e < nx * nx; e += 32) {
                    const int r = e / nx, q = e % nx;
                    if (q > r)
                        continue;
                    double v = 0.0;
                    for (int k = 0; k < m; ++k)
                        v += (double)sg[k] * YL[r * cs + k] * YL[q * cs + k];
                    tr[(size_t)tri_index(r / 8, q / 8) * kTileElems + (r % 8) * 8 + q % 8] += v;
                }
            }
        }
        if (!ok) {
            if (lane == 0)
                a.breakdown[blockIdx.x] = 1;
            return;
        }
        __syncwarp();
        // ---- write the stage back -------------------------------------------
        for (int e = lane; e < nux * nux; e += 32) {
            const int r = e / nux, k = e % nux;
            if (k <= r)
                *tile_el(g, st, r, k) = LH[e];
        }
        for (int e = lane; e < nx * nux; e += 32)
            *tile_el(g, st, top + e / nux, e % nux) = CP[e];
        __syncwarp();
    }
}

} // namespace

size_t update_smem_bytes(int nx, int nu, int cap) { return (size_t)Lay(nx, nu, cap).total * sizeof(double); }

bool launch_update_columns(cudaStream_t st, const UpdateArgs &a) {
    const size_t smem = update_smem_bytes(a.g.nx, a.g.nu, a.cap);
    if (smem > 227 * 1024)
        return false;
    static DeviceOnce once;
    once_per_device(once, [] {
        return cudaFuncSetAttribute(update_columns_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    update_columns_kernel<<<a.n, 32, smem, st>>>(a);
    return true;
}

} // namespace cyqb
