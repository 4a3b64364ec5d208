// Newton-system assembly for the QPALM inner loop (BASELINE config 4, SURVEY
// §8f row f2): restates the equality part of qpalm::assemble_newton
// (/root/reference/proj/src/qpalm.cpp:167-225) for a batch of instances,
//   R_j + D_j' Σ_j D_j + γ⁻¹ I,   S_j + D_j' Σ_j C_j,   Q_j + C_j' Σ_j C_j + γ⁻¹ I
// (stage 0 included, as synth.qpalm_sequence / the reference's
// factorization never read S_0, Q_0; the terminal Q_N takes C_N' Σ_N C_N),
// with the active set folded into Σ (σ = 0 for inactive rows).
//
// One warp per (instance, stage): [D_j C_j] (ny x nux) and σ_j are staged in
// shared memory (coalesced), G = [D C]' diag(σ) [D C] is formed on 8x8 FP64
// DMMA tiles (A operand = σ-scaled transposed rows, B operand = rows; the
// lower tiles only), and the augmented R / S / Q blocks are written
// row-major (both triangles) next to the unchanged A, B, f, r, q. Memory
// bound: it streams D, C, σ and the base Hessians once.
#include "kernels.h"

#include <string>

namespace cyqb {

namespace {

constexpr int kAugWarps = 4;
constexpr int kAugMaxY = 64, kAugMaxUX = 64; // ny, nu + nx limits (shared memory)

__global__ void __launch_bounds__(32 * kAugWarps) augment_kernel(
    int batch, int N, int nx, int nu, int ny, const double *R, const double *S, const double *Q,
    const double *D, const double *E, const double *sig, double gamma_inv, double *Ro, double *So,
    double *Qo, int per_warp) {
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long task = (long long)blockIdx.x * kAugWarps + wib;
    if (task >= (long long)batch * (N + 1))
        return;
    const int b = (int)(task / (N + 1)), j = (int)(task % (N + 1));
    const int nux = nu + nx, TT = (nux + 7) / 8, KS = (ny + 3) / 4;
    const int ldc = 8 * TT;                 // padded row length of [D C]
    double *Cm = sm + (size_t)wib * per_warp;
    double *sg = Cm + (size_t)4 * KS * ldc; // ny (padded to 4 KS)
    const bool has_d = j < N;
    // stage [D_j C_j] rows (zero padding rows / columns) and σ_j
    for (int e = lane; e < 4 * KS * ldc; e += 32) {
        const int i = e / ldc, m = e % ldc;
        double v = 0.0;
        if (i < ny && m < nux) {
            if (m < nu)
                v = has_d ? __ldg(D + (((size_t)b * N + j) * ny + i) * nu + m) : 0.0;
            else
                v = __ldg(E + (((size_t)b * (N + 1) + j) * ny + i) * nx + (m - nu));
        }
        Cm[e] = v;
    }
    for (int i = lane; i < 4 * KS; i += 32)
        sg[i] = i < ny ? __ldg(sig + ((size_t)b * (N + 1) + j) * ny + i) : 0.0;
    __syncwarp();
    const int rq = lane >> 2, cq = 2 * (lane & 3), kq = lane & 3;
    for (int ti = 0; ti < TT; ++ti)
        for (int tj = 0; tj <= ti; ++tj) {
            Frag acc{0.0, 0.0};
            for (int ks = 0; ks < KS; ++ks) {
                const int k = 4 * ks + kq;
                const double av = sg[k] * Cm[k * ldc + 8 * ti + rq]; // (σ C)'(m, k)
                const double bv = Cm[k * ldc + 8 * tj + rq];         // C(k, n)
                dmma(acc, av, bv);
            }
            // scatter G(r, c) (and its mirror) into R / S / Q with the base values
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = 8 * ti + rq, c = 8 * tj + cq + h;
                const double gv = h ? acc.b : acc.a;
                if (r >= nux || c >= nux || c > r)
                    continue;
                if (r < nu) { // R (j < N)
                    if (has_d) {
                        const size_t o = ((size_t)b * N + j) * nu * nu;
                        const double dg = (r == c) ? gamma_inv : 0.0;
                        Ro[o + r * nu + c] = __ldg(R + o + r * nu + c) + gv + dg;
                        if (r != c)
                            Ro[o + c * nu + r] = __ldg(R + o + c * nu + r) + gv;
                    }
                } else if (c < nu) { // S(c, r - nu) = G(c, r) = G(r, c)
                    if (has_d) {
                        const size_t o = ((size_t)b * N + j) * nu * nx;
                        So[o + c * nx + (r - nu)] = __ldg(S + o + c * nx + (r - nu)) + gv;
                    }
                } else { // Q
                    const int qr = r - nu, qc = c - nu;
                    const size_t o = ((size_t)b * (N + 1) + j) * nx * nx;
                    const double dg = (qr == qc && j >= 1) ? gamma_inv : 0.0;
                    Qo[o + qr * nx + qc] = __ldg(Q + o + qr * nx + qc) + gv + dg;
                    if (qr != qc)
                        Qo[o + qc * nx + qr] = __ldg(Q + o + qc * nx + qr) + gv;
                }
            }
        }
}

} // namespace

bool launch_augment(cudaStream_t st, int batch, int N, int nx, int nu, int ny, const double *R,
                    const double *S, const double *Q, const double *D, const double *C,
                    const double *sigma, double gamma_inv, double *R_out, double *S_out,
                    double *Q_out) {
    if (ny < 1 || ny > kAugMaxY || nx + nu > kAugMaxUX)
        return false;
    const int nux = nx + nu, ldc = 8 * ((nux + 7) / 8), ks = (ny + 3) / 4;
    const int per_warp = (4 * ks * ldc + 4 * ks + 1) & ~1;
    const long long tasks = (long long)batch * (N + 1);
    const int grid = (int)((tasks + kAugWarps - 1) / kAugWarps);
    const size_t smem = (size_t)kAugWarps * per_warp * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(augment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    augment_kernel<<<grid, 32 * kAugWarps, smem, st>>>(batch, N, nx, nu, ny, R, S, Q, D, C, sigma,
                                                       gamma_inv, R_out, S_out, Q_out, per_warp);
    return true;
}

} // namespace cyqb
