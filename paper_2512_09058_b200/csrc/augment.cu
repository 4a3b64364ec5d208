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
#include "riccati_common.cuh" // cp8 / cp_commit / cp_wait

#include <algorithm>
#include <string>

namespace cyqb {

namespace {

constexpr int kAugWarps = 8;
constexpr int kAugMaxY = 64, kAugMaxUX = 64; // ny, nu + nx limits (shared memory)

// out[i] = in[i] + G(row(i), col(i)) (+ gamma_inv on the diagonal), i over a
// contiguous row-major block of `rows x cols`, 16-byte coalesced when aligned
__device__ __forceinline__ void add_block(double *out, const double *in, const double *G, int ldg,
                                          int r0, int c0, int rows, int cols, double dg, int lane) {
    const int cnt = rows * cols;
    const bool al = (((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(in)) & 15) == 0) &&
                    (cols % 2 == 0);
    if (al) {
#pragma unroll 4
        for (int e = 2 * lane; e < cnt; e += 64) {
            const int r = e / cols, c = e % cols;
            const double2 v = __ldg(reinterpret_cast<const double2 *>(in + e));
            double2 o;
            o.x = v.x + G[(r0 + r) * ldg + c0 + c] + (r == c ? dg : 0.0);
            o.y = v.y + G[(r0 + r) * ldg + c0 + c + 1] + (r == c + 1 ? dg : 0.0);
            *reinterpret_cast<double2 *>(out + e) = o;
        }
    } else {
        for (int e = lane; e < cnt; e += 32) {
            const int r = e / cols, c = e % cols;
            out[e] = __ldg(in + e) + G[(r0 + r) * ldg + c0 + c] + (r == c ? dg : 0.0);
        }
    }
}

// CNU / CNX / CNY > 0: compile-time shape (all index arithmetic folds);
// 0: runtime shape
template <int CNU, int CNX, int CNY>
__global__ void __launch_bounds__(32 * kAugWarps) augment_kernel(
    int batch, int N, int nx_, int nu_, int ny_, const double *R, const double *S, const double *Q,
    const double *D, const double *E, const double *sig, double gamma_inv, double *Ro, double *So,
    double *Qo, int per_warp) {
    const int nx = CNX > 0 ? CNX : nx_, nu = CNU > 0 ? CNU : nu_, ny = CNY > 0 ? CNY : ny_;
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long task = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
    if (task >= (long long)batch * (N + 1))
        return;
    const int b = (int)(task / (N + 1)), j = (int)(task % (N + 1));
    const int nux = nu + nx, TT = (nux + 7) / 8, KS = (ny + 3) / 4;
    const int ldc = 8 * TT;                 // padded row length of [D C] and G
    double *Cm = sm + (size_t)wib * per_warp;
    double *sg = Cm + (size_t)4 * KS * ldc; // 4 KS
    double *G = sg + 4 * KS;                // ldc x ldc (symmetric, both triangles)
    const bool has_d = j < N;
    // stage [D_j C_j] rows and σ_j with cp.async (every copy in flight at
    // once); zero padding rows / columns written directly
    {
        const double *Dj = D + ((size_t)b * N + j) * ny * nu;
        const double *Ej = E + ((size_t)b * (N + 1) + j) * ny * nx;
#pragma unroll
        for (int e = lane; e < 4 * KS * ldc; e += 32) {
            const int i = e / ldc, m = e % ldc;
            if (i < ny && m < nu && has_d)
                ric::cp8(Cm + e, Dj + i * nu + m);
            else if (i < ny && m >= nu && m < nux)
                ric::cp8(Cm + e, Ej + i * nx + (m - nu));
            else
                Cm[e] = 0.0;
        }
        for (int i = lane; i < 4 * KS; i += 32) {
            if (i < ny)
                ric::cp8(sg + i, sig + ((size_t)b * (N + 1) + j) * ny + i);
            else
                sg[i] = 0.0;
        }
        ric::cp_commit();
        ric::cp_wait<0>();
    }
    __syncwarp();
    // G = [D C]' diag(σ) [D C] on DMMA tiles (lower tiles, mirrored into smem)
    const int rq = lane >> 2, cq = 2 * (lane & 3), kq = lane & 3;
#pragma unroll
    for (int ti = 0; ti < TT; ++ti)
#pragma unroll
        for (int tj = 0; tj <= ti; ++tj) {
            Frag acc{0.0, 0.0};
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int k = 4 * ks + kq;
                dmma(acc, sg[k] * Cm[k * ldc + 8 * ti + rq], Cm[k * ldc + 8 * tj + rq]);
            }
            // every entry written once, from its lower-triangle value (the
            // upper half of a diagonal tile differs in rounding: deterministic)
            const int r = 8 * ti + rq, c = 8 * tj + cq;
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (c + h <= r) {
                    const double v = h ? acc.b : acc.a;
                    G[r * ldc + c + h] = v;
                    G[(c + h) * ldc + r] = v;
                }
        }
    __syncwarp();
    // coalesced read-add-write of the stage's R, S, Q blocks
    if (has_d) {
        const size_t oR = ((size_t)b * N + j) * nu * nu, oS = ((size_t)b * N + j) * nu * nx;
        add_block(Ro + oR, R + oR, G, ldc, 0, 0, nu, nu, gamma_inv, lane);
        add_block(So + oS, S + oS, G, ldc, 0, nu, nu, nx, 0.0, lane);
    }
    const size_t oQ = ((size_t)b * (N + 1) + j) * nx * nx;
    add_block(Qo + oQ, Q + oQ, G, ldc, nu, nu, nx, nx, j >= 1 ? gamma_inv : 0.0, lane);
}

} // namespace

bool launch_augment(cudaStream_t st, int batch, int N, int nx, int nu, int ny, const double *R,
                    const double *S, const double *Q, const double *D, const double *C,
                    const double *sigma, double gamma_inv, double *R_out, double *S_out,
                    double *Q_out) {
    if (ny < 1 || ny > kAugMaxY || nx + nu > kAugMaxUX)
        return false;
    const int nux = nx + nu, ldc = 8 * ((nux + 7) / 8), ks = (ny + 3) / 4;
    const int per_warp = (4 * ks * ldc + 4 * ks + ldc * ldc + 1) & ~1;
    // warps per CTA: as many (up to 8) as shared memory holds -- the largest
    // shapes (nx + nu = 64, ny = 64: 66 KB per warp) run 3 per CTA
    constexpr size_t kSmemCap = 200 * 1024;
    const size_t per_warp_bytes = (size_t)per_warp * sizeof(double);
    const int nw = (int)std::min<size_t>(kAugWarps, kSmemCap / per_warp_bytes);
    if (nw < 1)
        return false;
    const long long tasks = (long long)batch * (N + 1);
    const int grid = (int)((tasks + nw - 1) / nw);
    const size_t smem = (size_t)nw * per_warp_bytes;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
        kern<<<grid, 32 * nw, smem, st>>>(batch, N, nx, nu, ny, R, S, Q, D, C, sigma, gamma_inv,
                                         R_out, S_out, Q_out, per_warp);
    };
    if (nu == 8 && nx == 16 && ny == 24)
        go(augment_kernel<8, 16, 24>); // BASELINE config 4
    else
        go(augment_kernel<0, 0, 0>);
    return true;
}

} // namespace cyqb
