// Augmented-Lagrangian gradients of the QPALM inner loop, batched
// (the step before the Newton system):
//   qpalm::eval_al_gradients (qpalm.cpp:106-165), with stage_constraint
//   (qpalm.cpp:39-53): per instance b and stage j = 0..N
//     g      = C_j x_j + D_j u_j            (j = N: C_term x_N)
//     yhat   = y + Σ (g - clamp(g + y / Σ, bl, bu))
//     ru_j   = r_j + R_j u_j + S_j x_j + D_j' yhat + γ⁻¹ (u_j - ubar_j)   (j < N)
//     cres_j = f_j + A_j x_j + B_j u_j - x_{j+1}                          (j < N)
//     qx_j   = q_j + Q_j x_j + S_j' u_j + C_j' yhat + γ⁻¹ (x_j - xbar_j)  (j >= 1;
//              j = N: q_N + Q_N x_N + C_term' yhat + γ⁻¹ (...))
// One warp per (instance, stage); u_j, x_j and yhat staged in shared memory,
// one output row per lane, each row a sequential fused multiply-add sum in
// the reference's order (its axpy accumulates row by row, qpalm.cpp:11-23).
// HBM-bound: every stage block of the problem is read once.
#include "kernels.h"

namespace cyqb {

namespace {

constexpr int kGradWarps = 4;

__global__ void __launch_bounds__(32 * kGradWarps) al_gradients_kernel(GradArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int N = a.N, nx = a.nx, nu = a.nu, ny = a.ny, lane = threadIdx.x & 31;
    const long long item = (long long)blockIdx.x * kGradWarps + (threadIdx.x >> 5);
    if (item >= (long long)a.batch * (N + 1))
        return;
    const int b = (int)(item / (N + 1)), j = (int)(item % (N + 1));
    double *us = sm + (size_t)(threadIdx.x >> 5) * (nu + nx + ny), *xs = us + nu, *yh = xs + nx;
    const bool st = j < N; // a stage with an input (else: the terminal)
    const size_t jb = (size_t)b * N + j, jx = (size_t)b * (N + 1) + j;
    for (int i = lane; i < nu; i += 32)
        us[i] = st ? a.u[jb * nu + i] : 0.0;
    for (int i = lane; i < nx; i += 32)
        xs[i] = a.x[jx * nx + i];
    __syncwarp();
    // yhat (qpalm.cpp:122-131)
    const double *Cj = a.C + jx * ny * nx, *Dj = st ? a.D + jb * ny * nu : nullptr;
    for (int i = lane; i < ny; i += 32) {
        double s1 = 0.0;
        for (int k = 0; k < nx; ++k)
            s1 = fma(__ldg(Cj + (size_t)i * nx + k), xs[k], s1);
        double gc = 0.0 + s1;
        if (st) {
            double s2 = 0.0;
            for (int k = 0; k < nu; ++k)
                s2 = fma(__ldg(Dj + (size_t)i * nu + k), us[k], s2);
            gc += s2;
        }
        const size_t o = jx * ny + i;
        const double y = __ldg(a.y + o), sg = __ldg(a.sigma + o);
        const double w = gc + y / sg;
        const double pr = fmin(fmax(w, __ldg(a.bl + o)), __ldg(a.bu + o));
        const double v = y + sg * (gc - pr);
        yh[i] = v;
        a.yhat[o] = v;
    }
    __syncwarp();
    if (st) {
        const double *Rj = a.R + jb * nu * nu, *Sj = a.S + jb * nu * nx;
        for (int i = lane; i < nu; i += 32) { // ru (qpalm.cpp:133-141)
            double ru = __ldg(a.r + jb * nu + i), s = 0.0;
            for (int k = 0; k < nu; ++k)
                s = fma(__ldg(Rj + (size_t)i * nu + k), us[k], s);
            ru += s;
            s = 0.0;
            for (int k = 0; k < nx; ++k)
                s = fma(__ldg(Sj + (size_t)i * nx + k), xs[k], s);
            ru += s;
            s = 0.0;
            for (int k = 0; k < ny; ++k)
                s = fma(__ldg(Dj + (size_t)k * nu + i), yh[k], s);
            ru += s;
            ru += a.gamma_inv * (us[i] - __ldg(a.ubar + jb * nu + i));
            a.ru[jb * nu + i] = ru;
        }
        const double *Aj = a.A + jb * nx * nx, *Bj = a.B + jb * nx * nu;
        for (int i = lane; i < nx; i += 32) { // dynamics residual (qpalm.cpp:142-148)
            double c = __ldg(a.f + jb * nx + i), s = 0.0;
            for (int k = 0; k < nx; ++k)
                s = fma(__ldg(Aj + (size_t)i * nx + k), xs[k], s);
            c += s;
            s = 0.0;
            for (int k = 0; k < nu; ++k)
                s = fma(__ldg(Bj + (size_t)i * nu + k), us[k], s);
            c += s;
            c -= a.x[(jx + 1) * nx + i];
            a.cres[jb * nx + i] = c;
        }
    }
    const double *Qj = a.Q + jx * nx * nx, *Sj = st ? a.S + jb * nu * nx : nullptr;
    for (int i = lane; i < nx; i += 32) { // qx (qpalm.cpp:150-163); qx[0] unused
        if (j == 0) {
            a.qx[jx * nx + i] = 0.0;
            continue;
        }
        double q = __ldg(a.q + jx * nx + i), s = 0.0;
        for (int k = 0; k < nx; ++k)
            s = fma(__ldg(Qj + (size_t)i * nx + k), xs[k], s);
        q += s;
        if (st) {
            s = 0.0;
            for (int k = 0; k < nu; ++k)
                s = fma(__ldg(Sj + (size_t)k * nx + i), us[k], s);
            q += s;
        }
        s = 0.0;
        for (int k = 0; k < ny; ++k)
            s = fma(__ldg(Cj + (size_t)k * nx + i), yh[k], s);
        q += s;
        q += a.gamma_inv * (xs[i] - __ldg(a.xbar + jx * nx + i));
        a.qx[jx * nx + i] = q;
    }
}

} // namespace

bool launch_al_gradients(cudaStream_t st, const GradArgs &a) {
    const size_t smem = (size_t)kGradWarps * (a.nu + a.nx + a.ny) * sizeof(double);
    if (smem > 48 * 1024)
        return false;
    const long long items = (long long)a.batch * (a.N + 1);
    al_gradients_kernel<<<(unsigned)((items + kGradWarps - 1) / kGradWarps), 32 * kGradWarps, smem, st>>>(a);
    return true;
}

} // namespace cyqb
