// Back substitution, compile-time (nu, nx) warp-per-chain fast path for the
// BASELINE shapes (nux <= 32, nx <= 32); same algorithm and output as
// backsub.cu (kkt_solve.cpp:185-307):
//   y_s   = [u'; x']_s - [LB ALQ]_s' lam_f
//   s = n-1:  x_s += L_Q^{-1} lam_b                      (T' lam_b)
//   s < n-1:  w  = -wl_s - ALQ_s' lam_f,  t = w - L_Q' (BA_{s+1} z_{s+1}),
//             lam^{j(s+1)} = -L_Q t,   x_s -= t
//   z_s   = LH_s^{-T} y_s
// Lane k owns vector entry k; the stage's stored pivot tiles, y, wl and
// BA_{s+1} are staged with cp.async (16-byte granules) one stage ahead into
// a per-warp double buffer; all tile addressing is compile-time except the
// lane's own column.
#include "kernels.h"
#include "riccati_common.cuh"

#include <cstdlib>

namespace cyqb {

using namespace cyqb::ric;

namespace {

template <int NU, int NX> struct BS {
    using S = Shp<NU, NX>;
    // shared-memory strides chosen for conflict-free lane access: tiles at a
    // 72-double stride (a row of consecutive tiles, 8 lanes each, lands on
    // disjoint banks), B and A rows at odd strides (lane i walking row i)
    // (measured: config 4 shape 8.47 -> 5.88 ms per step; at the config-1
    // shape the padded layout was neutral-to-slower, so it keeps the dense one)
    static constexpr bool PAD = NU * NX <= 128;
    static constexpr int TS = PAD ? kTileElems + 8 : kTileElems;
    static constexpr int BS_ = PAD ? (NU | 1) : NU, AS_ = PAD ? (NX | 1) : NX;
    // GBA shapes stage only the pivot-block tiles; the coupling rows (read
    // once, by y -= [LB ALQ]' lam_f) come straight from global memory
    static constexpr bool GBA_ = !PAD && S::NUX <= 32 && NX <= 32; // measured slower for the small (PAD) shapes
    static constexpr int NSTG = GBA_ ? S::CT * (S::CT + 1) / 2 : S::NPT;
    static constexpr int TILES = NSTG * TS;
    static constexpr int OFF_Y = TILES, OFF_WL = OFF_Y + ((S::NUX + 1) & ~1);
    // GBA: [B A]_{s+1} read straight from global (coalesced rows, lane =
    // column, butterfly reduce-scatter) instead of staged: 4.8 KB less shared
    // memory per warp at the config-1 shape -> 16 instead of 12 resident warps
    static constexpr bool GBA = GBA_;
    static constexpr int OFF_B = OFF_WL + ((NX + 1) & ~1);
    static constexpr int OFF_A = OFF_B + (GBA ? 0 : ((NX * BS_ + 1) & ~1));
    static constexpr int BUF = OFF_A + (GBA ? 0 : ((NX * AS_ + 1) & ~1));
    static constexpr int VEC = 64; // z (nux), lf/lb scratch
    // single buffer: more resident warps hide the loads (a double buffer
    // was measured slower at both the config-1 and config-4 shapes)
    static constexpr int NBUF = 1;
    static constexpr int PER_WARP = NBUF * BUF + VEC;
    // stored-tile offset of panel entry (r, col), r/col compile-time or not
    // the same entry in the global factor (dense 64-double tile stride)
    __host__ __device__ static constexpr int gat(int r, int col) {
        return ((r / 8) < S::CT ? S::T(r / 8, col / 8)
                                : S::CT * (S::CT + 1) / 2 + (r / 8 - S::CT) * S::CT + col / 8) *
                   kTileElems +
               (r % 8) * 8 + col % 8;
    }
    __host__ __device__ static constexpr int at(int r, int col) {
        return ((r / 8) < S::CT ? S::T(r / 8, col / 8)
                                : S::CT * (S::CT + 1) / 2 + (r / 8 - S::CT) * S::CT + col / 8) *
                   TS +
               (r % 8) * 8 + col % 8;
    }
};

template <int NU, int NX>
__device__ __forceinline__ void bs_stage(const BacksubArgs &a, double *buf, size_t chain, int b,
                                         int c, int s, int lane) {
    using S = Shp<NU, NX>;
    using L = BS<NU, NX>;
    const Geo &g = a.g;
    const int n = g.n, N = g.N;
    {
        const double *src = a.fac + (chain * n + s) * S::NPT * kTileElems;
        if constexpr (!L::PAD) {
            wcopy<L::TILES, 0>(buf, src, lane); // (GBA: the pivot-block tiles only)
        } else {
#pragma unroll
            for (int t = 0; t < L::NSTG; ++t)
                cp16(buf + t * L::TS + 2 * lane, src + t * kTileElems + 2 * lane);
        }
    }
    wcopy<S::NUX, 0>(buf + L::OFF_Y, a.y + (chain * n + s) * S::NUX, lane);
    if (s + 1 < n) {
        wcopy<NX, 0>(buf + L::OFF_WL, a.wl + (chain * n + s) * NX, lane);
        const int j1 = g.stage_of(c, s + 1);
        const bool in = j1 < N;
        const double *Bs = in ? a.p.B + ((size_t)b * N + j1) * NX * NU : nullptr;
        const double *As = (in && j1 != 0) ? a.p.A + ((size_t)b * N + j1) * NX * NX : nullptr;
        if constexpr (L::GBA) {
            (void)Bs;
            (void)As;
        } else if constexpr (!L::PAD) {
            wcopy<NX * NU, 0>(buf + L::OFF_B, Bs, lane);
            wcopy<NX * NX, 0>(buf + L::OFF_A, As, lane);
        } else {
#pragma unroll
            for (int e = lane; e < NX * NU; e += 32) {
                double *d = buf + L::OFF_B + (e / NU) * L::BS_ + e % NU;
                if (Bs)
                    cp8(d, Bs + e);
                else
                    *d = 0.0;
            }
#pragma unroll
            for (int e = lane; e < NX * NX; e += 32) {
                double *d = buf + L::OFF_A + (e / NX) * L::AS_ + e % NX;
                if (As)
                    cp8(d, As + e);
                else
                    *d = 0.0;
            }
        }
    }
    cp_commit();
}

} // namespace

template <int NU, int NX, int WPB>
__global__ void __launch_bounds__(32 * WPB) backsub_warp_kernel(BacksubArgs a) {
    using S = Shp<NU, NX>;
    using L = BS<NU, NX>;
    constexpr int NUX = S::NUX, TOP = S::TOP;
    extern __shared__ __align__(16) double sm[];
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const size_t chain = (size_t)blockIdx.x * WPB + wib;
    griddep_wait(); // the Schur kernel's multipliers
    if (chain >= (size_t)g.batch * g.P)
        return;
    const int b = (int)(chain / g.P), c = (int)(chain % g.P), n = g.n;
    double *base = sm + (size_t)wib * L::PER_WARP;
    double *bufs[2] = {base, base + (L::NBUF > 1 ? L::BUF : 0)};
    double *z = base + L::NBUF * L::BUF; // nux: z_{s+1}
    double *lf = z + 32;           // nx: lam_f (smem broadcast)

    const double lfk = lane < NX ? a.lamc[((size_t)b * g.P + c) * NX + lane] : 0.0;
    const double lbk = lane < NX ? a.lamc[((size_t)b * g.P + (c - 1 + g.P) % g.P) * NX + lane] : 0.0;
    if (lane < NX)
        lf[lane] = lfk;
    bs_stage<NU, NX>(a, bufs[0], chain, b, c, n - 1, lane);

    for (int s = n - 1; s >= 0; --s) {
        const double *buf = bufs[(n - 1 - s) & 1];
        const int k = lane; // this lane's entry of the nux-vector
        // y_k -= ([LB ALQ]' lam_f)_k: GBA shapes read the coupling rows from
        // global memory, issued before the wait for the staged pivot tiles
        double gk = 0.0;
        if constexpr (L::GBA) {
            const double *gfac = a.fac + (chain * n + s) * S::NPT * kTileElems;
#pragma unroll
            for (int q = 0; q < NX; ++q)
                gk += (k < NUX ? __ldg(gfac + L::gat(TOP + q, 0) + (k / 8) * kTileElems + k % 8) : 0.0) * lf[q];
        }
        if (L::NBUF > 1 && s > 0) {
            bs_stage<NU, NX>(a, bufs[(n - s) & 1], chain, b, c, s - 1, lane);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncwarp();
        const int j = g.stage_of(c, s), xi = g.x_index_of(c, s);
        // idg_k = 1 / LH_kk
        if constexpr (!L::GBA) {
#pragma unroll
            for (int q = 0; q < NX; ++q)
                gk += (k < NUX ? buf[L::at(TOP + q, 0) + (k / 8) * L::TS + k % 8] : 0.0) * lf[q];
        }
        double Y = (k < NUX) ? buf[L::OFF_Y + (k < NUX ? k : 0)] - gk : 0.0;
        const double idg = (k < NUX) ? 1.0 / buf[L::at(k < NUX ? k : 0, k < NUX ? k : 0)] : 0.0;
        if (s == n - 1) {
            // x += L_Q^{-1} lam_b  (T' lam_b, kkt_solve.cpp:218-223); lane i holds t_i
            double t = (lane < NX) ? lbk : 0.0;
#pragma unroll
            for (int kk = 0; kk < NX; ++kk) {
                const double idk = __shfl_sync(0xffffffffu, idg, NU + kk);
                const double xk = __shfl_sync(0xffffffffu, t, kk) * idk;
                if (lane == kk)
                    t = xk;
                else if (lane > kk && lane < NX)
                    t -= buf[L::at(NU + (lane < NX ? lane : 0), NU + kk)] * xk;
            }
            // move t_i (lane i) to Y_{nu+i} (lane nu+i)
            const double ti = __shfl_sync(0xffffffffu, t, (lane - NU) & 31);
            if (k >= NU && k < NUX)
                Y += ti;
        } else {
            const int j1 = g.stage_of(c, s + 1);
            // w_i = -wl_i - g_{nu+i}; zn_i = (B z_u + A z_x)_i ; lane i
            const double gx = __shfl_sync(0xffffffffu, gk, (lane + NU) & 31);
            double zn = 0.0;
            if constexpr (L::GBA) {
                // lane = column of [B A] (k < nux); row partials, then a
                // butterfly reduce-scatter leaves row i in lane i
                const bool in1 = j1 < g.N;
                const double *Bg = a.p.B + ((size_t)b * g.N + (in1 ? j1 : 0)) * NX * NU;
                const double *Ag = a.p.A + ((size_t)b * g.N + (in1 ? j1 : 0)) * NX * NX;
                const double zk = k < NUX ? z[k] : 0.0;
                const bool useA = in1 && j1 != 0;
                double pr[32];
#pragma unroll
                for (int r = 0; r < 32; ++r) {
                    double v = 0.0;
                    if (r < NX && in1) {
                        if (k < NU)
                            v = __ldg(Bg + r * NU + k);
                        else if (k < NUX && useA)
                            v = __ldg(Ag + r * NX + (k - NU));
                    }
                    pr[r] = v * zk;
                }
#pragma unroll
                for (int h = 16; h >= 1; h >>= 1) {
#pragma unroll
                    for (int r = 0; r < h; ++r) {
                        const bool up = (lane & h) != 0;
                        const double send = up ? pr[r] : pr[r + h];
                        const double keep = up ? pr[r + h] : pr[r];
                        pr[r] = keep + __shfl_xor_sync(0xffffffffu, send, h);
                    }
                }
                zn = lane < NX ? pr[0] : 0.0;
            } else if (lane < NX) {
#pragma unroll
                for (int q = 0; q < NU; ++q)
                    zn += buf[L::OFF_B + lane * L::BS_ + q] * z[q];
#pragma unroll
                for (int q = 0; q < NX; ++q)
                    zn += buf[L::OFF_A + lane * L::AS_ + q] * z[NU + q];
            }
            const double w = (lane < NX) ? -buf[L::OFF_WL + (lane < NX ? lane : 0)] - gx : 0.0;
            // t_i = w_i - sum_{k >= i} L_Q[k][i] zn_k
            double t = w;
#pragma unroll
            for (int kk = 0; kk < NX; ++kk) {
                const double znk = __shfl_sync(0xffffffffu, zn, kk);
                if (lane <= kk && lane < NX)
                    t -= buf[L::at(NU + kk, NU + (lane < NX ? lane : 0))] * znk;
            }
            // lam^{j(s+1)}_i = -sum_{k <= i} L_Q[i][k] t_k
            // (lane i walks its row from column i mod NX on: the per-lane
            // skew makes the column reads of one step hit distinct banks)
            double lam = 0.0;
#pragma unroll
            for (int m = 0; m < NX; ++m) {
                const int kk = L::PAD ? (lane + m) % NX : m;
                const double tk = __shfl_sync(0xffffffffu, t, kk);
                if (lane >= kk && lane < NX)
                    lam -= buf[L::at(NU + (lane < NX ? lane : 0), NU + kk)] * tk;
            }
            if (lane < NX && j1 < g.N)
                a.sol.lam[((size_t)b * g.N + j1) * NX + lane] = lam;
            const double ti = __shfl_sync(0xffffffffu, t, (lane - NU) & 31);
            if (k >= NU && k < NUX)
                Y -= ti;
        }
        // z = LH^{-T} Y : back substitution over the top block, lane k owns Y_k
#pragma unroll
        for (int r = NUX - 1; r >= 0; --r) {
            const double zr = __shfl_sync(0xffffffffu, Y * idg, r);
            if (lane == r)
                Y = zr;
            else if (lane < r)
                Y -= buf[L::at(r, 0) + (lane / 8) * L::TS + lane % 8] * zr;
        }
        __syncwarp();
        if (L::NBUF == 1 && s > 0) { // buffer consumed: fetch stage s-1
            __syncwarp();
            bs_stage<NU, NX>(a, bufs[0], chain, b, c, s - 1, lane);
        }
        if (k < NUX) {
            z[k] = Y;
            if (k < NU) {
                if (j < g.N)
                    a.sol.u[((size_t)b * g.N + j) * NU + k] = Y;
            } else if (xi <= g.N) {
                a.sol.x[((size_t)b * (g.N + 1) + xi) * NX + (k - NU)] = Y;
            }
        }
        __syncwarp();
    }
    if (c == 0 && lane < NX)
        a.sol.x[(size_t)b * (g.N + 1) * NX + lane] = __ldg(a.p.x_init + (size_t)b * NX + lane);
}

namespace {
template <int NU, int NX, int WPB> bool launch_b(const Geo &g, cudaStream_t st, const BacksubArgs &ba) {
    if (g.nu != NU || g.nx != NX)
        return false;
    const size_t smem = (size_t)WPB * BS<NU, NX>::PER_WARP * sizeof(double);
    static DeviceOnce once;
    once_per_device(once, [&] { return cudaFuncSetAttribute(backsub_warp_kernel<NU, NX, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    const int chains = g.batch * g.P;
    launch_pdl(backsub_warp_kernel<NU, NX, WPB>, dim3((chains + WPB - 1) / WPB), dim3(32 * WPB), smem, st, 1, ba);
    return true;
}
} // namespace

bool launch_backsub_warp(const Geo &g, cudaStream_t st, const BacksubArgs &ba) {
    return launch_b<10, 20, 4>(g, st, ba) || launch_b<8, 16, 4>(g, st, ba) ||
           launch_b<4, 12, 4>(g, st, ba) || launch_b<5, 10, 4>(g, st, ba);
}

} // namespace cyqb
