// Shared compile-time panel geometry and cp.async stage staging of the
// warp-level stage-panel Riccati kernels (riccati_warp.cu, riccati_pc.cu):
// R and Q straight into a tile-ordered image of the panel's pivot block,
// [B A] as one padded row-major block, S / [r; q] / f as plain vectors, and
// the compact, permuted x-column positions of W (see riccati_warp.cu).
#pragma once

#include "kkt_common.cuh"
#include "kernels.h"
#include "riccati_common.cuh"

#include <cstdint>

namespace cyqb {
namespace ric {

template <int NU, int NX> struct PanelShape {
    using S = Shp<NU, NX>;
    static constexpr int NUX = S::NUX, CT = S::CT, BT = S::BT, TT = S::TT, NT = S::NT;
    static constexpr int TOP = S::TOP, RHS = S::RHS, RT = RHS / 8, RR = RHS % 8;
    static constexpr int XT0 = S::XT0, NXT = S::NXT; // panel tile columns holding x columns
    static constexpr int NXF = NX / 8, REM = NX % 8;
    static constexpr bool HALF = REM > 0 && REM <= 4; // remainder on even positions only
    static constexpr int NXC = (NX + 7) / 8;           // compact W tile columns
    static constexpr int KQ = (NX + 3) / 4;            // V k-steps over x rows
    static constexpr int NXR = 4 * KQ;                 // padded x rows (LQ, BA)
    static constexpr int PW = 8 * CT;                  // padded panel width
    static constexpr int NIMG = CT * (CT + 1) / 2;     // image tiles
    // compact position of x-column kk / x-column at position p (-1 = none)
    __host__ __device__ static constexpr int pos(int kk) {
        return kk < 8 * NXF ? kk : 8 * NXF + (HALF ? 2 : 1) * (kk - 8 * NXF);
    }
    __host__ __device__ static constexpr int col_of(int p) {
        return p < 8 * NXF ? p
                           : (HALF ? ((((p - 8 * NXF) & 1) == 0 && (p - 8 * NXF) / 2 < REM)
                                          ? 8 * NXF + (p - 8 * NXF) / 2
                                          : -1)
                                   : ((p - 8 * NXF) < REM ? p : -1));
    }
};

// %laneid through a volatile asm: lane-dependent addresses derived from it
// are recomputed where used instead of being hoisted out of the stage loop
// (and spilled -- the long-scoreboard stalls of a first version)
__device__ __forceinline__ int lane_v() {
    int l;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

__device__ __forceinline__ bool aligned16(const void *p) {
    return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

// H_s: R -> panel (r, c), Q -> panel (NU + r, NU + c) of the tile image
// (lower tiles only), S raw, [r; q] -> imr. Padding stages get R = Q = I,
// S = 0, r = q = 0 (pad_problem, kkt_factor.cpp:27-47).
template <int NU, int NX>
__device__ __forceinline__ void stage_H(const Geo &g, const ProbView &p, int b, int j, int xi,
                                        double *img, double *imr, double *Sb) {
    using S = Shp<NU, NX>;
    const int N = g.N;
    const int lane = lane_v();
    const bool in = j < N, qin = xi <= N;
    auto at = [&](int r, int c) { return img + S::T(r / 8, c / 8) * kTileElems + (r % 8) * 8 + c % 8; };
    const double *Rs = in ? p.R + ((size_t)b * N + j) * NU * NU : nullptr;
    const double *Qs = qin ? p.Q + ((size_t)b * (N + 1) + xi) * NX * NX : nullptr;
    // R
    if (Rs && (NU % 2 == 0) && aligned16(Rs)) {
#pragma unroll
        for (int e = 2 * lane; e < NU * NU; e += 64) {
            const int r = e / NU, c = e % NU;
            if (c / 8 <= r / 8)
                cp16(at(r, c), Rs + e);
        }
    } else {
#pragma unroll
        for (int e = lane; e < NU * NU; e += 32) {
            const int r = e / NU, c = e % NU;
            if (c / 8 <= r / 8) {
                if (Rs)
                    cp8(at(r, c), Rs + e);
                else
                    *at(r, c) = r == c ? 1.0 : 0.0;
            }
        }
    }
    // Q
    if (Qs && (NU % 2 == 0) && (NX % 2 == 0) && aligned16(Qs)) {
#pragma unroll
        for (int e = 2 * lane; e < NX * NX; e += 64) {
            const int r = NU + e / NX, c = NU + e % NX;
            if (c / 8 <= r / 8)
                cp16(at(r, c), Qs + e);
        }
    } else {
#pragma unroll
        for (int e = lane; e < NX * NX; e += 32) {
            const int r = NU + e / NX, c = NU + e % NX;
            if (c / 8 <= r / 8) {
                if (Qs)
                    cp8(at(r, c), Qs + e);
                else
                    *at(r, c) = r == c ? 1.0 : 0.0;
            }
        }
    }
    wcopy<NU * NX, 0>(Sb, in ? p.S + ((size_t)b * N + j) * NU * NX : nullptr, lane);
    const double *rs = p.ru ? p.ru : p.r;
    const double *qs = p.qx ? p.qx : p.q;
    wcopy<NU, 0>(imr, in ? rs + ((size_t)b * N + j) * NU : nullptr, lane);
    wcopy<NX, 0>(imr + NU, qin ? qs + ((size_t)b * (N + 1) + xi) * NX : nullptr, lane);
}

// BA_j = [B A] -> rows of the padded block (A omitted for j = 0, zero for
// padding stages), f -> vector
template <int NU, int NX>
__device__ __forceinline__ void stage_BA(const Geo &g, const ProbView &p, int b, int j, double *ba,
                                         double *fb) {
    using W = PanelShape<NU, NX>;
    const int N = g.N;
    const int lane = lane_v();
    const bool in = j < N;
    const double *Bs = in ? p.B + ((size_t)b * N + j) * NX * NU : nullptr;
    const double *As = (in && j != 0) ? p.A + ((size_t)b * N + j) * NX * NX : nullptr;
    if (Bs && NU % 2 == 0 && aligned16(Bs)) {
#pragma unroll
        for (int e = 2 * lane; e < NX * NU; e += 64)
            cp16(ba + (e / NU) * W::PW + e % NU, Bs + e);
    } else {
#pragma unroll
        for (int e = lane; e < NX * NU; e += 32) {
            double *d = ba + (e / NU) * W::PW + e % NU;
            if (Bs)
                cp8(d, Bs + e);
            else
                *d = 0.0;
        }
    }
    if (As && NU % 2 == 0 && NX % 2 == 0 && aligned16(As)) {
#pragma unroll
        for (int e = 2 * lane; e < NX * NX; e += 64)
            cp16(ba + (e / NX) * W::PW + NU + e % NX, As + e);
    } else {
#pragma unroll
        for (int e = lane; e < NX * NX; e += 32) {
            double *d = ba + (e / NX) * W::PW + NU + e % NX;
            if (As)
                cp8(d, As + e);
            else
                *d = 0.0;
        }
    }
    const double *fs = p.fd ? p.fd : p.f;
    wcopy<NX, 0>(fb, in ? fs + ((size_t)b * N + j) * NX : nullptr, lane);
}

// Per-lane copy plan of the two scattered stagings -- R / Q into the tile
// image (lower tiles only) and [B A] into padded rows -- built once per CTA
// into shared memory: slot k of lane l holds the destination offset (in
// doubles, -1 = none) of source element G (l + 32 k). Staging a stage is then
// one 16-bit shared load and one cp.async per slot instead of the index
// arithmetic of stage_H / stage_BA (~2k cycles per stage at config 0, issued
// on the pivot chain's warp). G = 2 (16-byte copies) when every offset is
// even, else 1.
template <int NU, int NX> struct CopyPlan {
    using S = Shp<NU, NX>;
    using W = PanelShape<NU, NX>;
    static constexpr int G = (NU % 2 == 0 && NX % 2 == 0) ? 2 : 1;
    static constexpr int KR = (NU * NU / G + 31) / 32, KQ = (NX * NX / G + 31) / 32;
    static constexpr int KB = (NX * NU / G + 31) / 32, KA = KQ;
    static constexpr int OR = 0, OQ = KR, OB = OQ + KQ, OA = OB + KB, SLOTS = OA + KA;
    static constexpr int DOUBLES = (SLOTS * 32 * 2 + 15) / 16 * 2; // footprint (even)
    // the R / Q slots only (stage_H_plan), for kernels short of shared memory
    static constexpr int DOUBLES_H = ((KR + KQ) * 32 * 2 + 15) / 16 * 2;
    __device__ static int img_off(int r, int c) {
        return S::T(r / 8, c / 8) * kTileElems + (r % 8) * 8 + c % 8;
    }
    __device__ static void build(short *tab, int lane, bool with_ba = true) {
        for (int k = 0; k < KR; ++k) {
            const int e = G * (lane + 32 * k), r = e / NU, c = e % NU;
            tab[(OR + k) * 32 + lane] = (short)((e < NU * NU && c / 8 <= r / 8) ? img_off(r, c) : -1);
        }
        for (int k = 0; k < KQ; ++k) {
            const int e = G * (lane + 32 * k), r = NU + e / NX, c = NU + e % NX;
            tab[(OQ + k) * 32 + lane] = (short)((e < NX * NX && c / 8 <= r / 8) ? img_off(r, c) : -1);
        }
        if (!with_ba)
            return;
        for (int k = 0; k < KB; ++k) {
            const int e = G * (lane + 32 * k);
            tab[(OB + k) * 32 + lane] = (short)(e < NX * NU ? (e / NU) * W::PW + e % NU : -1);
        }
        for (int k = 0; k < KA; ++k) {
            const int e = G * (lane + 32 * k);
            tab[(OA + k) * 32 + lane] = (short)(e < NX * NX ? (e / NX) * W::PW + NU + e % NX : -1);
        }
    }
    template <int O, int K>
    __device__ static void run(const short *tab, double *dst, const double *src, int lane) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int o = tab[(O + k) * 32 + lane];
            if (o >= 0) {
                if (G == 2)
                    cp16(dst + o, src + 2 * (lane + 32 * k));
                else
                    cp8(dst + o, src + lane + 32 * k);
            }
        }
    }
};

// stage_H / stage_BA through the plan; stages that need fills (padding, A at
// j = 0) or unaligned sources take the general path
template <int NU, int NX>
__device__ __forceinline__ void stage_H_plan(const Geo &g, const ProbView &p, int b, int j, int xi,
                                             double *img, double *imr, double *Sb, const short *tab) {
    using CP = CopyPlan<NU, NX>;
    const int N = g.N;
    const double *Rs = j < N ? p.R + ((size_t)b * N + j) * NU * NU : nullptr;
    const double *Qs = xi <= N ? p.Q + ((size_t)b * (N + 1) + xi) * NX * NX : nullptr;
    if (!Rs || !Qs || (CP::G == 2 && !(aligned16(Rs) && aligned16(Qs)))) {
        stage_H<NU, NX>(g, p, b, j, xi, img, imr, Sb);
        return;
    }
    const int lane = lane_v();
    CP::template run<CP::OR, CP::KR>(tab, img, Rs, lane);
    CP::template run<CP::OQ, CP::KQ>(tab, img, Qs, lane);
    wcopy<NU * NX, 0>(Sb, p.S + ((size_t)b * N + j) * NU * NX, lane);
    const double *rs = p.ru ? p.ru : p.r;
    const double *qs = p.qx ? p.qx : p.q;
    wcopy<NU, 0>(imr, rs + ((size_t)b * N + j) * NU, lane);
    wcopy<NX, 0>(imr + NU, qs + ((size_t)b * (N + 1) + xi) * NX, lane);
}

template <int NU, int NX>
__device__ __forceinline__ void stage_BA_plan(const Geo &g, const ProbView &p, int b, int j, double *ba,
                                              double *fb, const short *tab) {
    using CP = CopyPlan<NU, NX>;
    const int N = g.N;
    const double *Bs = j < N ? p.B + ((size_t)b * N + j) * NX * NU : nullptr;
    const double *As = (j < N && j != 0) ? p.A + ((size_t)b * N + j) * NX * NX : nullptr;
    if (!Bs || !As || (CP::G == 2 && !(aligned16(Bs) && aligned16(As)))) {
        stage_BA<NU, NX>(g, p, b, j, ba, fb);
        return;
    }
    const int lane = lane_v();
    CP::template run<CP::OB, CP::KB>(tab, ba, Bs, lane);
    CP::template run<CP::OA, CP::KA>(tab, ba, As, lane);
    const double *fs = p.fd ? p.fd : p.f;
    wcopy<NX, 0>(fb, fs + ((size_t)b * N + j) * NX, lane);
}

} // namespace ric
} // namespace cyqb
