// Shared compile-time-shape helpers of the Riccati stage-panel kernels
// (riccati_warp.cu, riccati_pc.cu, riccati_cta.cu): tile geometry, cp.async staging of the
// stage data (R, S, Q, r, q / B, A, f) and the panel initialisation.
#pragma once

#include "kkt_common.cuh"
#include "kernels.h"

#include <cstdint>
#include <cstdio>

namespace cyqb {
namespace ric {

template <int NU, int NX> struct Shp {
    static constexpr int NUX = NU + NX;
    static constexpr int CT = (NUX + 7) / 8;      // pivot tile columns
    static constexpr int BT = (NX + 1 + 7) / 8;   // coupling + rhs tile rows
    static constexpr int TT = CT + BT;
    static constexpr int NT = TT * (TT + 1) / 2;
    static constexpr int XT0 = NU / 8, XT1 = (NUX - 1) / 8, NXT = XT1 - XT0 + 1;
    static constexpr int TOP = 8 * CT, RHS = TOP + NX;
    static constexpr int NLQ = NXT * (NXT + 1) / 2; // x-x tiles of L_Q
    static constexpr int NPT = CT * (CT + 1) / 2 + BT * CT;
    // staging (doubles)
    static constexpr int HB = NU * NU + NU * NX + NX * NX + NU + NX;
    static constexpr int BB = NX * NU + NX * NX + NX;
    static constexpr int HBp = (HB + 1) & ~1, BBp = (BB + 1) & ~1;
    static constexpr int SMEM_STAGED =
        (TT * NXT + NLQ) * kTileElems + HBp + BBp + 2 * ((NX + 1) & ~1) + kTileElems;
    // direct mode: stage data read from global (L2-prefetched one stage ahead)
    static constexpr int SMEM_DIRECT =
        (TT * NXT + NLQ) * kTileElems + 2 * ((NU + 1) & ~1) + kTileElems;
    __host__ __device__ static constexpr int T(int i, int j) { return i * (i + 1) / 2 + j; }
};

__device__ __forceinline__ void cp8(double *dst, const double *src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp16(double *dst, const double *src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int K> __device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

// ---- shared-memory mbarriers (hand-offs between warps of one CTA) ----------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(unsigned long long *mb, int count = 1) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
// this lane's arrival, triggered when its prior cp.async copies complete
__device__ __forceinline__ void mb_arrive_on_copies(unsigned long long *mb) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(mb)) : "memory");
}
// all lanes' prior shared-memory writes, then one (release) arrival
__device__ __forceinline__ void mb_signal(unsigned long long *mb, int lane) {
    __syncwarp();
    __threadfence_block();
    if (lane == 0)
        asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(mb)) : "memory");
    __syncwarp();
}
// suspend until the phase with parity `par` has completed (acquire)
#ifdef CYQ_MB_WATCHDOG // debug builds: a wait that never completes reports and traps
__device__ __forceinline__ void mb_wait(unsigned long long *mb, int par) {
    unsigned ok = 0;
    for (long long it = 0; !ok; ++it) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(smem_u32(mb)), "r"(par) : "memory");
        if (!ok && it == (1LL << 22) && (threadIdx.x & 31) == 0 && blockIdx.x < 2) {
            printf("mb_wait stuck: block %d warp %d barrier smem+%u parity %d\n", blockIdx.x, threadIdx.x >> 5,
                   smem_u32(mb), par);
            __trap();
        }
    }
}
#else
__device__ __forceinline__ void mb_wait(unsigned long long *mb, int par) {
    asm volatile("{\n .reg .pred p;\n"
                 "MB_WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
                 " @!p bra MB_WAIT_%=;\n}" ::"r"(smem_u32(mb)),
                 "r"(par)
                 : "memory");
}
#endif

// ---- shared-memory flags: a one-writer hand-off that is usually already
// there when its readers look. The writer's warp stores its data, then one
// lane releases the flag; readers spin on the expected value (an acquire
// load per look). Measured neutral against mbarrier try_wait on the config-3
// panel; kept because the value (stage + 1) needs no phase bookkeeping.
__device__ __forceinline__ void flag_set(unsigned *f, unsigned v, int lane) {
    __syncwarp();
    if (lane == 0)
        asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(f)), "r"(v) : "memory");
    __syncwarp();
}
// (every lane spins: with one lane polling and a __syncwarp the config-3 panel
// measured +0.9 ms, a nanosleep back-off between the looks was neutral)
#ifdef CYQ_MB_WATCHDOG // debug builds: a hand-off that never comes reports and traps
__device__ __forceinline__ void flag_wait(const unsigned *f, unsigned v) {
    unsigned r = ~v;
    for (long long it = 0; r != v; ++it) {
        asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(r) : "r"(smem_u32(f)) : "memory");
        if (r != v && it == (1LL << 24) && (threadIdx.x & 31) == 0 && blockIdx.x < 2) {
            printf("flag_wait stuck: block %d warp %d flag smem+%u = %u, expected %u\n", blockIdx.x,
                   threadIdx.x >> 5, smem_u32(f), r, v);
            __trap();
        }
    }
}
#else
__device__ __forceinline__ void flag_wait(const unsigned *f, unsigned v) {
    // (first look outside the loop: the rotated do-while form of the same
    // wait measured +0.35 ms on the config-3 panel)
    unsigned r;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(r) : "r"(smem_u32(f)) : "memory");
    while (r != v) {
        asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(r) : "r"(smem_u32(f)) : "memory");
    }
}
#endif

// async copy of cnt doubles (16-byte granules when both ends are aligned),
// or an identity / zero fill when src == nullptr
template <int CNT, int DIAG, int NTHR = 32>
__device__ __forceinline__ void wcopy(double *dst, const double *src, int lane) {
    if (src) {
        const bool al = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
        if (al) {
#pragma unroll
            for (int i = 2 * lane; i < (CNT & ~1); i += 2 * NTHR)
                cp16(dst + i, src + i);
            if ((CNT & 1) && lane == 0)
                cp8(dst + CNT - 1, src + CNT - 1);
        } else {
#pragma unroll
            for (int i = lane; i < CNT; i += NTHR)
                cp8(dst + i, src + i);
        }
    } else {
#pragma unroll
        for (int i = lane; i < CNT; i += NTHR)
            dst[i] = (DIAG > 0 && i / (DIAG > 0 ? DIAG : 1) == i % (DIAG > 0 ? DIAG : 1)) ? 1.0 : 0.0;
    }
}

template <int NU, int NX> struct Stage {
    double *R, *S, *Q, *r, *q; // H buffer
    double *B, *A, *f;         // BA buffer
};

template <int NU, int NX, int NTHR = 32>
__device__ __forceinline__ void load_H(const Geo &g, const ProbView &p, int b, int j, int xi,
                                       const Stage<NU, NX> &st, int lane) {
    const int N = g.N;
    const bool in = j < N;
    wcopy<NU * NU, NU, NTHR>(st.R, in ? p.R + ((size_t)b * N + j) * NU * NU : nullptr, lane);
    wcopy<NU * NX, 0, NTHR>(st.S, in ? p.S + ((size_t)b * N + j) * NU * NX : nullptr, lane);
    wcopy<NX * NX, NX, NTHR>(st.Q, xi <= N ? p.Q + ((size_t)b * (N + 1) + xi) * NX * NX : nullptr,
                       lane);
    const double *rs = p.ru ? p.ru : p.r;
    const double *qs = p.qx ? p.qx : p.q;
    wcopy<NU, 0, NTHR>(st.r, in ? rs + ((size_t)b * N + j) * NU : nullptr, lane);
    wcopy<NX, 0, NTHR>(st.q, xi <= N ? qs + ((size_t)b * (N + 1) + xi) * NX : nullptr, lane);
}

template <int NU, int NX, int NTHR = 32>
__device__ __forceinline__ void load_BA(const Geo &g, const ProbView &p, int b, int j,
                                        const Stage<NU, NX> &st, int lane) {
    const int N = g.N;
    const bool in = j < N;
    wcopy<NX * NU, 0, NTHR>(st.B, in ? p.B + ((size_t)b * N + j) * NX * NU : nullptr, lane);
    wcopy<NX * NX, 0, NTHR>(st.A, (in && j != 0) ? p.A + ((size_t)b * N + j) * NX * NX : nullptr,
                      lane);
    const double *fs = p.fd ? p.fd : p.f;
    wcopy<NX, 0, NTHR>(st.f, in ? fs + ((size_t)b * N + j) * NX : nullptr, lane);
}

__device__ __forceinline__ void pf_l2(const double *p, int bytes, int lane) {
    for (int o = lane * 128; o < bytes; o += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(reinterpret_cast<const char *>(p) + o));
}

// Direct mode: point at the global matrices of stage j (identity / zero
// constants for padding stages) and pull their lines into L2.
template <int NU, int NX>
__device__ __forceinline__ void point_H(const Geo &g, const ProbView &p, const double *cst, int b,
                                        int j, int xi, Stage<NU, NX> &st, int lane) {
    const int N = g.N;
    const double *eye_nu = cst, *eye_nx = cst + NU * NU, *zero = eye_nx + NX * NX;
    const bool in = j < N, qin = xi <= N;
    st.R = const_cast<double *>(in ? p.R + ((size_t)b * N + j) * NU * NU : eye_nu);
    st.S = const_cast<double *>(in ? p.S + ((size_t)b * N + j) * NU * NX : zero);
    st.Q = const_cast<double *>(qin ? p.Q + ((size_t)b * (N + 1) + xi) * NX * NX : eye_nx);
    st.r = const_cast<double *>(in ? (p.ru ? p.ru : p.r) + ((size_t)b * N + j) * NU : zero);
    st.q = const_cast<double *>(qin ? (p.qx ? p.qx : p.q) + ((size_t)b * (N + 1) + xi) * NX : zero);
    if (in) {
        pf_l2(st.R, NU * NU * 8, lane);
        pf_l2(st.S, NU * NX * 8, lane);
        pf_l2(st.r, NU * 8, lane);
    }
    if (qin) {
        pf_l2(st.Q, NX * NX * 8, lane);
        pf_l2(st.q, NX * 8, lane);
    }
}
template <int NU, int NX>
__device__ __forceinline__ void point_BA(const Geo &g, const ProbView &p, const double *cst, int b,
                                         int j, Stage<NU, NX> &st, int lane) {
    const int N = g.N;
    const double *zero = cst + NU * NU + NX * NX;
    const bool in = j < N;
    st.B = const_cast<double *>(in ? p.B + ((size_t)b * N + j) * NX * NU : zero);
    st.A = const_cast<double *>((in && j != 0) ? p.A + ((size_t)b * N + j) * NX * NX : zero);
    st.f = const_cast<double *>(in ? (p.fd ? p.fd : p.f) + ((size_t)b * N + j) * NX : zero);
    if (in) {
        pf_l2(st.B, NX * NU * 8, lane);
        if (j != 0)
            pf_l2(st.A, NX * NX * 8, lane);
        pf_l2(st.f, NX * 8, lane);
    }
}

// initial entry (r, col) of a pivot tile (compile-time tile, runtime lane).
// Branch-free: every candidate source is read with a clamped index and the
// result selected, so the panel initialisation is straight-line code that
// the scheduler can interleave (the tile row TI is a compile-time constant,
// so whole cases fold away).
template <int NU, int NX>
__device__ __forceinline__ double pinit(const Stage<NU, NX> &st, bool s0, bool j0, double sgn,
                                        const double *ru0, int ti, int r, int col) {
    using S = Shp<NU, NX>;
    if (8 * ti < S::TOP) { // top block: H_s (lower), identity padding
        const bool inb = r < S::NUX && col < S::NUX;
        const bool low = col <= r;
        const bool isR = inb && low && r < NU;
        const bool isS = inb && r >= NU && col < NU;
        const bool isQ = inb && low && r >= NU && col >= NU;
        const double vR = st.R[isR ? r * NU + col : 0];
        const double vS = st.S[isS ? col * NX + (r - NU) : 0];
        const double vQ = st.Q[isQ ? (r - NU) * NX + (col - NU) : 0];
        const double pad = (!inb && r == col) ? 1.0 : 0.0;
        return isR ? vR : isS ? (j0 ? 0.0 : vS) : isQ ? vQ : pad;
    } else {
        const int rb = r - S::TOP;
        const bool cin = col < S::NUX;
        const bool isB = s0 && rb < NX && col < NU;
        const bool isA = s0 && rb < NX && cin && col >= NU;
        const double vB = st.B[isB ? rb * NU + col : 0];
        const double vA = st.A[isA ? rb * NX + (col - NU) : 0];
        const bool isr = rb == NX && col < NU, isq = rb == NX && cin && col >= NU;
        const double vr = sgn * st.r[isr ? col : 0] - ((ru0 && isr) ? ru0[col] : 0.0);
        const double vq = sgn * st.q[isq ? col - NU : 0];
        return isB ? vB : isA ? vA : isr ? vr : isq ? vq : 0.0;
    }
}

} // namespace ric
} // namespace cyqb
