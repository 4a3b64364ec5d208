// C ABI (include/cyqlone_b200.h): contexts, device workspaces, launches.
//
// The batch entry points replace the reference's single-instance
// kkt::factor / solve / solve_problem (kkt_solver.hpp:118-128); the C++
// mirror (kkt_solver.cpp) wraps them with batch = 1. No CPU fallback: every
// path below launches the sm_100a kernels or reports CYQ_CUDA_ERR.
#include "../../include/cyqlone_b200.h"
#include "kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

using namespace cyqb;

struct cyq_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    // grow-only scratch for host-memory calls
    std::vector<std::pair<void **, size_t>> dummy;
    void *hbuf = nullptr;
    size_t hbuf_bytes = 0;
    void *wsbuf = nullptr;
    size_t wsbuf_bytes = 0;
    void *augbuf = nullptr; // augmented R, S, Q of cyq_solve_newton_batch's two-kernel path
    size_t augbuf_bytes = 0;
    void *lsbuf = nullptr; // line-search breakpoints + per-instance status
    size_t lsbuf_bytes = 0;
    unsigned long long *hfail = nullptr; // pinned per-instance failure keys (status readback)
    size_t hfail_n = 0;
    cudaStream_t copy_stream = nullptr; // host->device staging of chunked calls
    cudaStream_t side_stream = nullptr; // second compute stream (split device batches)
    // per-kernel timing (cyq_ctx_profile)
    bool profile = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
    std::vector<cudaEvent_t> pool;
    double ms[5] = {0, 0, 0, 0, 0};
    int64_t launches[5] = {0, 0, 0, 0, 0};
    int64_t kernels[5] = {0, 0, 0, 0, 0}; // kernel launches per kind
    LaunchOpts opts;                      // kernel selection (cyq_ctx_set_option)
    long long *phase = nullptr;           // phase clocks (CYQ_OPT_PHASE_PROF)
    // asynchronous status (CYQ_OPT_ASYNC_STATUS): pinned keys of the last call
    unsigned long long *hpend = nullptr;
    size_t hpend_n = 0;
    int64_t pend_batch = -1;
    // CUDA graph of the last repeated device pipeline (CYQ_OPT_GRAPHS)
    std::vector<unsigned long long> gkey_seen, gkey;
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t cap_stream = nullptr;
    int schur_path = -1; // Schur kernel of the last pipeline (see cyq_factor)
};

struct cyq_factor {
    cyq_ctx *ctx = nullptr;
    cyq_dims dims{};
    Geo g{};
    void *mem = nullptr; // one allocation: workspace (+ problem copy)
    size_t bytes = 0;
    FactorWS ws{};
    ProbView prob{}; // device copy of the problem (host-memory factor calls)
    bool owns_prob = false;
    LaunchOpts opts{}; // kernel selection at factor time (the solve reads its layouts)
    int schur_path = -1; // Schur kernel that factored it: 0 fused, 1 big, 2 per-level tiles, 3 scalar
};

namespace {

thread_local std::string g_last_err;

int set_err(cyq_ctx *ctx, int code, const std::string &msg) {
    if (ctx)
        ctx->err = msg;
    g_last_err = msg;
    return code;
}

#define CU(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return set_err(ctx, CYQ_CUDA_ERR,                                           \
                           std::string(#call) + ": " + cudaGetErrorString(e_));         \
    } while (0)

bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

// The runtime-shape kernels keep a stage's blocks (back substitution, forward
// sweep) or an instance's Schur rows in shared memory: shapes beyond it are
// rejected like the too-large stage panel in make_geo, never launched.
constexpr size_t kMaxDynSmem = 227 * 1024;
int smem_too_large(cyq_ctx *ctx, const char *what, size_t bytes) {
    char msg[160];
    snprintf(msg, sizeof msg, "stage shape too large: %s needs %zu KB of shared memory (max %zu)", what,
             bytes / 1024, kMaxDynSmem / 1024);
    return set_err(ctx, CYQ_INVALID_ARG, msg);
}

int make_geo(cyq_ctx *ctx, const cyq_dims *d, Geo &g) {
    if (!d || d->N < 1 || d->nx < 1 || d->nu < 1 || d->batch < 1)
        return set_err(ctx, CYQ_INVALID_ARG, "dims: N, nx, nu, batch must be >= 1");
    if (!pow2(d->P))
        return set_err(ctx, CYQ_INVALID_ARG, "P must be a power of two");
    g.N = (int)d->N;
    g.P = (int)d->P;
    g.Np = g.P * ((g.N + g.P - 1) / g.P);
    g.n = g.Np / g.P;
    g.nx = (int)d->nx;
    g.nu = (int)d->nu;
    g.nux = g.nx + g.nu;
    g.CT = (g.nux + 7) / 8;
    g.BT = (g.nx + 1 + 7) / 8;
    g.TT = g.CT + g.BT;
    g.XT0 = g.nu / 8;
    g.NXT = (g.nux - 1) / 8 - g.XT0 + 1;
    g.NPT = g.CT * (g.CT + 1) / 2 + g.BT * g.CT;
    g.NTT = g.BT * (g.BT + 1) / 2;
    g.batch = (int)d->batch;
    // FactorOptions::tail = pcr (kkt_factor.cpp:214-247): cyclic reduction
    // down to min(P, vlen) blocks, parallel cyclic reduction for the rest
    g.tail = ctx && ctx->opts.tail == CYQ_TAIL_PCR ? std::min(g.P, std::max(1, ctx->opts.vlen)) : 1;
    if (cyqb::riccati_smem_bytes(g) > 227 * 1024 || g.TT * (g.TT + 1) / 2 > 8 * 32)
        return set_err(ctx, CYQ_INVALID_ARG,
                       "stage panel too large (2 nx + nu > ~160 not supported)");
    return CYQ_OK;
}

struct WsSizes {
    size_t fac, y, wl, trail, schur, lamc, fail, consts, total;
};

WsSizes ws_sizes(const Geo &g) {
    WsSizes s;
    const size_t chains = (size_t)g.batch * g.P;
    auto al = [](size_t v) { return (v + 31) / 32 * 32; }; // 256-byte aligned
    s.fac = al(chains * g.n * g.NPT * kTileElems);
    s.y = al(chains * g.n * g.nux);
    s.wl = al(chains * g.n * g.nx);
    s.trail = al(chains * g.NTT * kTileElems);
    s.schur = al((size_t)g.batch * std::max<size_t>(std::max<size_t>(SchurLayout::make(g.P, g.nx).total,
                                                                      schur_fused_doubles(g)),
                                                    schur_big_doubles(g)));
    s.lamc = al((size_t)g.batch * g.P * g.nx);
    s.fail = al((size_t)g.batch); // 8-byte keys
    s.consts = al(riccati_consts_doubles(g));
    s.total = (s.fac + s.y + s.wl + s.trail + s.schur + s.lamc + s.fail + s.consts) *
              sizeof(double);
    return s;
}

FactorWS carve(void *base, const WsSizes &s) {
    FactorWS w;
    double *p = static_cast<double *>(base);
    w.fac = p;
    p += s.fac;
    w.y = p;
    p += s.y;
    w.wl = p;
    p += s.wl;
    w.trail = p;
    p += s.trail;
    w.schur = p;
    p += s.schur;
    w.lamc = p;
    p += s.lamc;
    w.fail = reinterpret_cast<unsigned long long *>(p);
    p += s.fail;
    w.consts = p;
    return w;
}

size_t prob_doubles(const Geo &g) {
    const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu;
    return B * (N * nx * nx + N * nx * nu + N * nu * nu + N * nu * nx + (N + 1) * nx * nx +
                N * nx + N * nu + (N + 1) * nx + nx);
}
size_t sol_doubles(const Geo &g) {
    const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu;
    return B * (N * nu + (N + 1) * nx + N * nx);
}

// Lays out a problem batch in one contiguous device buffer.
ProbView carve_prob(double *p, const Geo &g) {
    const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu;
    ProbView v{};
    double *q = p;
    auto take = [&](size_t cnt) {
        double *r = q;
        q += cnt;
        return r;
    };
    v.A = take(B * N * nx * nx);
    v.B = take(B * N * nx * nu);
    v.R = take(B * N * nu * nu);
    v.S = take(B * N * nu * nx);
    v.Q = take(B * (N + 1) * nx * nx);
    v.f = take(B * N * nx);
    v.r = take(B * N * nu);
    v.q = take(B * (N + 1) * nx);
    v.x_init = take(B * nx);
    return v;
}

int copy_prob_h2d(cyq_ctx *ctx, const Geo &g, const cyq_ocp_batch *h, const ProbView &d) {
    const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu;
    const std::pair<const double *, const double *> parts[] = {
        {h->A, d.A}, {h->B, d.B}, {h->R, d.R}, {h->S, d.S}, {h->Q, d.Q},
        {h->f, d.f}, {h->r, d.r}, {h->q, d.q}, {h->x_init, d.x_init}};
    const size_t cnt[] = {B * N * nx * nx, B * N * nx * nu, B * N * nu * nu, B * N * nu * nx,
                          B * (N + 1) * nx * nx, B * N * nx, B * N * nu, B * (N + 1) * nx,
                          B * nx};
    for (int i = 0; i < 9; ++i) {
        if (!parts[i].first)
            return set_err(ctx, CYQ_INVALID_ARG, "null problem array");
        CU(cudaMemcpyAsync(const_cast<double *>(parts[i].second), parts[i].first,
                           cnt[i] * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    return CYQ_OK;
}

ProbView view_of(const cyq_ocp_batch *p) {
    ProbView v{};
    v.A = p->A;
    v.B = p->B;
    v.R = p->R;
    v.S = p->S;
    v.Q = p->Q;
    v.f = p->f;
    v.r = p->r;
    v.q = p->q;
    v.x_init = p->x_init;
    return v;
}

// Warps per chain CTA and register tiles per warp (MAXT template).
void riccati_shape(const Geo &g, const LaunchOpts &o, int &nw, int &maxt) {
    const int nt = g.TT * (g.TT + 1) / 2;
    nw = o.panel_warps ? std::max(1, std::min(4, o.panel_warps)) : 4;
    int per = (nt + nw - 1) / nw;
    if (per > 16) { // large panels: the 256-thread, 32-tile-per-warp variant
        nw = 8;
        per = (nt + nw - 1) / nw;
    }
    // 8 warps only exist in the MAXT = 32 instantiation (launch bounds: 128
    // threads below it)
    maxt = nw == 8 ? 32 : per <= 4 ? 4 : per <= 8 ? 8 : per <= 16 ? 16 : 32;
}

template <int M> void launch_riccati_t(const Geo &g, int nw, cudaStream_t st, const RiccatiArgs &ra) {
    static DeviceOnce once;
    once_per_device(once, [] {
        return cudaFuncSetAttribute(riccati_panel_kernel_t<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    227 * 1024);
    });
    riccati_panel_kernel_t<M><<<ra.grid_chains(), 32 * nw, riccati_smem_bytes(g), st>>>(ra);
}

void launch_riccati(const Geo &g, const LaunchOpts &o, cudaStream_t st, const RiccatiArgs &ra) {
    int nw, maxt;
    riccati_shape(g, o, nw, maxt);
    switch (maxt) {
    case 4: launch_riccati_t<4>(g, nw, st, ra); break;
    case 8: launch_riccati_t<8>(g, nw, st, ra); break;
    case 16: launch_riccati_t<16>(g, nw, st, ra); break;
    default: launch_riccati_t<32>(g, nw, st, ra); break;
    }
}

cudaEvent_t take_event(cyq_ctx *ctx) {
    if (ctx->pool.empty()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    cudaEvent_t e = ctx->pool.back();
    ctx->pool.pop_back();
    return e;
}

// Brackets one launch with events when profiling is on.
struct Timed {
    cyq_ctx *ctx;
    int kind;
    cudaEvent_t a = nullptr, b = nullptr;
    int kernels = 1; // kernel launches inside the bracket (set by the caller)
    Timed(cyq_ctx *c, int k) : ctx(c), kind(k) {
        if (ctx->profile) {
            a = take_event(ctx);
            b = take_event(ctx);
            cudaEventRecord(a, ctx->stream);
        }
    }
    ~Timed() {
        if (ctx->profile) {
            cudaEventRecord(b, ctx->stream);
            ctx->ev.push_back({kind, {a, b}});
            ctx->kernels[kind] += kernels;
        }
    }
};

// Schur complement + cyclic reduction (factor and / or solve, per
// sa.do_factor / sa.do_solve): the fused one-kernel paths (schur_fused.cu,
// schur_big.cu) unless CYQ_OPT_SCHUR selects the per-level tile kernels or
// the scalar kernel, or no specialisation serves the shape.
int launch_schur(cyq_ctx *ctx, const Geo &g, const SchurArgs &sa, const LaunchOpts &o) {
    Timed t(ctx, 1);
    if (o.schur == 0 && launch_schur_fused(g, ctx->stream, sa, o)) {
        t.kernels = 1; // one fused kernel per batch
        ctx->schur_path = 0;
    } else if (o.schur == 0 && launch_schur_big(g, ctx->stream, sa)) {
        t.kernels = 1;
        ctx->schur_path = 1;
    } else if (sa.do_factor && o.schur != 2 && launch_schur_tiles(g, ctx->stream, sa)) {
        ctx->schur_path = 2;
        // DMMA-tile factorization levels, then the scalar kernel's solve
        t.kernels = 2 + SchurLayout::make(g.P, g.nx).levels + (sa.do_solve ? 1 : 0);
        if (sa.do_solve) {
            SchurArgs sv = sa;
            sv.do_factor = 0;
            const int nw = schur_warps_solve(g);
            if (schur_smem_for(g, nw) > kMaxDynSmem)
                return smem_too_large(ctx, "Schur/CR solve (P x nx)", schur_smem_for(g, nw));
            schur_cr_kernel<<<g.batch, 32 * nw, schur_smem_for(g, nw), ctx->stream>>>(sv);
        }
    } else if (sa.do_factor) {
        ctx->schur_path = 3;
        if (schur_smem_bytes(g) > kMaxDynSmem)
            return smem_too_large(ctx, "Schur/CR (P x nx)", schur_smem_bytes(g));
        schur_cr_kernel<<<g.batch, 32 * schur_warps(g), schur_smem_bytes(g), ctx->stream>>>(sa);
    } else {
        const int nw = schur_warps_solve(g);
        if (schur_smem_for(g, nw) > kMaxDynSmem)
            return smem_too_large(ctx, "Schur/CR solve (P x nx)", schur_smem_for(g, nw));
        schur_cr_kernel<<<g.batch, 32 * nw, schur_smem_for(g, nw), ctx->stream>>>(sa);
    }
    CU(cudaGetLastError());
    return CYQ_OK;
}

int launch_backsub(cyq_ctx *ctx, const Geo &g, const BacksubArgs &ba, const LaunchOpts &o) {
    Timed t(ctx, 2);
    if (o.backsub != 0 || (!launch_backsub_warp(g, ctx->stream, ba) && !launch_backsub_tile(g, ctx->stream, ba))) {
        const int wpb = backsub_wpb(g), chains = g.batch * g.P;
        if (backsub_smem_bytes(g) > kMaxDynSmem)
            return smem_too_large(ctx, "back substitution", backsub_smem_bytes(g));
        backsub_kernel<<<(chains + wpb - 1) / wpb, 32 * wpb, backsub_smem_bytes(g), ctx->stream>>>(ba);
    }
    CU(cudaGetLastError());
    return CYQ_OK;
}

// Profiling aid (CYQ_OPT_PHASE_PROF): chain 0's per-stage phase clocks of
// the stage panel and instance 0's Schur phases, to stderr.
int dump_phases(cyq_ctx *ctx, const Geo &g, const long long *ph, const long long *sph) {
    std::vector<long long> h(8 * (g.n + 1));
    CU(cudaMemcpyAsync(h.data(), ph, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    std::vector<long long> q(32);
    CU(cudaMemcpyAsync(q.data(), sph, 32 * sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int s = 0; s < g.n; ++s)
        fprintf(stderr, "phase s=%d init+WW %lld chol %lld store %lld mw %lld V %lld (wl %lld tiles %lld wait %lld rest %lld)\n", s,
                h[s * 8 + 1] - h[s * 8 + 0], h[s * 8 + 2] - h[s * 8 + 1], h[s * 8 + 3] - h[s * 8 + 2],
                h[s * 8 + 4] - h[s * 8 + 3], (s + 1 < g.n ? h[(s + 1) * 8] : h[g.n * 8]) - h[s * 8 + 4],
                h[s * 8 + 5] - h[s * 8 + 4], h[s * 8 + 6] - h[s * 8 + 5], h[s * 8 + 7] - h[s * 8 + 6],
                (s + 1 < g.n ? h[(s + 1) * 8] : h[g.n * 8]) - h[s * 8 + 7]);
#ifdef CYQ_TRACE
    if (g.nx == 64) { // riccati_cta column-loop trace: per (kb, warp) event clocks relative to the step start
        const int NW = 16, CT = 12;
        std::vector<long long> t(CT * NW * 8);
        CU(cudaMemcpy(t.data(), ph + 4096, t.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        long long t0 = t[0];
        for (int kb = 0; kb < CT; ++kb)
            for (int w = 0; w < NW; ++w) {
                const long long *e = &t[(kb * NW + w) * 8];
                fprintf(stderr, "trace kb=%d w=%d start %lld A %lld bar1 %lld pick %lld trail %lld bar2 %lld fac %lld\n", kb, w,
                        e[0] - t0, e[1] - e[0], e[2] - e[1], e[3] - e[2], e[4] - e[3], e[5] ? e[5] - e[0] : 0,
                        e[7] ? e[7] - e[0] : 0);
            }
        std::vector<long long> pt(CT * 8);
        CU(cudaMemcpy(pt.data(), ph + 6144, pt.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        for (int d = 0; d < CT; ++d) {
            const long long *e = &pt[d * 8];
            fprintf(stderr, "pivot d=%d start %lld wait+solve+update %lld factor %lld inverse %lld L-out %lld\n",
                    d, e[0] - t0, e[1] - e[0], e[3] - e[1], e[4] - e[3], e[5] - e[4]);
        }
    }
#endif
    if (q[31] > 1 && q[31] < 31) {
        fprintf(stderr, "schur phases (instance 0):");
        for (long long k = 1; k < q[31]; ++k)
            fprintf(stderr, " %lld", q[k] - q[k - 1]);
        fprintf(stderr, "  total %lld\n", q[q[31] - 1] - q[0]);
    }
    return CYQ_OK;
}

int launch_pipeline(cyq_ctx *ctx, const Geo &g, const ProbView &p, const FactorWS &ws,
                    const SolView *sol, bool do_solve) {
    static DeviceOnce once;
    CU(once_per_device(once, [] {
        cudaError_t e = cudaFuncSetAttribute(backsub_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        return e != cudaSuccess ? e
                                : cudaFuncSetAttribute(schur_cr_kernel,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    }));
    const LaunchOpts &o = ctx->opts;
    const int chains = g.batch * g.P;
    CU(cudaMemsetAsync(ws.fail, 0xFF, sizeof(unsigned long long) * g.batch, ctx->stream));
    const bool staged = riccati_staged(g);
    if (!staged) { // identity / zero constants for the direct-mode generic panel
        std::vector<double> h(riccati_consts_doubles(g), 0.0);
        for (int i = 0; i < g.nu; ++i)
            h[(size_t)i * g.nu + i] = 1.0;
        for (int i = 0; i < g.nx; ++i)
            h[(size_t)g.nu * g.nu + (size_t)i * g.nx + i] = 1.0;
        CU(cudaMemcpyAsync(ws.consts, h.data(), h.size() * sizeof(double),
                           cudaMemcpyHostToDevice, ctx->stream));
    }
    RiccatiArgs ra{g, p, ws.fac, ws.y, ws.wl, ws.trail, ws.fail, ws.consts, staged ? 1 : 0,
                   nullptr};
    if (o.phase_prof) {
        if (!ctx->phase)
            CU(cudaMalloc(&ctx->phase, 8 * 4096 * sizeof(long long)));
        CU(cudaMemsetAsync(ctx->phase, 0, 8 * 4096 * sizeof(long long), ctx->stream));
        ra.phase = ctx->phase;
    }
    {
        Timed t(ctx, 0);
        // kernel choice (CYQ_OPT_PANEL forces one; a forced kernel without a
        // specialisation for this shape falls back to the automatic order):
        // latency-bound launches (at most ~2 chains per SM: a single long
        // horizon, config 0 / 2) take the two-warp producer/consumer panel
        // (measured 0.078 -> 0.074 ms at config 2); batches the one-warp
        // compile-time-shape kernel, large tile-aligned blocks the CTA
        // kernel, every other shape the runtime-shape generic kernel
        bool done = false;
        if (p.aD) { // fused Newton-system augmentation: the warp kernel only
            if (!launch_riccati_warp(g, ctx->stream, ra, o))
                return set_err(ctx, CYQ_INVALID_ARG, "fused augmentation: no kernel for this shape");
            done = true;
        }
        if (!done) {
            switch (o.panel) {
            case CYQ_PANEL_WARP:
            case CYQ_PANEL_WARP_TMEM: done = launch_riccati_warp(g, ctx->stream, ra, o); break;
            case CYQ_PANEL_TWO_WARP: done = launch_riccati_pc(g, ctx->stream, ra); break;
            case CYQ_PANEL_CTA: done = launch_riccati_cta(g, ctx->stream, ra); break;
            case CYQ_PANEL_CTA_TMA: done = launch_riccati_cta(g, ctx->stream, ra, true); break;
            case CYQ_PANEL_GENERIC: launch_riccati(g, o, ctx->stream, ra); done = true; break;
            default: break;
            }
        }
        if (!done && (long long)chains <= 2LL * o.sms)
            done = launch_riccati_pc(g, ctx->stream, ra);
        if (!done)
            done = launch_riccati_warp(g, ctx->stream, ra, LaunchOpts{});
        if (!done)
            done = launch_riccati_cta(g, ctx->stream, ra);
        if (!done)
            launch_riccati(g, o, ctx->stream, ra);
    }
    CU(cudaGetLastError());
    SchurArgs sa{g, p, ws.fac, ws.y, ws.trail, ws.schur, ws.lamc,
                 sol ? sol->lam : nullptr, ws.fail, 1, do_solve ? 1 : 0};
    sa.phase = ra.phase ? ra.phase + 16 * (g.n + 1) + 8 : nullptr;
    int rc = launch_schur(ctx, g, sa, o);
    if (rc)
        return rc;
    if (ra.phase)
        dump_phases(ctx, g, ra.phase, sa.phase);
    if (do_solve) {
        rc = launch_backsub(ctx, g, BacksubArgs{g, p, ws.fac, ws.y, ws.wl, ws.lamc, *sol}, o);
        if (rc)
            return rc;
    }
    return CYQ_OK;
}

// kkt::solve over an existing factor: forward sweep (forward.cu), Schur/CR
// solve, back substitution. `p` carries the explicit rhs.
int launch_solve(cyq_ctx *ctx, const Geo &g, const ProbView &p, const FactorWS &ws,
                 const SolView &sol, const LaunchOpts &o) {
    static DeviceOnce once;
    CU(once_per_device(once, [] {
        return cudaFuncSetAttribute(forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    }));
    const int chains = g.batch * g.P;
    BacksubArgs ba{g, p, ws.fac, ws.y, ws.wl, ws.lamc, sol};
    {
        Timed t(ctx, 3);
        const int wpb = 2 * forward_smem_per_warp(g) <= 200 * 1024 ? 2 : 1;
        if ((size_t)wpb * forward_smem_per_warp(g) > kMaxDynSmem)
            return smem_too_large(ctx, "forward sweep", forward_smem_per_warp(g));
        forward_kernel<<<(chains + wpb - 1) / wpb, 32 * wpb, wpb * forward_smem_per_warp(g),
                         ctx->stream>>>(ba, ws.y, ws.wl, ws.trail);
    }
    CU(cudaGetLastError());
    SchurArgs sa{g, p, ws.fac, ws.y, ws.trail, ws.schur, ws.lamc, sol.lam, ws.fail, 0, 1};
    const int rc = launch_schur(ctx, g, sa, o);
    return rc ? rc : launch_backsub(ctx, g, ba, o);
}

int decode_status(cyq_ctx *ctx, const Geo &g, const unsigned long long *dfail,
                  cyq_status *status) {
    if (ctx->hfail_n < (size_t)g.batch) { // pinned: the readback is one DMA, no staging copy
        if (ctx->hfail)
            CU(cudaFreeHost(ctx->hfail));
        ctx->hfail = nullptr;
        ctx->hfail_n = 0;
        CU(cudaMallocHost(reinterpret_cast<void **>(&ctx->hfail), sizeof(unsigned long long) * g.batch));
        ctx->hfail_n = (size_t)g.batch;
    }
    unsigned long long *h = ctx->hfail;
    CU(cudaMemcpyAsync(h, dfail, sizeof(unsigned long long) * g.batch, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    int worst = CYQ_OK;
    for (int b = 0; b < g.batch; ++b) {
        cyq_status st{};
        st.instance = b;
        if (h[b] != ~0ull) {
            st.code = CYQ_PIVOT_FAIL;
            st.kind = (int)(h[b] >> 60);
            st.column_or_level = (int64_t)((h[b] >> 40) & 0xFFFFF);
            st.stage = (int64_t)((h[b] >> 20) & 0xFFFFF);
            st.pivot = (int64_t)(h[b] & 0xFFFFF);
            worst = CYQ_PIVOT_FAIL;
        }
        if (status)
            status[b] = st;
    }
    if (worst != CYQ_OK)
        set_err(ctx, worst, "factorization pivot failure (see status)");
    return worst;
}

// Status of a device-memory call: decoded now (host sync), or with
// CYQ_OPT_ASYNC_STATUS copied into pinned memory stream-ordered and decoded
// by cyq_ctx_wait_status.
int finish_status(cyq_ctx *ctx, const Geo &g, const unsigned long long *dfail, cyq_status *status) {
    if (!ctx->opts.async_status)
        return decode_status(ctx, g, dfail, status);
    if (ctx->hpend_n < (size_t)g.batch) {
        if (ctx->hpend)
            CU(cudaFreeHost(ctx->hpend));
        ctx->hpend = nullptr;
        ctx->hpend_n = 0;
        CU(cudaMallocHost(reinterpret_cast<void **>(&ctx->hpend), sizeof(unsigned long long) * g.batch));
        ctx->hpend_n = (size_t)g.batch;
    }
    CU(cudaMemcpyAsync(ctx->hpend, dfail, sizeof(unsigned long long) * g.batch, cudaMemcpyDeviceToHost,
                       ctx->stream));
    ctx->pend_batch = g.batch;
    return CYQ_OK;
}

int launch_pipeline(cyq_ctx *ctx, const Geo &g, const ProbView &p, const FactorWS &ws,
                    const SolView *sol, bool do_solve);

// launch_pipeline through a CUDA graph when the same device call (shape,
// pointers, options, solve or factor only) repeats: the first occurrence
// launches directly, the second is captured (on a private stream) and
// launched, later ones replay it -- one graph launch instead of a memset
// and three kernel launches per call. Not used while per-kernel profiling
// (events between the kernels) is on.
int run_pipeline(cyq_ctx *ctx, const Geo &g, const ProbView &p, const FactorWS &ws, const SolView *sol,
                 bool do_solve) {
    const LaunchOpts &o = ctx->opts;
    if (ctx->profile || !o.graphs || o.phase_prof || !riccati_staged(g))
        return launch_pipeline(ctx, g, p, ws, sol, do_solve);
    std::vector<unsigned long long> key;
    auto put = [&](const void *q, size_t bytes) {
        const unsigned char *c = static_cast<const unsigned char *>(q);
        for (size_t i = 0; i < bytes; i += 8) {
            unsigned long long v = 0;
            memcpy(&v, c + i, std::min<size_t>(8, bytes - i));
            key.push_back(v);
        }
    };
    put(&g, sizeof g);
    put(&p, sizeof p);
    put(&ws, sizeof ws);
    if (sol)
        put(sol, sizeof *sol);
    put(&o, sizeof o);
    key.push_back(do_solve);
    key.push_back(reinterpret_cast<unsigned long long>(ctx->stream));
    if (ctx->gexec && key == ctx->gkey) {
        CU(cudaGraphLaunch(ctx->gexec, ctx->stream));
        return CYQ_OK;
    }
    if (key != ctx->gkey_seen) { // first occurrence: direct launches
        ctx->gkey_seen = key;
        return launch_pipeline(ctx, g, p, ws, sol, do_solve);
    }
    if (!ctx->cap_stream)
        CU(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    const cudaStream_t user = ctx->stream;
    ctx->stream = ctx->cap_stream;
    CU(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = launch_pipeline(ctx, g, p, ws, sol, do_solve);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(ctx->cap_stream, &graph);
    ctx->stream = user;
    cudaGraphExec_t exec = nullptr;
    cudaError_t ei = cudaErrorUnknown;
    if (rc == CYQ_OK && ec == cudaSuccess && graph)
        ei = cudaGraphInstantiate(&exec, graph, 0);
    if (graph)
        cudaGraphDestroy(graph);
    if (rc != CYQ_OK)
        return rc;
    if (ei != cudaSuccess) { // not capturable: launch directly from now on
        cudaGetLastError();
        ctx->gkey_seen.clear();
        return launch_pipeline(ctx, g, p, ws, sol, do_solve);
    }
    if (ctx->gexec)
        cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = exec;
    ctx->gkey = key;
    CU(cudaGraphLaunch(ctx->gexec, ctx->stream));
    return CYQ_OK;
}

int ensure(cyq_ctx *ctx, void **buf, size_t *have, size_t need) {
    if (*have >= need)
        return CYQ_OK;
    if (*buf)
        CU(cudaFree(*buf));
    *buf = nullptr;
    *have = 0;
    CU(cudaMalloc(buf, need));
    *have = need;
    return CYQ_OK;
}

} // namespace

namespace cyqb {

cudaStream_t ctx_prepare(cyq_ctx *ctx) {
    cudaSetDevice(ctx->device);
    return ctx->stream;
}

} // namespace cyqb

extern "C" {

int cyq_ctx_create(int device, cyq_ctx **out) {
    cyq_ctx *ctx = nullptr;
    if (!out)
        return set_err(nullptr, CYQ_INVALID_ARG, "null out");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0)
        return set_err(nullptr, CYQ_NO_DEVICE, "no CUDA device");
    ctx = new cyq_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete ctx;
        return set_err(nullptr, CYQ_CUDA_ERR, cudaGetErrorString(e));
    }
    ctx->own_stream = true;
    cudaDeviceGetAttribute(&ctx->opts.sms, cudaDevAttrMultiProcessorCount, device);
    *out = ctx;
    return CYQ_OK;
}

int cyq_ctx_destroy(cyq_ctx *ctx) {
    if (!ctx)
        return CYQ_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream)
        cudaStreamSynchronize(ctx->stream);
    if (ctx->hbuf)
        cudaFree(ctx->hbuf);
    if (ctx->wsbuf)
        cudaFree(ctx->wsbuf);
    if (ctx->augbuf)
        cudaFree(ctx->augbuf);
    if (ctx->lsbuf)
        cudaFree(ctx->lsbuf);
    if (ctx->hfail)
        cudaFreeHost(ctx->hfail);
    if (ctx->phase)
        cudaFree(ctx->phase);
    if (ctx->hpend)
        cudaFreeHost(ctx->hpend);
    if (ctx->gexec)
        cudaGraphExecDestroy(ctx->gexec);
    if (ctx->cap_stream)
        cudaStreamDestroy(ctx->cap_stream);
    for (auto &e : ctx->ev) {
        cudaEventDestroy(e.second.first);
        cudaEventDestroy(e.second.second);
    }
    for (auto e : ctx->pool)
        cudaEventDestroy(e);
    if (ctx->own_stream && ctx->stream)
        cudaStreamDestroy(ctx->stream);
    if (ctx->copy_stream)
        cudaStreamDestroy(ctx->copy_stream);
    if (ctx->side_stream)
        cudaStreamDestroy(ctx->side_stream);
    delete ctx;
    return CYQ_OK;
}

int cyq_ctx_set_stream(cyq_ctx *ctx, void *s) {
    if (!ctx)
        return CYQ_INVALID_ARG;
    if (ctx->own_stream && ctx->stream)
        cudaStreamDestroy(ctx->stream);
    if (s) {
        ctx->stream = static_cast<cudaStream_t>(s);
        ctx->own_stream = false;
    } else {
        CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    return CYQ_OK;
}

int cyq_ctx_synchronize(cyq_ctx *ctx) {
    if (!ctx)
        return CYQ_INVALID_ARG;
    CU(cudaStreamSynchronize(ctx->stream));
    return CYQ_OK;
}

const char *cyq_ctx_last_error(cyq_ctx *ctx) {
    return ctx ? ctx->err.c_str() : g_last_err.c_str();
}

// Device-resident batch in K parts (CYQ_SPLIT=K, opt-in), alternating
// between the context stream and a side stream (joined back into the
// context stream): the tail of each kernel of one part overlaps kernels of
// the next (measured +2% at config 1 with K = 2).
static int split_device_pipeline(cyq_ctx *ctx, const Geo &g, const ProbView &pv, const SolView &sv,
                                 cyq_status *status, int K) {
    const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu;
    std::vector<size_t> b0s(K), hb(K);
    std::vector<Geo> gh(K, g);
    std::vector<WsSizes> wz(K);
    size_t total = 0;
    for (int h = 0; h < K; ++h) {
        b0s[h] = B * h / K;
        hb[h] = B * (h + 1) / K - b0s[h];
        gh[h].batch = (int)hb[h];
        wz[h] = ws_sizes(gh[h]);
        total += wz[h].total;
    }
    int rc = ensure(ctx, &ctx->wsbuf, &ctx->wsbuf_bytes, total);
    if (rc)
        return rc;
    if (!ctx->side_stream)
        CU(cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
    cudaEvent_t fork = take_event(ctx), join = take_event(ctx);
    CU(cudaEventRecord(fork, ctx->stream));
    CU(cudaStreamWaitEvent(ctx->side_stream, fork, 0));
    std::vector<FactorWS> wsh(K);
    {
        size_t off = 0;
        for (int h = 0; h < K; ++h) {
            wsh[h] = carve(static_cast<char *>(ctx->wsbuf) + off, wz[h]);
            off += wz[h].total;
        }
    }
    const cudaStream_t main = ctx->stream;
    for (int h = 0; h < K; ++h) {
        const size_t b0 = b0s[h];
        ProbView p = pv;
        const double **pp[9] = {&p.A, &p.B, &p.R, &p.S, &p.Q, &p.f, &p.r, &p.q, &p.x_init};
        const size_t per[9] = {N * nx * nx, N * nx * nu, N * nu * nu, N * nu * nx, (N + 1) * nx * nx,
                               N * nx, N * nu, (N + 1) * nx, nx};
        for (int i = 0; i < 9; ++i)
            *pp[i] += b0 * per[i];
        SolView s{sv.u + b0 * N * nu, sv.x + b0 * (N + 1) * nx, sv.lam + b0 * N * nx};
        ctx->stream = (h & 1) ? ctx->side_stream : main; // launches and their timing events
        rc = launch_pipeline(ctx, gh[h], p, wsh[h], &s, true);
        ctx->stream = main;
        if (rc)
            return rc;
    }
    CU(cudaEventRecord(join, ctx->side_stream));
    CU(cudaStreamWaitEvent(main, join, 0));
    ctx->pool.push_back(fork);
    ctx->pool.push_back(join);
    int worst = CYQ_OK;
    for (int h = 0; h < K; ++h) {
        const int r2 = decode_status(ctx, gh[h], wsh[h].fail, status ? status + b0s[h] : nullptr);
        if (status)
            for (size_t k = 0; k < hb[h]; ++k)
                status[b0s[h] + k].instance = (int64_t)(b0s[h] + k);
        if (r2 == CYQ_CUDA_ERR)
            return r2;
        worst = std::max(worst, r2);
    }
    if (worst != CYQ_OK)
        set_err(ctx, worst, "factorization pivot failure (see status)");
    return worst;
}

int cyq_solve_problem_batch(cyq_ctx *ctx, const cyq_dims *dims, const cyq_ocp_batch *prob,
                            const cyq_sol_batch *sol, cyq_status *status, int mem) {
    if (!ctx || !prob || !sol)
        return set_err(ctx, CYQ_INVALID_ARG, "null argument");
    Geo g;
    int rc = make_geo(ctx, dims, g);
    if (rc)
        return rc;
    CU(cudaSetDevice(ctx->device));
    const WsSizes wsz = ws_sizes(g);
    rc = ensure(ctx, &ctx->wsbuf, &ctx->wsbuf_bytes, wsz.total);
    if (rc)
        return rc;
    FactorWS ws = carve(ctx->wsbuf, wsz);
    if (mem == CYQ_MEM_DEVICE) {
        SolView sv{sol->u, sol->x, sol->lam};
        // opt-in (CYQ_SPLIT=K): the overlapped launches make each kernel's
        // own event-timed duration (the roofline's denominator) meaningless
        const int K = ctx->opts.split;
        if (g.batch >= 128 * K && K >= 2) {
            // K parts, each a full pipeline, on two alternating streams: the
            // kernels' tails (the Schur kernel's second wave above all)
            // overlap the next part's kernels
            return split_device_pipeline(ctx, g, view_of(prob), sv, status, K);
        }
        rc = run_pipeline(ctx, g, view_of(prob), ws, &sv, true);
        if (rc)
            return rc;
        return finish_status(ctx, g, ws.fail, status);
    }
    // host memory: the batch is split into chunks whose host->device copies
    // (copy stream) overlap the previous chunk's kernels (compute stream);
    // each chunk's solution is copied back on the compute stream.
    const size_t pd = prob_doubles(g), sd = sol_doubles(g);
    rc = ensure(ctx, &ctx->hbuf, &ctx->hbuf_bytes, (pd + sd) * sizeof(double));
    if (rc)
        return rc;
    if (!ctx->copy_stream)
        CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    double *base = static_cast<double *>(ctx->hbuf);
    const ProbView dp = carve_prob(base, g);
    const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu;
    const SolView svall{base + pd, base + pd + B * N * nu, base + pd + B * N * nu + B * (N + 1) * nx};
    // (more, smaller chunks for multi-GB problems: the copies are the bound and
    // the last chunk's kernels are the only part they do not hide)
    const int nch = B >= 256 ? (pd * sizeof(double) > (4ull << 30) ? 16 : 8) : (B >= 32 ? 4 : 1);
    const int per = (int)((B + nch - 1) / nch);
    Geo gc = g;
    gc.batch = per;
    const WsSizes wc = ws_sizes(gc);
    rc = ensure(ctx, &ctx->wsbuf, &ctx->wsbuf_bytes, (size_t)nch * wc.total);
    if (rc)
        return rc;
    const std::pair<const double *, size_t> hp[9] = {
        {prob->A, N * nx * nx}, {prob->B, N * nx * nu}, {prob->R, N * nu * nu},
        {prob->S, N * nu * nx}, {prob->Q, (N + 1) * nx * nx}, {prob->f, N * nx},
        {prob->r, N * nu},      {prob->q, (N + 1) * nx},     {prob->x_init, nx}};
    const double *dpa[9] = {dp.A, dp.B, dp.R, dp.S, dp.Q, dp.f, dp.r, dp.q, dp.x_init};
    for (int i = 0; i < 9; ++i)
        if (!hp[i].first)
            return set_err(ctx, CYQ_INVALID_ARG, "null problem array");
    std::vector<cudaEvent_t> evs;
    int worst = CYQ_OK;
    for (int ch = 0; ch < nch; ++ch) {
        const size_t b0 = (size_t)ch * per;
        if (b0 >= B)
            break;
        const size_t cb = std::min<size_t>(per, B - b0);
        for (int i = 0; i < 9; ++i)
            CU(cudaMemcpyAsync(const_cast<double *>(dpa[i]) + b0 * hp[i].second,
                               hp[i].first + b0 * hp[i].second, cb * hp[i].second * sizeof(double),
                               cudaMemcpyHostToDevice, ctx->copy_stream));
        cudaEvent_t ev = take_event(ctx);
        CU(cudaEventRecord(ev, ctx->copy_stream));
        CU(cudaStreamWaitEvent(ctx->stream, ev, 0));
        evs.push_back(ev);
        Geo gi = g;
        gi.batch = (int)cb;
        ProbView pv{};
        const double **pvp[9] = {&pv.A, &pv.B, &pv.R, &pv.S, &pv.Q, &pv.f, &pv.r, &pv.q, &pv.x_init};
        for (int i = 0; i < 9; ++i)
            *pvp[i] = dpa[i] + b0 * hp[i].second;
        SolView sv{svall.u + b0 * N * nu, svall.x + b0 * (N + 1) * nx, svall.lam + b0 * N * nx};
        FactorWS wsi = carve(static_cast<char *>(ctx->wsbuf) + (size_t)ch * wc.total, wc);
        rc = launch_pipeline(ctx, gi, pv, wsi, &sv, true);
        if (rc)
            return rc;
        CU(cudaMemcpyAsync(sol->u + b0 * N * nu, sv.u, cb * N * nu * sizeof(double),
                           cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(sol->x + b0 * (N + 1) * nx, sv.x, cb * (N + 1) * nx * sizeof(double),
                           cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(sol->lam + b0 * N * nx, sv.lam, cb * N * nx * sizeof(double),
                           cudaMemcpyDeviceToHost, ctx->stream));
    }
    for (int ch = 0; ch < nch; ++ch) {
        const size_t b0 = (size_t)ch * per;
        if (b0 >= B)
            break;
        Geo gi = g;
        gi.batch = (int)std::min<size_t>(per, B - b0);
        FactorWS wsi = carve(static_cast<char *>(ctx->wsbuf) + (size_t)ch * wc.total, wc);
        const int r2 = decode_status(ctx, gi, wsi.fail, status ? status + b0 : nullptr);
        if (status)
            for (size_t k = 0; k < (size_t)gi.batch; ++k)
                status[b0 + k].instance = (int64_t)(b0 + k);
        if (r2 == CYQ_CUDA_ERR)
            return r2;
        worst = std::max(worst, r2);
    }
    for (auto e : evs)
        ctx->pool.push_back(e);
    if (worst != CYQ_OK)
        set_err(ctx, worst, "factorization pivot failure (see status)");
    return worst;
}

int cyq_factor_batch(cyq_ctx *ctx, const cyq_dims *dims, const cyq_ocp_batch *prob, int mem,
                     cyq_factor **out, cyq_status *status) {
    if (!ctx || !prob || !out)
        return set_err(ctx, CYQ_INVALID_ARG, "null argument");
    Geo g;
    int rc = make_geo(ctx, dims, g);
    if (rc)
        return rc;
    CU(cudaSetDevice(ctx->device));
    cyq_factor *f = new cyq_factor();
    f->ctx = ctx;
    f->dims = *dims;
    f->g = g;
    f->opts = ctx->opts;
    const WsSizes wsz = ws_sizes(g);
    const size_t pbytes = prob_doubles(g) * sizeof(double);
    f->bytes = wsz.total + pbytes;
    cudaError_t e = cudaMalloc(&f->mem, f->bytes);
    if (e != cudaSuccess) {
        delete f;
        return set_err(ctx, CYQ_CUDA_ERR, cudaGetErrorString(e));
    }
    f->ws = carve(f->mem, wsz);
    f->prob = carve_prob(reinterpret_cast<double *>(static_cast<char *>(f->mem) + wsz.total), g);
    f->owns_prob = true;
    if (mem == CYQ_MEM_DEVICE) {
        const ProbView src = view_of(prob);
        const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu;
        const std::pair<const double *, const double *> parts[] = {
            {src.A, f->prob.A}, {src.B, f->prob.B}, {src.R, f->prob.R}, {src.S, f->prob.S},
            {src.Q, f->prob.Q}, {src.f, f->prob.f}, {src.r, f->prob.r}, {src.q, f->prob.q},
            {src.x_init, f->prob.x_init}};
        const size_t cnt[] = {B * N * nx * nx, B * N * nx * nu, B * N * nu * nu,
                              B * N * nu * nx, B * (N + 1) * nx * nx, B * N * nx, B * N * nu,
                              B * (N + 1) * nx, B * nx};
        for (int i = 0; i < 9; ++i)
            CU(cudaMemcpyAsync(const_cast<double *>(parts[i].second), parts[i].first,
                               cnt[i] * sizeof(double), cudaMemcpyDeviceToDevice,
                               ctx->stream));
    } else {
        rc = copy_prob_h2d(ctx, g, prob, f->prob);
        if (rc) {
            cyq_factor_destroy(f);
            return rc;
        }
    }
    rc = launch_pipeline(ctx, g, f->prob, f->ws, nullptr, false);
    f->schur_path = ctx->schur_path;
    if (rc == CYQ_OK)
        rc = decode_status(ctx, g, f->ws.fail, status);
    *out = f;
    return rc;
}

int cyq_solve_batch(cyq_ctx *ctx, const cyq_factor *f, const cyq_ocp_batch *prob,
                    const cyq_rhs_batch *rhs, const cyq_sol_batch *sol, int mem) {
    if (!ctx || !f || !rhs || !sol)
        return set_err(ctx, CYQ_INVALID_ARG, "null argument");
    (void)prob; // the factor keeps its own device copy of the problem
    const Geo &g = f->g;
    CU(cudaSetDevice(ctx->device));
    const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu;
    const size_t rd = B * (N * nu + (N + 1) * nx + N * nx);
    const size_t sd = sol_doubles(g);
    int rc = ensure(ctx, &ctx->hbuf, &ctx->hbuf_bytes, (rd + sd) * sizeof(double));
    if (rc)
        return rc;
    double *base = static_cast<double *>(ctx->hbuf);
    ProbView p = f->prob;
    SolView sv;
    if (mem == CYQ_MEM_DEVICE) {
        p.ru = rhs->ru;
        p.qx = rhs->qx;
        p.fd = rhs->fd;
        sv = SolView{sol->u, sol->x, sol->lam};
    } else {
        double *ru = base, *qx = ru + B * N * nu, *fd = qx + B * (N + 1) * nx;
        CU(cudaMemcpyAsync(ru, rhs->ru, B * N * nu * 8, cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaMemcpyAsync(qx, rhs->qx, B * (N + 1) * nx * 8, cudaMemcpyHostToDevice,
                           ctx->stream));
        CU(cudaMemcpyAsync(fd, rhs->fd, B * N * nx * 8, cudaMemcpyHostToDevice, ctx->stream));
        p.ru = ru;
        p.qx = qx;
        p.fd = fd;
        double *s0 = base + rd;
        sv = SolView{s0, s0 + B * N * nu, s0 + B * N * nu + B * (N + 1) * nx};
    }
    rc = launch_solve(ctx, g, p, f->ws, sv, f->opts);
    if (rc)
        return rc;
    if (mem != CYQ_MEM_DEVICE) {
        CU(cudaMemcpyAsync(sol->u, sv.u, B * N * nu * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(sol->x, sv.x, B * (N + 1) * nx * 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CU(cudaMemcpyAsync(sol->lam, sv.lam, B * N * nx * 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    return CYQ_OK;
}

int cyq_factor_update_batch(cyq_ctx *ctx, cyq_factor *f, const cyq_ocp_batch *p_new, int64_t ny,
                            const double *C, const double *D, const double *ds_stage, int64_t ny_term,
                            const double *C_term, const double *ds_term, double rho, int mem,
                            cyq_update_report *report) {
    if (!ctx || !f || !p_new || ny < 0 || ny_term < 0 || (ny > 0 && (!C || !D || !ds_stage)) ||
        (ny_term > 0 && (!C_term || !ds_term)))
        return set_err(ctx, CYQ_INVALID_ARG, "null argument");
    const Geo g = f->g;
    const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu, P = g.P;
    CU(cudaSetDevice(ctx->device));
    CU(cudaStreamSynchronize(ctx->stream));
    // ---- dSigma on the host: per-column ranks (kkt_update.cpp:392-409) -----
    std::vector<double> hds(B * N * (size_t)ny), hdt(B * (size_t)ny_term);
    if (mem == CYQ_MEM_DEVICE) {
        if (!hds.empty())
            CU(cudaMemcpy(hds.data(), ds_stage, hds.size() * 8, cudaMemcpyDeviceToHost));
        if (!hdt.empty())
            CU(cudaMemcpy(hdt.data(), ds_term, hdt.size() * 8, cudaMemcpyDeviceToHost));
    } else {
        std::copy(ds_stage, ds_stage + hds.size(), hds.begin());
        std::copy(ds_term, ds_term + hdt.size(), hdt.begin());
    }
    std::vector<int> upd, refac;
    std::vector<int64_t> rank(B * P, 0);
    int cap = 1;
    for (size_t b = 0; b < B; ++b)
        for (size_t c = 0; c < P; ++c) {
            int64_t r = 0;
            for (int s = 0; s < g.n; ++s) {
                const int j = g.stage_of((int)c, s);
                if (j < (int)N)
                    for (int64_t i = 0; i < ny; ++i)
                        r += hds[(b * N + j) * ny + i] != 0.0;
                if (j == 0)
                    for (int64_t i = 0; i < ny_term; ++i)
                        r += hdt[b * ny_term + i] != 0.0;
            }
            rank[b * P + c] = r;
            if (r == 0)
                continue;
            if ((double)r >= rho * (double)nx) {
                refac.push_back((int)(b * P + c));
            } else {
                upd.push_back((int)(b * P + c));
                cap = std::max<int>(cap, (int)r);
            }
        }
    if (report)
        for (size_t b = 0; b < B; ++b)
            report[b] = cyq_update_report{0, 0, 0, 0};
    if (upd.empty() && refac.empty())
        return CYQ_OK; // dSigma = 0: the factor already is the factor of p_new
    if (!upd.empty() && update_smem_bytes(g.nx, g.nu, cap) > 227 * 1024) { // too wide: refactorize
        refac.insert(refac.end(), upd.begin(), upd.end());
        upd.clear();
    }
    // ---- device copies: p_new -> the factor's problem, update data --------
    const size_t nC = B * N * ny * nx, nD = B * N * ny * nu, nds = B * N * ny, nCt = B * ny_term * nx,
                 nt = B * ny_term;
    const size_t scratch = (nC + nD + nds + nCt + nt) * 8 + (upd.size() + refac.size()) * 4 + upd.size() * 4 + 256;
    int rc = ensure(ctx, &ctx->augbuf, &ctx->augbuf_bytes, scratch);
    if (rc)
        return rc;
    double *dC = static_cast<double *>(ctx->augbuf), *dD = dC + nC, *dds = dD + nD, *dCt = dds + nds,
           *ddt = dCt + nCt;
    int *dlist = reinterpret_cast<int *>(ddt + nt), *dbreak = dlist + upd.size() + refac.size();
    const cudaMemcpyKind kind = mem == CYQ_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    {
        const ProbView src = view_of(p_new);
        const std::pair<const double *, const double *> parts[] = {
            {src.A, f->prob.A}, {src.B, f->prob.B}, {src.R, f->prob.R}, {src.S, f->prob.S},
            {src.Q, f->prob.Q}, {src.f, f->prob.f}, {src.r, f->prob.r}, {src.q, f->prob.q},
            {src.x_init, f->prob.x_init}};
        const size_t cnt[] = {B * N * nx * nx, B * N * nx * nu, B * N * nu * nu, B * N * nu * nx,
                              B * (N + 1) * nx * nx, B * N * nx, B * N * nu, B * (N + 1) * nx, B * nx};
        for (int i = 0; i < 9; ++i) {
            if (!parts[i].first)
                return set_err(ctx, CYQ_INVALID_ARG, "null problem array");
            CU(cudaMemcpyAsync(const_cast<double *>(parts[i].second), parts[i].first, cnt[i] * 8, kind,
                               ctx->stream));
        }
    }
    if (nC) {
        CU(cudaMemcpyAsync(dC, C, nC * 8, kind, ctx->stream));
        CU(cudaMemcpyAsync(dD, D, nD * 8, kind, ctx->stream));
        CU(cudaMemcpyAsync(dds, hds.data(), nds * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (nCt) {
        CU(cudaMemcpyAsync(dCt, C_term, nCt * 8, kind, ctx->stream));
        CU(cudaMemcpyAsync(ddt, hdt.data(), nt * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    CU(cudaMemsetAsync(f->ws.fail, 0xFF, sizeof(unsigned long long) * B, ctx->stream));
    // ---- low-rank column updates (update.cu) --------------------------------
    std::vector<int> broke;
    if (!upd.empty()) {
        CU(cudaMemcpyAsync(dlist, upd.data(), upd.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaMemsetAsync(dbreak, 0, upd.size() * 4, ctx->stream));
        UpdateArgs ua{g, f->prob, f->ws.fac, f->ws.trail, dlist, (int)upd.size(), dD, dC, dCt, dds, ddt,
                      (int)ny, (int)ny_term, cap, dbreak};
        {
            Timed t(ctx, 0);
            if (!launch_update_columns(ctx->stream, ua))
                return set_err(ctx, CYQ_INVALID_ARG, "update: stage shape too large");
        }
        CU(cudaGetLastError());
        std::vector<int> hb(upd.size());
        CU(cudaMemcpyAsync(hb.data(), dbreak, hb.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        std::vector<int> kept;
        for (size_t i = 0; i < upd.size(); ++i)
            (hb[i] ? refac : kept).push_back(upd[i]);
        upd.swap(kept);
    }
    // ---- refactorized columns: the panel kernels over the listed chains ----
    if (!refac.empty()) {
        int *dref = dlist + 0; // reuse the list slot (the update kernel is done reading it)
        CU(cudaMemcpyAsync(dref, refac.data(), refac.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
        RiccatiArgs ra{g, f->prob, f->ws.fac, f->ws.y, f->ws.wl, f->ws.trail, f->ws.fail, f->ws.consts, 1,
                       nullptr};
        ra.chain_list = dref;
        ra.n_list = (int)refac.size();
        if (!riccati_staged(g))
            return set_err(ctx, CYQ_INVALID_ARG, "update: refactorization needs the staged panel kernels");
        Timed t(ctx, 0);
        bool done = false;
        if ((long long)refac.size() <= 2LL * ctx->opts.sms)
            done = launch_riccati_pc(g, ctx->stream, ra);
        if (!done)
            done = launch_riccati_warp(g, ctx->stream, ra, LaunchOpts{});
        if (!done)
            done = launch_riccati_cta(g, ctx->stream, ra);
        if (!done)
            launch_riccati(g, ctx->opts, ctx->stream, ra);
    }
    CU(cudaGetLastError());
    // ---- Schur complement + CR factor re-formed from the updated columns ---
    SchurArgs sa{g, f->prob, f->ws.fac, f->ws.y, f->ws.trail, f->ws.schur, f->ws.lamc, nullptr,
                 f->ws.fail, 1, 0};
    rc = launch_schur(ctx, g, sa, f->opts);
    if (rc)
        return rc;
    f->schur_path = ctx->schur_path;
    if (report) {
        for (int ch : upd)
            ++report[ch / P].columns_updated;
        for (int ch : refac)
            ++report[ch / P].columns_refactored;
        for (size_t b = 0; b < B; ++b) {
            bool any = false;
            for (size_t c = 0; c < P; ++c)
                any = any || rank[b * P + c] > 0;
            report[b].schur_refactored = any;
        }
    }
    return decode_status(ctx, g, f->ws.fail, nullptr);
}

int cyq_factor_destroy(cyq_factor *f) {
    if (!f)
        return CYQ_OK;
    if (f->mem) {
        cudaSetDevice(f->ctx->device);
        cudaStreamSynchronize(f->ctx->stream);
        cudaFree(f->mem);
    }
    delete f;
    return CYQ_OK;
}

int cyq_factor_materialize(const cyq_factor *f, int64_t inst, double *LH, double *LB,
                           double *Acl, double *LA) {
    if (!f || inst < 0 || inst >= f->g.batch)
        return set_err(nullptr, CYQ_INVALID_ARG, "bad factor / instance");
    cyq_ctx *ctx = f->ctx;
    const Geo &g = f->g;
    const size_t per = (size_t)g.P * g.n * g.NPT * kTileElems;
    std::vector<double> h(per);
    CU(cudaMemcpy(h.data(), f->ws.fac + (size_t)inst * per, per * sizeof(double),
                  cudaMemcpyDeviceToHost));
    const int nu = g.nu, nx = g.nx, nux = g.nux, top = 8 * g.CT, P = g.P, n = g.n;
    auto at = [&](int c, int s, int r, int col) {
        const int ti = r / 8, tj = col / 8;
        const int st = ti < g.CT ? tri_index(ti, tj) : g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
        return h[(((size_t)c * n + s) * g.NPT + st) * kTileElems + (r % 8) * 8 + col % 8];
    };
    for (int s = 0; s < n; ++s)
        for (int c = 0; c < P; ++c) {
            if (LH)
                for (int r = 0; r < nux; ++r)
                    for (int k = 0; k < nux; ++k)
                        LH[(((size_t)s * P + c) * nux + r) * nux + k] = k <= r ? at(c, s, r, k) : 0.0;
            if (LB)
                for (int r = 0; r < nx; ++r)
                    for (int k = 0; k < nu; ++k)
                        LB[(((size_t)s * P + c) * nx + r) * nu + k] = at(c, s, top + r, k);
            // Acl = ALQ L_Q' ; LA = ALQ at the last stage
            for (int r = 0; r < nx; ++r)
                for (int k = 0; k < nx; ++k) {
                    double v = 0;
                    for (int m = 0; m <= k; ++m)
                        v += at(c, s, top + r, nu + m) * at(c, s, nu + k, nu + m);
                    if (Acl)
                        Acl[(((size_t)s * P + c) * nx + r) * nx + k] = v;
                    if (LA && s == n - 1)
                        LA[((size_t)c * nx + r) * nx + k] = at(c, s, top + r, nu + k);
                }
        }
    return CYQ_OK;
}

int cyq_ctx_set_option(cyq_ctx *ctx, int option, int64_t value) {
    if (!ctx)
        return set_err(nullptr, CYQ_INVALID_ARG, "null context");
    LaunchOpts &o = ctx->opts;
    auto bad = [&] { return set_err(ctx, CYQ_INVALID_ARG, "option value out of range"); };
    switch (option) {
    case CYQ_OPT_PANEL: if (value < 0 || value > 6) return bad(); o.panel = (int)value; break;
    case CYQ_OPT_SCHUR: if (value < 0 || value > 2) return bad(); o.schur = (int)value; break;
    case CYQ_OPT_SCHUR_WARPS:
        if (value != 0 && value != 2 && value != 4) return bad();
        o.schur_warps = (int)value;
        break;
    case CYQ_OPT_SCHUR_CLUSTER: o.schur_cluster = value != 0; break;
    case CYQ_OPT_SPLIT: if (value < 1 || value > 8) return bad(); o.split = (int)value; break;
    case CYQ_OPT_BACKSUB: if (value < 0 || value > 1) return bad(); o.backsub = (int)value; break;
    case CYQ_OPT_FUSED_AUGMENT: o.fused_aug = value != 0; break;
    case CYQ_OPT_PANEL_WARPS: if (value < 0 || value > 4) return bad(); o.panel_warps = (int)value; break;
    case CYQ_OPT_TAIL: if (value < 0 || value > 2) return bad(); o.tail = (int)value; break;
    case CYQ_OPT_PHASE_PROF: o.phase_prof = value != 0; break;
    case CYQ_OPT_ASYNC_STATUS: o.async_status = value != 0; break;
    case CYQ_OPT_VLEN:
        if (value < 1 || value > 1024 || (value & (value - 1)))
            return bad();
        o.vlen = (int)value;
        break;
    case CYQ_OPT_GRAPHS: o.graphs = value != 0; break;
    default: return set_err(ctx, CYQ_INVALID_ARG, "unknown option");
    }
    return CYQ_OK;
}

int cyq_ctx_wait_status(cyq_ctx *ctx, cyq_status *status, int64_t n) {
    if (!ctx)
        return set_err(nullptr, CYQ_INVALID_ARG, "null context");
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->pend_batch < 0)
        return CYQ_OK;
    int worst = CYQ_OK;
    for (int64_t b = 0; b < ctx->pend_batch; ++b) {
        const unsigned long long k = ctx->hpend[b];
        cyq_status st{};
        st.instance = b;
        if (k != ~0ull) {
            st.code = CYQ_PIVOT_FAIL;
            st.kind = (int)(k >> 60);
            st.column_or_level = (int64_t)((k >> 40) & 0xFFFFF);
            st.stage = (int64_t)((k >> 20) & 0xFFFFF);
            st.pivot = (int64_t)(k & 0xFFFFF);
            worst = CYQ_PIVOT_FAIL;
        }
        if (status && b < n)
            status[b] = st;
    }
    if (worst != CYQ_OK)
        set_err(ctx, worst, "factorization pivot failure (see status)");
    return worst;
}

int cyq_ctx_get_option(cyq_ctx *ctx, int option, int64_t *value) {
    if (!ctx || !value)
        return set_err(ctx, CYQ_INVALID_ARG, "null argument");
    const LaunchOpts &o = ctx->opts;
    const int v[CYQ_OPT_COUNT] = {o.panel,       o.schur,        o.schur_warps, o.schur_cluster,
                                  o.split,       o.backsub,      o.fused_aug,   o.panel_warps,
                                  o.tail,        o.phase_prof,   o.async_status, o.graphs,
                                  o.vlen};
    if (option < 0 || option >= CYQ_OPT_COUNT)
        return set_err(ctx, CYQ_INVALID_ARG, "unknown option");
    *value = v[option];
    return CYQ_OK;
}

int cyq_factor_materialize_schur(const cyq_factor *f, int64_t inst, double *T, double *Mfwd, double *Mbwd,
                                 double *W, double *schur_diag, double *schur_sub, double *cr_L,
                                 double *cr_U, double *cr_Y, double *cr_Lbase) {
    if (!f || inst < 0 || inst >= f->g.batch)
        return set_err(nullptr, CYQ_INVALID_ARG, "bad factor / instance");
    cyq_ctx *ctx = f->ctx;
    const Geo &g = f->g;
    SchurBlocks L{};
    const bool ok = f->schur_path == 0 ? schur_fused_blocks(g, L) : f->schur_path == 1 && schur_big_blocks(g, L);
    if (!ok)
        return set_err(ctx, CYQ_INVALID_ARG,
                       "materialize_schur: the factor's Schur path (per-level / scalar kernels) keeps no "
                       "persistent Schur blocks");
    const int P = g.P, nx = g.nx, XT = (nx + 7) / 8, n = g.n, nu = g.nu, top = 8 * g.CT;
    const size_t NF = (size_t)XT * XT, NL = (size_t)XT * (XT + 1) / 2;
    const size_t TF = 64 * NF, TLb = 64 * (L.full ? NF : NL);
    CU(cudaSetDevice(ctx->device));
    std::vector<double> ws((size_t)L.total), tr((size_t)P * g.NTT * kTileElems),
        fac((size_t)P * g.NPT * kTileElems);
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaMemcpy(ws.data(), f->ws.schur + (size_t)inst * L.total, ws.size() * 8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(tr.data(), f->ws.trail + (size_t)inst * P * g.NTT * kTileElems, tr.size() * 8,
                  cudaMemcpyDeviceToHost));
    for (int c = 0; c < P; ++c) // the last stage's pivot tiles of every column (L_Q, LA)
        CU(cudaMemcpy(fac.data() + (size_t)c * g.NPT * kTileElems,
                      f->ws.fac + (((size_t)inst * P + c) * n + (n - 1)) * g.NPT * kTileElems,
                      (size_t)g.NPT * kTileElems * 8, cudaMemcpyDeviceToHost));
    // element (r, k) of a tile-ordered block at `base`
    auto lower = [&](const double *base, int r, int k) {
        if (L.full)
            return base[((r / 8) * XT + k / 8) * 64 + (r % 8) * 8 + k % 8];
        return k <= r ? base[(tri_index(r / 8, k / 8)) * 64 + (r % 8) * 8 + k % 8] : 0.0;
    };
    auto full = [&](const double *base, int r, int k) { return base[((r / 8) * XT + k / 8) * 64 + (r % 8) * 8 + k % 8]; };
    // symmetric blocks keep their lower triangle (the upper tiles of a full
    // layout are not written)
    auto sym = [&](const double *base, int r, int k) { return lower(base, std::max(r, k), std::min(r, k)); };
    auto Tel = [&](int c, int r, int k) { // T_c = L_Q^{-T} (upper)
        const double *b = ws.data() + L.Tt + c * TLb;
        if (L.tt_is_inverse)
            return full(b, k, r);
        return k >= r ? b[(tri_index(k / 8, r / 8)) * 64 + (r % 8) * 8 + k % 8] : 0.0;
    };
    auto LAel = [&](int c, int r, int k) { // LA_c = ALQ of the last stage
        const int ti = (top + r) / 8, tj = (nu + k) / 8;
        const int t = g.CT * (g.CT + 1) / 2 + (ti - g.CT) * g.CT + tj;
        return fac[(size_t)c * g.NPT * kTileElems + t * 64 + ((top + r) % 8) * 8 + (nu + k) % 8];
    };
    auto Mfel = [&](int c, int r, int k) { // Mfwd_c = -(trailing coupling block)
        const int rr = std::max(r, k), kk = std::min(r, k);
        return -tr[((size_t)c * g.NTT + tri_index(rr / 8, kk / 8)) * 64 + (rr % 8) * 8 + kk % 8];
    };
    const size_t nn = (size_t)nx * nx;
    std::vector<double> Wv((size_t)P * nn), Mf((size_t)P * nn), Mb((size_t)P * nn);
    for (int c = 0; c < P; ++c)
        for (int r = 0; r < nx; ++r)
            for (int k = 0; k < nx; ++k) {
                double w = 0; // W_c = T_c LA_c'
                for (int m = 0; m < nx; ++m)
                    w += Tel(c, r, m) * LAel(c, k, m);
                Wv[c * nn + r * nx + k] = w;
                Mf[c * nn + r * nx + k] = Mfel(c, r, k);
                Mb[c * nn + r * nx + k] = sym(ws.data() + L.Mb + c * TLb, r, k);
                if (T)
                    T[c * nn + r * nx + k] = Tel(c, r, k);
            }
    if (W)
        memcpy(W, Wv.data(), Wv.size() * 8);
    if (Mfwd)
        memcpy(Mfwd, Mf.data(), Mf.size() * 8);
    if (Mbwd)
        memcpy(Mbwd, Mb.data(), Mb.size() * 8);
    // assemble_schur (kkt_factor.cpp:194-212): diag[c] = Mfwd_c + Mbwd_{c+1},
    // subdiag[c-1] = -W_c' (block (c, c-1)), subdiag[P-1] = 0
    for (int c = 0; c < P; ++c)
        for (size_t e = 0; e < nn; ++e) {
            if (schur_diag)
                schur_diag[c * nn + e] = Mf[c * nn + e] + Mb[((c + 1) % P) * nn + e];
            if (schur_sub) {
                const int r = (int)(e / nx), k = (int)(e % nx);
                schur_sub[c * nn + e] = c + 1 < P ? -Wv[(c + 1) * nn + k * nx + r] : 0.0;
            }
        }
    // CR levels: L (from the stored L^{-1}), U, Y per level slot; L_base
    auto inv_lower = [&](const double *Li, double *out) { // out = (Li)^{-1}, Li lower nx x nx
        for (int j = 0; j < nx; ++j)
            for (int i = 0; i < nx; ++i) {
                if (i < j) {
                    out[i * nx + j] = 0.0;
                    continue;
                }
                double s = i == j ? 1.0 : 0.0;
                for (int m = j; m < i; ++m)
                    s -= Li[i * nx + m] * out[m * nx + j];
                out[i * nx + j] = s / Li[i * nx + i];
            }
    };
    std::vector<double> tmp(nn);
    for (int l = 0; l < L.cr_levels; ++l) {
        const int half = (P >> l) / 2;
        const long long o0 = P - (P >> l);
        for (int mm = 0; mm < half; ++mm) {
            const size_t slot = (size_t)(o0 + mm);
            for (int r = 0; r < nx; ++r)
                for (int k = 0; k < nx; ++k) {
                    tmp[r * nx + k] = lower(ws.data() + L.Li + slot * TLb, r, k);
                    if (cr_U)
                        cr_U[slot * nn + r * nx + k] = full(ws.data() + L.U + slot * TF, r, k);
                    if (cr_Y)
                        cr_Y[slot * nn + r * nx + k] = full(ws.data() + L.Y + slot * TF, r, k);
                }
            if (cr_L)
                inv_lower(tmp.data(), cr_L + slot * nn);
        }
    }
    if (cr_Lbase) {
        if (g.tail <= 1) {
            for (int r = 0; r < nx; ++r)
                for (int k = 0; k < nx; ++k)
                    tmp[r * nx + k] = lower(ws.data() + L.Lb, r, k);
            inv_lower(tmp.data(), cr_Lbase);
        } else {
            memset(cr_Lbase, 0, nn * 8); // PCR tail: no single base block
        }
    }
    return CYQ_OK;
}

int cyq_ctx_profile(cyq_ctx *ctx, int enable) {
    if (!ctx)
        return CYQ_INVALID_ARG;
    ctx->profile = enable != 0;
    return CYQ_OK;
}

int cyq_ctx_profile_read(cyq_ctx *ctx, double *ms, int64_t *launches, int reset) {
    // launches[k] = kernel launches of kind k (several kernels may share one
    // timed bracket, e.g. the per-level CR kernels); ms[k] = their time
    if (!ctx)
        return CYQ_INVALID_ARG;
    CU(cudaStreamSynchronize(ctx->stream));
    for (auto &e : ctx->ev) {
        float t = 0;
        CU(cudaEventElapsedTime(&t, e.second.first, e.second.second));
        ctx->ms[e.first] += t;
        ctx->pool.push_back(e.second.first);
        ctx->pool.push_back(e.second.second);
    }
    ctx->ev.clear();
    for (int k = 0; k < 5; ++k) {
        if (ms)
            ms[k] = ctx->ms[k];
        if (launches)
            launches[k] = ctx->kernels[k];
        if (reset) {
            ctx->ms[k] = 0;
            ctx->kernels[k] = 0;
        }
    }
    return CYQ_OK;
}

int cyq_augment_hessians_batch(cyq_ctx *ctx, const cyq_dims *dims, int64_t ny, const double *R,
                               const double *S, const double *Q, const double *D, const double *C,
                               const double *sigma, double gamma_inv, double *R_out, double *S_out,
                               double *Q_out) {
    if (!ctx || !dims || !R || !S || !Q || !D || !C || !sigma || !R_out || !S_out || !Q_out)
        return set_err(ctx, CYQ_INVALID_ARG, "null argument");
    if (dims->N < 1 || dims->nx < 1 || dims->nu < 1 || dims->batch < 1 || ny < 1)
        return set_err(ctx, CYQ_INVALID_ARG, "dims: N, nx, nu, batch, ny must be >= 1");
    CU(cudaSetDevice(ctx->device));
    {
        Timed t(ctx, 4);
        if (!launch_augment(ctx->stream, (int)dims->batch, (int)dims->N, (int)dims->nx, (int)dims->nu,
                            (int)ny, R, S, Q, D, C, sigma, gamma_inv, R_out, S_out, Q_out))
            return set_err(ctx, CYQ_INVALID_ARG, "augment: ny <= 64 and nx + nu <= 64 supported");
    }
    CU(cudaGetLastError());
    return CYQ_OK;
}

int cyq_solve_newton_batch(cyq_ctx *ctx, const cyq_dims *dims, const cyq_ocp_batch *prob, int64_t ny,
                           const double *D, const double *C, const double *sigma, double gamma_inv,
                           const cyq_sol_batch *sol, cyq_status *status) {
    if (!ctx || !prob || !sol || !D || !C || !sigma)
        return set_err(ctx, CYQ_INVALID_ARG, "null argument");
    if (ny < 1 || ny > 64)
        return set_err(ctx, CYQ_INVALID_ARG, "ny must be in [1, 64]");
    Geo g;
    int rc = make_geo(ctx, dims, g);
    if (rc)
        return rc;
    CU(cudaSetDevice(ctx->device));
    const WsSizes wsz = ws_sizes(g);
    rc = ensure(ctx, &ctx->wsbuf, &ctx->wsbuf_bytes, wsz.total);
    if (rc)
        return rc;
    FactorWS ws = carve(ctx->wsbuf, wsz);
    ProbView pv = view_of(prob);
    if (riccati_warp_fuses_aug(g, (int)ny, ctx->opts)) {
        // assembly fused into the stage-panel loads: the augmented Hessians
        // never touch HBM
        pv.aD = D;
        pv.aC = C;
        pv.asig = sigma;
        pv.ny = (int)ny;
        pv.gamma_inv = gamma_inv;
    } else {
        // assembly kernel into context scratch, then the plain pipeline
        const size_t B = g.batch, N = g.N, nx = g.nx, nu = g.nu;
        const size_t nR = B * N * nu * nu, nS = B * N * nu * nx, nQ = B * (N + 1) * nx * nx;
        rc = ensure(ctx, &ctx->augbuf, &ctx->augbuf_bytes, (nR + nS + nQ) * sizeof(double));
        if (rc)
            return rc;
        double *Ro = static_cast<double *>(ctx->augbuf), *So = Ro + nR, *Qo = So + nS;
        {
            Timed t(ctx, 4);
            if (!launch_augment(ctx->stream, g.batch, g.N, g.nx, g.nu, (int)ny, pv.R, pv.S, pv.Q, D, C,
                                sigma, gamma_inv, Ro, So, Qo))
                return set_err(ctx, CYQ_INVALID_ARG, "augment: ny <= 64 and nx + nu <= 64 supported");
        }
        CU(cudaGetLastError());
        pv.R = Ro;
        pv.S = So;
        pv.Q = Qo;
    }
    SolView sv{sol->u, sol->x, sol->lam};
    rc = run_pipeline(ctx, g, pv, ws, &sv, true);
    if (rc)
        return rc;
    return finish_status(ctx, g, ws.fail, status);
}

int cyq_al_gradients_batch(cyq_ctx *ctx, const cyq_dims *dims, int64_t ny, const cyq_ocp_batch *prob,
                           const double *D, const double *C, const double *bl, const double *bu,
                           const double *u, const double *x, const double *y, const double *sigma,
                           const double *ubar, const double *xbar, double gamma_inv, double *ru,
                           double *qx, double *yhat, double *cres) {
    if (!ctx || !dims || !prob || !D || !C || !bl || !bu || !u || !x || !y || !sigma || !ubar || !xbar ||
        !ru || !qx || !yhat || !cres)
        return set_err(ctx, CYQ_INVALID_ARG, "null argument");
    if (dims->N < 1 || dims->nx < 1 || dims->nu < 1 || dims->batch < 1 || ny < 1)
        return set_err(ctx, CYQ_INVALID_ARG, "dims: N, nx, nu, batch, ny must be >= 1");
    CU(cudaSetDevice(ctx->device));
    GradArgs ga{(int)dims->batch, (int)dims->N, (int)dims->nx, (int)dims->nu, (int)ny,
                prob->R, prob->S, prob->Q, prob->A, prob->B, prob->f, prob->r, prob->q,
                D, C, bl, bu, u, x, y, sigma, ubar, xbar, gamma_inv, ru, qx, yhat, cres};
    {
        Timed t(ctx, 4);
        if (!launch_al_gradients(ctx->stream, ga))
            return set_err(ctx, CYQ_INVALID_ARG, "al_gradients: nx + nu + ny too large");
    }
    CU(cudaGetLastError());
    return CYQ_OK;
}

int cyq_line_search_batch(cyq_ctx *ctx, int64_t batch, int64_t m, const double *alpha,
                          const double *delta, const double *eta, const double *beta, double *tau,
                          int32_t *status, int64_t *iterations) {
    if (!ctx || !eta || !beta || !tau || (m > 0 && (!alpha || !delta)))
        return set_err(ctx, CYQ_INVALID_ARG, "null argument");
    if (batch < 1 || m < 0)
        return set_err(ctx, CYQ_INVALID_ARG, "batch >= 1 and m >= 0 required");
    CU(cudaSetDevice(ctx->device));
    const size_t tw = (size_t)batch * (size_t)(m > 0 ? m : 1) * 2 * sizeof(double);
    int rc = ensure(ctx, &ctx->lsbuf, &ctx->lsbuf_bytes, tw + (size_t)batch * sizeof(int));
    if (rc)
        return rc;
    int *dstat = reinterpret_cast<int *>(static_cast<char *>(ctx->lsbuf) + tw);
    LineSearchArgs la{batch, m, alpha, delta, eta, beta, tau, dstat,
                      reinterpret_cast<long long *>(iterations), static_cast<double *>(ctx->lsbuf)};
    {
        Timed t(ctx, 4);
        launch_line_search(ctx->stream, la);
    }
    CU(cudaGetLastError());
    std::vector<int> hs((size_t)batch);
    CU(cudaMemcpyAsync(hs.data(), dstat, hs.size() * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    int worst = CYQ_OK;
    for (int64_t k = 0; k < batch; ++k) {
        const int code = hs[(size_t)k] == 0 ? CYQ_OK : (hs[(size_t)k] == 1 ? CYQ_INVALID_ARG : CYQ_CUDA_ERR);
        if (status)
            status[k] = code;
        worst = std::max(worst, code);
    }
    if (worst == CYQ_INVALID_ARG)
        set_err(ctx, worst, "line_search_exact: not a descent direction (psi'(0) > 0) for some instance");
    return worst;
}

const char *cyq_version(void) {
    return "cyqlone_b200 0.1 sm_100a: riccati_panel_kernel (DMMA 8x8x4 f64 stage panels), "
           "schur_cr_kernel, backsub_kernel";
}

} // extern "C"
