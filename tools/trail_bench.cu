// Microbenchmark of the CTA panel's trailing-update inner loop (riccati_cta.cu):
// one CTA of NW warps per SM, every warp applying C_k -= L_i L_j' (two
// dependent DMMA.8x8x4 on one accumulator tile, operands two 512-byte tiles
// from shared memory) to its NT register tiles, in several loop shapes.
// Prints cycles per tile update per warp and the DMMA-pipe share
// (4 warps per SM sub-partition x 32 pipe cycles per update).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/trail_bench tools/trail_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Frag { double a, b; };
__device__ __forceinline__ void dmma(Frag &c, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c.a), "+d"(c.b) : "d"(a), "d"(b));
}
// volatile: the loads stay inside the timed loop, in program order with the DMMAs
__device__ __forceinline__ Frag ld_frag(const double *t, int lane) {
    Frag f;
    const unsigned a = (unsigned)__cvta_generic_to_shared(t) + 16 * lane;
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(f.a), "=d"(f.b) : "r"(a));
    return f;
}

constexpr int NT = 14, TT = 21;
__constant__ unsigned short c_list[16 * 32];

// MODE 0: load, 2 dependent DMMAs, next (no prefetch)
// MODE 1: operands of tile k+1 loaded before tile k's DMMAs (distinct registers)
// MODE 2: tiles in pairs: 4 operand tiles ahead, DMMAs interleaved a0 a1 b0 b1
// MODE 3: as 2 with a shared row operand per pair (3 loads per pair)
// MODE 4: DMMA only (operands loaded once)
// MODE 5: loads only (no DMMA; sum into acc by DADD on one element to keep them live)
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(long long *out, const int *idx, int iters, int stride, int cnt, int kbv) {
    extern __shared__ double sm0[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (TT + 8) * 64; i += blockDim.x)
        sm0[i] = 1e-3 * (i % 17);
    __syncthreads();
    int ti[NT], tj[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        ti[t] = idx[(warp * NT + t) * 2] * 64;
        tj[t] = idx[(warp * NT + t) * 2 + 1] * 64;
    }
    Frag acc[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t)
        acc[t] = Frag{1.0 + t, 2.0};
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const double *sm = sm0 + ((it * stride) & 0x1C0); // runtime offset: the loads stay in the loop
        if (MODE == 0) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const Frag li = ld_frag(sm + ti[t], lane), lj = ld_frag(sm + tj[t], lane);
                dmma(acc[t], -li.a, lj.a);
                dmma(acc[t], -li.b, lj.b);
            }
        } else if (MODE == 1) {
            Frag li = ld_frag(sm + ti[0], lane), lj = ld_frag(sm + tj[0], lane);
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                Frag ni{0, 0}, nj{0, 0};
                if (t + 1 < NT) {
                    ni = ld_frag(sm + ti[t + 1], lane);
                    nj = ld_frag(sm + tj[t + 1], lane);
                }
                dmma(acc[t], -li.a, lj.a);
                dmma(acc[t], -li.b, lj.b);
                li = ni;
                lj = nj;
            }
        } else if (MODE == 2 || MODE == 3) {
            Frag li0 = ld_frag(sm + ti[0], lane), lj0 = ld_frag(sm + tj[0], lane);
            Frag li1 = MODE == 3 ? li0 : ld_frag(sm + ti[1], lane), lj1 = ld_frag(sm + tj[1], lane);
#pragma unroll
            for (int t = 0; t < NT; t += 2) {
                Frag ni0{0, 0}, nj0{0, 0}, ni1{0, 0}, nj1{0, 0};
                if (t + 2 < NT) {
                    ni0 = ld_frag(sm + ti[t + 2], lane);
                    nj0 = ld_frag(sm + tj[t + 2], lane);
                    ni1 = MODE == 3 ? ni0 : ld_frag(sm + ti[t + 3], lane);
                    nj1 = ld_frag(sm + tj[t + 3], lane);
                }
                dmma(acc[t], -li0.a, lj0.a);
                dmma(acc[t + 1], -li1.a, lj1.a);
                dmma(acc[t], -li0.b, lj0.b);
                dmma(acc[t + 1], -li1.b, lj1.b);
                li0 = ni0; lj0 = nj0; li1 = ni1; lj1 = nj1;
            }
        } else if (MODE == 6) { // as the kernel: runtime count with a break per tile, prefetch-1
            Frag li = ld_frag(sm + ti[0], lane), lj = ld_frag(sm + tj[0], lane);
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (t >= cnt)
                    break;
                Frag ni{0, 0}, nj{0, 0};
                if (t + 1 < NT) {
                    ni = ld_frag(sm + ti[t + 1], lane);
                    nj = ld_frag(sm + tj[t + 1], lane);
                }
                dmma(acc[t], -li.a, lj.a);
                dmma(acc[t], -li.b, lj.b);
                li = ni;
                lj = nj;
            }
        } else if (MODE == 7 || MODE == 8) { // + tile ids from constant memory (+ predicated publish)
#define LTI(k) ((int)(c_list[warp * 32 + (k)] >> 8))
#define LTJ(k) ((int)(c_list[warp * 32 + (k)] & 255))
            int tjj = LTJ(0);
            Frag li = ld_frag(sm + LTI(0) * 64, lane), lj = ld_frag(sm + tjj * 64, lane);
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (t >= cnt)
                    break;
                Frag ni{0, 0}, nj{0, 0};
                int ntj = 0;
                if (t + 1 < NT) {
                    ntj = LTJ(t + 1);
                    ni = ld_frag(sm + LTI(t + 1) * 64, lane);
                    nj = ld_frag(sm + ntj * 64, lane);
                }
                dmma(acc[t], -li.a, lj.a);
                dmma(acc[t], -li.b, lj.b);
                if (MODE == 8 && tjj == kbv) {
                    double2 *d = reinterpret_cast<double2 *>(sm0 + (TT + 8) * 64 + LTI(t) * 64) + lane;
                    *d = make_double2(acc[t].a, acc[t].b);
                }
                li = ni;
                lj = nj;
                tjj = ntj;
            }
        } else if (MODE == 4) {
            const Frag li = ld_frag(sm + ti[0], lane), lj = ld_frag(sm + tj[0], lane);
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                dmma(acc[t], -li.a, lj.a);
                dmma(acc[t], -li.b, lj.b);
            }
        } else {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const Frag li = ld_frag(sm + ti[t], lane), lj = ld_frag(sm + tj[t], lane);
                acc[t].a += li.a;
                acc[t].b += lj.b;
            }
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int t = 0; t < NT; ++t)
        s += acc[t].a + acc[t].b;
    if (s == 1234.5678)
        out[1] = 1;
    if (threadIdx.x == 0 && blockIdx.x == 0)
        out[0] = t1 - t0;
}

template <int MODE> void run(const char *name, int nw, long long *out, const int *idx) {
    const int iters = 200;
    k<MODE><<<148, 32 * nw, (2 * TT + 8) * 64 * 8>>>(out, idx, 10, 64, NT, 100);
    cudaDeviceSynchronize();
    k<MODE><<<148, 32 * nw, (2 * TT + 8) * 64 * 8>>>(out, idx, iters, 64, NT, 100);
    cudaDeviceSynchronize();
    const double cyc = double(out[0]) / (iters * NT);
    const double per_sp = (nw / 4.0) * 32.0;
    printf("{\"mode\": \"%s\", \"warps\": %d, \"cycles_per_update_per_warp\": %.1f, \"dmma_pipe_share\": %.3f, "
           "\"smem_bytes_per_clk\": %.1f}\n",
           name, nw, cyc, MODE == 5 ? 0.0 : per_sp / cyc, MODE == 4 ? 0.0 : nw * 1024.0 / cyc * (MODE == 3 ? 0.75 : 1.0));
}

int main() {
    long long *out;
    int *idx;
    cudaMallocManaged(&out, 64);
    cudaMallocManaged(&idx, 16 * NT * 2 * sizeof(int));
    unsigned s = 12345;
    for (int i = 0; i < 16 * NT * 2; ++i) {
        s = s * 1664525u + 1013904223u;
        idx[i] = (s >> 8) % TT;
    }
    unsigned short h[16 * 32];
    for (int i = 0; i < 16 * 32; ++i) {
        s = s * 1664525u + 1013904223u;
        const int a = (s >> 8) % TT, b = (s >> 16) % TT;
        h[i] = (unsigned short)((a << 8) | b);
    }
    cudaMemcpyToSymbol(c_list, h, sizeof h);
    for (int nw : {16, 12}) {
        run<6>("break-per-tile", nw, out, idx);
        run<7>("break+const-table", nw, out, idx);
        run<8>("break+const-table+publish", nw, out, idx);
        run<0>("load-then-dmma", nw, out, idx);
        run<1>("prefetch-1", nw, out, idx);
        run<2>("pairs-interleaved", nw, out, idx);
        run<3>("pairs-shared-row", nw, out, idx);
        run<4>("dmma-only", nw, out, idx);
        run<5>("loads-only", nw, out, idx);
    }
    return 0;
}
