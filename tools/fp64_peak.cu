// FP64 roofline denominators for the B200 (sm_100a): DFMA and DMMA
// (mma.sync m8n8k4 f64) throughput, plus the latencies that bound the
// sequential parts of the KKT factorization (sqrt, rsqrt, div, shfl).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
// Output: one JSON object on stdout.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__,                  \
                    cudaGetErrorString(e));                                    \
            return 1;                                                          \
        }                                                                      \
    } while (0)

constexpr int kChains = 8;

__global__ void dfma_kernel(double *out, int iters, double a, double b) {
    double acc[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i)
        acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < kChains; ++i)
                acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < kChains; ++i)
        s += acc[i];
    if (s == 12345.678)
        out[0] = s;
}

__device__ __forceinline__ void dmma(double &c0, double &c1, double a,
                                     double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
                 "{%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_kernel(double *out, int iters, double a, double b) {
    double c[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i)
        c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int i = 0; i < NACC; ++i)
                dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i)
        s += c[i][0] + c[i][1];
    if (s == 12345.678)
        out[0] = s;
}

// DMMA and DFMA interleaved in one instruction stream: tells whether the
// FP64 tensor path and the FP64 FMA pipe are separate resources.
__global__ void mixed_kernel(double *out, int iters, double a, double b) {
    double c[8][2];
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
        acc[i] = i;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                dmma(c[i][0], c[i][1], a, b);
                // 8 DFMA warp-instructions = 256 FMAs, the work of one DMMA
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    acc[q] = fma(acc[q], a, b);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        s += c[i][0] + c[i][1] + acc[i];
    if (s == 12345.678)
        out[0] = s;
}

// Single-thread dependent-chain latencies (cycles).
__global__ void latency_kernel(long long *cyc, double *sink, double x0) {
    double x = x0;
    long long t0, t1;
    const int R = 256;
    // DFMA
    t0 = clock64();
    for (int i = 0; i < R; ++i)
        x = fma(x, 0.999, 1e-3);
    t1 = clock64();
    cyc[0] = (t1 - t0) / R;
    // sqrt
    t0 = clock64();
    for (int i = 0; i < R; ++i)
        x = sqrt(x) + 0.5;
    t1 = clock64();
    cyc[1] = (t1 - t0) / R;
    // rsqrt
    t0 = clock64();
    for (int i = 0; i < R; ++i)
        x = rsqrt(x) + 0.5;
    t1 = clock64();
    cyc[2] = (t1 - t0) / R;
    // div
    t0 = clock64();
    for (int i = 0; i < R; ++i)
        x = 1.5 / x + 0.25;
    t1 = clock64();
    cyc[3] = (t1 - t0) / R;
    // shfl of a double (two 32-bit shuffles)
    t0 = clock64();
    for (int i = 0; i < R; ++i)
        x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
    t1 = clock64();
    cyc[4] = (t1 - t0) / R;
    // DMMA dependent chain
    double c0 = x, c1 = x;
    t0 = clock64();
    for (int i = 0; i < R; ++i)
        dmma(c0, c1, 0.5, 0.25);
    t1 = clock64();
    cyc[5] = (t1 - t0) / R;
    sink[threadIdx.x] = x + c0 + c1;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    int sms = prop.multiProcessorCount;
    double *out;
    CK(cudaMalloc(&out, 1 << 20));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;

    // DFMA: each thread performs iters*16*kChains FMAs
    double best_dfma = 0;
    for (int threads : {256, 512}) {
        for (int bps : {2, 4, 8}) {
            int iters = 4000;
            int grid  = sms * bps;
            dfma_kernel<<<grid, threads>>>(out, 10, 1.0000001, 1e-9);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            dfma_kernel<<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            double fl = 2.0 * grid * threads * double(iters) * 16 * kChains;
            double tf = fl / (ms * 1e-3) / 1e12;
            if (tf > best_dfma)
                best_dfma = tf;
        }
    }
    // DMMA: per warp per mma 8*8*4 FMAs
    double best_dmma = 0;
    for (int threads : {128, 256, 512}) {
        for (int bps : {1, 2, 4}) {
            int iters = 2000;
            int grid  = sms * bps;
            dmma_kernel<8><<<grid, threads>>>(out, 10, 1.0, 1e-9);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            dmma_kernel<8><<<grid, threads>>>(out, iters, 1.0, 1e-9);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            double warps = double(grid) * threads / 32;
            double fl    = 2.0 * warps * iters * 4 * 8 * 256;
            double tf    = fl / (ms * 1e-3) / 1e12;
            if (tf > best_dmma)
                best_dmma = tf;
        }
    }
    // mixed DMMA + DFMA (equal FMA counts); FLOPs counted for both
    double best_mixed = 0;
    for (int threads : {128, 256}) {
        for (int bps : {2, 4}) {
            int iters = 1000;
            int grid  = sms * bps;
            mixed_kernel<<<grid, threads>>>(out, 10, 1.0, 1e-9);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            mixed_kernel<<<grid, threads>>>(out, iters, 1.0, 1e-9);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            double warps = double(grid) * threads / 32;
            double fl    = 2.0 * warps * iters * 4 * 8 * (256 + 8 * 32);
            double tf    = fl / (ms * 1e-3) / 1e12;
            if (tf > best_mixed)
                best_mixed = tf;
        }
    }
    long long *cyc;
    CK(cudaMallocManaged(&cyc, 16 * sizeof(long long)));
    latency_kernel<<<1, 32>>>(cyc, out, 2.0);
    CK(cudaDeviceSynchronize());
    latency_kernel<<<1, 32>>>(cyc, out, 2.0);
    CK(cudaDeviceSynchronize());
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\"sms\": %d, \"clock_mhz\": %d, \"dfma_tflops\": %.3f, "
           "\"dmma_tflops\": %.3f, \"mixed_dmma_dfma_tflops\": %.3f, \"lat_cycles\": {\"dfma\": %lld, "
           "\"sqrt\": %lld, \"rsqrt\": %lld, \"div\": %lld, \"shfl_f64\": %lld, "
           "\"dmma\": %lld}}\n",
           sms, clk_khz / 1000, best_dfma, best_dmma, best_mixed, cyc[0], cyc[1], cyc[2],
           cyc[3], cyc[4], cyc[5]);
    return 0;
}
