// FP64 peak microbenchmark for B200 (sm_100a): DFMA vector pipe and the
// FP64 tensor path (mma.sync DMMA m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
//   ./fp64_peak        -> one JSON line per kernel (TFLOP/s, FMA = 2 flops)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double a, double b)
{
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
           x6 = x0 + 6, x7 = x0 + 7;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma884_kernel(double *out, int iters)
{
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][2] = {};
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma1684_kernel(double *out, int iters)
{
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-4, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][4] = {};
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                         : "d"(a0), "d"(a1), "d"(b));
    }
    double s = 0;
    for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16816_kernel(double *out, int iters)
{
    double a[8], b[4];
    for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-3 + q;
    for (int q = 0; q < 4; ++q) b[q] = 1.0 - threadIdx.x * 1e-4 * q;
    double c[2][4] = {};
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 2; ++u)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                         "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                         : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]),
                           "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
    for (int u = 0; u < 2; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float timeit(F launch)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main_mixed();
int main()
{
    main_mixed();
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    double *out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    const int it = 4096;
    float ms = timeit([&] { dfma_kernel<<<blocks, threads>>>(out, it, 0.999, 1e-3); });
    double fl = 2.0 * blocks * threads * (double)it * 16 * 8;
    printf("{\"kernel\": \"dfma\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);
    ms = timeit([&] { dmma884_kernel<<<blocks, threads>>>(out, it); });
    fl = 2.0 * 8 * 8 * 4 * (blocks * threads / 32) * (double)it * 4;
    printf("{\"kernel\": \"dmma_m8n8k4\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);
    ms = timeit([&] { dmma1684_kernel<<<blocks, threads>>>(out, it); });
    fl = 2.0 * 16 * 8 * 4 * (blocks * threads / 32) * (double)it * 4;
    printf("{\"kernel\": \"dmma_m16n8k4\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);
    ms = timeit([&] { dmma16816_kernel<<<blocks, threads>>>(out, it); });
    fl = 2.0 * 16 * 8 * 16 * (blocks * threads / 32) * (double)it * 2;
    printf("{\"kernel\": \"dmma_m16n8k16\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}

// --- concurrency probe: DFMA warps and DMMA warps in the same kernel ---
__global__ void mixed_kernel(double *out, int iters, int mode)
{
    // mode 0: all warps DFMA, 1: all DMMA, 2: even warps DFMA / odd warps DMMA
    const int w = threadIdx.x >> 5;
    const bool do_mma = mode == 1 || (mode == 2 && (w & 1));
    double s = 0;
    if (do_mma) {
        double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
        double c[4][2] = {};
        for (int k = 0; k < iters; ++k) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
        }
        for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1];
    } else {
        double x[8];
        for (int q = 0; q < 8; ++q) x[q] = threadIdx.x + q;
        // 8 lanes-FMA per thread x 16 x 8 = same FMA count per iteration as 4 DMMA/warp
        for (int k = 0; k < iters; ++k) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int q = 0; q < 8; ++q) x[q] = fma(x[q], 0.999, 1e-3);
        }
        for (int q = 0; q < 8; ++q) s += x[q];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main_mixed()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    double *out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    const int it = 4096;
    for (int mode = 0; mode < 3; ++mode) {
        float ms = timeit([&] { mixed_kernel<<<blocks, threads>>>(out, it, mode); });
        // per warp per iteration: DFMA warp = 32 lanes x 32 FMA = 1024 FMA; DMMA warp = 4 x 256 = 1024 FMA
        double fl = 2.0 * 1024.0 * (blocks * threads / 32) * (double)it;
        printf("{\"kernel\": \"mixed_mode%d\", \"tflops\": %.2f, \"ms\": %.3f}\n", mode, fl / ms / 1e9, ms);
    }
    return 0;
}
