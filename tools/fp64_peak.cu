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

int main()
{
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
