// Dependent-chain latency of FP64 ops on one warp (cycles per op), sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double *out, long long *cyc, double a, double b, int iters)
{
    double x = threadIdx.x * 1e-3 + 1.0;
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 64; ++u) {
            if (OP == 0) x = fma(x, a, b);
            if (OP == 1) x = x + b;
            if (OP == 2) x = x * a;
            if (OP == 3) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
            if (OP == 4) x = fmax(x, b) * a;   // DMNMX + DMUL
            if (OP == 5) { asm volatile("{.reg .pred p; setp.gt.f64 p, %1, %2; selp.f64 %0, %1, %2, p;}" : "=d"(x) : "d"(x), "d"(b)); }
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main()
{
    double *out; long long *cyc, h;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
    const char *names[] = {"dfma", "dadd", "dmul", "mufu.rcp64h", "dmnmx+dmul", "dsetp+sel"};
    const int iters = 1000;
#define RUN(K) chain<K><<<1, 32>>>(out, cyc, 0.999999, 1e-9, iters); chain<K><<<1, 32>>>(out, cyc, 0.999999, 1e-9, iters); \
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("{\"op\": \"%s\", \"cycles_per_dep_op\": %.2f}\n", names[K], (double)h / (iters * 64.0));
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5)
    return 0;
}
