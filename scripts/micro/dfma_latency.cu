// Micro-benchmark: dependent-issue latency and per-SM throughput of DFMA /
// DADD and the latency of a 64-bit shuffle on sm_100a (clock64 around
// unrolled chains).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma scripts/micro/dfma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double *out, long long *cyc, double a, double b, int iters)
{
    double x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void shfl_chain(double *out, long long *cyc, int iters)
{
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) x = __shfl_up_sync(0xffffffffu, x, 1) + 1.0;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int ILP>
void run(int warps, const char *name)
{
    double *out; long long *cyc;
    cudaMalloc(&out, sizeof(double) * 32 * warps);
    cudaMalloc(&cyc, sizeof(long long));
    const int iters = 1000;
    chain<ILP><<<1, 32 * warps>>>(out, cyc, 1.0000001, 1e-9, iters);
    chain<ILP><<<1, 32 * warps>>>(out, cyc, 1.0000001, 1e-9, iters);
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double per = (double)c / (16.0 * iters);
    printf("%s warps/SM %2d ILP %d: %.2f cycles per dependent step, %.2f cycles per warp-DFMA per SM sub-partition\n",
           name, warps, ILP, per, per / ILP / ((warps + 3) / 4));
    cudaFree(out); cudaFree(cyc);
}

int main()
{
    run<1>(1, "DFMA"); run<2>(1, "DFMA"); run<4>(1, "DFMA"); run<8>(1, "DFMA");
    run<1>(4, "DFMA"); run<4>(4, "DFMA"); run<8>(4, "DFMA");
    run<1>(12, "DFMA"); run<4>(12, "DFMA"); run<8>(16, "DFMA");
    double *out; long long *cyc;
    cudaMalloc(&out, 256); cudaMalloc(&cyc, 8);
    shfl_chain<<<1, 32>>>(out, cyc, 1000);
    shfl_chain<<<1, 32>>>(out, cyc, 1000);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("64-bit SHFL + DADD dependent step: %.2f cycles\n", (double)c / 16000.0);
    return 0;
}
