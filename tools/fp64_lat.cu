// FP64 latency / per-warp throughput micro (diagnostics): dependent DFMA chains (1..8
// independent chains per thread), rsqrt.approx.f64 chains, and 1..4 warps per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_lat tools/fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k_fma(double* out, long long* cyc, int iters, double a, double b) {
    double x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C, int OP>
__global__ void k_op(double* out, long long* cyc, int iters, double a, double b) {
    double x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = 1.0 + threadIdx.x * 1e-3 + c;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (OP == 0) x[c] = x[c] * a;
            else if (OP == 1) x[c] = x[c] + b;
            else x[c] = x[c] * x[c];
        }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
__global__ void k_rsq(double* out, long long* cyc, int iters) {
    double x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = 1.0 + threadIdx.x * 1e-3 + c;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double y;
            asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[c]));
            x[c] = y + 1.0;
        }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 1024);
    const int it = 4096;
    for (int op = 0; op < 3; ++op) {
        long long c;
        if (op == 0) k_op<4, 0><<<1, 512>>>(out, cyc, it, 0.9999999, 1e-9);
        if (op == 1) k_op<4, 1><<<1, 512>>>(out, cyc, it, 0.9999999, 1e-9);
        if (op == 2) k_op<4, 2><<<1, 512>>>(out, cyc, it, 0.9999999, 1e-9);
        cudaDeviceSynchronize();
        cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
        printf("%s chains 4 threads 512: %.3f warp-instr/cycle/SM\n", op == 0 ? "dmul(x,uniform)" : op == 1 ? "dadd(x,uniform)" : "dmul(x,x)",
               4.0 * it * 16 / double(c));
    }
    for (int th : {512}) {
        k_fma<1><<<1, th>>>(out, cyc, it, 1.0000001, 1e-9);
        cudaDeviceSynchronize();
#define RUNF(C)                                                                                      \
    {                                                                                                \
        k_fma<C><<<1, th>>>(out, cyc, it, 1.0000001, 1e-9);                                          \
        cudaDeviceSynchronize();                                                                     \
        long long c;                                                                                 \
        cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);                                       \
        printf("dfma chains %d threads %4d: %.2f cycles/step, %.3f warp-DFMA/cycle/SM\n", C, th,   \
               double(c) / it, double(C) * it * (th / 32) / double(c));                             \
    }
        RUNF(1) RUNF(2) RUNF(4) RUNF(8)
#define RUNR(C)                                                                                      \
    {                                                                                                \
        k_rsq<C><<<1, th>>>(out, cyc, it);                                                           \
        cudaDeviceSynchronize();                                                                     \
        long long c;                                                                                 \
        cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);                                       \
        printf("rsq+add chains %d threads %4d: %.2f cycles/step, %.3f warp-RSQ/cycle/SM\n", C, th, \
               double(c) / it, double(C) * it * (th / 32) / double(c));                             \
    }
        RUNR(1) RUNR(4)
    }
    return 0;
}
