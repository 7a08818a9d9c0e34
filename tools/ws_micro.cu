// Isolated timing of k_pc_ws's half-tile DMMA GEMM (gemm_half, 8 MMA warps, 3 n-tiles)
// at N = 200: every CTA repeats the update of one half `reps` times from its own smem F
// block.  Compare cycles/half with the pipe bound (19 tiles x 50 k-steps x 16 cycles per
// SMSP = 15.2k).  Optional FP load: 8 more warps run a DFMA/rsqrt chain loop meanwhile
// (argv[1] = 1) to measure how much the shared FP64 pipe slows the GEMM.
#include <cstdio>
#include <vector>
#include "../paper_2301_03989_b200/csrc/pc_slots2.cu"
using namespace pswarm_dev;

template <int MAIN, int XMW, bool HASX>
__global__ void __launch_bounds__(WS_THREADS, 1) k_half_loop(const double2* upack, int nkp, int N, int reps, int fp_load,
                                                     double* sink, long long* cycles) {
    extern __shared__ __align__(16) double fbuf[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 2 * nkp * FKS; i += blockDim.x) fbuf[i] = 1e-3 * (i % 97);
    __syncthreads();
    HalfPlan hp;
    hp.main = MAIN;
    hp.mb = MAIN * MMA_WARPS;
    hp.extras = ((N + 7) / 8 - hp.mb) * 3;
    double s = 0.0;
    if (warp < MMA_WARPS) {
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            double acc[MAIN][3][2], xacc[XMW][2];
            gemm_half<MAIN, XMW>(upack, nkp, fbuf, hp, warp, lane, acc, xacc);
#pragma unroll
            for (int i = 0; i < MAIN; ++i)
#pragma unroll
                for (int p = 0; p < 3; ++p) s += acc[i][p][0] + acc[i][p][1];
#pragma unroll
            for (int x = 0; x < XMW; ++x) s += xacc[x][0] + xacc[x][1];
            asm volatile("bar.sync 1, %0;" ::"n"(MMA_THREADS));
        }
        long long t1 = clock64();
        if (tid == 0) cycles[blockIdx.x] = t1 - t0;
    } else {
      if (fp_load) {
        // FP group stand-in: 4 independent rsqrt + Newton + FMA chains per thread
        double x[4] = {1.1 + tid, 2.2 + tid, 3.3 + tid, 4.4 + tid}, y[4] = {0, 0, 0, 0};
        for (int r = 0; r < reps * 60; ++r)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double q = rsqrt_newton(x[k], rsqrt_seed(x[k]));
                y[k] = fma(q * q, q, y[k]);
                x[k] = fma(x[k], 1.0000001, 1e-9);
            }
        s = y[0] + y[1] + y[2] + y[3];
      }
    }
    sink[blockIdx.x * blockDim.x + tid] = s;
}

#ifndef MICRO_MAIN
#define MICRO_MAIN 3
#define MICRO_XMW 1
#endif
constexpr int MM = MICRO_MAIN, XM = MICRO_XMW;

int main(int argc, char** argv) {
    const int fp_load = argc > 1 ? atoi(argv[1]) : 0;
    const int N = argc > 2 ? atoi(argv[2]) : 200, nkp = (N + 7) / 8, mt = (N + 1 + 7) / 8;
    std::vector<double> hu(static_cast<size_t>(mt) * nkp * 64);
    for (size_t i = 0; i < hu.size(); ++i) hu[i] = 1e-4 * ((i * 2654435761u) % 1000);
    double2* du; cudaMalloc(&du, hu.size() * 8); cudaMemcpy(du, hu.data(), hu.size() * 8, cudaMemcpyHostToDevice);
    double* sink; cudaMalloc(&sink, 148 * WS_THREADS * 8);
    long long* cyc; cudaMalloc(&cyc, 148 * 8);
    const size_t smem = 2 * nkp * FKS * 8;
    cudaFuncSetAttribute(k_half_loop<MM, XM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_half_loop<MM, XM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 200;
    for (int it = 0; it < 3; ++it) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        if (N % 64 == 0 && N < 256) k_half_loop<MM, XM, false><<<148, WS_THREADS, smem>>>(du, nkp, N, reps, fp_load, sink, cyc);
        else k_half_loop<MM, XM, true><<<148, WS_THREADS, smem>>>(du, nkp, N, reps, fp_load, sink, cyc);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> hc(148); cudaMemcpy(hc.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0; double avg = 0; for (auto c : hc) { mx = c > mx ? c : mx; avg += c / 148.0; }
        const double flops = 148.0 * reps * N * 24 * N * 2.0;
        std::printf("{\"N\": %d, \"fp_load\": %d, \"reps\": %d, \"ms\": %.3f, \"cycles_per_half_avg\": %.0f, \"cycles_per_half_max\": %.0f, "
                    "\"useful_tflops\": %.2f, \"err\": \"%s\"}\n", N, fp_load, reps, ms, avg / reps, (double)mx / reps,
                    flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
