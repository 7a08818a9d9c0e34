// Isolated timing of the slot kernel's DMMA tile GEMM (warp_gemm of pc_device.cuh):
// every CTA repeats the N=200 update `reps` times on its own smem F block, so the
// cycles/tick of the GEMM phase can be compared with the 31.2k-cycle DMMA bound.
#include <cstdio>
#include <vector>
#include "../paper_2301_03989_b200/csrc/pc_device.cuh"
using namespace pswarm_dev;

template <int XM>
__global__ void __launch_bounds__(384, 1) k_gemm_loop(const double2* upack, int nkp, GemmPlan gp, int reps,
                                                     double* sink, long long* cycles) {
    extern __shared__ __align__(16) double fbuf[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 8 * nkp * COLS; i += blockDim.x) fbuf[i] = 1e-3 * (i % 97);
    __syncthreads();
    double s = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        const APrefetch<XM> pre = gemm_prefetch<XM>(upack, nkp, gp, warp, lane);
        double acc[2][6][2], xacc[XM][2];
        warp_gemm<XM>(upack, nkp, fbuf, gp, warp, lane, pre, acc, xacc);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int n = 0; n < 6; ++n) s += acc[i][n][0] + acc[i][n][1];
#pragma unroll
        for (int x = 0; x < XM; ++x) s += xacc[x][0] + xacc[x][1];
        __syncthreads();
    }
    long long t1 = clock64();
    sink[blockIdx.x * blockDim.x + tid] = s;
    if (tid == 0) cycles[blockIdx.x] = t1 - t0;
}

GemmPlan plan200() {
    GemmPlan gp{};
    gp.mtiles = 26; gp.warps = 12; gp.main = 2; gp.mb = 24; gp.extras = 12; gp.xmax = 2;
    return gp;
}

int main() {
    const int nkp = 25, mt = 26;
    std::vector<double> hu(static_cast<size_t>(mt) * nkp * 64);
    for (size_t i = 0; i < hu.size(); ++i) hu[i] = 1e-4 * ((i * 2654435761u) % 1000);
    double2* du; cudaMalloc(&du, hu.size() * 8); cudaMemcpy(du, hu.data(), hu.size() * 8, cudaMemcpyHostToDevice);
    double* sink; cudaMalloc(&sink, 148 * 384 * 8);
    long long* cyc; cudaMalloc(&cyc, 148 * 8);
    const size_t smem = 8 * nkp * COLS * 8;
    cudaFuncSetAttribute(k_gemm_loop<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 200;
    for (int it = 0; it < 3; ++it) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_gemm_loop<2><<<148, 384, smem>>>(du, nkp, plan200(), reps, sink, cyc);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> hc(148); cudaMemcpy(hc.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0; double avg = 0; for (auto c : hc) { mx = c > mx ? c : mx; avg += c / 148.0; }
        const double flops = 148.0 * reps * 208 * 48 * 200 * 2.0;
        std::printf("{\"reps\": %d, \"ms\": %.3f, \"cycles_per_tick_avg\": %.0f, \"cycles_per_tick_max\": %.0f, "
                    "\"tflops\": %.2f, \"err\": \"%s\"}\n", reps, ms, avg / reps, (double)mx / reps,
                    flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
