// Pipe-sharing micro (diagnostics): 8 warps run k_pc_ws's half-tile DMMA GEMM back to
// back while FPW other warps run independent FP64 rsqrt/FMA chains until the GEMM warps
// finish.  Reports GEMM cycles per half and the FP64 warp-instruction rate the FP warps
// achieved meanwhile: does adding FP warps buy FP throughput under the DMMA stream?
#include <cstdio>
#include <vector>
#include "../paper_2301_03989_b200/csrc/pc_slots2.cu"
using namespace pswarm_dev;

template <int FPW, int MODE>
__global__ void __launch_bounds__(256 + 32 * FPW, 1) k_mix(const double2* upack, int nkp, int N, int reps,
                                                          double* sink, long long* cycles, unsigned long long* fp_iters) {
    extern __shared__ __align__(16) double fbuf[];
    __shared__ volatile int done;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 2 * nkp * FKS; i += blockDim.x) fbuf[i] = 1e-3 * (i % 97);
    if (tid == 0) done = 0;
    __syncthreads();
    if (warp < MMA_WARPS) {
        if constexpr (FPW > 8) asm volatile("setmaxnreg.inc.sync.aligned.u32 128;");
        HalfPlan hp;
        hp.main = 3;
        hp.mb = 3 * MMA_WARPS;
        hp.extras = ((N + 7) / 8 - hp.mb) * 3;
        double s = 0.0;
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            double acc[3][3][2], xacc[1][2];
            gemm_half<3, 1>(upack, nkp, fbuf, hp, warp, lane, acc, xacc);
            for (int i = 0; i < 3; ++i)
                for (int p = 0; p < 3; ++p) s += acc[i][p][0] + acc[i][p][1];
            s += xacc[0][0];
            asm volatile("bar.sync 1, 256;");
        }
        long long t1 = clock64();
        if (tid == 0) {
            cycles[blockIdx.x] = t1 - t0;
            done = 1;
        }
        sink[blockIdx.x * blockDim.x + tid] = s;
    } else {
        if constexpr (FPW > 8) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        double x[4] = {1.1 + tid, 2.2 + tid, 3.3 + tid, 4.4 + tid}, y[4] = {0, 0, 0, 0};
        unsigned u[4] = {1u + tid, 2u + tid, 3u + tid, 4u + tid};
        const volatile unsigned* sidx = reinterpret_cast<const volatile unsigned*>(fbuf);
        unsigned long long it = 0;
        while (!done) {
            if constexpr (MODE == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {  // 6 FP64 instructions per chain step
                    const double q = rsqrt_newton(x[k], rsqrt_seed(x[k]));
                    y[k] = fma(q * q, q, y[k]);
                    x[k] = fma(x[k], 1.0000001, 1e-9);
                }
            } else if constexpr (MODE == 1) {
#pragma unroll
                for (int k = 0; k < 4; ++k)  // 6 integer ALU instructions per chain step
#pragma unroll
                    for (int r = 0; r < 3; ++r) u[k] = (u[k] * 2654435761u + 12345u) ^ (u[k] >> 7);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)  // dependent shared loads (+ index arithmetic)
#pragma unroll
                    for (int r = 0; r < 6; ++r) u[k] = sidx[(u[k] + lane) & 1023] & 1023;
            }
            ++it;
        }
        if (lane == 0) atomicAdd(fp_iters, it);
        sink[blockIdx.x * blockDim.x + tid] = y[0] + y[1] + y[2] + y[3] + u[0] + u[1] + u[2] + u[3];
    }
}

template <int FPW, int MODE>
void run(const double2* du, int nkp, int N) {
    double* sink; cudaMalloc(&sink, 148 * 1024 * 8);
    long long* cyc; cudaMalloc(&cyc, 148 * 8);
    unsigned long long* it; cudaMalloc(&it, 8); cudaMemset(it, 0, 8);
    const size_t smem = 2 * nkp * FKS * 8;
    cudaFuncSetAttribute(k_mix<FPW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 200;
    k_mix<FPW, MODE><<<148, 256 + 32 * FPW, smem>>>(du, nkp, N, reps, sink, cyc, it);
    cudaMemset(it, 0, 8);
    k_mix<FPW, MODE><<<148, 256 + 32 * FPW, smem>>>(du, nkp, N, reps, sink, cyc, it);
    cudaDeviceSynchronize();
    std::vector<long long> hc(148); cudaMemcpy(hc.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
    unsigned long long hi; cudaMemcpy(&hi, it, 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (auto c : hc) avg += c / 148.0;
    // FP64 warp instructions issued by the FP warps per SM-cycle (24 per loop iteration)
    const double fp_rate = hi * 24.0 / 148.0 / avg;
    std::fflush(stdout);
    std::printf("{\"mode\": \"%s\", \"fp_warps\": %d, \"gemm_cycles_per_half\": %.0f, \"warp_instr_per_cycle_per_sm\": %.3f, \"err\": \"%s\"}\n",
                MODE == 0 ? "fp64" : (MODE == 1 ? "int" : "lds"), FPW, avg / reps, fp_rate,
                cudaGetErrorString(cudaGetLastError()));
    std::fflush(stdout);
}

int main() {
    const int N = 200, nkp = 25, mt = 26;
    std::vector<double> hu(static_cast<size_t>(mt) * nkp * 64);
    for (size_t i = 0; i < hu.size(); ++i) hu[i] = 1e-4 * ((i * 2654435761u) % 1000);
    double2* du; cudaMalloc(&du, hu.size() * 8); cudaMemcpy(du, hu.data(), hu.size() * 8, cudaMemcpyHostToDevice);
    run<0, 0>(du, nkp, N);
    run<8, 0>(du, nkp, N);
    run<8, 1>(du, nkp, N);
    run<8, 2>(du, nkp, N);
    return 0;
}
