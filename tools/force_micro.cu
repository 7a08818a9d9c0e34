// Force micro (diagnostics): k_pc_uni's force phase in isolation — 400 of 512 threads run
// force_pair<2> over staged synthetic state/ephemeris (N = 200, B = 8), cycles per call.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr
//      -Iinclude -Ipaper_2301_03989_b200/csrc -o tools/force_micro tools/force_micro.cu
#include <cstdio>
#include <vector>
#include "../paper_2301_03989_b200/csrc/pc_slots2.cu"
using namespace pswarm_dev;

template <int NS, int ITEMS_PER_HALF_PAIR>
__global__ void __launch_bounds__(512, 1) k_force(ForceData fd, int N, int reps, long long* cyc, double* sink) {
    extern __shared__ __align__(16) double sm[];
    const int B = fd.n_bodies, half = N / 2;
    double* ybuf = sm;                         // N * YS2
    double* fb = ybuf + N * YS2;               // 2 halves of 64 * FKS
    double* eph = fb + 2 * 64 * FKS;           // 3B N + 3N
    __shared__ int sing[SLOTS];
    const int tid = threadIdx.x;
    for (int i = tid; i < N * YS2; i += blockDim.x) ybuf[i] = (i % 6 < 3) ? 1.2e8 + 1e3 * (i % 977) : 20.0;
    for (int i = tid; i < N * 3 * B + 3 * N; i += blockDim.x) eph[i] = 1.0e8 * (1 + (i % 13)) + 7e6 * (i % 5);
    if (tid < SLOTS) sing[tid] = INT_MAX;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        for (int w = tid; w < 2 * ITEMS_PER_HALF_PAIR * half; w += blockDim.x) {
            const int h = w / (ITEMS_PER_HALF_PAIR * half), rr = w % (ITEMS_PER_HALF_PAIR * half);
            force_pair<NS>(fd, ybuf, fb + h * 64 * FKS, sing, eph, eph + N * 3 * B, 1, N, 0xF, h, rr % half, N,
                           (rr / half) * NS);
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
    sink[blockIdx.x * 512 + tid] = fb[tid];
}

__global__ void __launch_bounds__(512, 1) k_scale(ForceData fd, int N, int reps, long long* cyc, double* sink) {
    extern __shared__ __align__(16) double sm[];
    const int B = fd.n_bodies, half = N / 2;
    double* ybuf = sm;
    double* fb = ybuf + N * YS2;
    double* eph = fb + 2 * 64 * FKS;
    __shared__ int sing[SLOTS];
    const int tid = threadIdx.x;
    for (int i = tid; i < N * YS2; i += blockDim.x) ybuf[i] = (i % 6 < 3) ? 1.2e8 + 1e3 * (i % 977) : 20.0;
    for (int i = tid; i < N * 3 * B + 3 * N; i += blockDim.x) eph[i] = 1.0e8 * (1 + (i % 13)) + 7e6 * (i % 5);
    if (tid < SLOTS) sing[tid] = INT_MAX;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        const int w = tid % (2 * half);
        force_pair<2>(fd, ybuf, fb + (tid / 256) * 64 * FKS, sing, eph, eph + N * 3 * B, 1, N, 0xF, 0, w % half, N,
                      (w / half) * 2);
        __syncthreads();
    }
    const long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
    sink[blockIdx.x * 512 + tid] = fb[tid];
}

int main() {
    const int N = 200, B = 8;
    std::vector<double> mu(B, 1e5);
    double* dmu; cudaMalloc(&dmu, B * 8); cudaMemcpy(dmu, mu.data(), B * 8, cudaMemcpyHostToDevice);
    ForceData fd{};
    fd.n_bodies = B;
    fd.central_mu = 1.32712440018e11;
    fd.body_mu = dmu;
    fd.floor_km = 1.0;
    fd.floor2_hi = 1.0;
    fd.floor2_hi_bits = 0x3ff0000000000000ll;
    long long* cyc; cudaMalloc(&cyc, 148 * 8);
    double* sink; cudaMalloc(&sink, 148 * 512 * 8);
    const size_t smem = (N * YS2 + 2 * 64 * FKS + N * 3 * B + 3 * N) * 8;
    auto run = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<148, 512, smem>>>(fd, N, 20, cyc, sink);
        kern<<<148, 512, smem>>>(fd, N, 20, cyc, sink);
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        std::printf("%-28s %6lld cycles per force phase (both halves)  err=%s\n", name, c,
                    cudaGetErrorString(cudaGetLastError()));
    };
    run(k_force<2, 2>, "force_pair<2> x 400 thr");
    run(k_force<1, 4>, "force_pair<1> x 800 items");
    // scaling: every thread one force_pair<2> call, 1..4 warps per SMSP
    for (int th : {128, 256, 384, 512}) {
        auto kern = k_scale;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<148, th, smem>>>(fd, N, 20, cyc, sink);
        kern<<<148, th, smem>>>(fd, N, 20, cyc, sink);
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        std::printf("scale threads %3d (one force_pair<2> each): %6lld cycles\n", th, c);
    }
    return 0;
}
