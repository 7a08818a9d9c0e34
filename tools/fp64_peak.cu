// FP64 peak microbenchmark for B200 (sm_100a): DMMA.8x8x4 (mma.sync m8n8k4 f64)
// and DFMA throughput, plus a fragment-layout self-check of mma.m8n8k4.f64.
// The roofline denominator for the Picard update / force kernels is the
// larger of the two measured rates (both pipes are FP64).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); std::exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double c[CHAINS][2];
  #pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  const double a = seed * (threadIdx.x + 1);
  const double b = 1.0 / (threadIdx.x + 3);
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < CHAINS; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
  #pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double c[CHAINS];
  #pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = seed * i;
  const double a = 1.0 + 1e-9 * threadIdx.x;
  const double b = 1e-12;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
  #pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Half the warps issue DMMA chains, the other half DFMA chains: if the tensor
// (DMMA) and FP64 (DFMA) pipes are separate, the aggregate exceeds either alone.
__global__ void mixed_loop(double* out, int iters, double seed) {
  const int warp = threadIdx.x >> 5;
  double s = 0.0;
  if (warp & 1) {
    double c[8][2];
    for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
    const double a = seed * (threadIdx.x + 1), b = 1.0 / (threadIdx.x + 3);
    for (int it = 0; it < iters; ++it) {
      #pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double c[8];
    for (int i = 0; i < 8; ++i) c[i] = seed * i;
    const double a = 1.0 + 1e-9 * threadIdx.x, b = 1e-12;
    for (int it = 0; it < iters * 4; ++it) {
      #pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
    }
    for (int i = 0; i < 8; ++i) s += c[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// A (8x4) row-major, B (4x8) "col", C 8x8: verify assumed fragment layout.
__global__ void layout_check(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x;
  const double a = A[(lane >> 2) * 4 + (lane & 3)];      // A[g][q]
  const double b = B[(lane & 3) * 8 + (lane >> 2)];      // B[q][g]
  double c0 = 0.0, c1 = 0.0;
  dmma(c0, c1, a, b);
  C[(lane >> 2) * 8 + 2 * (lane & 3) + 0] = c0;          // C[g][2q]
  C[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = c1;          // C[g][2q+1]
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  std::printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", p.name, p.multiProcessorCount, clk_khz);

  // layout check
  {
    std::vector<double> A(32), B(32), C(64), R(64, 0.0);
    for (int i = 0; i < 32; ++i) { A[i] = 1.0 + i; B[i] = 0.5 * i - 3.0; }
    for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) for (int k = 0; k < 4; ++k) R[r * 8 + c] += A[r * 4 + k] * B[k * 8 + c];
    double *dA, *dB, *dC;
    CK(cudaMalloc(&dA, 256)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dC, 512));
    CK(cudaMemcpy(dA, A.data(), 256, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), 256, cudaMemcpyHostToDevice));
    layout_check<<<1, 32>>>(dA, dB, dC);
    CK(cudaMemcpy(C.data(), dC, 512, cudaMemcpyDeviceToHost));
    double worst = 0.0;
    for (int i = 0; i < 64; ++i) worst = std::fmax(worst, std::fabs(C[i] - R[i]));
    std::printf(", \"layout_max_abs_err\": %.3e", worst);
  }

  double* out; CK(cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int sms = p.multiProcessorCount;

  auto bench = [&](const char* name, auto launch, double flops) {
    launch(); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); best = std::fmin(best, ms);
    }
    std::printf(", \"%s_tflops\": %.3f", name, flops / (best * 1e-3) / 1e12);
  };

  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    const int threads = 32 * warps;
    const int blocks = sms * 2;
    char nm[64]; std::snprintf(nm, sizeof nm, "dmma_w%d", warps);
    bench(nm, [&] { dmma_loop<8><<<blocks, threads>>>(out, iters, 1e-3); },
          double(blocks) * warps * iters * 8 * 512.0);
  }
  for (int threads : {256, 512}) {
    const int blocks = sms * 4;
    char nm[64]; std::snprintf(nm, sizeof nm, "dfma_t%d", threads);
    bench(nm, [&] { dfma_loop<8><<<blocks, threads>>>(out, iters, 1e-3); },
          double(blocks) * threads * iters * 8 * 2.0);
  }
  // mixed: per DMMA warp 8*512 flops/iter; per DFMA warp 4*8*2*32 = 2048 flops/iter
  for (int warps : {8, 16}) {
    const int blocks = sms * 2;
    char nm[64]; std::snprintf(nm, sizeof nm, "mixed_w%d", warps);
    const double per_block = (warps / 2) * (8 * 512.0) + (warps / 2) * (4 * 8 * 2 * 32.0);
    bench(nm, [&] { mixed_loop<<<blocks, 32 * warps>>>(out, iters, 1e-3); }, double(blocks) * per_block * iters);
  }
  std::printf("}\n");
  return 0;
}
