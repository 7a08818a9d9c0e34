// tcgen05 kind::i8 probe (diagnostics): D[M=128][N] (s32, TMEM) = A[128][K] . B[N][K]^T, both
// operands int8 K-major without swizzle in shared memory (8-row x 16-byte core matrices), checked
// against a host integer GEMM; then R back-to-back accumulating MMAs timed with clock64.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_i8_micro tools/tc_i8_micro.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

constexpr int M = 128, K = 128;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// canonical K-major no-swizzle offset of (row r, byte k) for an operand with K bytes per row
__host__ __device__ __forceinline__ int kmaj(int r, int k, int kbytes) {
    return (r >> 3) * (kbytes * 8) + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version 1 (sm_100)
    return d;         // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
    return (2u << 4)      // D s32
           | (1u << 7)    // A signed
           | (1u << 10)   // B signed
           | (0u << 15)   // A K-major
           | (0u << 16)   // B K-major
           | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

template <int N>
__global__ void k_probe(const int8_t* A, const int8_t* B, int* D, int reps, long long* cyc, int swap_lbo) {
    extern __shared__ __align__(1024) unsigned char sm[];
    int8_t* sa = reinterpret_cast<int8_t*>(sm);
    int8_t* sb = sa + M * K;
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < M * K; i += blockDim.x) sa[kmaj(i / K, i % K, K)] = A[i];
    for (int i = tid; i < N * K; i += blockDim.x) sb[kmaj(i / K, i % K, K)] = B[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "n"(N <= 32 ? 32 : N <= 64 ? 64 : 128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy operand writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    const uint32_t lbo = swap_lbo ? K * 8 : 128, sbo = swap_lbo ? 128 : K * 8;
    long long t0 = 0, t1 = 0;
    if (tid == 0) {
        const uint32_t id = idesc_i8(M, N);
        t0 = clock64();
        for (int r = 0; r < reps; ++r)
            for (int ks = 0; ks < K / 32; ++ks) {
                const uint64_t da = sdesc(su32(sa) + ks * 256, lbo, sbo);
                const uint64_t db = sdesc(su32(sb) + ks * 256, lbo, sbo);
                const uint32_t acc = (r | ks) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
                    "l"(da), "l"(db), "r"(id), "r"(acc));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                         : "=r"(done) : "r"(su32(&mbar)), "r"(0));
        t1 = clock64();
        cyc[0] = t1 - t0;
    }
    __syncthreads();
    {  // other threads: wait on the same phase
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                         : "=r"(done) : "r"(su32(&mbar)), "r"(0));
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // drain: warp w reads lanes 32w..32w+31 (row = tid), 8 columns per load
    const int row = tid;
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tm + (static_cast<uint32_t>(warp * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int e = 0; e < 8; ++e) D[row * N + c0 + e] = static_cast<int>(v[e]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(N <= 32 ? 32 : N <= 64 ? 64 : 128));
}


// A-operand streaming: every CTA (one per SM) streams NCH chunks of A (104 rows x 32 K bytes in
// the canonical layout, 3,328 B, L2-resident source) through an R-slot shared-memory ring with
// cp.async.bulk + mbarriers, one M128 x NB x K32 MMA per chunk (B resident), and reports cycles
// per chunk: is the U-digit stream of an emulated-FP64 update latency-bound with a small ring?
constexpr int CH = 104 * 32;
template <int R, int NB>
__global__ void k_stream(const int8_t* A, int nsrc, int nch, long long* cyc, int* sink, int do_mma) {
    extern __shared__ __align__(1024) unsigned char sm[];
    int8_t* ring = reinterpret_cast<int8_t*>(sm);
    int8_t* sb = ring + R * 4096;
    __shared__ __align__(8) uint64_t full[R], empty[R];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < NB * 32; i += blockDim.x) sb[kmaj(i / 32, i % 32, 32)] = static_cast<int8_t>(i % 7 - 3);
    // (the ring is not pre-filled: async-proxy writes only)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int r = 0; r < R; ++r) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[r])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[r])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) {  // the whole warp runs the loop (lane 0 issues): no lane parked at a CTA barrier
        const bool l0 = (tid & 31) == 0;
        const uint32_t tm = tbase, id = idesc_i8(M, NB);
        auto wait = [&](uint64_t* b, uint32_t ph) {  // test_wait spin (no suspend window)
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred q;\n\tmbarrier.test_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                             : "=r"(done) : "r"(su32(b)), "r"(ph));
        };
        auto issue = [&](int c) {  // chunk c into slot c % R
            const int r = c % R;
            if (!l0) return;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[r])), "r"(CH));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(ring + r * 4096)), "l"(A + static_cast<size_t>(nsrc > 56 ? blockIdx.x * 56 + c % 56 : (c * 7 + blockIdx.x) % nsrc) * CH), "r"(CH), "r"(su32(&full[r])) : "memory");
        };
        const long long t0 = clock64();
        for (int c = 0; c < R && c < nch; ++c) issue(c);  // then chunk j + R refills slot j
        for (int c = 0; c < nch; ++c) {
            wait(&full[c % R], (c / R) & 1);
            if (do_mma) asm volatile("tcgen05.fence::after_thread_sync;");
            const uint64_t da = sdesc(su32(ring + (c % R) * 4096), 128, 256);
            const uint64_t db = sdesc(su32(sb), 128, 256);
            if (do_mma && l0) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
                    "l"(da), "l"(db), "r"(id), "r"(c ? 1u : 0u));
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[c % R])));
            } else if (l0) {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[c % R])));
            }
            __syncwarp();
            // refill the slot of chunk j = c - R/2 (its MMA was issued R/2 chunks ago): R/2 MMAs stay
            // queued while the issuer waits, R/2 copies are in flight
            const int j = c - R / 2;
            if (j >= 0 && j + R < nch) {
                wait(&empty[j % R], (j / R) & 1);
                issue(j + R);
            }
        }
        wait(&empty[(nch - 1) % R], ((nch - 1) / R) & 1);
        const long long t1 = clock64();
        if (l0) cyc[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tbase));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (tid == 0) sink[blockIdx.x] = static_cast<int>(v);
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(256));
    }
}

template <int R, int NB>
static void stream(int nch, int do_mma = 1, int nsrc = 56, int grid = 148) {
    int8_t* da;
    long long* dc;
    int* ds;
    CK(cudaMalloc(&da, static_cast<size_t>(nsrc) * CH));
    CK(cudaMemset(da, 1, static_cast<size_t>(nsrc) * CH));
    CK(cudaMalloc(&dc, grid * 8));
    CK(cudaMalloc(&ds, grid * 4));
    const int smem = R * 4096 + NB * 32;
    CK(cudaFuncSetAttribute(k_stream<R, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int rep = 0; rep < 2; ++rep) k_stream<R, NB><<<grid, 128, smem>>>(da, nsrc, nch, dc, ds, do_mma);
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(grid);
    CK(cudaMemcpy(c.data(), dc, grid * 8, cudaMemcpyDeviceToHost));
    double mean = 0;
    for (auto x : c) mean += double(x) / grid;
    printf("stream ring %d, N%d, mma %d, %s source: %.0f cycles per chunk (%d CTAs, %d chunks each)\n", R, NB, do_mma,
           nsrc > 56 ? "per-CTA" : "shared", mean / nch, grid, nch);
    cudaFree(da);
    cudaFree(dc);
    cudaFree(ds);
}

// L2 -> SM read bandwidth with plain 16-byte loads: every CTA (one per SM, T threads) sweeps a
// private L2-resident region `reps` times; bytes per cycle per SM.
template <int T>
__global__ void k_ldg(const int4* src, size_t per_cta16, int reps, long long* cyc, int* sink) {
    const int4* p = src + blockIdx.x * per_cta16;
    int acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll 4
        for (size_t i = threadIdx.x; i < per_cta16; i += T) {
            const int4 v = __ldcg(p + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678) sink[0] = acc;
}

template <int T>
static void ldg_bw(size_t per_cta_bytes, int reps) {
    const int grid = 148;
    int4* d;
    long long* dc;
    int* ds;
    CK(cudaMalloc(&d, per_cta_bytes * grid));
    CK(cudaMemset(d, 1, per_cta_bytes * grid));
    CK(cudaMalloc(&dc, grid * 8));
    CK(cudaMalloc(&ds, 4));
    for (int rep = 0; rep < 2; ++rep) k_ldg<T><<<grid, T>>>(d, per_cta_bytes / 16, reps, dc, ds);
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(grid);
    CK(cudaMemcpy(c.data(), dc, grid * 8, cudaMemcpyDeviceToHost));
    double mean = 0;
    for (auto x : c) mean += double(x) / grid;
    printf("ldg %d threads, %zu KB per CTA x %d: %.1f B/cycle/SM (%.2f TB/s at 1.9 GHz, 148 SMs)\n", T, per_cta_bytes / 1024, reps,
           double(per_cta_bytes) * reps / mean, double(per_cta_bytes) * reps / mean * 148 * 1.9e9 / 1e12);
    cudaFree(d);
    cudaFree(dc);
    cudaFree(ds);
}

// one CTA: a single 1-D bulk copy of `bytes` (L2-resident source) -> cycles (size dependence of the
// bulk-copy rate: per-copy overhead vs bytes per cycle)
__global__ void k_bulk_one(const int8_t* src, int bytes, long long* cyc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms L2
            const long long t0 = clock64();
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(sm)), "l"(src), "r"(bytes), "r"(su32(&bar)) : "memory");
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                             : "=r"(done) : "r"(su32(&bar)), "r"(rep & 1));
            cyc[rep] = clock64() - t0;
        }
    }
}

static void bulk_one(int bytes) {
    int8_t* d;
    long long* dc;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(d, 3, bytes));
    CK(cudaMalloc(&dc, 16));
    CK(cudaFuncSetAttribute(k_bulk_one, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    k_bulk_one<<<1, 32, 200 * 1024>>>(d, bytes, dc);
    CK(cudaDeviceSynchronize());
    long long c[2];
    CK(cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost));
    printf("bulk one copy %6d B: %lld cycles (%.1f B/cycle) [cold %lld]\n", bytes, c[1], double(bytes) / c[1], c[0]);
    cudaFree(d);
    cudaFree(dc);
}

// one CTA: k back-to-back 1-D bulk copies of `bytes` each (distinct sources and destinations),
// either on ONE mbarrier (expect_tx k*bytes) or on k separate mbarriers waited in order
__global__ void k_bulk_many(const int8_t* src, int bytes, int k, int separate, long long* cyc, int stride, int variant) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bars[32];
    __shared__ uint32_t tb;
    // variant 1: TMEM allocated first (as a tcgen05 kernel would); 2: 128-thread CTA, others parked at a barrier
    if (variant == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tb)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 32; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        for (int rep = 0; rep < 2; ++rep) {
            const long long t0 = clock64();
            if (!separate)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[0])), "r"(bytes * k));
            for (int i = 0; i < k; ++i) {
                uint64_t* b = separate ? &bars[i] : &bars[0];
                if (separate)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 su32(sm + i * 4096)), "l"(src + static_cast<size_t>((i * stride) % 56) * bytes), "r"(bytes), "r"(su32(b)) : "memory");
            }
            for (int i = 0; i < (separate ? k : 1); ++i) {
                uint32_t done = 0;
                while (!done)
                    asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                                 : "=r"(done) : "r"(su32(&bars[i])), "r"(rep & 1));
            }
            cyc[rep] = clock64() - t0;
        }
    }
    if (variant == 2) __syncthreads();
    if (variant == 1) {
        __syncwarp();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(256));
    }
}
static void bulk_many(int k, int separate, int stride = 1, int variant = 0) {
    const int bytes = 3328;
    int8_t* d;
    long long* dc;
    CK(cudaMalloc(&d, bytes * 56));
    CK(cudaMemset(d, 3, bytes * 56));
    CK(cudaMalloc(&dc, 16));
    CK(cudaFuncSetAttribute(k_bulk_many, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    k_bulk_many<<<1, variant == 2 ? 128 : 32, 200 * 1024>>>(d, bytes, k, separate, dc, stride, variant);
    CK(cudaDeviceSynchronize());
    long long c[2];
    CK(cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost));
    printf("bulk %2d x %d B, %s, stride %d, variant %d: %lld cycles (%.0f per copy)\n", k, bytes,
           separate ? "separate mbarriers" : "one mbarrier", stride, variant, c[1], double(c[1]) / k);
    cudaFree(d);
    cudaFree(dc);
}

template <int N>
static int run(int swap) {
    std::vector<int8_t> a(M * K), b(N * K);
    srand(7);
    for (auto& x : a) x = static_cast<int8_t>(rand() % 256 - 128);
    for (auto& x : b) x = static_cast<int8_t>(rand() % 256 - 128);
    int8_t *da, *db;
    int* dd;
    long long* dc;
    CK(cudaMalloc(&da, a.size()));
    CK(cudaMalloc(&db, b.size()));
    CK(cudaMalloc(&dd, M * N * 4));
    CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice));
    const int smem = M * K + N * K;
    CK(cudaFuncSetAttribute(k_probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_probe<N><<<1, 128, smem>>>(da, db, dd, 1, dc, swap);
    CK(cudaDeviceSynchronize());
    std::vector<int> d(M * N);
    CK(cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            int s = 0;
            for (int k = 0; k < K; ++k) s += a[m * K + k] * b[n * K + k];
            if (s != d[m * N + n] && bad++ < 3) printf("  N=%d swap=%d mismatch (%d,%d): %d vs %d\n", N, swap, m, n, d[m * N + n], s);
        }
    long long cyc = 0;
    const int reps = 256;
    k_probe<N><<<1, 128, smem>>>(da, db, dd, reps, dc, swap);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("N=%d swap=%d: %s (%d bad); %.1f cycles per MMA (M128 N%d K32), %.0f MAC/cycle\n", N, swap,
           bad ? "MISMATCH" : "exact", bad, double(cyc) / (reps * K / 32), N, double(M) * N * K * reps / cyc);
    cudaFree(da);
    cudaFree(db);
    cudaFree(dd);
    cudaFree(dc);
    return bad;
}

int main() {
    int bad = 0;
    bad += run<48>(0);
    if (bad) bad = run<48>(1);
    run<32>(0);
    run<64>(0);
    run<128>(0);
    stream<3, 192>(1120);
    stream<4, 192>(1120);
    stream<8, 192>(1120);
    stream<16, 192>(1120);
    stream<4, 48>(1120);
    stream<8, 48>(1120);
    stream<4, 48>(1120, 0);
    stream<16, 48>(1120, 0);
    stream<4, 48>(1120, 0, 148 * 56);
    stream<16, 48>(1120, 0, 148 * 56);
    stream<16, 192>(1120, 1, 148 * 56);
    stream<16, 48>(1120, 0, 56, 1);
    stream<16, 48>(16, 0, 56, 1);
    stream<16, 48>(1, 0, 56, 1);
    stream<16, 48>(16, 0, 56, 148);
    stream<4, 48>(1120, 0, 56, 1);
    for (int b : {3328, 16384, 65536, 196608}) bulk_one(b);
    for (int k : {1, 4, 16, 32}) { bulk_many(k, 0); bulk_many(k, 1); }
    bulk_many(16, 1, 7);
    bulk_many(16, 0, 7);
    bulk_many(16, 1, 7, 1);
    bulk_many(16, 1, 7, 2);
    ldg_bw<512>(186 * 1024, 20);
    ldg_bw<256>(186 * 1024, 20);
    ldg_bw<512>(1024 * 1024, 4);
    return 0;
}
