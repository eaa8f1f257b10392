// Round 2 microbenchmark: random 32-byte record gathers into shared memory inside cell-sized
// spans (25000 records), the collide's phase-1 pattern, four ways, alone and followed by a
// contiguous store of the chunk (the collide's output traffic):
//   ldgsts   two 16-byte cp.async per record by one thread (the product's way)
//   pairs    lanes 2r / 2r+1 copy the two halves of one record in the same instruction
//   bulk1d   one 32-byte TMA bulk copy (cp.async.bulk ... mbarrier::complete_tx) per record
//   ld256    one 256-bit register load per record, then two 16-byte shared stores
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bulk_gather bulk_gather.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

constexpr int kChunk = 1536;
constexpr int kThreads = 256;

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(void* s, const void* g)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(s)), "l"(g) : "memory");
}

__device__ int g_pf_waves = 0;    // MODE 4: L2 bulk prefetch this many waves (gridDim chunks) ahead

template <int MODE, bool STORE>
__global__ void __launch_bounds__(kThreads) k_gather(const double* __restrict__ rec, const int32_t* __restrict__ idx,
                                                     int64_t n, double* __restrict__ outp)
{
    extern __shared__ __align__(128) double st[];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x & 31;
    if (MODE == 2 && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t nch = n / kChunk;
    double acc = 0.0;
    unsigned phase = 0;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
        const int32_t* ix = idx + c * kChunk;
        if (MODE == 4) {
            // sequential DRAM reads: prefetch into L2 the chunk-aligned 48 KB of the record array
            // that chunk c + waves * grid will gather from (its cell span), then gather as MODE 1
            const int64_t cp = c + static_cast<int64_t>(g_pf_waves) * gridDim.x;
            if (threadIdx.x == 0 && cp < nch)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rec + 4 * cp * kChunk), "r"(kChunk * 32)
                             : "memory");
        }
        if (MODE == 0) {
            for (int e = threadIdx.x; e < kChunk; e += kThreads) {
                const double* g = rec + 4 * static_cast<int64_t>(ix[e]);
                cp16(st + 4 * e, g);
                cp16(st + 4 * e + 2, g + 2);
            }
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
        } else if (MODE == 1 || MODE == 4) {
            // 2 * kChunk half-records, lane pairs share a record
            for (int h = threadIdx.x; h < 2 * kChunk; h += kThreads) {
                const int e = h >> 1, half = h & 1;
                cp16(st + 4 * e + 2 * half, rec + 4 * static_cast<int64_t>(ix[e]) + 2 * half);
            }
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
        } else if (MODE == 2) {
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(kChunk * 32)
                             : "memory");
            __syncthreads();
            for (int e = threadIdx.x; e < kChunk; e += kThreads)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];"
                             ::"r"(sa(st + 4 * e)), "l"(rec + 4 * static_cast<int64_t>(ix[e])), "r"(sa(&bar))
                             : "memory");
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(sa(&bar)), "r"(phase) : "memory");
            phase ^= 1u;
        } else {
            constexpr int R = kChunk / kThreads;
            double a[R], b[R], cc[R], d[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double* g = rec + 4 * static_cast<int64_t>(ix[threadIdx.x + r * kThreads]);
                asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                             : "=d"(a[r]), "=d"(b[r]), "=d"(cc[r]), "=d"(d[r]) : "l"(g));
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int e = threadIdx.x + r * kThreads;
                reinterpret_cast<double2*>(st)[2 * e] = make_double2(a[r], b[r]);
                reinterpret_cast<double2*>(st)[2 * e + 1] = make_double2(cc[r], d[r]);
            }
        }
        __syncthreads();
        if (STORE) {
            double* o = outp + 4 * c * kChunk;
            for (int e = threadIdx.x; e < 2 * kChunk; e += kThreads)
                reinterpret_cast<double2*>(o)[e] = reinterpret_cast<const double2*>(st)[e];
        } else {
            for (int e = threadIdx.x; e < kChunk; e += kThreads) acc += st[4 * e] + st[4 * e + 3];
        }
        __syncthreads();
    }
    if (acc == 1.2345) outp[0] = acc;
    (void)lane;
}

template <int MODE, bool STORE>
float timeit(const double* rec, const int32_t* idx, int64_t n, double* outp, int ctas, int smem)
{
    cudaFuncSetAttribute(k_gather<MODE, STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_gather<MODE, STORE><<<148 * ctas, kThreads, smem>>>(rec, idx, n, outp);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) k_gather<MODE, STORE><<<148 * ctas, kThreads, smem>>>(rec, idx, n, outp);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
}

int main()
{
    const int64_t n = 100000000 / kChunk * kChunk;
    double *rec, *outp;
    int32_t* idx;
    cudaMalloc(&rec, n * 32);
    cudaMalloc(&outp, n * 32);
    cudaMalloc(&idx, n * 4);
    cudaMemset(rec, 0, n * 32);
    std::vector<int32_t> h(n);
    std::mt19937_64 rng(1);
    for (int64_t i = 0; i < n; ++i) h[i] = static_cast<int32_t>(i);
    for (int64_t b = 0; b < n; b += 25000) std::shuffle(h.begin() + b, h.begin() + std::min(n, b + 25000), rng);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    const int smem = kChunk * 32;
    const char* names[4] = {"ldgsts 2x16B", "lane pairs  ", "bulk1d 32B  ", "ld.v4.f64   "};
    for (int waves : {0, 1, 2, 4}) {
        cudaMemcpyToSymbol(g_pf_waves, &waves, sizeof(int));
        for (int ctas : {4, 6}) {
            const float g = timeit<4, false>(rec, idx, n, outp, ctas, smem), gs = timeit<4, true>(rec, idx, n, outp, ctas, smem);
            printf("%d CTAs/SM lane pairs + L2 prefetch %d wave(s) ahead: gathers %.3f ms, gathers + stores %.3f ms  err=%s\n",
                   ctas, waves, g, gs, cudaGetErrorString(cudaGetLastError()));
        }
    }
    for (int ctas : {4, 6}) {
        float g[4], gs[4];
        g[0] = timeit<0, false>(rec, idx, n, outp, ctas, smem); gs[0] = timeit<0, true>(rec, idx, n, outp, ctas, smem);
        g[1] = timeit<1, false>(rec, idx, n, outp, ctas, smem); gs[1] = timeit<1, true>(rec, idx, n, outp, ctas, smem);
        g[2] = timeit<2, false>(rec, idx, n, outp, ctas, smem); gs[2] = timeit<2, true>(rec, idx, n, outp, ctas, smem);
        g[3] = timeit<3, false>(rec, idx, n, outp, ctas, smem); gs[3] = timeit<3, true>(rec, idx, n, outp, ctas, smem);
        for (int k = 0; k < 4; ++k)
            printf("%d CTAs/SM %s: gathers %.3f ms, gathers + contiguous stores %.3f ms  err=%s\n", ctas, names[k], g[k],
                   gs[k], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
