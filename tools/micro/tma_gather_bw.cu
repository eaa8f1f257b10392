// Microbenchmark: random 32-byte record gathers into shared memory, as k_collide_large's
// phase 1 does them (indices shuffled inside windows of `span` records, i.e. a cell slice),
// issued (a) as two 16-byte cp.async (LDGSTS) per record by every thread, or (b) as
// Blackwell TMA tile::gather4 (4 records per instruction, completion on an mbarrier).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_gather_bw tma_gather_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

constexpr int kChunk = 1536;     // records per CTA chunk (= 2 x 768 pairs)
constexpr int kThreads = 256;

__device__ __forceinline__ void cp16(void* s, const void* g)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g)
                 : "memory");
}

__global__ void __launch_bounds__(kThreads) k_ldgsts(const double* __restrict__ rec, const int32_t* __restrict__ idx,
                                                     int64_t n, double* __restrict__ out)
{
    extern __shared__ __align__(16) double st[];
    double acc = 0.0;
    const int64_t nch = n / kChunk;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
        for (int e = threadIdx.x; e < kChunk; e += kThreads) {
            const double* g = rec + 4 * static_cast<int64_t>(idx[c * kChunk + e]);
            cp16(st + 4 * e, g);
            cp16(st + 4 * e + 2, g + 2);
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
        __syncthreads();
        for (int e = threadIdx.x; e < kChunk; e += kThreads) acc += st[4 * e] + st[4 * e + 3];
        __syncthreads();
    }
    if (acc == 1.2345) out[0] = acc;
}

// (c) 256-bit register loads (one LDG.E.256 request per record), then 2 x st.shared.v2
__global__ void __launch_bounds__(kThreads) k_ld256(const double* __restrict__ rec, const int32_t* __restrict__ idx,
                                                    int64_t n, double* __restrict__ out)
{
    extern __shared__ __align__(16) double st[];
    double acc = 0.0;
    const int64_t nch = n / kChunk;
    constexpr int R = kChunk / kThreads;      // 6 records per thread
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
        double a[R], b[R], cc[R], d[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int e = threadIdx.x + r * kThreads;
            const double* g = rec + 4 * static_cast<int64_t>(idx[c * kChunk + e]);
            asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a[r]), "=d"(b[r]), "=d"(cc[r]), "=d"(d[r]) : "l"(g));
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int e = threadIdx.x + r * kThreads;
            reinterpret_cast<double2*>(st + 4 * e)[0] = make_double2(a[r], b[r]);
            reinterpret_cast<double2*>(st + 4 * e)[1] = make_double2(cc[r], d[r]);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < kChunk; e += kThreads) acc += st[4 * e] + st[4 * e + 3];
        __syncthreads();
    }
    if (acc == 1.2345) out[0] = acc;
}

__global__ void __launch_bounds__(kThreads) k_gather4(const __grid_constant__ CUtensorMap tmap,
                                                      const int32_t* __restrict__ idx, int64_t n,
                                                      double* __restrict__ out)
{
    extern __shared__ __align__(16) double st_raw[];
    // TMA destinations must be 128-byte aligned: round the dynamic smem base up
    double* st = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(st_raw) + 127) & ~uintptr_t(127));
    __shared__ __align__(8) uint64_t bar;
    const unsigned sbar = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double acc = 0.0;
    uint32_t phase = 0;
    const int64_t nch = n / kChunk;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sbar), "r"(kChunk * 32) : "memory");
        __syncthreads();
        if (threadIdx.x < 32) {          // one warp issues the chunk's kChunk/4 gather4 instructions
            for (int g = threadIdx.x; g < kChunk / 4; g += 32) {
                const int32_t* ip = idx + c * kChunk + 4 * g;
                const unsigned dst = (unsigned)__cvta_generic_to_shared(st + 16 * g);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
                    "l"(&tmap), "r"(0), "r"(ip[0]), "r"(ip[1]), "r"(ip[2]), "r"(ip[3]), "r"(sbar)
                    : "memory");
            }
        }
        // wait for the transaction bytes
        asm volatile(
            "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(
                sbar),
            "r"(phase)
            : "memory");
        phase ^= 1;
        for (int e = threadIdx.x; e < kChunk; e += kThreads) acc += st[4 * e] + st[4 * e + 3];
        __syncthreads();
    }
    if (acc == 1.2345) out[0] = acc;
}

// random 32-byte record WRITES (the cold k_scatter pattern): records come from a sequential
// stream; (a) st.global.v4.f64 per record per thread; (b) staged in smem per warp, then one
// lane issues TMA tile::scatter4 per 4 records.
__global__ void __launch_bounds__(kThreads) k_st256(const int32_t* __restrict__ idx, int64_t n, double* __restrict__ rec)
{
    for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
        const double a = (double)i, b = 2.0 * i, c = 3.0 * i, d = 4.0 * i;
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(rec + 4 * (int64_t)idx[i]), "d"(a), "d"(b), "d"(c),
                     "d"(d) : "memory");
    }
}

__global__ void __launch_bounds__(kThreads) k_scatter4(const __grid_constant__ CUtensorMap tmap,
                                                       const int32_t* __restrict__ idx, int64_t n)
{
    extern __shared__ __align__(16) double sraw[];
    double* st = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sraw) + 127) & ~uintptr_t(127));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* my = st + w * 32 * 4 * 2;          // two 1 KB buffers per warp
    int buf = 0;
    for (int64_t i0 = (blockIdx.x * (int64_t)kThreads) + w * 32; i0 < n; i0 += (int64_t)gridDim.x * kThreads) {
        const int64_t i = i0 + lane;
        double* slot = my + buf * 128 + 4 * lane;
        // the buffer written two iterations ago must have been read by the TMA engine
        if ((lane & 3) == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // per-thread groups
        __syncwarp();
        slot[0] = (double)i; slot[1] = 2.0 * i; slot[2] = 3.0 * i; slot[3] = 4.0 * i;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        const int32_t d = (i < n) ? idx[i] : 0;
        const int32_t d1 = __shfl_down_sync(0xFFFFFFFFu, d, 1);
        const int32_t d2 = __shfl_down_sync(0xFFFFFFFFu, d, 2);
        const int32_t d3 = __shfl_down_sync(0xFFFFFFFFu, d, 3);
        if ((lane & 3) == 0) {
            const unsigned src = (unsigned)__cvta_generic_to_shared(slot);
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                         ::"l"(&tmap), "r"(0), "r"(d), "r"(d1), "r"(d2), "r"(d3), "r"(src) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        buf ^= 1;
    }
    if ((lane & 3) == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// gather (LDGSTS) + contiguous output of the same bytes, per chunk: (A) st.global.v2 by every
// thread from shared memory, (B) one TMA bulk store (cp.async.bulk.global.shared::cta) of the chunk
template <bool TMA_STORE>
__global__ void __launch_bounds__(kThreads) k_gather_store(const double* __restrict__ rec,
                                                           const int32_t* __restrict__ idx, int64_t n,
                                                           double* __restrict__ outp)
{
    extern __shared__ __align__(16) double sraw2[];
    double* st = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sraw2) + 127) & ~uintptr_t(127));
    const int64_t nch = n / kChunk;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
        if (TMA_STORE && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        for (int e = threadIdx.x; e < kChunk; e += kThreads) {
            const double* g = rec + 4 * static_cast<int64_t>(idx[c * kChunk + e]);
            cp16(st + 4 * e, g);
            cp16(st + 4 * e + 2, g + 2);
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
        __syncthreads();
        double* o = outp + 4 * c * kChunk;
        if (TMA_STORE) {
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o),
                             "r"((unsigned)__cvta_generic_to_shared(st)), "r"(kChunk * 32) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else {
            for (int e = threadIdx.x; e < 2 * kChunk; e += kThreads)
                reinterpret_cast<double2*>(o)[e] = reinterpret_cast<const double2*>(st)[e];
        }
    }
    if (TMA_STORE && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main()
{
    const int64_t n = 100000000 / kChunk * kChunk;
    double* rec;
    int32_t* idx;
    double* out;
    cudaMalloc(&rec, n * 32);
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 8);
    {   // distinct nonzero records
        std::vector<double> hr(4 * (n / 16));
        for (size_t i = 0; i < hr.size(); ++i) hr[i] = 1.0 + static_cast<double>(i % 9973);
        for (int k = 0; k < 16; ++k) cudaMemcpy(rec + 4 * (n / 16) * k, hr.data(), hr.size() * 8, cudaMemcpyHostToDevice);
    }
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q);
    if (!encode) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    CUtensorMap tmap;
    const cuuint64_t dims[2] = {4, static_cast<cuuint64_t>(n)};
    const cuuint64_t strides[1] = {32};
    const cuuint32_t box[2] = {4, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, rec, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc %d\n", (int)r);
    std::vector<int32_t> h(n);
    std::mt19937_64 rng(1);
    const int smem = kChunk * 32 + 128;
    cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int64_t S : {int64_t(25000), int64_t(1) << 20, n}) {
        for (int64_t i = 0; i < n; ++i) h[i] = static_cast<int32_t>(i);
        for (int64_t b = 0; b < n; b += S) std::shuffle(h.begin() + b, h.begin() + std::min(n, b + S), rng);
        cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int ctas : {4, 6}) {
            float ms[2];
            for (int k = 0; k < 2; ++k) {
                for (int rep = 0; rep < 2; ++rep) {
                    if (rep == 1) cudaEventRecord(a);
                    if (k == 0) k_ldgsts<<<148 * ctas, kThreads, smem>>>(rec, idx, n, out);
                    else k_gather4<<<148 * ctas, kThreads, smem>>>(tmap, idx, n, out);
                    if (rep == 1) cudaEventRecord(b);
                }
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms[k], a, b);
            }
            {
                float m3 = 0;
                cudaFuncSetAttribute(k_ld256, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                for (int rep = 0; rep < 2; ++rep) {
                    if (rep == 1) cudaEventRecord(a);
                    k_ld256<<<148 * ctas, kThreads, smem>>>(rec, idx, n, out);
                    if (rep == 1) cudaEventRecord(b);
                }
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&m3, a, b);
                printf("span %10lld, %d CTAs/SM: LDG.256 %.3f ms\n", (long long)S, ctas, m3);
            }
            printf("span %10lld, %d CTAs/SM: LDGSTS %.3f ms (%.0f GB/s)  TMA gather4 %.3f ms (%.0f GB/s)  err=%s\n",
                   (long long)S, ctas, ms[0], n * 32.0 / ms[0] / 1e6, ms[1], n * 32.0 / ms[1] / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    {   // gathers (cell-sized spans) + output stores of the same bytes to a second 3.2 GB array
        double* outp;
        cudaMalloc(&outp, n * 32);
        for (int64_t i = 0; i < n; ++i) h[i] = static_cast<int32_t>(i);
        for (int64_t b = 0; b < n; b += 25000) std::shuffle(h.begin() + b, h.begin() + std::min(n, b + 25000), rng);
        cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(k_gather_store<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_gather_store<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float ms[2];
        for (int k = 0; k < 2; ++k) {
            for (int rep = 0; rep < 2; ++rep) {
                if (rep == 1) cudaEventRecord(a);
                if (k == 0) k_gather_store<false><<<148 * 4, kThreads, smem>>>(rec, idx, n, outp);
                else k_gather_store<true><<<148 * 4, kThreads, smem>>>(rec, idx, n, outp);
                if (rep == 1) cudaEventRecord(b);
            }
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms[k], a, b);
        }
        printf("gather (25000 spans) + contiguous store of the chunk: st.global %.3f ms, TMA bulk store %.3f ms  err=%s\n",
               ms[0], ms[1], cudaGetErrorString(cudaGetLastError()));
        cudaFree(outp);
    }
    {   // L2-resident gathers: 1e8 random gathers out of a 48 MB (1.5M-record) array
        const int64_t small = 1536000;
        for (int64_t i = 0; i < n; ++i) h[i] = static_cast<int32_t>(rng() % small);
        cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int ctas : {4, 6}) {
            float ms = 0;
            for (int rep = 0; rep < 2; ++rep) {
                if (rep == 1) cudaEventRecord(a);
                k_ldgsts<<<148 * ctas, kThreads, smem>>>(rec, idx, n, out);
                if (rep == 1) cudaEventRecord(b);
            }
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            float ms2 = 0;
            cudaFuncSetAttribute(k_ld256, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            for (int rep = 0; rep < 2; ++rep) {
                if (rep == 1) cudaEventRecord(a);
                k_ld256<<<148 * ctas, kThreads, smem>>>(rec, idx, n, out);
                if (rep == 1) cudaEventRecord(b);
            }
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms2, a, b);
            printf("L2-resident (48 MB) random gathers, %d CTAs/SM: LDGSTS %.3f ms (%.2f G records/s)  LDG.256 %.3f ms "
                   "(%.2f G records/s) err=%s\n", ctas, ms, n / ms / 1e6, ms2, n / ms2 / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
        // sequential gathers (idx = i): the DRAM streaming reference
        for (int64_t i = 0; i < n; ++i) h[i] = static_cast<int32_t>(i);
        cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
            if (rep == 1) cudaEventRecord(a);
            k_ldgsts<<<148 * 4, kThreads, smem>>>(rec, idx, n, out);
            if (rep == 1) cudaEventRecord(b);
        }
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("sequential records (3.2 GB from DRAM): LDGSTS %.3f ms (%.0f GB/s)\n", ms, n * 32.0 / ms / 1e6);
    }
    cudaFuncSetAttribute(k_scatter4, cudaFuncAttributeMaxDynamicSharedMemorySize, kThreads / 32 * 32 * 32 * 2 + 128);
    for (int64_t S : {int64_t(25000), int64_t(1) << 20, n}) {
        for (int64_t i = 0; i < n; ++i) h[i] = static_cast<int32_t>(i);
        for (int64_t b = 0; b < n; b += S) std::shuffle(h.begin() + b, h.begin() + std::min(n, b + S), rng);
        cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float ms[2];
        for (int k = 0; k < 2; ++k) {
            for (int rep = 0; rep < 2; ++rep) {
                if (rep == 1) cudaEventRecord(a);
                if (k == 0) k_st256<<<148 * 8, kThreads>>>(idx, n, rec);
                else k_scatter4<<<148 * 4, kThreads, kThreads / 32 * 32 * 32 * 2 + 128>>>(tmap, idx, n);
                if (rep == 1) cudaEventRecord(b);
            }
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms[k], a, b);
        }
        // check: record at idx[5] holds 5
        double chk[4];
        cudaMemcpy(chk, rec + 4 * (int64_t)h[5], 32, cudaMemcpyDeviceToHost);
        printf("scatter span %10lld: st.v4 %.3f ms (%.0f GB/s)  TMA scatter4 %.3f ms (%.0f GB/s)  check %g %g err=%s\n",
               (long long)S, ms[0], n * 32.0 / ms[0] / 1e6, ms[1], n * 32.0 / ms[1] / 1e6, chk[0], chk[3],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
