// Microbenchmark (round 2): can a cluster exchange a cell's particles through
// distributed shared memory fast enough to replace the random L2 gathers?
//  (a) 32-byte records stored into remote CTAs' shared memory as two 16-byte
//      st.shared::cluster.v2.f64 — random rank + random slot, warp-uniform rank,
//      warp-uniform rank with contiguous slots, and local-only for reference;
//  (b) bulk copies smem -> remote smem (cp.async.bulk.shared::cluster, mbarrier
//      complete_tx), 8 x 12 KB per CTA per round, cluster barrier per round.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o dsmem_store_bw dsmem_store_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kCl = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

__device__ __forceinline__ void st_cl16(uint32_t a, double x, double y)
{
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}

__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// MODE 0 random rank per lane, random slot; 1 own rank, random slot; 2 warp-uniform random rank,
// random slot; 3 warp-uniform random rank, contiguous 32 slots; 4 plain st.shared local random
template <int MODE>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(256) k_store(int iters, int slots, double* out)
{
    extern __shared__ __align__(16) double sm[];
    const uint32_t me = cluster_rank();
    for (int i = threadIdx.x; i < slots * 4; i += blockDim.x) sm[i] = 0.0;
    cluster_sync();
    uint32_t x = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u + 12345u;
    uint32_t xw = (blockIdx.x * 64 + (threadIdx.x >> 5)) * 2246822519u + 777u;
    const uint32_t base = smem_u32(sm);
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        xw ^= xw << 13; xw ^= xw >> 17; xw ^= xw << 5;
        uint32_t r, w;
        if (MODE == 0) { r = (x >> 28) & (kCl - 1); w = (x & 0xFFFFFF) % slots; }
        else if (MODE == 1) { r = me; w = (x & 0xFFFFFF) % slots; }
        else if (MODE == 2) { r = (xw >> 28) & (kCl - 1); w = (x & 0xFFFFFF) % slots; }
        else if (MODE == 3) { r = (xw >> 28) & (kCl - 1); w = ((xw & 0xFFFFFF) % (slots / 32)) * 32 + lane; }
        else { r = me; w = (x & 0xFFFFFF) % slots; }
        const double v = static_cast<double>(it);
        if (MODE == 4) {
            double2* p = reinterpret_cast<double2*>(sm + 4 * w);
            p[0] = make_double2(v, v);
            p[1] = make_double2(v, v);
        } else {
            const uint32_t a = mapa(base + 32u * w, r);
            st_cl16(a, v, v);
            st_cl16(a + 16u, v, v);
        }
    }
    cluster_sync();
    if (sm[threadIdx.x] == 1.2345) out[0] = sm[threadIdx.x];
}

// (b) bulk: send region [kCl][chunk] -> receivers' recv region [kCl][chunk] at my rank's slot
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(128) k_bulk(int iters, int chunk, double* out)
{
    extern __shared__ __align__(128) unsigned char smb[];
    __shared__ __align__(8) uint64_t bar;
    unsigned char* send = smb;
    unsigned char* recv = smb + static_cast<size_t>(kCl) * chunk;
    const uint32_t me = cluster_rank();
    for (int i = threadIdx.x; i < kCl * chunk / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(send)[i] = i;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync();
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                         "r"(kCl * chunk) : "memory");
        }
        cluster_sync();   // every receiver armed before any sender completes bytes on it
        if (threadIdx.x < kCl) {
            const uint32_t d = (me + threadIdx.x) % kCl;
            const uint32_t dst = mapa(smem_u32(recv + static_cast<size_t>(me) * chunk), d);
            const uint32_t rb = mapa(smem_u32(&bar), d);
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                "r"(smem_u32(send + static_cast<size_t>(d) * chunk)), "r"(chunk), "r"(rb)
                : "memory");
        }
        // wait for my receive phase
        asm volatile(
            "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
            "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(&bar)),
            "r"(phase)
            : "memory");
        phase ^= 1u;
    }
    cluster_sync();
    if (recv[threadIdx.x] == 123 && out) out[0] = 1.0;
}

int main()
{
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int slots = 3200;              // 100 KB of 32-byte records per CTA
    const int iters = 2048;
    const int blocks = 296 / kCl * kCl;  // 2 CTAs per SM
    auto run_store = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, slots * 32);
        kern<<<blocks, 256, slots * 32>>>(iters, slots, out);
        cudaEventRecord(a);
        kern<<<blocks, 256, slots * 32>>>(iters, slots, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double recs = static_cast<double>(blocks) * 256 * iters;
        printf("%-44s %.3f ms  %7.1f G records/s  %.3f records/clk/SM (1.965 GHz)  err=%s\n", name, ms,
               recs / ms / 1e6, recs / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    };
    run_store(k_store<0>, "remote st.v2 x2, random rank/slot");
    run_store(k_store<1>, "st.shared::cluster own rank, random slot");
    run_store(k_store<2>, "remote, warp-uniform rank, random slot");
    run_store(k_store<3>, "remote, warp-uniform rank, contiguous slots");
    run_store(k_store<4>, "local st.shared random slot");
    for (int chunk : {4096, 12288}) {
        const size_t sm = 2ull * kCl * chunk;
        cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
        const int bl = 148 / kCl * kCl * (sm <= 100 * 1024 ? 2 : 1);
        const int it = 400;
        k_bulk<<<bl, 128, sm>>>(it, chunk, out);
        cudaEventRecord(a);
        k_bulk<<<bl, 128, sm>>>(it, chunk, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = static_cast<double>(bl) * kCl * chunk * it;
        printf("bulk smem->dsmem chunk %6d B, %d CTAs: %.3f ms  %.1f GB/s total  %.2f B/clk/SM  err=%s\n", chunk, bl, ms,
               bytes / ms / 1e6, bytes / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
