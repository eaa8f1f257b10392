// Round 2 microbenchmark: do random 32-byte record writes (and random 8-byte SoA writes) run at
// DRAM-streaming speed when every write lands inside an L2-sized window that the whole GPU
// fills before moving on?  n = 1e8 records read sequentially (32 B each) and written to
// dest = window base + a keyed random bijection of the index inside the window (W records).
// W = n is the fully random scatter (the cold k_scatter's pattern).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o window_scatter window_scatter.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t h)
{
    h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
    return h;
}

// bijection on [0, W) for W a power of two: 4-round Feistel on the two halves of the bits
__device__ __forceinline__ uint32_t perm_w(uint32_t x, uint32_t logw, uint32_t key)
{
    const uint32_t hb = logw >> 1, lb = logw - hb;
    const uint32_t lm = (1u << lb) - 1u, hm = (1u << hb) - 1u;
    uint32_t L = x & lm, R = x >> lb;
    for (int r = 0; r < 4; ++r) {
        if (r & 1) R ^= mix(L ^ (key + 77u * r)) & hm;
        else L ^= mix(R ^ (key + 77u * r)) & lm;
    }
    return L | (R << lb);
}

// mode 0: 32-B record out; mode 1: SoA out (3 x 8 B rows + 4 B cell)
__global__ void k_scatter(const double4* __restrict__ src, int64_t n, uint32_t logw, double4* __restrict__ dst,
                          double* __restrict__ soa, int32_t* __restrict__ cell, int mode)
{
    const int64_t W = 1ll << logw;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double4 r = src[i];
        const int64_t base = i & ~(W - 1);
        const int64_t d = base + perm_w(static_cast<uint32_t>(i & (W - 1)), logw, 0x1234567u);
        if (mode == 0) {
            dst[d] = r;
        } else {
            soa[d] = r.x; soa[n + d] = r.y; soa[2 * n + d] = r.z; cell[d] = static_cast<int32_t>(__double_as_longlong(r.w));
        }
    }
}

int main()
{
    const int64_t n = 1ll << 27;      // 134M records = 4.3 GB (power of two so windows tile it)
    double4 *src, *dst; double* soa; int32_t* cell;
    cudaMalloc(&src, n * 32); cudaMalloc(&dst, n * 32); cudaMalloc(&soa, n * 24); cudaMalloc(&cell, n * 4);
    cudaMemset(src, 0, n * 32);
    for (int mode = 0; mode < 2; ++mode)
        for (uint32_t logw : {27u, 24u, 22u, 21u, 20u, 19u, 18u, 16u, 12u}) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            k_scatter<<<148 * 8, 256>>>(src, n, logw, dst, soa, cell, mode);
            cudaEventRecord(a);
            for (int r = 0; r < 3; ++r) k_scatter<<<148 * 8, 256>>>(src, n, logw, dst, soa, cell, mode);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
            const double bytes = n * (32.0 + (mode ? 28.0 : 32.0));
            printf("%s window %8lld records (%7.1f MB out): %.3f ms  %.0f GB/s (read+write)  err=%s\n",
                   mode ? "SoA   " : "record", 1ll << logw, (1ll << logw) * (mode ? 28.0 : 32.0) / 1e6, ms,
                   bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
