// Microbenchmark: random 16-byte loads from distributed shared memory of an
// 8-CTA cluster (the gather pattern of a cluster-staged collide), vs local smem.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int CLUSTER>
__global__ void __cluster_dims__(CLUSTER, 1, 1) k_dsmem(int iters, int words, int remote, double* out)
{
    extern __shared__ double2 sm[];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = make_double2(i, blockIdx.x);
    cl.sync();
    uint32_t x = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u + 12345u;
    double acc = 0;
    const unsigned me = cl.block_rank();
    for (int it = 0; it < iters; ++it) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        const unsigned r = remote ? (x >> 24) % CLUSTER : me;
        const int w = (x & 0xFFFFFF) % words;
        const double2* p = cl.map_shared_rank(sm, r);
        const double2 v = p[w];
        acc += v.x + v.y;
    }
    cl.sync();
    if (acc == 1.2345) out[0] = acc;
}

int main()
{
    double* out; cudaMalloc(&out, 8);
    const int words = 100 * 1024 / 16;      // 100 KB per CTA
    const int iters = 4096;
    for (int remote = 0; remote < 2; ++remote) {
        auto kern = k_dsmem<8>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        const int blocks = 148 * 2 / 8 * 8;   // ~2 CTAs per SM
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        kern<<<blocks, 256, 100 * 1024>>>(iters, words, remote, out);
        cudaEventRecord(a);
        kern<<<blocks, 256, 100 * 1024>>>(iters, words, remote, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double loads = (double)blocks * 256 * iters;
        printf("%s: %.3f ms  %.2f G loads/s total, %.2f loads/clk/SM (1.965 GHz), err=%s\n", remote ? "DSMEM random rank" : "local smem   ",
               ms, loads / ms / 1e6, loads / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
