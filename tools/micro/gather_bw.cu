// Microbenchmark: gathering 32-byte records from src[idx[i]] (idx = identity shuffled in
// blocks of `span` records) and streaming them out SoA — the collide's access pattern —
// vs. sequential.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void k_gather(const double* __restrict__ src, const int32_t* __restrict__ idx, int64_t n, double* __restrict__ out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = idx[i];
        double a, b, c, d;
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(src + 4 * s));
        out[i] = a; out[n + i] = b; out[2 * n + i] = c;
    }
}

int main()
{
    const int64_t n = 100000000;
    double* src; int32_t* idx; double* out;
    cudaMalloc(&src, n * 32); cudaMalloc(&idx, n * 4); cudaMalloc(&out, 3 * n * 8);
    cudaMemset(src, 0, n * 32);
    std::vector<int32_t> h(n);
    std::mt19937_64 rng(1);
    const int64_t spans[] = {0, 1 << 15, 1 << 18, 1 << 20, 1 << 22, 1 << 24, n};
    for (int64_t S : spans) {
        for (int64_t i = 0; i < n; ++i) h[i] = (int32_t)i;
        if (S > 0)
            for (int64_t b = 0; b < n; b += S) std::shuffle(h.begin() + b, h.begin() + std::min(n, b + S), rng);
        cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int w = 0; w < 2; ++w) k_gather<<<148 * 8, 256>>>(src, idx, n, out);
        cudaEventRecord(a);
        const int R = 5;
        for (int r = 0; r < R; ++r) k_gather<<<148 * 8, 256>>>(src, idx, n, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= R;
        const double bytes = n * (32.0 + 4.0 + 24.0);
        printf("span %12lld records (%8.1f MB): %.3f ms  %.0f GB/s (r+w)\n", (long long)S, S * 32.0 / 1e6, ms, bytes / ms / 1e6);
    }
    return 0;
}
