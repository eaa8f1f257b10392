// Microbenchmark: streaming 32-byte records to destinations drawn at random
// within a window of `span` bytes (the k_move write pattern), vs sequential.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scatter_bw scatter_bw.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void k_scatter(const double* __restrict__ v, const int32_t* __restrict__ dest, int64_t n, double* __restrict__ out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = dest[i];
        const double x = v[i], y = v[n + i], z = v[2 * n + i];
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" :: "l"(out + 4 * d), "d"(x), "d"(y), "d"(z), "d"(0.0) : "memory");
    }
}

int main()
{
    const int64_t n = 100000000;
    double* v; int32_t* dest; double* out;
    cudaMalloc(&v, 3 * n * 8); cudaMalloc(&dest, n * 4); cudaMalloc(&out, n * 32);
    cudaMemset(v, 0, 3 * n * 8);
    std::vector<int32_t> h(n);
    std::mt19937_64 rng(1);
    // dest = a permutation where consecutive inputs go to random places in [0, n) but
    // restricted so that a window of W consecutive inputs maps into a span of S records
    const int64_t spans[] = {0, 1 << 20, 1 << 22, 1 << 24, 1 << 26, n};
    for (int64_t S : spans) {
        for (int64_t i = 0; i < n; ++i) h[i] = (int32_t)i;
        if (S > 0) {
            // shuffle within blocks of S records: writes of a window of inputs hit a span of S*32 bytes
            for (int64_t b = 0; b < n; b += S) {
                int64_t e = std::min(n, b + S);
                std::shuffle(h.begin() + b, h.begin() + e, rng);
            }
        }
        cudaMemcpy(dest, h.data(), n * 4, cudaMemcpyHostToDevice);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int w = 0; w < 2; ++w) k_scatter<<<148 * 8, 256>>>(v, dest, n, out);
        cudaEventRecord(a);
        const int R = 5;
        for (int r = 0; r < R; ++r) k_scatter<<<148 * 8, 256>>>(v, dest, n, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= R;
        const double bytes = n * (24.0 + 4.0 + 32.0);
        printf("span %12lld records (%8.1f MB): %.3f ms  %.0f GB/s (r+w)\n", (long long)S, S * 32.0 / 1e6, ms, bytes / ms / 1e6);
    }
    return 0;
}
