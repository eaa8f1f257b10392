// Random-order writes/reads of C-byte chunks over a 3.2 GB array (each chunk written/read once),
// C = 32..1024: does the cost of random record traffic depend on the chunk size?
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

// each warp moves one C-byte chunk per iteration cooperatively (lanes cover 32 B each)
__global__ void k_wr(const int32_t* __restrict__ perm, int64_t nchunks, int C, double* __restrict__ out, int write)
{
    const int lane = threadIdx.x & 31;
    const int per = C / 32;             // 32-byte pieces per chunk
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int cpw = 32 / per;          // chunks per warp-iteration
    for (int64_t c0 = wid * cpw; c0 < nchunks; c0 += nw * cpw) {
        const int64_t c = c0 + lane / per;
        if (c >= nchunks) continue;
        const int64_t d = (int64_t)perm[c] * C + (lane % per) * 32;
        double* p = (double*)((char*)out + d);
        if (write) {
            asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};" :: "l"(p), "d"(1.0) : "memory");
        } else {
            double a, b, e, f;
            asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(e), "=d"(f) : "l"(p));
            if (a == 12345.0) out[0] = b + e + f;
        }
    }
}

int main()
{
    const int64_t bytes = 3200000000ll;
    double* out; int32_t* perm;
    cudaMalloc(&out, bytes); cudaMalloc(&perm, (bytes / 32) * 4);
    cudaMemset(out, 0, bytes);
    std::mt19937_64 rng(1);
    for (int C : {32, 64, 128, 256, 512, 1024}) {
        const int64_t nc = bytes / C;
        std::vector<int32_t> h(nc);
        for (int64_t i = 0; i < nc; ++i) h[i] = (int32_t)i;
        std::shuffle(h.begin(), h.end(), rng);
        cudaMemcpy(perm, h.data(), nc * 4, cudaMemcpyHostToDevice);
        for (int write = 0; write < 2; ++write) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            k_wr<<<148 * 8, 256>>>(perm, nc, C, out, write);
            cudaEventRecord(a);
            for (int r = 0; r < 3; ++r) k_wr<<<148 * 8, 256>>>(perm, nc, C, out, write);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
            printf("chunk %5d B  %s: %.3f ms  %.0f GB/s data\n", C, write ? "write" : "read ", ms, bytes / ms / 1e6);
        }
    }
    return 0;
}
