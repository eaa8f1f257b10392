// Accuracy of the sm_100a fp64 approximation instructions (rsqrt.approx / rcp.approx) and of
// one / two Newton steps on them, over log-uniform inputs: max relative error vs IEEE 1/sqrt, 1/x.
#include <cstdio>
#include <cmath>
#include <cstdint>
__global__ void k(int n, double* err)
{
    double e[6] = {0, 0, 0, 0, 0, 0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint64_t h = 0x9E3779B97F4A7C15ull * (i + 1); h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
        const double x = exp2(-40.0 + 80.0 * (double)(h >> 11) * 0x1.0p-53);
        double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
        const double ex = 1.0 / sqrt(x);
        const double hx = 0.5 * x;
        double y1 = fma(y, fma(-hx * y, y, 0.5), y);
        double y2 = fma(y1, fma(-hx * y1, y1, 0.5), y1);
        e[0] = fmax(e[0], fabs(y / ex - 1)); e[1] = fmax(e[1], fabs(y1 / ex - 1)); e[2] = fmax(e[2], fabs(y2 / ex - 1));
        double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        const double er = 1.0 / x;
        double r1 = fma(r, fma(-x, r, 1.0), r);
        double r2 = fma(r1, fma(-x, r1, 1.0), r1);
        e[3] = fmax(e[3], fabs(r / er - 1)); e[4] = fmax(e[4], fabs(r1 / er - 1)); e[5] = fmax(e[5], fabs(r2 / er - 1));
    }
    for (int q = 0; q < 6; ++q) {
        unsigned long long* p = reinterpret_cast<unsigned long long*>(err + q);
        atomicMax(p, __double_as_longlong(e[q]));   // positive doubles order like their bits
    }
}
int main()
{
    double* d; cudaMalloc(&d, 6 * sizeof(double)); cudaMemset(d, 0, 6 * sizeof(double));
    k<<<1184, 256>>>(1 << 26, d);
    double h[6]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("rsqrt.approx %.3e  +1 NR %.3e  +2 NR %.3e\nrcp.approx   %.3e  +1 NR %.3e  +2 NR %.3e\n", h[0], h[1], h[2], h[3], h[4], h[5]);
    return 0;
}
