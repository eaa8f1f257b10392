// Prototype (round 2): the cell-exchange collide.  A cluster of 8 CTAs owns one
// cell at a time.  Phase 1: each CTA reads its contiguous share of the cell's
// (cell-sorted) SoA velocities, computes every slot's pair-order position
// p = pi^-1(s) (keyed Feistel, R1) and writes a 32-byte record into a per-cluster
// L2 scratch, grouped by destination segment (exact run offsets from a count
// exchange over DSMEM).  Phase 2: each CTA reads its segments' records (one
// contiguous run each), places them in shared memory by p, and collides
// adjacent pairs; the output is written in pair order, coalesced.  No random
// global access anywhere: the random placement happens in local shared memory.
// mode 0: identity (data movement only, validated on the host); 1: Philox +
// AS241 + TA77 per pair (the real arithmetic).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o cluster_xchg cluster_xchg.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2508_06771_b200/csrc/cc_device.cuh"

constexpr int kCl = 8;
constexpr int kThr = 256;
constexpr int kSmax = 2048;     // records per segment (stage capacity)
constexpr int kCmax = 4;        // segments per CTA -> N <= 8 * 4 * 2048 = 65536
constexpr int kKmax = kCl * kCmax;
constexpr int kU = kSmax / kThr;   // records per thread per segment

struct __align__(16) Sm {
    double stage[4 * kSmax];              // 64 KB: placed records of the current segment
    uint32_t ps[kCmax * kSmax];           // 32 KB: p of my slots
    int32_t cnt[kKmax][kKmax];            // [src segment][dst segment]
    int32_t cur[kCmax][kKmax];            // my run cursors
    int32_t cell;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cl_s32(uint32_t a, int32_t v)
{
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
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

__device__ __forceinline__ uint32_t feistel_Einv(const cc::Feistel& f, uint32_t y)
{
    const uint32_t amask = (1u << f.bL) - 1u;
    uint32_t L = y & amask, R = y >> f.bL;
#pragma unroll
    for (int r = 7; r >= 0; --r) {
        if ((r & 1) == 0) {
            L ^= cc::fmix32_small(R, f.kp[r]) & amask;
        } else {
            const uint32_t t = __umulhi(cc::fmix32_small(L, f.kp[r]), f.m);
            R = (R >= t) ? R - t : R + f.m - t;
        }
    }
    return L + (R << f.bL);
}

__device__ __forceinline__ uint32_t feistel_pi_inv(const cc::Feistel& f, uint32_t s)
{
    uint32_t x = feistel_Einv(f, s);
    while (x >= f.N) x = feistel_Einv(f, x);
    return x;
}

template <int MODE, int DISCARD, int PF>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kThr, 2)
k_xchg(const double* __restrict__ v, int64_t ldv, const int32_t* __restrict__ off, int M, double* __restrict__ vout,
       int32_t* __restrict__ cout, int32_t* __restrict__ pout, double* __restrict__ scratch, int* __restrict__ counter,
       double C, double* __restrict__ sink)
{
    extern __shared__ __align__(16) unsigned char smraw[];
    Sm& S_ = *reinterpret_cast<Sm*>(smraw);
    const uint32_t rank = cluster_rank();
    const int tid = threadIdx.x;
    double* scr = scratch + static_cast<int64_t>(blockIdx.x / kCl) * (4ll * kCl * kCmax * kSmax);
    double accm = 0.0;
    for (;;) {
        if (rank == 0 && tid == 0) {
            const int j = atomicAdd(counter, 1);
            for (uint32_t d = 0; d < kCl; ++d) st_cl_s32(mapa(smem_u32(&S_.cell), d), j);
        }
        cluster_sync();
        const int j = S_.cell;
        if (j >= M) break;
        const int32_t o = off[j], N = off[j + 1] - o;
        const int c = (N + kCl * kSmax - 1) / (kCl * kSmax);
        int32_t S = (N + kCl * c - 1) / (kCl * c);
        S = (S + 3) & ~3;                          // segment starts 128-byte aligned in the scratch
        const int K = (N + S - 1) / S;
        const cc::U4 keys = cc::philox4x32_10(cc::U4{0u, static_cast<uint32_t>(j), 7u, 1u}, 42u, 0u);
        const cc::Feistel f = cc::make_feistel(static_cast<uint32_t>(N), keys);
        for (int i = tid; i < kCmax * kKmax; i += kThr) (&S_.cur[0][0])[i] = 0;
        if (PF && tid < 3 * c) {          // my v slices -> L2 while the Feistel runs
            const int t = tid / 3, comp = tid % 3;
            const int g = t * kCl + static_cast<int>(rank);
            const int32_t s0 = g * S, s1 = min(s0 + S, N);
            if (s1 > s0) {
                const double* a = v + comp * ldv + o + s0;
                const uintptr_t lo = reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15);
                const uintptr_t hi = (reinterpret_cast<uintptr_t>(v + comp * ldv + o + s1) + 15) & ~uintptr_t(15);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(static_cast<uint32_t>(hi - lo)) : "memory");
            }
        }
        __syncthreads();
        // phase 1a: p of my slots, counts per destination segment
        for (int t = 0; t < c; ++t) {
            const int g = t * kCl + static_cast<int>(rank);
            const int32_t s0 = g * S, s1 = min(s0 + S, N);
            for (int32_t s = s0 + tid; s < s1; s += kThr) {
                const uint32_t p = feistel_pi_inv(f, static_cast<uint32_t>(s));
                S_.ps[t * kSmax + (s - s0)] = p;
                const uint32_t dg = p / static_cast<uint32_t>(S);
                const uint32_t peers = __match_any_sync(__activemask(), dg);
                if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&S_.cur[t][dg], __popc(peers));
            }
        }
        __syncthreads();
        // publish my counts to every CTA of the cluster
        for (int i = tid; i < c * K * kCl; i += kThr) {
            const int d = i / (c * K), r = i % (c * K), t = r / K, dg = r % K;
            const int g = t * kCl + static_cast<int>(rank);
            if (g < K) st_cl_s32(mapa(smem_u32(&S_.cnt[g][dg]), d), S_.cur[t][dg]);
        }
        cluster_sync();
        // run bases: dst segment dg starts at dg * S; my run after every lower source segment's
        for (int i = tid; i < c * K; i += kThr) {
            const int t = i / K, dg = i % K;
            const int g = t * kCl + static_cast<int>(rank);
            int32_t b = dg * S;
            for (int gs = 0; gs < g; ++gs) b += S_.cnt[gs][dg];
            S_.cur[t][dg] = b;
        }
        __syncthreads();
        // phase 1b: records into the scratch runs (loads batched: kU per thread in flight)
        for (int t = 0; t < c; ++t) {
            const int g = t * kCl + static_cast<int>(rank);
            const int32_t s0 = g * S, s1 = min(s0 + S, N);
            double x[kU], y[kU], z[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int32_t s = min(s0 + tid + u * kThr, s1 - 1);
                x[u] = __ldg(v + o + s); y[u] = __ldg(v + ldv + o + s); z[u] = __ldg(v + 2 * ldv + o + s);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int32_t s = s0 + tid + u * kThr;
                if (s < s1) {
                    const uint32_t p = S_.ps[t * kSmax + (s - s0)];
                    const uint32_t dg = p / static_cast<uint32_t>(S);
                    const int32_t q = atomicAdd(&S_.cur[t][dg], 1);
                    const double w = __longlong_as_double((static_cast<long long>(p - dg * S) << 32) |
                                                          static_cast<uint32_t>(o + s));
                    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(scr + 4ll * q), "d"(x[u]), "d"(y[u]),
                                 "d"(z[u]), "d"(w)
                                 : "memory");
                }
            }
        }
        cluster_sync();
        // phase 2: my segments
        for (int t = 0; t < c; ++t) {
            const int g = t * kCl + static_cast<int>(rank);
            if (g >= K) break;
            const int32_t p0 = g * S, Sg = min(S, N - p0);
            {
                double rx[kU], ry[kU], rz[kU], rw[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const int32_t e = min(tid + u * kThr, Sg - 1);
                    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                                 : "=d"(rx[u]), "=d"(ry[u]), "=d"(rz[u]), "=d"(rw[u]) : "l"(scr + 4ll * (p0 + e)));
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    if (tid + u * kThr < Sg) {
                        const uint32_t pos = static_cast<uint32_t>(__double_as_longlong(rw[u]) >> 32);
                        double2* st = reinterpret_cast<double2*>(S_.stage + 4 * pos);
                        st[0] = make_double2(rx[u], ry[u]);
                        st[1] = make_double2(rz[u], rw[u]);
                    }
                }
            }
            __syncthreads();
            if (DISCARD) {
                const int lines = (Sg * 32) / 128;
                for (int l = tid; l < lines; l += kThr)
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(scr + 4ll * p0 + 16ll * l) : "memory");
            }
            for (int32_t k = tid; 2 * k < Sg; k += kThr) {
                const int32_t pa = o + p0 + 2 * k;
                const double2 a01 = *reinterpret_cast<const double2*>(S_.stage + 8 * k);
                const double2 a23 = *reinterpret_cast<const double2*>(S_.stage + 8 * k + 2);
                double ax = a01.x, ay = a01.y, az = a23.x;
                const int32_t ia = static_cast<int32_t>(__double_as_longlong(a23.y));
                if (2 * k + 1 < Sg) {
                    const double2 b01 = *reinterpret_cast<const double2*>(S_.stage + 8 * k + 4);
                    const double2 b23 = *reinterpret_cast<const double2*>(S_.stage + 8 * k + 6);
                    double bx = b01.x, by = b01.y, bz = b23.x;
                    const int32_t ib = static_cast<int32_t>(__double_as_longlong(b23.y));
                    if (MODE == 1) {
                        const cc::U4 r = cc::philox4x32_10(cc::U4{static_cast<uint32_t>(p0 / 2 + k), static_cast<uint32_t>(j), 7u, 0u}, 42u, 0u);
                        cc::ta_update(ax, ay, az, bx, by, bz, C, cc::u01(r.x, r.y), cc::u01(r.z, r.w));
                        accm += ax + bx + ay * ay + by * by;
                    }
                    *reinterpret_cast<double2*>(vout + pa) = make_double2(ax, bx);
                    *reinterpret_cast<double2*>(vout + ldv + pa) = make_double2(ay, by);
                    *reinterpret_cast<double2*>(vout + 2 * ldv + pa) = make_double2(az, bz);
                    *reinterpret_cast<int2*>(cout + pa) = make_int2(j, j);
                    *reinterpret_cast<int2*>(pout + pa) = make_int2(ia, ib);
                } else {
                    vout[pa] = ax; vout[ldv + pa] = ay; vout[2 * ldv + pa] = az;
                    cout[pa] = j; pout[pa] = ia;
                }
            }
            __syncthreads();
        }
    }
    if (accm == 1.2345) sink[0] = accm;
}

// the DRAM floor of the same traffic: read v (24 B), write v + cell + perm (32 B), streaming
__global__ void k_stream(const double* __restrict__ v, int64_t ldv, int64_t n, double* __restrict__ vout,
                         int32_t* __restrict__ cout, int32_t* __restrict__ pout)
{
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        vout[i] = v[i]; vout[ldv + i] = v[ldv + i]; vout[2 * ldv + i] = v[2 * ldv + i];
        cout[i] = 1; pout[i] = static_cast<int32_t>(i);
    }
}

int main(int argc, char** argv)
{
    const int M = 4096, Nc = argc > 1 ? atoi(argv[1]) : 25000;
    const int64_t n = static_cast<int64_t>(M) * Nc;
    std::vector<double> hv(3 * n);
    for (int64_t i = 0; i < 3 * n; ++i) hv[i] = static_cast<double>(i % 1000003) * 1.5 + 0.25;
    std::vector<int32_t> hoff(M + 1);
    for (int j = 0; j <= M; ++j) hoff[j] = j * Nc;
    double *v, *vo, *scr, *sink;
    int32_t *off, *co, *po;
    int* counter;
    cudaMalloc(&v, 24 * n);
    cudaMalloc(&vo, 24 * n);
    cudaMalloc(&co, 4 * n);
    cudaMalloc(&po, 4 * n);
    cudaMalloc(&off, 4 * (M + 1));
    cudaMalloc(&counter, 4);
    cudaMalloc(&sink, 8);
    int maxCl = 0;
    const size_t smem = sizeof(Sm);
    cudaMemcpy(v, hv.data(), 24 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(off, hoff.data(), 4 * (M + 1), cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](auto kern, const char* name, bool check) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kCl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(kThr);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(kCl * 64);
        cudaOccupancyMaxActiveClusters(&maxCl, kern, &cfg);
        cfg.gridDim = dim3(kCl * maxCl);
        static bool alloc = false;
        if (!alloc) { cudaMalloc(&scr, static_cast<size_t>(maxCl) * 32 * kCl * kCmax * kSmax); alloc = true; }
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            cudaMemset(counter, 0, 4);
            cudaEventRecord(a);
            cudaLaunchKernelEx(&cfg, kern, static_cast<const double*>(v), static_cast<int64_t>(n),
                               static_cast<const int32_t*>(off), M, vo, co, po, scr, counter, 1e-3, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep > 0) best = std::min(best, ms);
        }
        printf("%-36s clusters %d  %.3f ms  %.1f GB/s (56 B/particle)  err=%s\n", name, maxCl, best,
               56.0 * n / best / 1e6, cudaGetErrorString(cudaGetLastError()));
        if (check) {
            std::vector<double> ho(3 * n);
            std::vector<int32_t> hp(n);
            cudaMemcpy(ho.data(), vo, 24 * n, cudaMemcpyDeviceToHost);
            cudaMemcpy(hp.data(), po, 4 * n, cudaMemcpyDeviceToHost);
            long bad = 0;
            for (int j = 0; j < M; j += 97) {
                std::vector<char> seen(Nc, 0);
                for (int p = 0; p < Nc; ++p) {
                    const int64_t q = static_cast<int64_t>(j) * Nc + p;
                    const int32_t i = hp[q];
                    if (i < j * Nc || i >= (j + 1) * Nc || seen[i - j * Nc]) { ++bad; continue; }
                    seen[i - j * Nc] = 1;
                    for (int cc_ = 0; cc_ < 3; ++cc_) bad += ho[cc_ * n + q] != hv[cc_ * n + i];
                }
            }
            printf("  check: %ld mismatches\n", bad);
        }
    };
    run(k_xchg<0, 0, 0>, "exchange, identity", true);
    run(k_xchg<0, 1, 1>, "exchange, identity, discard, L2 pf", true);
    run(k_xchg<0, 0, 1>, "exchange, identity, L2 pf", false);
    run(k_xchg<1, 0, 1>, "exchange + Philox/AS241/TA, L2 pf", false);
    run(k_xchg<1, 1, 1>, "exchange + TA, discard, L2 pf", false);
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a);
        k_stream<<<148 * 8, 256>>>(v, n, n, vo, co, po);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0) best = std::min(best, ms);
    }
    printf("%-36s %.3f ms  %.1f GB/s\n", "streaming floor (24 B in, 32 B out)", best, 56.0 * n / best / 1e6);
    return 0;
}
