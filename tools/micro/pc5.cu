// Prototype (round 2), design B v3 (v2 + next-item metadata prefetch, Feistel ILP,
// ranks from the count pass, warp-per-sub-run loads, thread-0 release): persistent producer / consumer exchange
// through L2 (see pc_xchg.cu for v1).  Changes: power-of-two segments
// (S = 2048: d = p >> 11, pos = p & 2047), P1 writes straight from registers
// into 128-byte-aligned buckets of a padded per-segment scratch region (warp-
// aggregated cursors), P2 discards every scratch line it consumed
// (discard.global.L2: no write-back of the exchange to DRAM), Feistel keys and
// segment -> cell from tables.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o pc2 pc2.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2508_06771_b200/csrc/cc_device.cuh"

#ifndef OCC
#define OCC 3
#endif
#ifndef THR
#define THR 256
#endif
constexpr int kThr = THR;
#ifndef KLOG
#define KLOG 11
#endif
constexpr int kLog = KLOG;
constexpr int kSeg = 1 << kLog;           // slots per segment
constexpr int kKmax = 32;                 // segments per cell
constexpr int kCap = kSeg + 4 * kKmax;    // padded records per segment region
constexpr int kB = 4;

struct __align__(16) Sm {
    double buf[4 * kSeg];                 // P2 placement stage (64 KB)
    uint32_t ps[kSeg];                    // P1 p of the segment's slots
    int32_t cnt[kKmax];
    int32_t cur[kKmax];
    int32_t pre[kKmax + 1];
    int32_t lo[kKmax];
    int32_t prep[2 * kKmax];
    int32_t item;
    int4 meta[2];                      // {o, N, j, g}
    uint4 mkey;
    int32_t cur_t;
};

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

__device__ __forceinline__ void st_v4(double* p, double a, double b, double c, double d)
{
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void ld_v4_cg(const double* p, double& a, double& b, double& c, double& d)
{
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}


struct __align__(16) Meta {
    int32_t o, N, j, g;
    uint32_t k0, k1, k2, k3;
};

template <int NV>
__device__ __forceinline__ void feistel_Einv_multi(const cc::Feistel& f, uint32_t (&x)[NV])
{
    const uint32_t amask = (1u << f.bL) - 1u;
    uint32_t L[NV], R[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) { L[v] = x[v] & amask; R[v] = x[v] >> f.bL; }
#pragma unroll
    for (int r = 7; r >= 0; --r) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            if ((r & 1) == 0) {
                L[v] ^= cc::fmix32_small(R[v], f.kp[r]) & amask;
            } else {
                const uint32_t t = __umulhi(cc::fmix32_small(L[v], f.kp[r]), f.m);
                R[v] = (R[v] >= t) ? R[v] - t : R[v] + f.m - t;
            }
        }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) x[v] = L[v] + (R[v] << f.bL);
}

__device__ __forceinline__ int item_of(int t, int T, int Lw, bool& p1)
{
    if (t < Lw) { p1 = true; return t; }
    const int u = t - Lw;
    if (u < 2 * (T - Lw)) { p1 = (u & 1) == 0; return p1 ? Lw + u / 2 : u / 2; }
    p1 = false;
    return u - (T - Lw);
}

constexpr int kPer = kSeg / kThr;        // slots per thread in P1 (8)

template <int MODE, int DISCARD>
__global__ void __launch_bounds__(kThr, OCC)
k_pc(const double* __restrict__ v, int64_t ldv, const Meta* __restrict__ meta, int M, int T, int Lw,
     double* __restrict__ vout, int32_t* __restrict__ cout, int32_t* __restrict__ pout, double* __restrict__ scr,
     int32_t* __restrict__ hdr, int* __restrict__ done, int* __restrict__ ticket, double C, double* __restrict__ sink)
{
    extern __shared__ __align__(16) unsigned char smraw[];
    Sm& S_ = *reinterpret_cast<Sm*>(smraw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    double accm = 0.0;
    long long prof[6] = {0, 0, 0, 0, 0, 0};
    // prologue: ticket + metadata of the first item, ticket of the second
    if (tid == 0) {
        const int t = atomicAdd(ticket, 1);
        S_.cur_t = t;
        if (t < 2 * T) {
            bool p1;
            const int idx = item_of(t, T, Lw, p1);
            const Meta m = meta[idx];
            S_.meta[0] = make_int4(m.o, m.N, m.j, m.g);
            S_.mkey = make_uint4(m.k0, m.k1, m.k2, m.k3);
        }
        S_.item = atomicAdd(ticket, 1);
    }
    __syncthreads();
    for (;;) {
        const int t = S_.cur_t;
        if (t >= 2 * T) break;
        long long c0 = clock64();
        bool p1;
        const int idx = item_of(t, T, Lw, p1);
        const int4 mm = S_.meta[0];
        const uint4 mk = S_.mkey;
        const int32_t o = mm.x, N = mm.y, j = mm.z, g = mm.w;
        const int K = (N + kSeg - 1) >> kLog;
        const int32_t sb = idx - g;
        // next item's metadata: issued now (thread 0), consumed at the end of this item
        const int tn = S_.item;
        Meta mn;
        if (tid == 0 && tn < 2 * T) {
            bool q;
            mn = meta[item_of(tn, T, Lw, q)];
        }
        __syncthreads();
        if (p1) {
            const int32_t s0 = g << kLog, Sg = min(kSeg, N - s0);
            const cc::Feistel f = cc::make_feistel(static_cast<uint32_t>(N), cc::U4{mk.x, mk.y, mk.z, mk.w});
            if (tid < kKmax) S_.cnt[tid] = 0;
            // the segment's velocity rows -> shared memory (8-byte cp.async, all in flight during the Feistel)
            for (int32_t e = tid; e < 3 * Sg; e += kThr) {
                const int c = e / Sg, i = e - c * Sg;
                const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(S_.buf + c * kSeg + i));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(v + c * ldv + o + s0 + i) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            __syncthreads();
            {
                uint32_t x[kPer];
#pragma unroll
                for (int u = 0; u < kPer; ++u) x[u] = (tid + u * kThr < Sg) ? static_cast<uint32_t>(s0 + tid + u * kThr) : 0u;
                feistel_Einv_multi(f, x);
#pragma unroll
                for (int u = 0; u < kPer; ++u) {
                    while (x[u] >= f.N) x[u] = feistel_Einv(f, x[u]);
                    const int32_t e = tid + u * kThr;
                    const bool ok = e < Sg;
                    const uint32_t d = ok ? (x[u] >> kLog) : 0xFFFFFFFFu;
                    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
                    const int leader = __ffs(peers) - 1;
                    int32_t b = 0;
                    if (ok && lane == leader) b = atomicAdd(&S_.cnt[d], __popc(peers));
                    b = __shfl_sync(0xFFFFFFFFu, b, leader);
                    if (ok) S_.ps[e] = (x[u] & 0xFFFFu) | (static_cast<uint32_t>(b + __popc(peers & lt)) << 16);
                }
            }
            __syncthreads();
            if (tid < 32) {
                const int32_t x = tid < K ? S_.cnt[tid] : 0;
                const int32_t xa = (x + 3) & ~3;
                int32_t s = xa;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const int32_t y = __shfl_up_sync(0xFFFFFFFFu, s, dd);
                    if (tid >= dd) s += y;
                }
                if (tid < K) {
                    S_.cur[tid] = s - xa;
                    hdr[static_cast<int64_t>(idx) * (2 * kKmax) + tid] = s - xa;
                    hdr[static_cast<int64_t>(idx) * (2 * kKmax) + kKmax + tid] = x;
                }
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
            double* reg = scr + 4ll * kCap * idx;
            for (int32_t e = tid; e < Sg; e += kThr) {
                const uint32_t pr = S_.ps[e];
                const uint32_t p = pr & 0xFFFFu;
                const int32_t r = S_.cur[p >> kLog] + static_cast<int32_t>(pr >> 16);
                const double w = __longlong_as_double((static_cast<long long>(p & (kSeg - 1)) << 32) |
                                                      static_cast<uint32_t>(o + s0 + e));
                st_v4(reg + 4ll * r, S_.buf[e], S_.buf[kSeg + e], S_.buf[2 * kSeg + e], w);
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(done + j, 1);
                prof[0] += clock64() - c0; prof[1] += 1;
            }
        } else {
            const int d = g;
            if (tid == 0) {
                for (;;) {
                    int x;
                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(x) : "l"(done + j) : "memory");
                    if (x >= K) break;
                    __nanosleep(100);
                }
            }
            __syncthreads();
            long long c1 = clock64();
            if (tid < 32) {
                int32_t len = 0, l0 = 0;
                if (tid < K) {
                    const int32_t* h = hdr + static_cast<int64_t>(sb + tid) * (2 * kKmax);
                    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(l0) : "l"(h + d));
                    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(len) : "l"(h + kKmax + d));
                    l0 += (sb + tid) * kCap;
                }
                int32_t s = len;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const int32_t y = __shfl_up_sync(0xFFFFFFFFu, s, dd);
                    if (tid >= dd) s += y;
                }
                S_.lo[tid] = l0;
                S_.cnt[tid] = len;
                S_.prep[tid] = s - len;
                if (tid == 31) S_.pre[0] = s;
            }
            __syncthreads();
            const int32_t Sd = S_.pre[0];
            // every record of the segment in flight at once: 16-byte cp.async into the staging buffer
            for (int gg = warp; gg < K; gg += kThr / 32) {
                const int32_t len = S_.cnt[gg], st0 = S_.prep[gg];
                const double* base = scr + 4ll * S_.lo[gg];
                for (int32_t e = lane; e < 2 * len; e += 32) {
                    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(S_.buf + 4 * st0 + 2 * e));
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(base + 2 * e) : "memory");
                }
            }
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
            __syncthreads();
            // placement map: pair-order position -> staging index
            for (int32_t e = tid; e < Sd; e += kThr)
                S_.ps[static_cast<uint32_t>(__double_as_longlong(S_.buf[4 * e + 3]) >> 32)] = static_cast<uint32_t>(e);
            if (DISCARD) {
                for (int gg = warp; gg < K; gg += kThr / 32) {
                    const int lines = (S_.cnt[gg] + 3) >> 2;
                    for (int l = lane; l < lines; l += 32)
                        asm volatile("discard.global.L2 [%0], 128;" ::"l"(scr + 4ll * S_.lo[gg] + 16ll * l) : "memory");
                }
            }
            __syncthreads();
            long long c2 = clock64();
            const int32_t p0 = d << kLog;
            for (int32_t k = tid; 2 * k < Sd; k += kThr) {
                const int32_t pa = o + p0 + 2 * k;
                const double* A_ = S_.buf + 4 * S_.ps[2 * k];
                const double2 a01 = *reinterpret_cast<const double2*>(A_);
                const double2 a23 = *reinterpret_cast<const double2*>(A_ + 2);
                double ax = a01.x, ay = a01.y, az = a23.x;
                const int32_t ia = static_cast<int32_t>(__double_as_longlong(a23.y));
                if (2 * k + 1 < Sd) {
                    const double* B_ = S_.buf + 4 * S_.ps[2 * k + 1];
                    const double2 b01 = *reinterpret_cast<const double2*>(B_);
                    const double2 b23 = *reinterpret_cast<const double2*>(B_ + 2);
                    double bx = b01.x, by = b01.y, bz = b23.x;
                    const int32_t ib = static_cast<int32_t>(__double_as_longlong(b23.y));
                    if (MODE == 1) {
                        const cc::U4 r = cc::philox4x32_10(
                            cc::U4{static_cast<uint32_t>(p0 / 2 + k), static_cast<uint32_t>(j), 7u, 0u}, 42u, 0u);
                        const double z_ = cc::ppnd16_central(cc::u01(r.x, r.y));
                        cc::ta_update_z(ax, ay, az, bx, by, bz, C, z_, cc::u01(r.z, r.w));
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
            if (tid == 0) { prof[2] += c1 - c0; prof[3] += c2 - c1; prof[4] += clock64() - c2; prof[5] += 1; }
        }
        // hand over: next item's metadata, the ticket after it
        __syncthreads();
        if (tid == 0) {
            S_.cur_t = tn;
            if (tn < 2 * T) {
                S_.meta[0] = make_int4(mn.o, mn.N, mn.j, mn.g);
                S_.mkey = make_uint4(mn.k0, mn.k1, mn.k2, mn.k3);
                S_.item = atomicAdd(ticket, 1);
            }
        }
        __syncthreads();
    }
    if (accm == 1.2345) sink[0] = accm;
    if (tid == 0) for (int q = 0; q < 6; ++q) atomicAdd(reinterpret_cast<unsigned long long*>(sink) + 1 + q, static_cast<unsigned long long>(prof[q]));
}

__global__ void k_stream(const double* __restrict__ v, int64_t ldv, int64_t n, double* __restrict__ vout,
                         int32_t* __restrict__ cout, int32_t* __restrict__ pout)
{
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        vout[i] = v[i]; vout[ldv + i] = v[ldv + i]; vout[2 * ldv + i] = v[2 * ldv + i];
        cout[i] = 1; pout[i] = static_cast<int32_t>(i);
    }
}

__global__ void k_keys(cc::U4* keys, int M)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < M) keys[j] = cc::philox4x32_10(cc::U4{0u, static_cast<uint32_t>(j), 7u, 1u}, 42u, 0u);
}

int main(int argc, char** argv)
{
    const int M = 4096, Nc = argc > 1 ? atoi(argv[1]) : 25000;
    const int one = argc > 2 ? atoi(argv[2]) : -1;
    const int64_t n = static_cast<int64_t>(M) * Nc;
    std::vector<double> hv(3 * n);
    for (int64_t i = 0; i < 3 * n; ++i) hv[i] = static_cast<double>(i % 1000003) * 1.5 + 0.25;
    const int K = (Nc + kSeg - 1) / kSeg;
    std::vector<int32_t> hoff(M + 1), hseg(M + 1), hsc;
    for (int j = 0; j <= M; ++j) { hoff[j] = j * Nc; hseg[j] = j * K; }
    for (int j = 0; j < M; ++j) for (int g = 0; g < K; ++g) hsc.push_back(j);
    std::vector<Meta> hmeta;
    const int T = M * K;
    double *v, *vo, *scr, *sink;
    int32_t *off, *seg, *sc, *co, *po, *hdr;
    int *done, *ticket;
    cc::U4* keys;
    cudaMalloc(&v, 24 * n);
    cudaMalloc(&vo, 24 * n);
    cudaMalloc(&scr, 32ll * kCap * T);
    cudaMalloc(&co, 4 * n);
    cudaMalloc(&po, 4 * n);
    cudaMalloc(&off, 4 * (M + 1));
    cudaMalloc(&seg, 4 * (M + 1));
    cudaMalloc(&sc, 4 * T);
    cudaMalloc(&hdr, 4ll * T * 2 * kKmax);
    cudaMalloc(&done, 4 * M);
    cudaMalloc(&ticket, 4);
    cudaMalloc(&sink, 64);
    cudaMalloc(&keys, sizeof(cc::U4) * M);
    k_keys<<<(M + 255) / 256, 256>>>(keys, M);
    cudaMemcpy(v, hv.data(), 24 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(off, hoff.data(), 4 * (M + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(seg, hseg.data(), 4 * (M + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(sc, hsc.data(), 4 * T, cudaMemcpyHostToDevice);
    {
        std::vector<cc::U4> hk(M);
        cudaDeviceSynchronize();
        cudaMemcpy(hk.data(), keys, sizeof(cc::U4) * M, cudaMemcpyDeviceToHost);
        for (int j = 0; j < M; ++j)
            for (int g = 0; g < K; ++g) hmeta.push_back(Meta{hoff[j], Nc, j, g, hk[j].x, hk[j].y, hk[j].z, hk[j].w});
    }
    Meta* meta;
    cudaMalloc(&meta, sizeof(Meta) * T);
    cudaMemcpy(meta, hmeta.data(), sizeof(Meta) * T, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t smem = sizeof(Sm);
    auto run = [&](auto kern, const char* name, bool check, int Lw) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThr, smem);
        const int grid = occ * 148;
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            cudaMemsetAsync(done, 0, 4 * M);
            cudaMemsetAsync(ticket, 0, 4);
            cudaEventRecord(a);
            kern<<<grid, kThr, smem>>>(v, n, meta, M, T, Lw, vo, co, po, scr, hdr, done, ticket, 1e-3, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep > 0) best = std::min(best, ms);
        }
        printf("%-34s occ %d Lw %5d  %.3f ms  %.1f GB/s (56 B/particle)  err=%s\n", name, occ, Lw, best,
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
                    for (int c = 0; c < 3; ++c) bad += ho[c * n + q] != hv[c * n + i];
                }
            }
            printf("  check: %ld mismatches\n", bad);
        }
    };
    if (one == 9) {
        cudaMemset(sink, 0, 64);
        run(k_pc<1, 1>, "TA, discard (profiled)", false, 512);
        unsigned long long h[7];
        cudaMemcpy(h, sink, 56, cudaMemcpyDeviceToHost);
        // 6 reps were run: averages per item
        printf("P1 items %llu: %.0f cyc/item;  P2 items %llu: wait %.0f, load+place %.0f, compute+store %.0f cyc/item\n",
               h[2], (double)h[1] / h[2], h[6], (double)h[3] / h[6], (double)h[4] / h[6], (double)h[5] / h[6]);
        return 0;
    }
    if (one >= 0) {
        if (one == 0) run(k_pc<0, 1>, "identity, discard", false, 512);
        else run(k_pc<1, 1>, "TA, discard", false, 512);
        return 0;
    }
    run(k_pc<0, 1>, "identity, discard", true, 512);
    for (int Lw : {512, 768, 1024, 1536, 2048}) run(k_pc<1, 1>, "TA (central), discard", false, Lw * (kSeg == 1024 ? 2 : 1));
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
    printf("%-34s %.3f ms  %.1f GB/s\n", "streaming floor (24 B in, 32 B out)", best, 56.0 * n / best / 1e6);
    return 0;
}
