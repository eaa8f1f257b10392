// cc_kernels.cu — sm_100a kernels and C ABI of the e–e Coulomb collision
// operator (arXiv 2508.06771 step S1; Table 5).
//
// Pipeline of one coulomb_collide() call (all on the caller's stream):
//   k_count        CCS1: per-tile cell histograms  -> tcount[T][M+1],
//                  invalid-id flag, descent count (picks the binning mode)
//   k_scan_tiles   CCS2, part 1: per cell, exclusive scan over tiles
//   k_scan_cells   CCS2, part 2: off[] (cell offsets), chunk_off[]
//   k_cell_setup   per cell: TA constant C_j (R5/R6/R7), Feistel keys (R1, R3),
//                  the chunk table and the R1b segment order (absolute segment
//                  starts of every block)
//   k_scatter      CCS3 as a STABLE counting sort: per-warp
//                  sub-ranges, match.any ranks, no global atomics; by binning
//                  mode: nothing (sorted input), the input index of each stable
//                  slot (nearly sorted), or the particle as one 32-byte record
//                  {vx, vy, vz, (perm, cell)} (random order) into ws_v
//   k_collide_small  N_j <= 64: one warp per cell; pi_j by sort-by-key (R1)
//   k_collide_large  N_j > 64: R1b (default) one CTA per block of whole
//                  segments, copied into shared memory and paired there by
//                  tau_b; R1 (CC_CELL_UNIFORM) cell-aligned chunks of pairs
//                  gathered by the whole-cell Feistel pi_j; CCS4 Philox per
//                  pair; CCS5 TA update; output in pair order, SoA; fused
//                  per-chunk moment partials (post- and pre-collision)
//   k_copy_dead    dead particles after the live ones, input order
//   k_finalize_cells / k_finalize_diag   deterministic reductions of the
//                  partials -> moments_out [M][7], diag_out [16]
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "../../include/coulomb.h"
#include "cc_device.cuh"

// Ablation switch for performance studies only (tools/ablate.sh); 0 in every
// build of the product: bit 0 skips the TA math, bit 1 pairs slots 2k, 2k+1
// (no Feistel), bit 2 skips CCS4 (Philox + AS241), bit 3 skips the index modes' stage copies.
#ifndef CC_ABLATE
#define CC_ABLATE 0
#endif

// Bounds-asserting build (-DCC_DEBUG_BOUNDS, tools/debug_bounds.sh) for the index and segment
// arithmetic of R1b and the binning modes (compute-sanitizer is unavailable on the GPU pool);
// compiled out of the product.
#ifdef CC_DEBUG_BOUNDS
#include <cassert>
#define CC_DBG_ASSERT(c) assert(c)
#else
#define CC_DBG_ASSERT(c) ((void)0)
#endif

namespace {

#ifndef CC_COUNT_THREADS
#define CC_COUNT_THREADS 256
#endif
constexpr int kCountThreads = CC_COUNT_THREADS;
#ifndef CC_SUB
#define CC_SUB 4096
#endif
constexpr int kSub = CC_SUB;             // elements per warp sub-range in k_scatter
// k_scatter shape (design-study knobs, tools/scatter_shape.sh)
#ifndef CC_SCATTER_UA
#define CC_SCATTER_UA 16
#endif
#ifndef CC_SCATTER_UB
#define CC_SCATTER_UB 4
#endif
#ifndef CC_SCATTER_BUDGET_KB
#define CC_SCATTER_BUDGET_KB 96
#endif
#ifndef CC_SCATTER_CTAS
#define CC_SCATTER_CTAS 2
#endif
#ifndef CC_SCATTER_PREFETCH
#define CC_SCATTER_PREFETCH 1
#endif
constexpr bool kScatterPrefetch = CC_SCATTER_PREFETCH != 0;   // next batch's cell ids loaded one batch ahead
constexpr int kScatterUnrollA = CC_SCATTER_UA;   // cell loads in flight per lane, counting pass
constexpr int kScatterUnrollB = CC_SCATTER_UB;   // (cell, v) loads in flight per lane, scatter pass
#ifndef CC_SCATTER_UP
#define CC_SCATTER_UP 4
#endif
constexpr int kScatterUnrollP = CC_SCATTER_UP;   // ids per lane per batch, index-only scatter pass (kModePerm)
// k_collide_large shape (tools/collide_shape.sh overrides them for design studies)
#ifndef CC_COLLIDE_THREADS
#define CC_COLLIDE_THREADS 64
#endif
#ifndef CC_CHUNK
#define CC_CHUNK 192
#endif
#ifndef CC_COLLIDE_CTAS
#define CC_COLLIDE_CTAS 12
#endif
// unroll factors of k_collide_large's phase-1 (Feistel + gathers) and phase-2b (TA + stores) item loops
#ifndef CC_P1_UNROLL
#define CC_P1_UNROLL 1
#endif
#ifndef CC_P2B_UNROLL
#define CC_P2B_UNROLL 3
#endif
constexpr int kP1Unroll = CC_P1_UNROLL, kP2BUnroll = CC_P2B_UNROLL;
constexpr int kCollideThreads = CC_COLLIDE_THREADS;
constexpr int kChunk = CC_CHUNK;         // items (pairs or sitter) per k_collide_large CTA
constexpr int kRec = 12;                 // chunk record: S1' (3), S2' (3) post-collision; raw pre-collision v (3), |v|^2; pad
constexpr int kSmallRec = 16;            // small-cell record: S1', S2' about the exact mean, the mean (3), pad, pre (12..15)
constexpr int kCellSum = 8;              // per-cell raw sums: post-collision v (3), |v|^2; pre-collision v (3), |v|^2
constexpr int kScatterSmemBudget = CC_SCATTER_BUDGET_KB * 1024;   // per-warp counters of one CTA
#ifndef CC_SCATTER_MAXW
#define CC_SCATTER_MAXW 12
#endif
constexpr int kMaxScatterWarps = CC_SCATTER_MAXW;
static_assert(kMaxScatterWarps * kSub <= 65536, "per-warp 16-bit cell counters must hold a whole tile");

// ------------------------------------------------------------------ layout
struct Layout {
    int W = 1, sub = kSub, tile = kSub, T = 0;
    int chunk = kChunk;                  // pairs per k_collide_large CTA (multiple of kCollideThreads)
    int64_t max_chunks = 0;
    size_t o_err = 0, o_tcount = 0, o_cnt = 0, o_off = 0, o_chunk = 0, o_C = 0, o_keys = 0;
    size_t o_seg = 0, o_perm = 0, o_small = 0, o_recs = 0, o_cellsum = 0, o_ref = 0, o_chunkcell = 0, o_trec = 0, o_wsv = 0, total = 0;
};

size_t align256(size_t x) { return (x + 255u) & ~static_cast<size_t>(255u); }

int scatter_warps(int32_t M)
{
    int W = kScatterSmemBudget / (2 * (M + 2));
    if (W > kMaxScatterWarps) W = kMaxScatterWarps;
    if (W < 1) W = 1;
    return W;
}

Layout make_layout(int64_t n, int32_t M)
{
    Layout L;
    L.W = scatter_warps(M);
    // small inputs: shorter warp sub-ranges and collide chunks so that the binning tiles and the
    // collide CTAs still fill the GPU (C2/C3-sized calls); C4-sized calls keep kSub / kChunk
    constexpr int64_t kTargetTiles = 2 * 148 * 2, kTargetChunks = CC_COLLIDE_CTAS * 148;
    while (L.sub > 256 && (n + static_cast<int64_t>(L.W) * L.sub - 1) / (static_cast<int64_t>(L.W) * L.sub) < kTargetTiles)
        L.sub /= 2;
    while (L.chunk > kCollideThreads && (n / 2) / L.chunk < kTargetChunks) L.chunk -= kCollideThreads;
    {
        // whole waves of binning tiles (k_scatter: CC_SCATTER_CTAS CTAs on each of the 148 SMs): the
        // warp sub-range is trimmed, in steps of 128 ids, so that the tiles just fill the last wave
        const int64_t wave = static_cast<int64_t>(CC_SCATTER_CTAS) * 148;
        const int64_t t0 = (n + static_cast<int64_t>(L.W) * L.sub - 1) / (static_cast<int64_t>(L.W) * L.sub);
        if (t0 > wave) {
            const int64_t waves = (t0 + wave - 1) / wave;
            const int64_t per = static_cast<int64_t>(L.W) * waves * wave;
            const int64_t sub = ((n + per - 1) / per + 127) / 128 * 128;
            if (sub >= 256 && sub <= L.sub) L.sub = static_cast<int>(sub);
        }
    }
    L.tile = L.W * L.sub;
    L.T = static_cast<int>((n + L.tile - 1) / L.tile);
    L.max_chunks = (n + M) / 2 / L.chunk + M + 1;
    size_t o = 0;
    L.o_err = o;      o = align256(o + 64 * sizeof(int32_t));
    L.o_tcount = o;   o = align256(o + static_cast<size_t>(L.T > 0 ? L.T : 1) * (M + 1) * sizeof(int32_t));
    L.o_cnt = o;      o = align256(o + static_cast<size_t>(M + 1) * sizeof(int32_t));
    L.o_off = o;      o = align256(o + static_cast<size_t>(M + 1) * sizeof(int32_t));
    L.o_chunk = o;    o = align256(o + static_cast<size_t>(M + 1) * sizeof(int32_t));
    L.o_C = o;        o = align256(o + static_cast<size_t>(M) * sizeof(double));
    L.o_keys = o;     o = align256(o + static_cast<size_t>(M) * sizeof(cc::U4));
    L.o_small = o;    o = align256(o + static_cast<size_t>(M) * kSmallRec * sizeof(double));
    L.o_recs = o;     o = align256(o + static_cast<size_t>(L.max_chunks) * kRec * sizeof(double));
    L.o_cellsum = o;  o = align256(o + static_cast<size_t>(M) * kCellSum * sizeof(double));
    L.o_ref = o;      o = align256(o + static_cast<size_t>(M) * 4 * sizeof(double));
    L.o_trec = o;     o = align256(o + static_cast<size_t>(M) * kRec * sizeof(double));
    L.o_chunkcell = o; o = align256(o + static_cast<size_t>(L.max_chunks) * sizeof(int4));
    L.o_seg = o;      o = align256(o + static_cast<size_t>(L.max_chunks) * cc::kBlockSegs * sizeof(int32_t));  // R1b
    L.o_perm = o;     o = align256(o + static_cast<size_t>(n > 0 ? n : 1) * sizeof(int32_t));   // CC_PRESERVE_ORDER
    L.o_wsv = o;      o = align256(o + static_cast<size_t>(n > 0 ? n : 1) * 4 * sizeof(double));
    L.total = o;
    return L;
}

template <typename T>
T* at(void* base, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(base) + off); }

// ------------------------------------------------------------------ 256-bit global access
__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d)
{
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

__device__ __forceinline__ void st256(double* p, double a, double b, double c, double d)
{
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
                 : "memory");
}

__device__ __forceinline__ double pack_pc(int32_t perm, int32_t cell)
{
    return __longlong_as_double((static_cast<long long>(static_cast<uint32_t>(cell)) << 32) |
                                static_cast<uint32_t>(perm));
}

__device__ __forceinline__ int32_t unpack_perm(double w)
{
    return static_cast<int32_t>(static_cast<uint32_t>(__double_as_longlong(w)));
}

// ------------------------------------------------------------------ CCS1: count
// flags[0]: sticky invalid-id flag; flags[1]: "input not cell-sorted"; flags[2]: the
// number of descents (positions whose cell key is below the previous one's), which
// selects the binning mode (bin_mode); flags[1..2] are cleared before each call.  Sorted means live ids non-decreasing in input
// order with every dead/invalid particle after the last live one; then the
// stable order is the identity and k_scatter packs the records in place.
// Each thread takes 4 consecutive ids (one 16-byte load when the array is
// 16-byte aligned); the order check takes the previous id from the neighbour
// lane (only lane 0 reloads one), so every id is read once; a warp whose 128
// ids are one cell (sorted input) adds them with a single shared atomic instead
// of 128 same-address ones.
__device__ __forceinline__ int32_t count_key(int32_t c, int M)
{
    return static_cast<uint32_t>(c) < static_cast<uint32_t>(M) ? c : M;
}

// Binning mode of a call, decided on the device from k_count's flags:
//  kModeSorted  input already cell-sorted (dead last): the stable order is the identity,
//               nothing is moved; the collide reads v_in at the stable slot itself;
//  kModePerm    nearly sorted (descents at most 1/kPermModeDiv of a random order's expected
//               n (M - 1) / (2 M) — i.e. up to ~25% for many cells; the steady state of a PIC loop
//               that feeds the operator its own output): the scatter writes only the input
//               index of each stable slot (4 bytes, the paper's "track and sort particle
//               indices"); the collide reads v_in through it — mostly contiguous runs;
//  kModeRec     otherwise (randomly ordered input): the scatter moves each particle as a
//               32-byte record {vx, vy, vz, perm} and the collide reads the records.
// Index modes are used only with R1b (index_modes != 0); R1 always takes kModeRec.
constexpr int kModeRec = 0, kModePerm = 1, kModeSorted = 2;
#ifndef CC_PERM_MODE_DIV
#define CC_PERM_MODE_DIV 2
#endif
// (design studies: 0 = kModePerm for every unsorted input).  Measured at C4: the
// index mode beats the record mode at 2-20% movers (2.50-2.79 vs 3.17-3.19 ms/step at 10-20%).
constexpr int kPermModeDiv = CC_PERM_MODE_DIV;
__device__ __forceinline__ int bin_mode(const int32_t* flags, int n, int M, int index_modes)
{
    if (!index_modes) return kModeRec;
    if (__ldg(flags + 1) == 0) return kModeSorted;
#ifdef CC_STUDY_NOREC
    return kModePerm;                    // design study only: the R1b collide without its record path
#endif
    // descents <= (n (M-1) / (2M)) / kPermModeDiv, in integers
    return static_cast<int64_t>(__ldg(flags + 2)) * 2 * M * kPermModeDiv <= static_cast<int64_t>(n) * (M - 1) ? kModePerm
                                                                                                      : kModeRec;
}

__global__ void __launch_bounds__(kCountThreads)
k_count(const int32_t* __restrict__ cell, int n, int M, int tile, int32_t* __restrict__ tcount,
        int32_t* __restrict__ flags)
{
    extern __shared__ int32_t hist[];   // [M+1], bin M = dead or invalid
    for (int i = threadIdx.x; i <= M; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const int64_t start = static_cast<int64_t>(blockIdx.x) * tile;
    const int64_t end = min(start + tile, static_cast<int64_t>(n));
    const int lane = threadIdx.x & 31;
    int bad = 0, unsorted = 0;          // unsorted: this thread's descents (k[i] < k[i-1])
    // full 8-id groups (a tile starts at a multiple of 8: tile = W x sub, sub a multiple of 128):
    // one 32-byte load per lane keeps twice the bytes of a 16-byte load in flight per warp
    const int64_t vend = start + ((end - start) & ~static_cast<int64_t>(7));
    const uintptr_t al = reinterpret_cast<uintptr_t>(cell);
    for (int64_t i0 = start; i0 < vend; i0 += 8 * static_cast<int64_t>(blockDim.x)) {
        const int64_t i = i0 + 8 * static_cast<int64_t>(threadIdx.x);
        const bool ok = i < vend;
        const unsigned act = __ballot_sync(0xFFFFFFFFu, ok);
        if (!ok) break;
        int32_t c[8];
        if ((al & 31u) == 0) {
            unsigned long long a, b, d, e;
            asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(d), "=l"(e) : "l"(cell + i));
            c[0] = static_cast<int32_t>(a); c[1] = static_cast<int32_t>(a >> 32);
            c[2] = static_cast<int32_t>(b); c[3] = static_cast<int32_t>(b >> 32);
            c[4] = static_cast<int32_t>(d); c[5] = static_cast<int32_t>(d >> 32);
            c[6] = static_cast<int32_t>(e); c[7] = static_cast<int32_t>(e >> 32);
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) c[u] = __ldg(cell + i + u);
        }
        int32_t k[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            // an id is valid iff -1 <= c < M, i.e. (unsigned)(c + 1) <= M
            bad |= static_cast<uint32_t>(c[u] + 1) > static_cast<uint32_t>(M);
            k[u] = count_key(c[u], M);
        }
        int32_t prev = __shfl_up_sync(act, k[7], 1);
        if (lane == 0) prev = (i > 0) ? count_key(__ldg(cell + i - 1), M) : 0;
        unsorted += k[0] < prev;
#pragma unroll
        for (int u = 1; u < 8; ++u) unsorted += k[u] < k[u - 1];
        const int32_t kl = __shfl_sync(act, k[0], 0);
        bool same = true;
#pragma unroll
        for (int u = 0; u < 8; ++u) same = same && (k[u] == kl);
        if (__all_sync(act, same)) {
            if (lane == 0) atomicAdd(&hist[kl], 8 * __popc(act));
            continue;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) atomicAdd(&hist[k[u]], 1);
    }
    for (int64_t i = vend + threadIdx.x; i < end; i += blockDim.x) {     // tail (< 8 ids)
        const int32_t c = __ldg(cell + i);
        bad |= static_cast<uint32_t>(c + 1) > static_cast<uint32_t>(M);
        const int32_t k = count_key(c, M);
        if (i > 0) unsorted += k < count_key(__ldg(cell + i - 1), M);
        atomicAdd(&hist[k], 1);
    }
    __shared__ int32_t desc_sm;
    if (threadIdx.x == 0) desc_sm = 0;
    const int any_bad = __syncthreads_or(bad);
    const int wdesc = __reduce_add_sync(0xFFFFFFFFu, unsorted);
    if (lane == 0 && wdesc) atomicAdd(&desc_sm, wdesc);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (any_bad) atomicOr(flags, 1);
        if (desc_sm) { atomicOr(flags + 1, 1); atomicAdd(flags + 2, desc_sm); }
    }
    int32_t* row = tcount + static_cast<int64_t>(blockIdx.x) * (M + 1);
    for (int i = threadIdx.x; i <= M; i += blockDim.x) row[i] = hist[i];
}

// ------------------------------------------------------------------ CCS2 part 1
// grid: ceil((M+1)/32) CTAs of 32x16 threads; lane = bin, warp row = tile range.
// Loads are issued 8 at a time (independent addresses) to keep DRAM busy.
constexpr int kScanRows = 32;
__global__ void __launch_bounds__(32 * kScanRows)
k_scan_tiles(int32_t* __restrict__ tcount, int T, int M1, int32_t* __restrict__ cnt)
{
    __shared__ int32_t part[kScanRows][33];
    const int lane = threadIdx.x, wy = threadIdx.y;
    const int c = blockIdx.x * 32 + lane;
    const int per = (T + kScanRows - 1) / kScanRows;
    const int t0 = min(wy * per, T), t1 = min(t0 + per, T);
    const bool ok = c < M1;
    int32_t s = 0;
    int t = t0;
    for (; t + 8 <= t1; t += 8) {
        int32_t x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = ok ? tcount[static_cast<int64_t>(t + u) * M1 + c] : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) s += x[u];
    }
    for (; t < t1; ++t) s += ok ? tcount[static_cast<int64_t>(t) * M1 + c] : 0;
    part[wy][lane] = s;
    __syncthreads();
    int32_t pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kScanRows; ++w) {
        const int32_t x = part[w][lane];
        pre += (w < wy) ? x : 0;
        tot += x;
    }
    if (ok) {
        int32_t run = pre;
        t = t0;
        for (; t + 8 <= t1; t += 8) {
            int32_t x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = tcount[static_cast<int64_t>(t + u) * M1 + c];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                tcount[static_cast<int64_t>(t + u) * M1 + c] = run;
                run += x[u];
            }
        }
        for (; t < t1; ++t) {
            int32_t* p = tcount + static_cast<int64_t>(t) * M1 + c;
            const int32_t x = *p;
            *p = run;
            run += x;
        }
        if (wy == 0) cnt[c] = tot;
    }
}

// ------------------------------------------------------------------ CCS2 part 2
struct CellConst {
    double K;            // e^4 dt / (8 pi eps0^2 m_r^2)
    double weight;
    double volume;
    const double* volume_arr;
    double ln_lambda;
    const double* ln_lambda_arr;
};

__device__ __forceinline__ int32_t n_chunks(int32_t N, int32_t chunk)
{
    if (N <= cc::kSmallCell) return 0;
    const int32_t items = (N + 1) / 2;
    return (items + chunk - 1) / chunk;
}

// single CTA of 1024 threads
__global__ void __launch_bounds__(1024)
k_scan_cells(const int32_t* __restrict__ cnt, int M, int32_t* __restrict__ off, int32_t* __restrict__ chunk_off,
             int chunk)
{
    __shared__ int32_t wsum_a[32], wsum_b[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int per = (M + nt - 1) / nt;
    const int j0 = min(tid * per, M), j1 = min(j0 + per, M);
    int32_t a = 0, b = 0;
    for (int j = j0; j < j1; ++j) { a += cnt[j]; b += n_chunks(cnt[j], chunk); }
    // block exclusive scan of (a, b)
    const int lane = tid & 31, wid = tid >> 5;
    int32_t ia = a, ib = b;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int32_t xa = __shfl_up_sync(0xFFFFFFFFu, ia, d);
        const int32_t xb = __shfl_up_sync(0xFFFFFFFFu, ib, d);
        if (lane >= d) { ia += xa; ib += xb; }
    }
    if (lane == 31) { wsum_a[wid] = ia; wsum_b[wid] = ib; }
    __syncthreads();
    if (wid == 0) {
        int32_t va = (lane < nt / 32) ? wsum_a[lane] : 0;
        int32_t vb = (lane < nt / 32) ? wsum_b[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t xa = __shfl_up_sync(0xFFFFFFFFu, va, d);
            const int32_t xb = __shfl_up_sync(0xFFFFFFFFu, vb, d);
            if (lane >= d) { va += xa; vb += xb; }
        }
        wsum_a[lane] = va;
        wsum_b[lane] = vb;
    }
    __syncthreads();
    int32_t ra = ia - a + (wid > 0 ? wsum_a[wid - 1] : 0);
    int32_t rb = ib - b + (wid > 0 ? wsum_b[wid - 1] : 0);
    for (int j = j0; j < j1; ++j) {
        const int32_t N = cnt[j];
        off[j] = ra;
        chunk_off[j] = rb;
        ra += N;
        rb += n_chunks(N, chunk);
    }
    if (tid == nt - 1) { off[M] = ra; chunk_off[M] = rb; }
}

// Per-cell constants (one CTA of kSetupThreads per cell): TA constant C_j (R5-R7) and the
// Feistel keys (R1, R3) from thread 0, and the chunk -> cell table of k_collide_large
// written by the CTA (coalesced).  R1b (seg != NULL, chunk = kBlock / 2): a cell of
// N > kBlock slots also gets its segment order sigma, written as each block's kBlockSegs
// first stable slots (absolute: the cell offset included) in seg[chunk * kBlockSegs + g];
// the tail segment, if any, is the last entry.  Sigma's Feistel form is a pure function of
// the position, so the CTA's threads share a C4 cell's 781 positions (6 each).  Cells of
// 64 < N <= kBlock (one block) get their consecutive segments, so the collide reads one table.
constexpr int kSetupThreads = 128;
__global__ void __launch_bounds__(kSetupThreads)
k_cell_setup(const int32_t* __restrict__ cnt, const int32_t* __restrict__ chunk_off, int M,
             int4* __restrict__ chunk_cell, double* __restrict__ Cj, cc::U4* __restrict__ keys,
             CellConst cc_, uint32_t cell_base, uint32_t step, uint32_t s0, uint32_t s1,
             const uint32_t* __restrict__ step_dev, const int32_t* __restrict__ off, int chunk,
             int32_t* __restrict__ seg)
{
    __shared__ int32_t sig_sm[cc::kSmallCell];
    const int j = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31;
    if (step_dev) step += *step_dev;              // graph replay: effective step read on the device
    const uint32_t G = cell_base + static_cast<uint32_t>(j);
    const int32_t Nj = cnt[j], oj = off[j], c0 = chunk_off[j], c1 = chunk_off[j + 1];
    if (t == 0) {
        const double V = cc_.volume_arr ? cc_.volume_arr[j] : cc_.volume;
        const double lnL = cc_.ln_lambda_arr ? cc_.ln_lambda_arr[j] : cc_.ln_lambda;
        const double nj = static_cast<double>(Nj) * cc_.weight / V;
        Cj[j] = fmax(cc_.K * nj * lnL, 0.0);
        keys[j] = cc::philox4x32_10(cc::U4{0u, G, step, 1u}, s0, s1);
    }
    // per chunk {cell, cell's first slot, N, first item}: k_collide_large starts from one load
    for (int32_t c = c0 + t; c < c1; c += kSetupThreads) chunk_cell[c] = make_int4(j, oj, Nj, (c - c0) * chunk);
    if (seg && Nj > cc::kSmallCell) {
        int32_t* out = seg + static_cast<int64_t>(c0) * cc::kBlockSegs;
        const uint32_t Sf = static_cast<uint32_t>(Nj) / cc::kSeg;
        if (Nj <= cc::kBlock) {
            if (t < cc::kBlockSegs) out[t] = oj + t * cc::kSeg;     // one block: the stable slots in order
            return;
        }
        // R1b segment order sigma: R1's construction over the S_f full segments (sort purpose 6
        // for S_f <= 64, Feistel purpose 5 above); the tail segment goes last
        if (Sf <= static_cast<uint32_t>(cc::kSmallCell)) {
            if (t < 32) {
                cc::small_cell_perm(Sf, G, step, s0, s1, lane, sig_sm, 0u, 6u);
                for (uint32_t p = lane; p < Sf; p += 32) out[p] = oj + sig_sm[p] * cc::kSeg;
            }
        } else {
            const cc::Feistel f = cc::make_feistel(Sf, cc::philox4x32_10(cc::U4{0u, G, step, 5u}, s0, s1));
            for (uint32_t p = t; p < Sf; p += kSetupThreads) out[p] = oj + static_cast<int32_t>(cc::feistel_pi(f, p)) * cc::kSeg;
        }
        if (t == 0 && Sf * cc::kSeg < static_cast<uint32_t>(Nj)) out[Sf] = oj + static_cast<int32_t>(Sf) * cc::kSeg;
    }
}

// ------------------------------------------------------------------ CCS3: stable scatter
// Tile = W warps x kSub elements; warp w owns the contiguous sub-range w of the
// tile, so "input order" = (tile, warp, step, lane).  Per-warp 16-bit counters
// (two per 32-bit word) give each element its rank among equal-cell
// predecessors: the leader of each match.any group advances its cell's counter
// with one shared-memory atomic and broadcasts the old value to the group, so
// successive groups never wait on each other.  Loads are issued in batches
// (kScatterUnrollA / B per lane) to keep several KB per warp in flight.
// Predicated shared-memory atomics (no branch, so a batch of them issues
// back to back; same-address atomics of one warp execute in program order).
__device__ __forceinline__ uint32_t atom_add_if(bool pred, uint32_t* addr, uint32_t val)
{
    uint32_t old = 0;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(addr));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p atom.shared.add.u32 %0, [%1], %3;\n\t}"
                 : "+r"(old) : "r"(a), "r"(static_cast<unsigned>(pred)), "r"(val) : "memory");
    return old;
}

__device__ __forceinline__ void red_add_if(bool pred, uint32_t* addr, uint32_t val)
{
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(addr));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p red.shared.add.u32 [%0], %2;\n\t}"
                 :: "r"(a), "r"(static_cast<unsigned>(pred)), "r"(val) : "memory");
}

template <bool HAS_V>
__device__ __forceinline__ void load_batch(const double* __restrict__ v, int64_t ldv, const int32_t* __restrict__ cell,
                                           int64_t i, double& x, double& y, double& z, int32_t& c)
{
    c = __ldg(cell + i);
    if (HAS_V) { x = __ldg(v + i); y = __ldg(v + ldv + i); z = __ldg(v + 2 * ldv + i); }
    else { x = y = z = 0.0; }
}

// k_scatter pass B over one warp's sub-range [s0, s1): each id's rank among equal-cell
// predecessors, its destination slot, and the move: the 32-byte record (RECS) or the input
// index alone (kModePerm, no velocity loads, so more ids per batch).  The next batch's ids
// are loaded before this batch is ranked, its velocities at the top of its own iteration.
template <int UB, bool RECS, bool HAS_V>
__device__ __forceinline__ void scatter_pass_b(const double* __restrict__ v, int64_t ldv, const int32_t* __restrict__ cell,
                                               int64_t s0, int64_t s1, int M, uint32_t* my, const int32_t* base,
                                               int lane, double* __restrict__ wsv, int32_t* __restrict__ sperm, int n)
{
    const uint32_t lt = (1u << lane) - 1u;
    int32_t cB[UB];
    auto fetchB = [&](int64_t i0) {
#pragma unroll
        for (int u = 0; u < UB; ++u) cB[u] = __ldg(cell + min(i0 + 32 * u + lane, s1 - 1));
    };
    if (kScatterPrefetch && s0 < s1) fetchB(s0);
    for (int64_t i0 = s0; i0 < s1; i0 += 32 * UB) {
        int32_t key[UB];
        double x[UB], y[UB], z[UB];
        if (!kScatterPrefetch) fetchB(i0);
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            const int64_t i = i0 + 32 * u + lane;
            const int64_t ic = min(i, s1 - 1);
            if (HAS_V && RECS) { x[u] = __ldg(v + ic); y[u] = __ldg(v + ldv + ic); z[u] = __ldg(v + 2 * ldv + ic); }
            else { x[u] = y[u] = z[u] = 0.0; }
            const int32_t c = cB[u];
            key[u] = (i >= s1) ? -1 - lane : ((c >= 0 && c < M) ? c : M);
        }
        if (kScatterPrefetch && i0 + 32 * UB < s1) fetchB(i0 + 32 * UB);
        uint32_t peers[UB], old[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) peers[u] = __match_any_sync(0xFFFFFFFFu, key[u]);
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            const int32_t b = max(key[u], 0);
            old[u] = atom_add_if(key[u] >= 0 && lane == __ffs(peers[u]) - 1, my + (b >> 1),
                                 static_cast<uint32_t>(__popc(peers[u])) << ((b & 1) << 4));
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            const int32_t b = key[u];
            const uint32_t o = __shfl_sync(0xFFFFFFFFu, (old[u] >> ((max(b, 0) & 1) << 4)) & 0xFFFFu,
                                           __ffs(peers[u]) - 1);
            if (b >= 0) {
                const int32_t dest = base[b] + static_cast<int32_t>(o) + __popc(peers[u] & lt);
                const int64_t i = i0 + 32 * u + lane;
                if (RECS)
                    st256(wsv + 4 * static_cast<int64_t>(dest), x[u], y[u], z[u],
                          pack_pc(static_cast<int32_t>(i), b < M ? b : -1));
                else
                    sperm[dest] = static_cast<int32_t>(i);
                CC_DBG_ASSERT(dest >= 0 && dest < n && i < s1);
            }
        }
    }
}

template <bool HAS_V>
__global__ void __launch_bounds__(32 * kMaxScatterWarps, CC_SCATTER_CTAS)
k_scatter(const double* __restrict__ v, int64_t ldv, const int32_t* __restrict__ cell, int n, int M,
          int W, int sub, const int32_t* __restrict__ tbase, const int32_t* __restrict__ off,
          double* __restrict__ wsv, const int32_t* __restrict__ flags, int index_modes)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // binning mode (bin_mode): sorted -> nothing to move; perm -> 4-byte input indices only
    const int mode = flags ? bin_mode(flags, n, M, index_modes) : kModeRec;
    if (mode == kModeSorted) return;
    const bool recs = mode == kModeRec;
    int32_t* __restrict__ sperm = reinterpret_cast<int32_t*>(wsv);   // kModePerm: input index per stable slot
    if (flags && flags[1] == 0) {
        // input already cell-sorted: the stable order is the identity, so the
        // records are written in place (a streaming SoA -> 32-byte-record pack)
        const int64_t t0 = static_cast<int64_t>(blockIdx.x) * W * sub;
        const int64_t t1 = min(t0 + static_cast<int64_t>(W) * sub, static_cast<int64_t>(n));
        for (int64_t i0 = t0 + static_cast<int64_t>(w) * 32 * kScatterUnrollB; i0 < t1;
             i0 += static_cast<int64_t>(W) * 32 * kScatterUnrollB) {
            double x[kScatterUnrollB], y[kScatterUnrollB], z[kScatterUnrollB];
            int32_t c[kScatterUnrollB];
#pragma unroll
            for (int u = 0; u < kScatterUnrollB; ++u)
                load_batch<HAS_V>(v, ldv, cell, min(i0 + 32 * u + lane, t1 - 1), x[u], y[u], z[u], c[u]);
#pragma unroll
            for (int u = 0; u < kScatterUnrollB; ++u) {
                const int64_t i = i0 + 32 * u + lane;
                const bool live = c[u] >= 0 && c[u] < M;
                if (i < t1) st256(wsv + 4 * i, x[u], y[u], z[u], pack_pc(static_cast<int32_t>(i), live ? c[u] : -1));
            }
        }
        return;
    }
    const int M1 = M + 1;
    const int MW = (M1 + 1) / 2;           // 32-bit words per warp row
    int32_t* base = reinterpret_cast<int32_t*>(smem);                       // [M1]
    uint32_t* wcnt = reinterpret_cast<uint32_t*>(smem + sizeof(int32_t) * M1);  // [W][MW] packed u16 pairs
    for (int i = threadIdx.x; i < W * MW; i += blockDim.x) wcnt[i] = 0u;
    // CTA base = cell offset + tile offset (independent of pass A: its loads overlap pass A's)
    const int32_t* trow = tbase + static_cast<int64_t>(blockIdx.x) * M1;
    for (int c = threadIdx.x; c < M1; c += blockDim.x) base[c] = off[c] + trow[c];   // off[M] = L: dead last
    __syncthreads();

    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * W * sub + static_cast<int64_t>(w) * sub;
    const int64_t s1 = min(s0 + sub, static_cast<int64_t>(n));
    uint32_t* my = wcnt + w * MW;
    const uint32_t lt = (1u << lane) - 1u;

    // pass A: per-warp counts of the sub-range (loads batched, branch-free); counting is order-free,
    // so lane l takes the kScatterUnrollA consecutive ids [i0 + l UA, ...) with 32-byte loads and
    // "row" u of the match is the u-th id of every lane; the next batch's ids are loaded before
    // this batch is counted (CC_SCATTER_PREFETCH)
    static_assert(kScatterUnrollA % 8 == 0, "pass A loads 8 ids per 32-byte load");
    const bool vec32 = (reinterpret_cast<uintptr_t>(cell) & 31u) == 0;
    int32_t cN[kScatterUnrollA];
    auto fetchA = [&](int64_t i0) {
        const int64_t b = i0 + static_cast<int64_t>(kScatterUnrollA) * lane;
        if (vec32 && b + kScatterUnrollA <= s1) {
#pragma unroll
            for (int h = 0; h < kScatterUnrollA / 8; ++h) {
                unsigned long long a0, a1, a2, a3;
                asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                    : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(cell + b + 8 * h));
                cN[8 * h + 0] = static_cast<int32_t>(a0); cN[8 * h + 1] = static_cast<int32_t>(a0 >> 32);
                cN[8 * h + 2] = static_cast<int32_t>(a1); cN[8 * h + 3] = static_cast<int32_t>(a1 >> 32);
                cN[8 * h + 4] = static_cast<int32_t>(a2); cN[8 * h + 5] = static_cast<int32_t>(a2 >> 32);
                cN[8 * h + 6] = static_cast<int32_t>(a3); cN[8 * h + 7] = static_cast<int32_t>(a3 >> 32);
            }
        } else {
#pragma unroll
            for (int u = 0; u < kScatterUnrollA; ++u) cN[u] = __ldg(cell + min(b + u, s1 - 1));
        }
    };
    if (kScatterPrefetch && s0 < s1) fetchA(s0);
    for (int64_t i0 = s0; i0 < s1; i0 += 32 * kScatterUnrollA) {
        int32_t key[kScatterUnrollA];
        if (!kScatterPrefetch) fetchA(i0);
#pragma unroll
        for (int u = 0; u < kScatterUnrollA; ++u) {
            const int64_t i = i0 + static_cast<int64_t>(kScatterUnrollA) * lane + u;
            const int32_t c = cN[u];
            key[u] = (i >= s1) ? -1 - lane : ((c >= 0 && c < M) ? c : M);
        }
        if (kScatterPrefetch && i0 + 32 * kScatterUnrollA < s1) fetchA(i0 + 32 * kScatterUnrollA);
        uint32_t peers[kScatterUnrollA];
#pragma unroll
        for (int u = 0; u < kScatterUnrollA; ++u) peers[u] = __match_any_sync(0xFFFFFFFFu, key[u]);
#pragma unroll
        for (int u = 0; u < kScatterUnrollA; ++u) {
            const int32_t b = max(key[u], 0);
            red_add_if(key[u] >= 0 && lane == __ffs(peers[u]) - 1, my + (b >> 1),
                       static_cast<uint32_t>(__popc(peers[u])) << ((b & 1) << 4));
        }
    }
    __syncthreads();
    // exclusive scan over warps per cell
    for (int c = threadIdx.x; c < M1; c += blockDim.x) {
        const uint32_t sh = (static_cast<uint32_t>(c) & 1u) << 4;
        uint32_t run = 0;
        for (int ww = 0; ww < W; ++ww) {
            uint32_t* wd = wcnt + ww * MW + (c >> 1);
            const uint32_t x = (*wd >> sh) & 0xFFFFu;
            // the two halves of a word belong to cells c and c^1, handled by
            // different threads: update only our half with an atomic
            atomicAdd(wd, (run - x) << sh);    // half := run (mod 2^16, no carry: run, x < 2^16)
            run += x;
        }
    }
    __syncthreads();

    // pass B: ranks, destinations, 32-byte records or 4-byte indices (loads batched, branch-free)
    if (recs) scatter_pass_b<kScatterUnrollB, true, HAS_V>(v, ldv, cell, s0, s1, M, my, base, lane, wsv, sperm, n);
    else scatter_pass_b<kScatterUnrollP, false, false>(v, ldv, cell, s0, s1, M, my, base, lane, wsv, sperm, n);
}

// ------------------------------------------------------------------ CCS4 + CCS5 items
// NEXT f2 push geometry (cc_grid with L_a = n_a d_a precomputed)
struct PushGrid {
    int dims;
    int n[3];
    double d[3], L[3];
    uint32_t periodic;
};

// S2c drift of one position row a (R22-R24), explicitly rounded as in the oracle:
// x' = x + dt v', periodic wrap or absorption, cell index along a.  Returns x'.
__device__ __forceinline__ double drift_axis(const PushGrid& g, int a, double x, double v, double dt, bool& alive,
                                             int64_t& G, int64_t& stride)
{
    double xa = __dadd_rn(x, __dmul_rn(dt, v));
    const double L = g.L[a];
    if (!isfinite(xa)) {
        alive = false;                          // R23: a non-finite position is absorbed
    } else if (g.periodic & (1u << a)) {
        // R23: more than one period away -> the exact remainder (fmod is exact), so each
        // loop below runs at most once (no unbounded wrap)
        if (xa < -L || xa >= 2.0 * L) xa = fmod(xa, L);
        while (xa < 0.0) xa = __dadd_rn(xa, L);
        while (xa >= L) xa = __dsub_rn(xa, L);
    } else if (xa < 0.0 || xa >= L) {
        alive = false;
    }
    if (alive) {
        int64_t i = static_cast<int64_t>(floor(__ddiv_rn(xa, g.d[a])));
        if (i > g.n[a] - 1) i = g.n[a] - 1;
        G += i * stride;
    }
    stride *= g.n[a];
    return xa;
}

struct CollideArgs {
    const double* wsv;          // cell-sorted 32-byte records (cold input)
    int64_t ldv;                // row stride of v_out
    const int32_t* cnt;
    const int32_t* off;
    const int32_t* chunk_off;
    const int4* chunk_cell;     // [max_chunks] {cell, cell's first slot, N, first item} (valid below chunk_off[M])
    const double* Cj;
    const cc::U4* keys;
    double* v_out;
    int32_t* cell_out;
    int32_t* perm_out;
    double* recs;
    double* small_recs;
    double* cellref;            // [M][4] shift of large cells (pre-collision v of the first slot)
    int M;
    uint32_t model;             // CC_ODD_TRIPLET | CC_NANBU (NEXT f1 collision-model variants)
    double* trec;               // [M][kRec] triplet moment records of large odd cells (triplet mode)
    int pair_vec;               // outputs aligned for 16-byte (v) / 8-byte (cell, perm) pair stores
    uint32_t cell_base, step, s0, s1;
    const uint32_t* step_dev;   // NULL, or DEVICE offset added to `step` (cc_params.step_dev)
    int chunk;                  // pairs per k_collide_large CTA (<= kChunk, multiple of kCollideThreads)
    int blocked;                // R1b pairing (default); 0: R1 over the whole cell (CC_CELL_UNIFORM)
    int index_modes;            // bin_mode may pick kModeSorted / kModePerm (R1b calls)
    const int32_t* flags;       // k_count's flags (bin_mode)
    int n;
    const double* v_in;         // the caller's SoA input (read directly in the index modes)
    int64_t ldvi;
    int vec16;                  // v_in 16-byte aligned and ldvi even (16-byte copies of aligned runs)
    const int32_t* seg;         // R1b: [chunks][kBlockSegs] first stable slot of each block segment
    // fused S2b + S2c push of the outputs (cc_params.push; NEXT f2): x_in is read at the
    // particle's input index, x_out / v_out / cell_out written at the output slot
    int push;
    PushGrid pg;
    const double* E;
    int64_t ldE;
    double kick, dt;
    const double* x_in;
    int64_t ldxi;
    double* x_out;
    int64_t ldxo;
};

__device__ __forceinline__ uint32_t eff_step(const CollideArgs& A)
{
    return A.step + (A.step_dev ? __ldg(A.step_dev) : 0u);
}

// Post-collision moment accumulator about a per-cell shift r:
// [0..2] sum (v - r), [3..5] sum (v - r)^2.  (Pre-collision sums come from
// k_scatter, which holds every particle in registers anyway.)
struct Acc {
    double a[6];
    __device__ void zero()
    {
#pragma unroll
        for (int q = 0; q < 6; ++q) a[q] = 0.0;
    }
    __device__ void post(double x, double y, double z, double rx, double ry, double rz)
    {
        const double dx = x - rx, dy = y - ry, dz = z - rz;
        a[0] += dx; a[1] += dy; a[2] += dz;
        a[3] = fma(dx, dx, a[3]); a[4] = fma(dy, dy, a[4]); a[5] = fma(dz, dz, a[5]);
    }
};

struct Rec {
    double x, y, z, w;     // w = (perm, cell) bit pattern
};

// Stable slot s of the current call: its 32-byte record in ws_v.
__device__ __forceinline__ Rec load_slot(const CollideArgs& A, int64_t s)
{
    Rec r;
    ld256(A.wsv + 4 * s, r.x, r.y, r.z, r.w);
    return r;
}

__device__ __forceinline__ int call_mode(const CollideArgs& A) { return bin_mode(A.flags, A.n, A.M, A.index_modes); }

// Stable slot s in any binning mode: the record (kModeRec), or v_in at the slot's input
// index (kModeSorted: the slot itself; kModePerm: the index k_scatter wrote).
__device__ __forceinline__ Rec load_slot_m(const CollideArgs& A, int mode, int64_t s)
{
    if (mode == kModeRec) return load_slot(A, s);
    const int64_t i = (mode == kModeSorted) ? s : static_cast<int64_t>(__ldg(reinterpret_cast<const int32_t*>(A.wsv) + s));
    Rec r;
    r.x = __ldg(A.v_in + i);
    r.y = __ldg(A.v_in + A.ldvi + i);
    r.z = __ldg(A.v_in + 2 * A.ldvi + i);
    r.w = pack_pc(static_cast<int32_t>(i), 0);
    return r;
}

// raw pre-collision sums v (3), |v|^2 (the diagnostics' "before" terms)
__device__ __forceinline__ void pre_add(double (&pre)[4], double x, double y, double z)
{
    pre[0] += x; pre[1] += y; pre[2] += z;
    pre[3] = fma(x, x, fma(y, y, fma(z, z, pre[3])));
}

// Fused push of one particle (cell j = its LOCAL collision cell, -1 dead): kick v (if E),
// drift its position read at input index l, write x_out[.][p]; returns the post-push
// GLOBAL cell (or -1).  The arithmetic is k_push's (drift_axis), so the result is
// bit-identical to coulomb_collide followed by cc_push.
__device__ __forceinline__ int32_t push_one(const CollideArgs& A, int32_t p, int32_t j, int32_t l, double& vx,
                                            double& vy, double& vz)
{
    const PushGrid& g = A.pg;
    double v3[3] = {vx, vy, vz};
    if (j < 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
            if (a < g.dims) A.x_out[a * A.ldxo + p] = __ldg(A.x_in + a * A.ldxi + l);
        return -1;
    }
    if (A.E) {
#pragma unroll
        for (int c = 0; c < 3; ++c) v3[c] = __dadd_rn(v3[c], __dmul_rn(A.kick, __ldg(A.E + c * A.ldE + j)));
        vx = v3[0]; vy = v3[1]; vz = v3[2];
    }
    bool alive = true;
    int64_t G = 0, stride = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a)
        if (a < g.dims)
            A.x_out[a * A.ldxo + p] = drift_axis(g, a, __ldg(A.x_in + a * A.ldxi + l), v3[a], A.dt, alive, G, stride);
    return alive ? static_cast<int32_t>(G) : -1;
}

template <bool PUSH = false>
__device__ __forceinline__ void write_out(const CollideArgs& A, int32_t p, int32_t j, const Rec& r)
{
    double x = r.x, y = r.y, z = r.z;
    int32_t cj = j;
    if (PUSH) cj = push_one(A, p, j, unpack_perm(r.w), x, y, z);
    A.v_out[p] = x;
    A.v_out[A.ldv + p] = y;
    A.v_out[2 * A.ldv + p] = z;
    A.cell_out[p] = cj;
    if (A.perm_out) A.perm_out[p] = unpack_perm(r.w);
}

// Both members of pair k: slots pa, pa+1 of every output row.  With an even
// pa and aligned outputs this is one 16-byte store per velocity row and one
// 8-byte store for the cell ids and for perm.
// fused push: start the position loads of input particle l early (L1 prefetch, no registers)
__device__ __forceinline__ void prefetch_x(const CollideArgs& A, int32_t l)
{
#pragma unroll
    for (int a = 0; a < 3; ++a)
        if (a < A.pg.dims) asm volatile("prefetch.global.L1 [%0];" ::"l"(A.x_in + a * A.ldxi + l));
}

// small kernels (k_collide_small, k_triplets, k_copy_dead): runtime choice
__device__ __forceinline__ void write_out_any(const CollideArgs& A, int32_t p, int32_t j, const Rec& r)
{
    if (A.push) write_out<true>(A, p, j, r);
    else write_out<false>(A, p, j, r);
}

// PUSH (k_collide_large<.., true>): both members are pushed first (push_one writes x_out),
// then the same paired stores carry the kicked velocities and post-push cells.
template <bool PUSH = false>
__device__ __forceinline__ void write_pair_out(const CollideArgs& A, int32_t pa, int32_t j, Rec a, Rec b)
{
    int32_t ca = j, cb = j;
    if (PUSH) {
        ca = push_one(A, pa, j, unpack_perm(a.w), a.x, a.y, a.z);
        cb = push_one(A, pa + 1, j, unpack_perm(b.w), b.x, b.y, b.z);
    }
    if (A.pair_vec && (pa & 1) == 0) {
        *reinterpret_cast<double2*>(A.v_out + pa) = make_double2(a.x, b.x);
        *reinterpret_cast<double2*>(A.v_out + A.ldv + pa) = make_double2(a.y, b.y);
        *reinterpret_cast<double2*>(A.v_out + 2 * A.ldv + pa) = make_double2(a.z, b.z);
        *reinterpret_cast<int2*>(A.cell_out + pa) = make_int2(ca, cb);
        if (A.perm_out) *reinterpret_cast<int2*>(A.perm_out + pa) = make_int2(unpack_perm(a.w), unpack_perm(b.w));
    } else {
        A.v_out[pa] = a.x; A.v_out[A.ldv + pa] = a.y; A.v_out[2 * A.ldv + pa] = a.z;
        A.v_out[pa + 1] = b.x; A.v_out[A.ldv + pa + 1] = b.y; A.v_out[2 * A.ldv + pa + 1] = b.z;
        A.cell_out[pa] = ca;
        A.cell_out[pa + 1] = cb;
        if (A.perm_out) { A.perm_out[pa] = unpack_perm(a.w); A.perm_out[pa + 1] = unpack_perm(b.w); }
    }
}

// CCS4: one Philox call per pair, ctr = (k, G, step, 0) -> (u1, u2) (R3).
__device__ __forceinline__ void pair_uniforms(const CollideArgs& A, int32_t j, uint32_t k, uint32_t step, double& u1,
                                              double& u2)
{
    const cc::U4 r = cc::philox4x32_10(cc::U4{k, A.cell_base + static_cast<uint32_t>(j), step, 0u}, A.s0, A.s1);
    u1 = cc::u01(r.x, r.y);
    u2 = cc::u01(r.z, r.w);
}

template <int NV>
__device__ __forceinline__ void warp_reduce(double (&a)[NV])
{
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) a[q] += __shfl_down_sync(0xFFFFFFFFu, a[q], d);
}

// R19: TA77 odd-count triplet — (1,2), (2,3), (3,1) in order, each with C/2,
// randoms Philox(ctr = (q, G, step, 3)) for sub-collision q; r[] in place.
__device__ __forceinline__ void triplet_update(const CollideArgs& A, uint32_t G, double C, uint32_t step, Rec (&r)[3])
{
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const cc::U4 x = cc::philox4x32_10(cc::U4{static_cast<uint32_t>(q), G, step, 3u}, A.s0, A.s1);
        Rec& a = r[q];
        Rec& b = r[(q + 1) % 3];
        cc::collide_model(a.x, a.y, a.z, b.x, b.y, b.z, 0.5 * C, cc::u01(x.x, x.y), cc::u01(x.z, x.w), A.model);
    }
}

// N_j <= 64: one warp per cell; item k = lane.  The warp holds the whole cell,
// so its moment record is an exact two-pass one about the post-collision mean.
__global__ void __launch_bounds__(256)
k_collide_small(CollideArgs A)
{
    __shared__ int32_t pi_sm[8][cc::kSmallCell];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int j = blockIdx.x * 8 + w;
    if (j >= A.M) return;
    const int32_t N = A.cnt[j];
    if (N == 0 || N > cc::kSmallCell) return;
    const int32_t o = A.off[j];
    const uint32_t G = A.cell_base + static_cast<uint32_t>(j);
    const uint32_t step = eff_step(A);
    const int mode = call_mode(A);
    double pre[4] = {0.0, 0.0, 0.0, 0.0};
    cc::small_cell_perm(static_cast<uint32_t>(N), G, step, A.s0, A.s1, lane, pi_sm[w]);
    const double C = A.Cj[j];
    Acc acc;
    acc.zero();
    const uint32_t items = static_cast<uint32_t>(N + 1) / 2;
    const uint32_t k = static_cast<uint32_t>(lane);
    const bool triplet = (A.model & cc::kOddTriplet) && N >= 3 && (N & 1);
    Rec mine[3];                  // this lane's post-collision particles (pair, sitter or triplet)
    int nmine = 0;
    if (triplet && k == items - 2) {
        // R19: the last three of the pair order collide as a TA77 triplet
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            mine[q] = load_slot_m(A, mode, o + pi_sm[w][N - 3 + q]);
            pre_add(pre, mine[q].x, mine[q].y, mine[q].z);
        }
        triplet_update(A, G, C, step, mine);
#pragma unroll
        for (int q = 0; q < 3; ++q) write_out_any(A, o + N - 3 + q, j, mine[q]);
        nmine = 3;
    } else if (k < items && !(triplet && k == items - 1)) {
        const int32_t pa = o + 2 * static_cast<int32_t>(k);
        mine[0] = load_slot_m(A, mode, o + pi_sm[w][2 * k]);
        pre_add(pre, mine[0].x, mine[0].y, mine[0].z);
        nmine = 1;
        if (2 * k + 1 < static_cast<uint32_t>(N)) {
            mine[1] = load_slot_m(A, mode, o + pi_sm[w][2 * k + 1]);
            pre_add(pre, mine[1].x, mine[1].y, mine[1].z);
            double u1, u2;
            pair_uniforms(A, j, k, step, u1, u2);
            cc::collide_model(mine[0].x, mine[0].y, mine[0].z, mine[1].x, mine[1].y, mine[1].z, C, u1, u2, A.model);
            write_out_any(A, pa + 1, j, mine[1]);
            nmine = 2;
        }
        write_out_any(A, pa, j, mine[0]);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
        if (q < nmine) acc.post(mine[q].x, mine[q].y, mine[q].z, 0.0, 0.0, 0.0);
    warp_reduce(acc.a);
    // pass 2: sums about the exact mean, from the lane's own particles (registers; the
    // output may be in input order, CC_PRESERVE_ORDER)
    const double inv = 1.0 / static_cast<double>(N);
    const double mx = __shfl_sync(0xFFFFFFFFu, acc.a[0], 0) * inv;
    const double my = __shfl_sync(0xFFFFFFFFu, acc.a[1], 0) * inv;
    const double mz = __shfl_sync(0xFFFFFFFFu, acc.a[2], 0) * inv;
    Acc q;
    q.zero();
#pragma unroll
    for (int t = 0; t < 3; ++t)
        if (t < nmine) q.post(mine[t].x, mine[t].y, mine[t].z, mx, my, mz);
    warp_reduce(q.a);
    warp_reduce(pre);
    if (lane == 0) {
        double* r = A.small_recs + static_cast<int64_t>(j) * kSmallRec;
#pragma unroll
        for (int c = 0; c < 6; ++c) r[c] = q.a[c];
        r[6] = mx; r[7] = my; r[8] = mz;
        r[9] = r[10] = r[11] = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) r[12 + c] = pre[c];
    }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem_src) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}

// Gather stable slot s's 32-byte record into shared memory.
__device__ __forceinline__ void stage_slot(const CollideArgs& A, int64_t s, double* dst)
{
    const double* g = A.wsv + 4 * s;
    cp_async16(dst, g);
    cp_async16(dst + 2, g + 2);
}

// A staged particle: interleaved 32-byte records (kModeRec) or, in the index modes, the
// planar stage x[kBlock], y[kBlock], z[kBlock], input index (int32)[kBlock].
__device__ __forceinline__ Rec stage_rec(const double* stage, bool planar, uint32_t u)
{
    if (planar)
        return Rec{stage[u], stage[cc::kBlock + u], stage[2 * cc::kBlock + u],
                   pack_pc(reinterpret_cast<const int32_t*>(stage + 3 * cc::kBlock)[u], 0)};
    const double2 a01 = *reinterpret_cast<const double2*>(stage + 4 * u);
    const double2 a23 = *reinterpret_cast<const double2*>(stage + 4 * u + 2);
    return Rec{a01.x, a01.y, a23.x, a23.y};
}

// N_j > 64: one CTA per cell-aligned chunk of kChunk items, two phases:
//  1. (R1) every thread computes pi_j(2k), pi_j(2k+1) (keyed Feistel) for its
//     items and issues cp.async gathers of both records into shared memory —
//     the whole chunk's gathers are in flight at once; (R1b) see BLOCKED below;
//  2. items are processed two per thread per round: Philox (CCS4), the central
//     AS241 branch in place and the tail branch (~15% of draws) compacted
//     across the warp and evaluated once per 32 tails, then TA (CCS5), and the
//     pair-ordered, coalesced SoA output plus the moment partials.
constexpr int kItemsPerThread = kChunk / kCollideThreads;
constexpr int kWarpItems = 32 * kItemsPerThread;            // items of one warp per chunk
constexpr size_t kCollideSmem = 2ull * kChunk * 4 * sizeof(double);
static_assert(kChunk % kCollideThreads == 0, "chunk must be a whole number of thread items");

static_assert(kChunk >= cc::kBlock / 2, "one k_collide_large CTA holds an R1b block (stage and thread items)");

// BLOCKED (R1b, the default pairing): the CTA owns block b = i0 / (kBlock/2) of its cell.
// Phase 1 copies the block's segments (whole 32-record runs of the cell-sorted records,
// in the block's segment order; cells of N <= kBlock are one block of consecutive slots)
// into the stage with contiguous 16-byte cp.async — a warp instruction moves 512
// consecutive bytes — and computes tau_b of each item's two block slots; phase 2 reads
// the pair's records from the stage at those slots.  No random global access.
#ifndef CC_BLOCKED_CTAS
#define CC_BLOCKED_CTAS 10
#endif
template <bool NANBU, bool PUSH, bool BLOCKED>
__global__ void __launch_bounds__(kCollideThreads, BLOCKED ? CC_BLOCKED_CTAS : CC_COLLIDE_CTAS)
k_collide_large(CollideArgs A)
{
    extern __shared__ __align__(16) double stage[];       // R1: [2][kChunk][4]; R1b: [kBlock][4]
    __shared__ int32_t pi_small[BLOCKED ? cc::kSmallCell : 1];
    __shared__ __align__(16) double ref_sm[4];             // R1b: the cell's first stable slot (moment shift)
    __shared__ double zq[kCollideThreads / 32][kWarpItems];  // normal variate z = Phi^-1(u1) per item
    __shared__ double u2q[kCollideThreads / 32][kWarpItems]; // u2 per item
    __shared__ int16_t tq[kCollideThreads / 32][kWarpItems]; // compacted AS241-tail (Nanbu: Newton) items
    __shared__ double aq[NANBU ? kCollideThreads / 32 : 1][NANBU ? kWarpItems : 1];  // Nanbu A per item
    __shared__ double red[kCollideThreads / 32][10];
    const int c = blockIdx.x;
    if (c >= __ldg(A.chunk_off + A.M)) return;      // grid is an upper bound on the chunk count
    const int4 cm = __ldg(A.chunk_cell + c);
    const int j = cm.x;
    const int32_t N = cm.z, o = cm.y;
    const uint32_t step = eff_step(A);
    const uint32_t items = static_cast<uint32_t>(N + 1) / 2;
    const uint32_t i0 = static_cast<uint32_t>(cm.w);
    const uint32_t i1 = min(i0 + static_cast<uint32_t>(A.chunk), items);
    const bool triplet = (A.model & cc::kOddTriplet) && (N & 1);   // N > 64 here
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int mode = BLOCKED ? call_mode(A) : kModeRec;
    int32_t nb = 0;                                        // R1b: slots of this CTA's block
    uint32_t xs[kItemsPerThread][2];                      // R1b: block slots of each item's pair
    if (BLOCKED) {
        const uint32_t b = i0 / static_cast<uint32_t>(cc::kBlock / 2);
        nb = min(N - static_cast<int32_t>(b) * cc::kBlock, cc::kBlock);
        const int nseg = (nb + cc::kSeg - 1) / cc::kSeg;
        int32_t sg[cc::kBlockSegs];                       // absolute first stable slot of each segment
        {
            const int4* sp = reinterpret_cast<const int4*>(A.seg + static_cast<int64_t>(c) * cc::kBlockSegs);
#pragma unroll
            for (int g4 = 0; g4 < cc::kBlockSegs / 4; ++g4) {
                const int4 q = __ldg(sp + g4);
                sg[4 * g4] = q.x; sg[4 * g4 + 1] = q.y; sg[4 * g4 + 2] = q.z; sg[4 * g4 + 3] = q.w;
            }
        }
#ifdef CC_DEBUG_BOUNDS
        for (int g = 0; g < nseg; ++g) {
            const int32_t len = min(cc::kSeg, nb - g * cc::kSeg);
            CC_DBG_ASSERT(sg[g] >= o && sg[g] + len <= o + N && (sg[g] - o) % cc::kSeg == 0);
        }
#endif
        if (mode == kModeRec) {
            // 16-byte pieces: segment g = pieces [64 g, 64 g + 64), record (piece mod 64) / 2
#pragma unroll
            for (int g = 0; g < cc::kBlockSegs; ++g) {
                if (g < nseg) {
                    for (int p = threadIdx.x; p < 2 * cc::kSeg; p += kCollideThreads) {
                        const int r = p >> 1, h = p & 1;
                        if (g * cc::kSeg + r < nb)
                            cp_async16(stage + 4 * (g * cc::kSeg + r) + 2 * h,
                                       A.wsv + 4 * (static_cast<int64_t>(sg[g]) + r) + 2 * h);
                    }
                }
            }
            if (threadIdx.x < 2) cp_async16(ref_sm + 2 * threadIdx.x, A.wsv + 4 * static_cast<int64_t>(o) + 2 * threadIdx.x);
        }
        // index modes: the input indices are loaded first and the copies issued after tau_b,
        // so the index loads' latency hides behind the Feistel rounds
        static_assert(kCollideThreads % cc::kSeg == 0, "a warp covers whole segments");
        constexpr int kPer = cc::kBlock / kCollideThreads;
        int32_t idx[kPer];
        int32_t iref = o;                                  // input index of the cell's first stable slot
        if (mode != kModeRec) {
            if (mode == kModePerm && threadIdx.x < 3) iref = __ldg(reinterpret_cast<const int32_t*>(A.wsv) + o);
            // index modes: block slot u = stable slot o + sg[u / 32] + u % 32 = input index
            // (kModeSorted) or the index k_scatter wrote (kModePerm); its three velocity
            // components are copied from the SoA input (a warp reads 32 mostly consecutive
            // indices: three coalesced 256-byte runs), w = the input index
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int u = static_cast<int>(threadIdx.x) + q * kCollideThreads;
                // segment of u: q * (kCollideThreads / 32) + w, selected without dynamic indexing
                int32_t st0 = 0;
#pragma unroll
                for (int ww = 0; ww < kCollideThreads / cc::kSeg; ++ww)
                    if (ww == w) st0 = sg[q * (kCollideThreads / cc::kSeg) + ww];
                const int64_t sl = static_cast<int64_t>(st0) + lane;
                idx[q] = (u < nb) ? (mode == kModeSorted ? static_cast<int32_t>(sl)
                                                         : __ldg(reinterpret_cast<const int32_t*>(A.wsv) + sl))
                                  : -1;
                CC_DBG_ASSERT(idx[q] >= -1 && idx[q] < A.n && (u >= nb || idx[q] >= 0));
            }
        }
        const uint32_t G = A.cell_base + static_cast<uint32_t>(j);
        if (nb > cc::kSmallCell) {
            const cc::Feistel f = cc::make_feistel(static_cast<uint32_t>(nb), cc::philox4x32_10(cc::U4{b, G, step, 1u}, A.s0, A.s1));
#pragma unroll
            for (int q = 0; q < kItemsPerThread; ++q) {
                const uint32_t e = threadIdx.x + q * kCollideThreads;
                uint32_t x[2] = {2 * e, 2 * e + 1};
                if (i0 + e < i1 && !(CC_ABLATE & 2)) {
                    cc::feistel_E_multi(f, x);
                    while (x[0] >= f.N) x[0] = cc::feistel_E(f, x[0]);
                    if (2 * e + 1 < static_cast<uint32_t>(nb))
                        while (x[1] >= f.N) x[1] = cc::feistel_E(f, x[1]);
                }
                xs[q][0] = x[0];
                xs[q][1] = x[1];
                CC_DBG_ASSERT(i0 + e >= i1 || (x[0] < static_cast<uint32_t>(nb) &&
                                               (2 * e + 1 >= static_cast<uint32_t>(nb) || x[1] < static_cast<uint32_t>(nb))));
            }
        } else {
            // the last block of a large cell holds <= 64 slots: R1's sort-by-key form
            if (w == 0) cc::small_cell_perm(static_cast<uint32_t>(nb), G, step, A.s0, A.s1, lane, pi_small,
                                           b * static_cast<uint32_t>(cc::kBlock / 4), 2u);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < kItemsPerThread; ++q) {
                const uint32_t e = threadIdx.x + q * kCollideThreads;
                xs[q][0] = (2 * e < static_cast<uint32_t>(nb)) ? pi_small[2 * e] : 0u;
                xs[q][1] = (2 * e + 1 < static_cast<uint32_t>(nb)) ? pi_small[2 * e + 1] : 0u;
            }
        }
        if (mode != kModeRec) {
            // planar stage (consecutive lanes -> consecutive 8-byte words: no bank conflicts)
            int32_t* pw = reinterpret_cast<int32_t*>(stage + 3 * cc::kBlock);
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int u = static_cast<int>(threadIdx.x) + q * kCollideThreads;
                // a warp's 32 slots are one segment; when their input indices are one even-aligned
                // run (always for sorted input in an even-offset cell; about half the segments of
                // steady input) the three 256-byte rows move as 16-byte copies
                const int32_t i0w = __shfl_sync(0xFFFFFFFFu, idx[q], 0);
                const bool run = A.vec16 && __all_sync(0xFFFFFFFFu, idx[q] == i0w + lane) && (i0w & 1) == 0;
                if (CC_ABLATE & 8) {
                } else if (run) {
                    const int seg0 = u - lane;                   // planar position of the segment
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const int pc = lane + 32 * r;            // 48 pieces: row pc / 16, pair pc % 16
                        if (pc < 48) {
                            const int row = pc >> 4, h = pc & 15;
                            cp_async16(stage + row * cc::kBlock + seg0 + 2 * h, A.v_in + row * A.ldvi + i0w + 2 * h);
                        }
                    }
                } else if (idx[q] >= 0) {
                    const double* src = A.v_in + idx[q];
                    cp_async8(stage + u, src);
                    cp_async8(stage + cc::kBlock + u, src + A.ldvi);
                    cp_async8(stage + 2 * cc::kBlock + u, src + 2 * A.ldvi);
                }
                if (idx[q] >= 0) pw[u] = idx[q];
            }
            if (threadIdx.x < 3) cp_async8(ref_sm + threadIdx.x, A.v_in + iref + threadIdx.x * A.ldvi);
        }
    }
    // phase 1 (R1): pi_j (keyed Feistel) of each item's two slots in lock step
    // (rare cycle walks afterwards), gathers issued item by item
    if (!BLOCKED) {
        const cc::Feistel f = cc::make_feistel(static_cast<uint32_t>(N), A.keys[j]);
#pragma unroll kP1Unroll
        for (int q = 0; q < kItemsPerThread; ++q) {
            const uint32_t k = i0 + threadIdx.x + q * kCollideThreads;
            if (k < i1) {
                const uint32_t e = k - i0;
                uint32_t x[2] = {2 * k, 2 * k + 1};
                if (!(CC_ABLATE & 2)) cc::feistel_E_multi(f, x);
                while (x[0] >= f.N) x[0] = cc::feistel_E(f, x[0]);       // cycle walking (rare)
                stage_slot(A, o + static_cast<int64_t>(x[0]), stage + 4 * e);
                if (2 * k + 1 < static_cast<uint32_t>(N)) {
                    while (x[1] >= f.N) x[1] = cc::feistel_E(f, x[1]);
                    stage_slot(A, o + static_cast<int64_t>(x[1]), stage + 4 * (kChunk + e));
                }
            }
        }
    }
    // phase 2a (overlaps the gathers): CCS4 Philox per pair and AS241; the
    // central branch in place, the tails compacted across the warp
    {
        const uint32_t lt = (1u << lane) - 1u;
        int qn = 0;
        double u1[kItemsPerThread], u2[kItemsPerThread];
#pragma unroll
        for (int t = 0; t < kItemsPerThread; ++t) {    // independent Philox calls, interleaved
            if (CC_ABLATE & 4) { u1[t] = 0.3; u2[t] = 0.7; continue; }
            pair_uniforms(A, j, i0 + threadIdx.x + t * kCollideThreads, step, u1[t], u2[t]);
        }
#pragma unroll
        for (int t = 0; t < kItemsPerThread; ++t) {
            const uint32_t k = i0 + threadIdx.x + t * kCollideThreads;
            const bool pair = (k < i1) && (2 * k + 1 < static_cast<uint32_t>(N));
            const bool nanbu = NANBU;                       // Nanbu samples from u1 itself (phase 2b)
            const bool tail = pair && !nanbu && !cc::ppnd16_is_central(u1[t]);
            const int slot = t * 32 + lane;
            zq[w][slot] = nanbu ? u1[t] : tail ? cc::ppnd16_tail_arg(u1[t]) : cc::ppnd16_central(u1[t]);
            u2q[w][slot] = u2[t];
            const uint32_t tm = __ballot_sync(0xFFFFFFFFu, tail);
            if (tail) tq[w][qn + __popc(tm & lt)] = static_cast<int16_t>(slot);
            qn += __popc(tm);
        }
        __syncwarp();
        for (int e = lane; e < qn; e += 32) {
            const int slot = tq[w][e];
            zq[w][slot] = cc::ppnd16_tail(zq[w][slot]);
        }
    }
    // shift for the moment partials: pre-collision v of the cell's first stable slot
    Rec ref;
    if (!BLOCKED) ref = load_slot(A, o);
    const double C = A.Cj[j];
    const double sqC = sqrt(C);
    cp_async_wait_all();
    __syncthreads();
    if (BLOCKED) ref = Rec{ref_sm[0], ref_sm[1], ref_sm[2], 0.0};
    if (i0 == 0 && threadIdx.x == 0) {
        double* cr = A.cellref + 4 * static_cast<int64_t>(j);
        cr[0] = ref.x; cr[1] = ref.y; cr[2] = ref.z; cr[3] = 0.0;
    }
    // raw pre-collision sums of the particles this thread updates (diagnostics)
    double pre[4] = {0.0, 0.0, 0.0, 0.0};
#ifdef CC_STUDY_NOREC
    const bool planar = BLOCKED;
#else
    const bool planar = mode != kModeRec;
#endif

    // phase 2b: CCS5 TA update out of shared memory, pair-ordered coalesced output
    if (NANBU) {
        // Nanbu: A(s) of every pair first.  The cheap cases are set in place; pairs that need the
        // inverse-Langevin Newton solve are compacted across the warp (tq, unused by Nanbu in
        // phase 2a) and solved with all lanes busy, instead of each warp iterating for its
        // slowest lane.  aq[slot] holds A (or x = e^-s until solved).
        const uint32_t lt = (1u << lane) - 1u;
        int qn = 0;
#pragma unroll 1
        for (int t = 0; t < kItemsPerThread; ++t) {
            const uint32_t k = i0 + threadIdx.x + t * kCollideThreads;
            const uint32_t e = k - i0;
            const int slot = t * 32 + lane;
            bool newton = false;
            if (k < i1 && !(triplet && k + 2 >= items) && 2 * k + 1 < static_cast<uint32_t>(N)) {
                const uint32_t ia = BLOCKED ? xs[t][0] : e, ib = BLOCKED ? xs[t][1] : kChunk + e;
                const Rec a = stage_rec(stage, planar, ia), b = stage_rec(stage, planar, ib);
                double Av, x;
                newton = !cc::nanbu_A_direct(cc::nanbu_s(a.x, a.y, a.z, b.x, b.y, b.z, C), Av, x);
                aq[w][slot] = newton ? x : Av;
            }
            const uint32_t nm = __ballot_sync(0xFFFFFFFFu, newton);
            if (newton) tq[w][qn + __popc(nm & lt)] = static_cast<int16_t>(slot);
            qn += __popc(nm);
        }
        __syncwarp();
        for (int q = lane; q < qn; q += 32) {
            const int slot = tq[w][q];
            aq[w][slot] = cc::nanbu_newton(aq[w][slot]);
        }
        __syncwarp();
    }
    Acc acc;
    acc.zero();
    // (Nanbu's sampler is several transcendentals long: one copy of the loop body keeps the
    // kernel inside the instruction cache)
    constexpr int kUnroll2b = NANBU ? 1 : kP2BUnroll;
#pragma unroll kUnroll2b
    for (int t = 0; t < kItemsPerThread; ++t) {
        const uint32_t k = i0 + threadIdx.x + t * kCollideThreads;
        if (k < i1 && !(triplet && k + 2 >= items)) {     // the triplet's two items: k_triplets
            const uint32_t e = k - i0;
            const int32_t pa = o + 2 * static_cast<int32_t>(k);
            const uint32_t ia = BLOCKED ? xs[t][0] : e, ib = BLOCKED ? xs[t][1] : kChunk + e;
            Rec a = stage_rec(stage, planar, ia);
            pre_add(pre, a.x, a.y, a.z);
            if (2 * k + 1 < static_cast<uint32_t>(N)) {
                Rec b = stage_rec(stage, planar, ib);
                pre_add(pre, b.x, b.y, b.z);
                if (PUSH) {                                // the push's position gathers, in flight
                    prefetch_x(A, unpack_perm(a.w));       // during the collision arithmetic
                    prefetch_x(A, unpack_perm(b.w));
                }
                const int slot = t * 32 + lane;
                if (NANBU)
                    cc::nanbu_apply(a.x, a.y, a.z, b.x, b.y, b.z, aq[w][slot], zq[w][slot], u2q[w][slot]);
                else if (!(CC_ABLATE & 1))
                    cc::ta_update_zs(a.x, a.y, a.z, b.x, b.y, b.z, sqC, zq[w][slot], u2q[w][slot]);
                write_pair_out<PUSH>(A, pa, j, a, b);
                acc.post(b.x, b.y, b.z, ref.x, ref.y, ref.z);
            } else {
                write_out<PUSH>(A, pa, j, a);
            }
            acc.post(a.x, a.y, a.z, ref.x, ref.y, ref.z);
        }
    }
    warp_reduce(acc.a);
    warp_reduce(pre);
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 6; ++q) red[w][q] = acc.a[q];
#pragma unroll
        for (int q = 0; q < 4; ++q) red[w][6 + q] = pre[q];
    }
    __syncthreads();
    if (threadIdx.x < kRec) {
        double sum = 0.0;
        if (threadIdx.x < 10)
#pragma unroll
            for (int ww = 0; ww < kCollideThreads / 32; ++ww) sum += red[ww][threadIdx.x];
        A.recs[static_cast<int64_t>(c) * kRec + threadIdx.x] = sum;
    }
}

// R1b: the stable slot (relative to the cell) at pair-order position q of a cell of
// N > kBlock slots, from the segment table k_cell_setup wrote (one thread, off the hot path)
__device__ __noinline__ uint32_t blocked_slot(const CollideArgs& A, int j, int32_t N, uint32_t q)
{
    const uint32_t b = q / cc::kBlock, r = q % cc::kBlock;
    const uint32_t nb = static_cast<uint32_t>(min(N - static_cast<int32_t>(b) * cc::kBlock, cc::kBlock));
    const uint32_t G = A.cell_base + static_cast<uint32_t>(j), step = eff_step(A);
    uint32_t u;
    if (nb > static_cast<uint32_t>(cc::kSmallCell)) {
        const cc::Feistel f = cc::make_feistel(nb, cc::philox4x32_10(cc::U4{b, G, step, 1u}, A.s0, A.s1));
        u = cc::feistel_pi(f, r);
    } else {
        u = cc::small_select(nb, r, G, step, A.s0, A.s1, b * (cc::kBlock / 4), 2u);
    }
    const int32_t c = A.chunk_off[j] + static_cast<int32_t>(b);
    const uint32_t slot = static_cast<uint32_t>(A.seg[static_cast<int64_t>(c) * cc::kBlockSegs + u / cc::kSeg] - A.off[j]) + u % cc::kSeg;
    CC_DBG_ASSERT(u < nb && slot < static_cast<uint32_t>(N));
    return slot;
}

// Triplet mode, N_j > 64 and odd: thread per cell runs R19 on the last three
// slots of the pair order and writes their moment partials (about the cell's
// shift) to trec[j]; every other large cell gets a zero record.
__global__ void k_triplets(CollideArgs A)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= A.M) return;
    const int32_t N = A.cnt[j];
    if (N <= cc::kSmallCell) return;
    double* tr = A.trec + static_cast<int64_t>(j) * kRec;
    Acc acc;
    acc.zero();
    double pre[4] = {0.0, 0.0, 0.0, 0.0};
    if (N & 1) {
        const int32_t o = A.off[j];
        Rec r[3];
        if (A.blocked && N > cc::kBlock) {
#pragma unroll 1
            for (int q = 0; q < 3; ++q)
                r[q] = load_slot_m(A, call_mode(A), o + static_cast<int64_t>(blocked_slot(A, j, N, static_cast<uint32_t>(N - 3 + q))));
        } else {
            const cc::Feistel f = cc::make_feistel(static_cast<uint32_t>(N), A.keys[j]);
#pragma unroll
            for (int q = 0; q < 3; ++q) r[q] = load_slot(A, o + static_cast<int64_t>(cc::feistel_pi(f, N - 3 + q)));
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) pre_add(pre, r[q].x, r[q].y, r[q].z);
        triplet_update(A, A.cell_base + static_cast<uint32_t>(j), A.Cj[j], eff_step(A), r);
        const double* cr = A.cellref + 4 * static_cast<int64_t>(j);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            write_out_any(A, o + N - 3 + q, j, r[q]);
            acc.post(r[q].x, r[q].y, r[q].z, cr[0], cr[1], cr[2]);
        }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) tr[q] = acc.a[q];
#pragma unroll
    for (int q = 0; q < 4; ++q) tr[6 + q] = pre[q];
    tr[10] = tr[11] = 0.0;
}

// CC_PRESERVE_ORDER, pass 1: output position p -> a 32-byte record {v, cell} at the
// particle's input position perm[p] in the (now free) record array.
__global__ void k_unpermute(const double* __restrict__ v, int64_t ldv, const int32_t* __restrict__ cell,
                            const int32_t* __restrict__ perm, int64_t n, double* __restrict__ wsv)
{
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = perm[p];
        st256(wsv + 4 * i, v[p], v[ldv + p], v[2 * ldv + p], __longlong_as_double(static_cast<long long>(cell[p])));
    }
}

// pass 2: the records, now in input order, back to the SoA outputs (streaming); perm = identity
__global__ void k_unpack(const double* __restrict__ wsv, int64_t n, double* __restrict__ v, int64_t ldv,
                         int32_t* __restrict__ cell, int32_t* __restrict__ perm)
{
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double x, y, z, w;
        ld256(wsv + 4 * i, x, y, z, w);
        v[i] = x;
        v[ldv + i] = y;
        v[2 * ldv + i] = z;
        cell[i] = static_cast<int32_t>(__double_as_longlong(w));
        if (perm) perm[i] = static_cast<int32_t>(i);
    }
}

// Dead (and invalid) particles: slots [L, n), copied unchanged.
__global__ void k_copy_dead(CollideArgs A, int n)
{
    const int32_t L = A.off[A.M];
    const int mode = call_mode(A);
    for (int64_t p = L + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const Rec r = load_slot_m(A, mode, p);
        write_out_any(A, static_cast<int32_t>(p), -1, r);
    }
}

// ------------------------------------------------------------------ moments and diagnostics
struct MomConst {
    double weight, volume;
    const double* volume_arr;
    double m_over_e;
};

// moments from shifted sums: mean = ref + S1/N, T = (m/e) (S2/N - (S1/N)^2)
__device__ __forceinline__ void moments_from_sums(const double* s, double N, double rx, double ry,
                                                  double rz, double V, const MomConst& mc, double* o)
{
    const double inv = 1.0 / N;
    const double d[3] = {s[0] * inv, s[1] * inv, s[2] * inv};
    const double r[3] = {rx, ry, rz};
    o[0] = N * mc.weight / V;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        o[1 + q] = r[q] + d[q];
        o[4 + q] = mc.m_over_e * (s[3 + q] * inv - d[q] * d[q]);
    }
}

__global__ void k_finalize_cells(const int32_t* __restrict__ cnt, const int32_t* __restrict__ chunk_off,
                                 const double* __restrict__ recs, const double* __restrict__ small_recs,
                                 const double* __restrict__ cellref, const double* __restrict__ trec, int M,
                                 MomConst mc, double* __restrict__ moments_out, double* __restrict__ cellsum)
{
    // warp per cell: the lanes add the cell's chunk records in a fixed strided order, then a
    // fixed shuffle tree (deterministic); lane 0 finishes the cell
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= M) return;
    const int32_t N = cnt[j];
    double s[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};    // post S1', S2' (6), raw pre (4)
    double rx = 0, ry = 0, rz = 0;
    if (N > cc::kSmallCell) {
        for (int32_t c = chunk_off[j] + lane; c < chunk_off[j + 1]; c += 32)
#pragma unroll
            for (int q = 0; q < 10; ++q) s[q] += recs[static_cast<int64_t>(c) * kRec + q];
#pragma unroll
        for (int q = 0; q < 10; ++q)
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) s[q] += __shfl_down_sync(0xFFFFFFFFu, s[q], d);
    }
    if (lane != 0) return;
    if (N > 0) {
        if (N <= cc::kSmallCell) {
            const double* r = small_recs + static_cast<int64_t>(j) * kSmallRec;
#pragma unroll
            for (int q = 0; q < 6; ++q) s[q] = r[q];
#pragma unroll
            for (int q = 0; q < 4; ++q) s[6 + q] = r[12 + q];
            rx = r[6]; ry = r[7]; rz = r[8];
        } else {
            const double* cr = cellref + 4 * static_cast<int64_t>(j);
            rx = cr[0]; ry = cr[1]; rz = cr[2];
            if (trec)
#pragma unroll
                for (int q = 0; q < 10; ++q) s[q] += trec[static_cast<int64_t>(j) * kRec + q];
        }
    }
    if (moments_out) {
        double* o = moments_out + static_cast<int64_t>(j) * CC_MOMENTS_LEN;
        if (N > 0) {
            const double V = mc.volume_arr ? mc.volume_arr[j] : mc.volume;
            moments_from_sums(s, static_cast<double>(N), rx, ry, rz, V, mc, o);
        } else {
#pragma unroll
            for (int q = 0; q < CC_MOMENTS_LEN; ++q) o[q] = 0.0;
        }
    }
    // raw post-collision sums: sum v = N r + S1', sum v^2 = S2' + 2 r S1' + N r^2
    const double Nd = static_cast<double>(N);
    const double r[3] = {rx, ry, rz};
    double* cs = cellsum + static_cast<int64_t>(j) * kCellSum;
    double e = 0.0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        cs[q] = fma(Nd, r[q], s[q]);
        e += s[3 + q] + 2.0 * r[q] * s[q] + Nd * r[q] * r[q];
    }
    cs[3] = e;
#pragma unroll
    for (int q = 0; q < 4; ++q) cs[4 + q] = s[6 + q];
}

// single CTA of 1024 threads: fixed-order reductions over cells and tiles
__global__ void __launch_bounds__(1024)
k_finalize_diag(const int32_t* __restrict__ cnt, const double* __restrict__ cellsum, int M,
                double* __restrict__ diag)
{
    __shared__ double red[32][12];
    double s[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) s[q] = 0.0;
    // unrolled so each thread's loads are in flight together (same per-thread summation order)
#pragma unroll 4
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
        const int32_t N = cnt[j];
        s[0] += N;
        s[1] += N / 2;
        s[2] += N & 1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            s[7 + q] += cellsum[static_cast<int64_t>(j) * kCellSum + q];
            s[3 + q] += cellsum[static_cast<int64_t>(j) * kCellSum + 4 + q];
        }
    }
    if (threadIdx.x == 0) s[11] = cnt[M];
#pragma unroll
    for (int q = 0; q < 12; ++q)
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) s[q] += __shfl_down_sync(0xFFFFFFFFu, s[q], d);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 12; ++q) red[w][q] = s[q];
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[12];
        for (int q = 0; q < 12; ++q) t[q] = 0.0;
        for (int ww = 0; ww < static_cast<int>(blockDim.x / 32); ++ww)
            for (int q = 0; q < 12; ++q) t[q] += red[ww][q];
        diag[0] = t[0];
        diag[1] = t[11];
        diag[2] = t[1];
        diag[3] = t[2];
        for (int q = 0; q < 8; ++q) diag[4 + q] = t[3 + q];
        for (int q = 12; q < 16; ++q) diag[q] = 0.0;
    }
}

// ------------------------------------------------------------------ test-hook kernels
__global__ void k_extract_perm(const double* __restrict__ wsv, int n, int32_t* __restrict__ perm)
{
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p < n) {
        double x, y, z, w;
        ld256(wsv + 4 * p, x, y, z, w);
        perm[p] = unpack_perm(w);
    }
}

// one CTA per cell; pair base = sum_{i<j} floor(N_i/2) computed in-block (test hook only)
__global__ void __launch_bounds__(256)
k_pairs(const int32_t* __restrict__ off, int M, uint32_t cell_base, uint32_t step, uint32_t s0,
        uint32_t s1, int32_t* __restrict__ out, int64_t max_pairs, int blocked)
{
    __shared__ int64_t red[8];
    __shared__ int32_t pi_sm[cc::kSmallCell];
    const int j = blockIdx.x;
    int64_t part = 0;
    for (int i = threadIdx.x; i < j; i += blockDim.x) part += (off[i + 1] - off[i]) / 2;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) part += __shfl_down_sync(0xFFFFFFFFu, part, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    int64_t pb = 0;
    for (int w = 0; w < 8; ++w) pb += red[w];
    const int32_t o = off[j], N = off[j + 1] - off[j];
    if (N < 2) return;
    const uint32_t G = cell_base + static_cast<uint32_t>(j);
    if (N <= cc::kSmallCell) {
        if (threadIdx.x < 32) {
            cc::small_cell_perm(static_cast<uint32_t>(N), G, step, s0, s1, threadIdx.x, pi_sm);
            for (int k = threadIdx.x; k < N / 2; k += 32) {
                const int64_t g = pb + k;
                if (g < max_pairs) {
                    out[2 * g] = o + pi_sm[2 * k];
                    out[2 * g + 1] = o + pi_sm[2 * k + 1];
                }
            }
        }
        return;
    }
    if (blocked && N > cc::kBlock) {
        // R1b computed from its definition pair by pair (test hook: no segment table)
        const uint32_t Sf = static_cast<uint32_t>(N) / cc::kSeg;
        const cc::Feistel fs = cc::make_feistel(Sf > 1 ? Sf : 2u, cc::philox4x32_10(cc::U4{0u, G, step, 5u}, s0, s1));
        for (int k = threadIdx.x; k < N / 2; k += blockDim.x) {
            const int64_t g = pb + k;
            if (g >= max_pairs) continue;
#pragma unroll 1
            for (int m = 0; m < 2; ++m) {
                const uint32_t q = 2u * k + m, b = q / cc::kBlock, r = q % cc::kBlock;
                const uint32_t nb = min(static_cast<uint32_t>(N) - b * cc::kBlock, static_cast<uint32_t>(cc::kBlock));
                uint32_t u;
                if (nb > static_cast<uint32_t>(cc::kSmallCell))
                    u = cc::feistel_pi(cc::make_feistel(nb, cc::philox4x32_10(cc::U4{b, G, step, 1u}, s0, s1)), r);
                else
                    u = cc::small_select(nb, r, G, step, s0, s1, b * (cc::kBlock / 4), 2u);
                const uint32_t p = b * cc::kBlockSegs + u / cc::kSeg;     // position in the segment sequence
                uint32_t seg0;
                if (p >= Sf) seg0 = Sf * cc::kSeg;                          // the tail segment
                else if (Sf <= static_cast<uint32_t>(cc::kSmallCell)) seg0 = cc::small_select(Sf, p, G, step, s0, s1, 0u, 6u) * cc::kSeg;
                else seg0 = cc::feistel_pi(fs, p) * cc::kSeg;
                out[2 * g + m] = o + static_cast<int32_t>(seg0 + u % cc::kSeg);
            }
        }
        return;
    }
    const cc::U4 keys = cc::philox4x32_10(cc::U4{0u, G, step, 1u}, s0, s1);
    const cc::Feistel f = cc::make_feistel(static_cast<uint32_t>(N), keys);
    for (int k = threadIdx.x; k < N / 2; k += blockDim.x) {
        const int64_t g = pb + k;
        if (g < max_pairs) {
            out[2 * g] = o + static_cast<int32_t>(cc::feistel_pi(f, 2u * k));
            out[2 * g + 1] = o + static_cast<int32_t>(cc::feistel_pi(f, 2u * k + 1u));
        }
    }
}

__global__ void k_philox(const uint32_t* __restrict__ ctr, uint32_t s0, uint32_t s1,
                         uint32_t* __restrict__ out, int64_t m)
{
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= m) return;
    const cc::U4 r = cc::philox4x32_10(cc::U4{ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]}, s0, s1);
    out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
}

__global__ void k_ppnd16(const double* __restrict__ u, double* __restrict__ z, int64_t m)
{
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < m) z[i] = cc::ppnd16(u[i]);
}

__global__ void k_ta_pairs(double* __restrict__ va, double* __restrict__ vb, const double* __restrict__ C,
                           const double* __restrict__ u1, const double* __restrict__ u2, int64_t m)
{
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= m) return;
    double ax = va[i], ay = va[m + i], az = va[2 * m + i];
    double bx = vb[i], by = vb[m + i], bz = vb[2 * m + i];
    cc::ta_update(ax, ay, az, bx, by, bz, C[i], u1[i], u2[i]);
    va[i] = ax; va[m + i] = ay; va[2 * m + i] = az;
    vb[i] = bx; vb[m + i] = by; vb[2 * m + i] = bz;
}

// P2C hook: one CTA per cell, shifted single pass (ref = first slot), fixed order.
__global__ void __launch_bounds__(256)
k_moments(const double* __restrict__ v, int64_t ldv, const int32_t* __restrict__ off, int M, MomConst mc,
          double* __restrict__ out)
{
    __shared__ double red[8][6];
    const int j = blockIdx.x;
    const int32_t a = off[j], b = off[j + 1], N = b - a;
    double* o = out + static_cast<int64_t>(j) * CC_MOMENTS_LEN;
    if (N <= 0) {
        if (threadIdx.x < CC_MOMENTS_LEN) o[threadIdx.x] = 0.0;
        return;
    }
    const double rx = v[a], ry = v[ldv + a], rz = v[2 * ldv + a];
    double s[6] = {0, 0, 0, 0, 0, 0};
    for (int32_t p = a + threadIdx.x; p < b; p += blockDim.x) {
        const double dx = v[p] - rx, dy = v[ldv + p] - ry, dz = v[2 * ldv + p] - rz;
        s[0] += dx; s[1] += dy; s[2] += dz;
        s[3] += dx * dx; s[4] += dy * dy; s[5] += dz * dz;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) s[q] += __shfl_down_sync(0xFFFFFFFFu, s[q], d);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int q = 0; q < 6; ++q) red[threadIdx.x >> 5][q] = s[q];
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[6] = {0, 0, 0, 0, 0, 0};
        for (int w = 0; w < 8; ++w)
            for (int q = 0; q < 6; ++q) t[q] += red[w][q];
        const double V = mc.volume_arr ? mc.volume_arr[j] : mc.volume;
        moments_from_sums(t, static_cast<double>(N), rx, ry, rz, V, mc, o);
    }
}

__global__ void k_gather(const double* __restrict__ v, int64_t ldv, const int32_t* __restrict__ cell,
                         const int32_t* __restrict__ idx, int64_t m, int32_t shift, double* __restrict__ vo,
                         int64_t ldo, int32_t* __restrict__ co)
{
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx[p];
        vo[p] = v[i];
        vo[ldo + p] = v[ldv + i];
        vo[2 * ldo + p] = v[2 * ldv + i];
        const int32_t c = cell[i];
        co[p] = (c >= 0) ? c - shift : -1;
    }
}

// ------------------------------------------------------------------ NEXT f4: atomic P2C (S3a)
// The paper's particle-to-cell kernel: a block reduction over
// UNSORTED particles by atomics, with each cell split into `sub` auxiliary
// sub-bins omega_jm to spread atomic congestion, then V^j = sum_m V^jm.
// Raw sums per (cell, sub-bin): {N, sum v_x, v_y, v_z, sum v_x^2, v_y^2, v_z^2};
// the sub-bin of particle p is (p / 32) mod sub (one per warp-aligned group of
// 32 particles).  fp64 global atomics (red.add.f64): results agree with a
// sequential sum to rounding, not bitwise (order).  A warp whose 32 particles
// all sit in one cell (cell-sorted input) first reduces them with shuffles and
// issues one set of 7 atomics instead of 32 — the congestion the paper's
// sub-bins address, removed at the source.
constexpr int kRaw = 7;

__global__ void __launch_bounds__(256)
k_p2c_atomic(const double* __restrict__ v, int64_t ldv, const int32_t* __restrict__ cell, int64_t n, int M, int sub,
             double* __restrict__ acc)
{
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t g = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; g * 32 < n; g += nwarps) {
        const int64_t p = g * 32 + lane;
        const int32_t j = p < n ? __ldg(cell + p) : -1;
        const bool ok = j >= 0 && j < M;
        double x = 0.0, y = 0.0, z = 0.0;
        if (ok) { x = __ldg(v + p); y = __ldg(v + ldv + p); z = __ldg(v + 2 * ldv + p); }
        const int32_t j0 = __shfl_sync(0xFFFFFFFFu, j, 0);
        const int64_t bin = g % sub;
        if (__all_sync(0xFFFFFFFFu, ok && j == j0)) {
            double r[kRaw] = {1.0, x, y, z, x * x, y * y, z * z};
#pragma unroll
            for (int q = 0; q < kRaw; ++q)
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) r[q] += __shfl_xor_sync(0xFFFFFFFFu, r[q], d);
            if (lane < kRaw) {
                double val = r[0];
#pragma unroll
                for (int q = 1; q < kRaw; ++q) val = (lane == q) ? r[q] : val;
                atomicAdd(acc + (static_cast<int64_t>(j0) * sub + bin) * kRaw + lane, val);
            }
        } else if (ok) {
            double* a = acc + (static_cast<int64_t>(j) * sub + bin) * kRaw;
            atomicAdd(a + 0, 1.0);
            atomicAdd(a + 1, x);
            atomicAdd(a + 2, y);
            atomicAdd(a + 3, z);
            atomicAdd(a + 4, x * x);
            atomicAdd(a + 5, y * y);
            atomicAdd(a + 6, z * z);
        }
    }
}

// thread per cell: raw[j] = sum over its sub-bins in fixed order
__global__ void k_p2c_reduce(const double* __restrict__ acc, int M, int sub, double* __restrict__ raw)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    double s[kRaw] = {0, 0, 0, 0, 0, 0, 0};
    for (int m = 0; m < sub; ++m)
#pragma unroll
        for (int q = 0; q < kRaw; ++q) s[q] += acc[(static_cast<int64_t>(j) * sub + m) * kRaw + q];
#pragma unroll
    for (int q = 0; q < kRaw; ++q) raw[static_cast<int64_t>(j) * kRaw + q] = s[q];
}

// thread per cell: raw sums (possibly all-reduced over replicated ranks) -> moments [M][7]
__global__ void k_p2c_moments(const double* __restrict__ raw, int M, MomConst mc, double* __restrict__ out)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const double* r = raw + static_cast<int64_t>(j) * kRaw;
    double* o = out + static_cast<int64_t>(j) * CC_MOMENTS_LEN;
    if (!(r[0] > 0.0)) {
#pragma unroll
        for (int q = 0; q < CC_MOMENTS_LEN; ++q) o[q] = 0.0;
        return;
    }
    const double V = mc.volume_arr ? mc.volume_arr[j] : mc.volume;
    moments_from_sums(r + 1, r[0], 0.0, 0.0, 0.0, V, mc, o);
}

// ------------------------------------------------------------------ NEXT f3: recombination C5
// Table 4 RS0-RS5 on a collision call's cell-sorted output, one CTA
// per cell.  The paper builds per-cell catalyte lists with atomics over
// unsorted particles (RS1, "the majority of time") and pops them atomically
// (RS3); here the particles already sit cell-major in a fresh random order
// (the pair order, R14), so RS1 is a block scan and the matching is the
// deterministic rank match of R26: i-th primary <-> i-th non-primary.
constexpr int kRecWin = 1024;   // primaries matched per pass over the cell (windowed path)
constexpr int kRecList = 512;   // primaries per warp held by the one-pass list path

// RS4 + RS5 for primary at a and its catalyte at c (R27, R28): the catalyte keeps its direction
// and takes the primary's kinetic energy plus the binding energy; the primary dies (a marker that
// keeps the sort key until k_recombine_finish)
__device__ __forceinline__ void rc_pair(double* __restrict__ v, int64_t ldv, int32_t* __restrict__ cell, int64_t a,
                                        int64_t c, double vb2, int j)
{
    const double px = v[a], py = v[ldv + a], pz = v[2 * ldv + a];
    const double cx = v[c], cy = v[ldv + c], cz = v[2 * ldv + c];
    const double c2 = __dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz));
    const double p2 = __dadd_rn(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)), __dmul_rn(pz, pz));
    const double t2 = __dadd_rn(__dadd_rn(c2, p2), vb2);
    double ux = cx, uy = cy, uz = cz, s2 = c2;
    if (c2 == 0.0) { ux = px; uy = py; uz = pz; s2 = p2; }
    if (s2 == 0.0) { ux = 1.0; uy = 0.0; uz = 0.0; s2 = 1.0; }
    const double f = __dsqrt_rn(__ddiv_rn(t2, s2));
    v[c] = __dmul_rn(ux, f); v[ldv + c] = __dmul_rn(uy, f); v[2 * ldv + c] = __dmul_rn(uz, f);
    cell[a] = -2 - j;
}

__device__ __forceinline__ bool rc_primary(int32_t q, uint32_t G, uint32_t step, uint32_t s0, uint32_t s1, double prob)
{
    const cc::U4 x = cc::philox4x32_10(cc::U4{static_cast<uint32_t>(q), G, step, 4u}, s0, s1);
    return cc::u01(x.x, x.y) < prob;
}

// Search key of a slot of the cell-sorted collision output.  A primary killed by this
// call is first marked -2 - j (not -1): the marker keeps the key j, so the binary
// searches of CTAs that start later still see a sorted array (writing -1
// directly let a late CTA's search land on a killed slot of a lower cell).
// k_recombine_finish turns the markers into -1 after every CTA is done.
__device__ __forceinline__ int32_t rc_key(int32_t c, int M)
{
    if (c <= -2) return -2 - c;
    return (c < 0 || c >= M) ? M : c;
}

__global__ void __launch_bounds__(256)
k_recombine(double* __restrict__ v, int64_t ldv, int32_t* __restrict__ cell, int64_t n, int M, uint32_t cell_base,
            const double* __restrict__ prob, double vb2, uint32_t step, uint32_t s0, uint32_t s1,
            unsigned long long* __restrict__ stats)
{
    __shared__ int64_t s_lo, s_hi;
    __shared__ int32_t s_wsum[8];
    __shared__ int32_t ppos[kRecWin], cpos[kRecWin];
    __shared__ int32_t plist[8][kRecList];          // per-warp primaries (list path)
    __shared__ int32_t prim[8 * kRecList];          // all primaries of the cell, position order
    const int j = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) {             // the cell's slot range: binary search in the cell-sorted ids
        int64_t a = 0, b = n;
        while (a < b) { const int64_t m = (a + b) >> 1; if (rc_key(cell[m], M) < j) a = m + 1; else b = m; }
        s_lo = a;
        b = n;
        while (a < b) { const int64_t m = (a + b) >> 1; if (rc_key(cell[m], M) <= j) a = m + 1; else b = m; }
        s_hi = a;
    }
    __syncthreads();
    const int64_t lo = s_lo;
    const int32_t N = static_cast<int32_t>(s_hi - lo);
    const double pr = prob[j];
    if (N == 0 || !(pr > 0.0)) return;
    const uint32_t G = cell_base + static_cast<uint32_t>(j);
    // RS0: the primaries.  Warp w draws the contiguous positions [w C, (w+1) C) and appends its
    // primaries in position order to its list (so the lists, in warp order, are the cell's
    // primaries in position order); a list that overflows sends the cell to the windowed path
    const int32_t C = (N + 7) / 8;
    const int32_t q0w = min(w * C, N), q1w = min(q0w + C, N);
    int32_t np = 0;
    for (int32_t q = q0w + lane; q - lane < q1w; q += 32) {
        const bool isp = q < q1w && rc_primary(q, G, step, s0, s1, pr);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, isp);
        const int32_t at = np + __popc(bal & ((1u << lane) - 1u));
        if (isp && at < kRecList) plist[w][at] = q;
        np += __popc(bal);
    }
    if (lane == 0) s_wsum[w] = np;
    __syncthreads();
    int32_t P = 0, before = 0, longest = 0;
    for (int i = 0; i < 8; ++i) {
        before += (i < w) ? s_wsum[i] : 0;
        P += s_wsum[i];
        longest = max(longest, s_wsum[i]);
    }
    const int32_t m = min(P, N - P);
    if (longest <= kRecList) {
        // list path: prim[k] = k-th primary position; the i-th catalyte (non-primary in position
        // order) is c_i = i + #{k : prim[k] - k <= i}, found by binary search on the
        // non-decreasing prim[k] - k
        for (int32_t t = lane; t < np; t += 32) prim[before + t] = plist[w][t];
        __syncthreads();
        for (int32_t i = threadIdx.x; i < m; i += blockDim.x) {
            int32_t a = 0, b = P;                 // first k with prim[k] - k > i
            while (a < b) { const int32_t h = (a + b) >> 1; if (prim[h] - h <= i) a = h + 1; else b = h; }
            rc_pair(v, ldv, cell, lo + prim[i], lo + i + a, vb2, j);
        }
    } else {
    // RS1-RS5 in windows of kRecWin ranks: positions of primaries / catalytes of rank in the window
    for (int32_t w0 = 0; w0 < m; w0 += kRecWin) {
        __syncthreads();
        int32_t base = 0;               // primaries before the current 256-position chunk
        for (int32_t q0 = 0; q0 < N; q0 += blockDim.x) {
            const int32_t q = q0 + threadIdx.x;
            const bool isp = q < N && rc_primary(q, G, step, s0, s1, pr);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, isp);
            __syncthreads();
            if (lane == 0) s_wsum[w] = __popc(bal);
            __syncthreads();
            int32_t before = base;
            for (int i = 0; i < w; ++i) before += s_wsum[i];
            const int32_t rp = before + __popc(bal & ((1u << lane) - 1u));   // primary rank of q
            if (q < N) {
                const int32_t r = isp ? rp : q - rp;                           // catalyte rank = q - rp
                if (r >= w0 && r < w0 + kRecWin && r < m) (isp ? ppos : cpos)[r - w0] = q;
            }
            for (int i = 0; i < 8; ++i) base += s_wsum[i];
        }
        __syncthreads();
        for (int32_t i = threadIdx.x; i < min(kRecWin, m - w0); i += blockDim.x)
            rc_pair(v, ldv, cell, lo + ppos[i], lo + cpos[i], vb2, j);
    }
    }
    if (threadIdx.x == 0) {
        atomicAdd(stats + 0, static_cast<unsigned long long>(m));
        atomicAdd(stats + 1, static_cast<unsigned long long>(P - m));
        atomicAdd(stats + 2, static_cast<unsigned long long>(P));
    }
}

// second pass: the kill markers of k_recombine -> -1 (R28: dead)
__global__ void k_recombine_finish(int32_t* __restrict__ cell, int64_t n)
{
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (cell[i] <= -2) cell[i] = -1;
}

// ------------------------------------------------------------------ NEXT f2: push (S2b + S2c)
// Thread per particle (grid-stride).  Every product and sum is an explicitly
// rounded IEEE operation (__dmul_rn / __dadd_rn / __ddiv_rn), as in the
// oracle (compiled without FMA contraction), so the result is bit-exact.
// HAS_E = false (field-free): v is read but not rewritten (v + 0 == v).
// Only the position rows a < DIMS are read and written.
template <bool HAS_E, int DIMS>
__global__ void __launch_bounds__(256)
k_push(const double* __restrict__ xin, int64_t ldxi, const int32_t* __restrict__ perm, double* __restrict__ xo,
       int64_t ldxo, double* __restrict__ v, int64_t ldv, int32_t* __restrict__ cell, int64_t n, PushGrid g,
       const double* __restrict__ E, int64_t ldE, double qm, double dt)
{
    const double kick = __dmul_rn(dt, qm);
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t src = perm ? static_cast<int64_t>(__ldg(perm + p)) : p;
        const int32_t j = cell[p];
        double x[DIMS];
#pragma unroll
        for (int a = 0; a < DIMS; ++a) x[a] = __ldg(xin + a * ldxi + src);
        if (j < 0) {
#pragma unroll
            for (int a = 0; a < DIMS; ++a) xo[a * ldxo + p] = x[a];
            continue;
        }
        double vn[DIMS];
#pragma unroll
        for (int c = 0; c < (HAS_E ? 3 : DIMS); ++c) {
            double vc = v[c * ldv + p];
            if (HAS_E) {
                vc = __dadd_rn(vc, __dmul_rn(kick, __ldg(E + c * ldE + j)));
                v[c * ldv + p] = vc;
            }
            if (c < DIMS) vn[c] = vc;
        }
        bool alive = true;
        int64_t G = 0, stride = 1;
#pragma unroll
        for (int a = 0; a < DIMS; ++a) xo[a * ldxo + p] = drift_axis(g, a, x[a], vn[a], dt, alive, G, stride);
        cell[p] = alive ? static_cast<int32_t>(G) : -1;
    }
}

template <bool HAS_E>
void launch_push(unsigned blocks, cudaStream_t st, const double* x_in, int64_t ldx_in, const int32_t* perm,
                 double* x_out, int64_t ldx_out, double* v, int64_t ldv, int32_t* cell, int64_t n, const PushGrid& g,
                 const double* E, int64_t ldE, double qm, double dt)
{
    if (g.dims == 1)
        k_push<HAS_E, 1><<<blocks, 256, 0, st>>>(x_in, ldx_in, perm, x_out, ldx_out, v, ldv, cell, n, g, E, ldE, qm, dt);
    else if (g.dims == 2)
        k_push<HAS_E, 2><<<blocks, 256, 0, st>>>(x_in, ldx_in, perm, x_out, ldx_out, v, ldv, cell, n, g, E, ldE, qm, dt);
    else
        k_push<HAS_E, 3><<<blocks, 256, 0, st>>>(x_in, ldx_in, perm, x_out, ldx_out, v, ldv, cell, n, g, E, ldE, qm, dt);
}

__global__ void k_step_advance(uint32_t* step, uint32_t inc) { *step += inc; }

__global__ void k_owner(const int32_t* __restrict__ cell, int64_t n, const int32_t* __restrict__ bounds, int P,
                        int32_t* __restrict__ owner)
{
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t c = cell[i];
        int32_t r = -1;
        if (c >= bounds[0] && c < bounds[P]) {
            int lo = 0, hi = P;       // bounds[lo] <= c < bounds[hi]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (bounds[mid] <= c) lo = mid; else hi = mid;
            }
            r = lo;
        }
        owner[i] = r;
    }
}

__global__ void k_coulomb_log(const double* __restrict__ m, int M, double* __restrict__ out)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const double* r = m + static_cast<int64_t>(j) * CC_MOMENTS_LEN;
    const double n_cm = r[0] * 1e-6;
    const double T = (r[4] + r[5] + r[6]) / 3.0;
    double l = 2.0;
    if (n_cm > 0.0 && T > 0.0) {
        const double lt = log(T);
        l = 23.5 - (0.5 * log(n_cm) - 1.25 * lt) - sqrt(1e-5 + (lt - 2.0) * (lt - 2.0) / 16.0);
        if (!(l >= 2.0)) l = 2.0;
    }
    out[j] = l;
}

__global__ void k_diag_sum_ranks(const double* __restrict__ g, int P, double* __restrict__ out)
{
    const int q = threadIdx.x;
    if (q >= CC_DIAG_LEN) return;
    double s = 0.0;
    for (int r = 0; r < P; ++r) s += g[r * CC_DIAG_LEN + q];
    out[q] = s;
}

// ------------------------------------------------------------------ host helpers
bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

bool overlaps(const void* a, size_t na, const void* b, size_t nb)
{
    if (!a || !b || na == 0 || nb == 0) return false;
    const char* pa = static_cast<const char*>(a);
    const char* pb = static_cast<const char*>(b);
    return pa < pb + nb && pb < pa + na;
}

int launch_ok()
{
    return cudaGetLastError() == cudaSuccess ? CC_OK : CC_ECUDA;
}

// Opt a kernel into `bytes` of dynamic shared memory (above the 48 KB default).
template <typename K>
int want_smem(K kernel, size_t bytes)
{
    // (static shared memory counts against the 48 KB default too, so always opt in)
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)) !=
        cudaSuccess) {
        cudaGetLastError();
        return CC_ECUDA;
    }
    return CC_OK;
}

void mark(void* const* ev, int i, cudaStream_t st)
{
    if (ev && ev[i]) cudaEventRecord(static_cast<cudaEvent_t>(ev[i]), st);
}

int run_binning(const double* v_in, int64_t ldv, const int32_t* cell_in, int n, int M, const Layout& L,
                void* ws, const CellConst& k, uint32_t cell_base, uint32_t step, uint64_t seed,
                cudaStream_t st, void* const* ev, bool allow_sorted_skip, const uint32_t* step_dev = nullptr,
                bool blocked = false)
{
    // R1b: one k_collide_large CTA per block of kBlock slots (kBlock / 2 pair items); R1: L.chunk
    const int chunk = blocked ? cc::kBlock / 2 : L.chunk;
    int32_t* err = at<int32_t>(ws, L.o_err);
    mark(ev, 0, st);                     // the timed region starts before the flag reset
    if (cudaMemsetAsync(err + 1, 0, 2 * sizeof(int32_t), st) != cudaSuccess) return CC_ECUDA;   // unsorted flag, descents
    int32_t* tcount = at<int32_t>(ws, L.o_tcount);
    int32_t* cnt = at<int32_t>(ws, L.o_cnt);
    int32_t* off = at<int32_t>(ws, L.o_off);
    int32_t* chunk_off = at<int32_t>(ws, L.o_chunk);
    double* Cj = at<double>(ws, L.o_C);
    cc::U4* keys = at<cc::U4>(ws, L.o_keys);
    double* wsv = at<double>(ws, L.o_wsv);
    const int M1 = M + 1;
    const size_t smem = sizeof(int32_t) * M1 + sizeof(uint32_t) * static_cast<size_t>(L.W) * ((M1 + 1) / 2);
    int rc = want_smem(k_count, sizeof(int32_t) * M1);
    if (!rc) rc = want_smem(k_scatter<true>, smem);
    if (!rc) rc = want_smem(k_scatter<false>, smem);
    if (rc) return rc;
    const int32_t* skip = allow_sorted_skip ? err : nullptr;
    const int index_modes = (allow_sorted_skip && blocked) ? 1 : 0;
    k_count<<<L.T, kCountThreads, sizeof(int32_t) * M1, st>>>(cell_in, n, M, L.tile, tcount, err);
    mark(ev, 1, st);
    k_scan_tiles<<<(M1 + 31) / 32, dim3(32, kScanRows), 0, st>>>(tcount, L.T, M1, cnt);
    k_scan_cells<<<1, 1024, 0, st>>>(cnt, M, off, chunk_off, chunk);
    k_cell_setup<<<M, kSetupThreads, 0, st>>>(cnt, chunk_off, M, at<int4>(ws, L.o_chunkcell), Cj, keys, k,
                                                   cell_base, step, static_cast<uint32_t>(seed),
                                                   static_cast<uint32_t>(seed >> 32), step_dev, off, chunk,
                                                   blocked ? at<int32_t>(ws, L.o_seg) : nullptr);
    mark(ev, 2, st);
    if (v_in)
        k_scatter<true><<<L.T, 32 * L.W, smem, st>>>(v_in, ldv, cell_in, n, M, L.W, L.sub, tcount, off, wsv, skip,
                                                     index_modes);
    else
        k_scatter<false><<<L.T, 32 * L.W, smem, st>>>(nullptr, 0, cell_in, n, M, L.W, L.sub, tcount, off, wsv, skip,
                                                      0);
    return launch_ok();
}

CellConst cell_const(const cc_params& p, double dt)
{
    CellConst k;
    const double e2 = p.charge * p.charge;
    const double mr = 0.5 * p.mass;
    k.K = e2 * e2 * dt / (8.0 * M_PI * p.eps0 * p.eps0 * mr * mr);
    k.weight = p.weight;
    k.volume = p.cell_volume;
    k.volume_arr = p.cell_volume_arr;
    k.ln_lambda = p.ln_lambda;
    k.ln_lambda_arr = p.ln_lambda_arr;
    return k;
}

template <bool BLOCKED>
int launch_collide_large(const CollideArgs& A, unsigned grid, bool nanbu, bool push, cudaStream_t st)
{
    int rc = want_smem(k_collide_large<false, false, BLOCKED>, kCollideSmem);
    if (!rc) rc = want_smem(k_collide_large<true, false, BLOCKED>, kCollideSmem);
    if (!rc) rc = want_smem(k_collide_large<false, true, BLOCKED>, kCollideSmem);
    if (!rc) rc = want_smem(k_collide_large<true, true, BLOCKED>, kCollideSmem);
    if (rc) return rc;
    if (push) {
        if (nanbu) k_collide_large<true, true, BLOCKED><<<grid, kCollideThreads, kCollideSmem, st>>>(A);
        else k_collide_large<false, true, BLOCKED><<<grid, kCollideThreads, kCollideSmem, st>>>(A);
    } else {
        if (nanbu) k_collide_large<true, false, BLOCKED><<<grid, kCollideThreads, kCollideSmem, st>>>(A);
        else k_collide_large<false, false, BLOCKED><<<grid, kCollideThreads, kCollideSmem, st>>>(A);
    }
    return CC_OK;
}

bool finite_pos(double x) { return std::isfinite(x) && x > 0.0; }

// Host-side argument checks of coulomb_collide (scalars and cc_params), shared with the
// host-buffer entry so that it rejects bad arguments before enqueueing any copy.
int check_call(const cc_params& p, int64_t n, int32_t cells, int64_t ldv, double dt, uint64_t step)
{
    if (n < 0 || cells < 1 || ldv < n || !(dt > 0.0) || step >= (1ull << 32)) return CC_EINVAL;
    if (n >= (1ll << 31) || cells > CC_MAX_CELLS) return CC_ECOUNT;
    if (!finite_pos(p.mass) || !finite_pos(p.charge) || !finite_pos(p.eps0) || !std::isfinite(p.weight) ||
        p.weight < 0.0 || (!p.cell_volume_arr && !finite_pos(p.cell_volume)) ||
        (!p.ln_lambda_arr && !std::isfinite(p.ln_lambda)) ||
        (p.flags & ~(CC_ODD_TRIPLET | CC_NANBU | CC_PRESERVE_ORDER | CC_CELL_UNIFORM)) != 0)
        return CC_EINVAL;
    if (p.push) {                            // fused push (NEXT f2): same checks as cc_push
        const cc_push_params& q = *p.push;
        if (!q.grid || q.grid->dims < 1 || q.grid->dims > 3 || !std::isfinite(q.q_over_m) ||
            (p.flags & CC_PRESERVE_ORDER) || (n > 0 && (!q.x_in || !q.x_out)) || q.ldx_in < n || q.ldx_out < n ||
            (q.E && q.ldE < cells))
            return CC_EINVAL;
        int64_t total = 1;
        for (int a = 0; a < q.grid->dims; ++a) {
            if (q.grid->n[a] < 1 || !finite_pos(q.grid->d[a])) return CC_EINVAL;
            total *= q.grid->n[a];
        }
        if (total >= (1ll << 31)) return CC_EINVAL;
    }
    return CC_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

void cc_default_params(cc_params* p)
{
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->mass = 9.1093837015e-31;
    p->charge = 1.602176634e-19;
    p->eps0 = 8.8541878128e-12;
    p->weight = 1.0;
    p->cell_volume = 1.0;
    p->ln_lambda = 10.0;
}

size_t cc_workspace_bytes(int64_t n, int32_t cells)
{
    if (n < 0 || cells < 1) return 0;
    return make_layout(n, cells).total;
}

const char* cc_strerror(int code)
{
    switch (code) {
        case CC_OK: return "ok";
        case CC_EINVAL: return "invalid argument";
        case CC_EWORKSPACE: return "workspace too small or misaligned";
        case CC_ECUDA: return "CUDA launch failed";
        case CC_ECELL: return "cell id outside [-1, cells)";
        case CC_ECOUNT: return "n >= 2^31 or cells > CC_MAX_CELLS";
        case CC_ENCCL: return "NCCL error";
        default: return "unknown error";
    }
}

int coulomb_collide(const double* v_in, int64_t ldv, const int32_t* cell_in, double* v_out,
                    int32_t* cell_out, int32_t* perm_out, int64_t n, int32_t cells, uint32_t cell_base,
                    double dt, const cc_params* params, uint64_t seed, uint64_t step,
                    double* moments_out, double* diag_out, void* workspace, size_t workspace_bytes,
                    void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    cc_params p;
    if (params) p = *params; else cc_default_params(&p);
    if (const int rc = check_call(p, n, cells, ldv, dt, step)) return rc;
    if (!workspace || !aligned(workspace, 256)) return CC_EWORKSPACE;
    const Layout L = make_layout(n, cells);
    if (workspace_bytes < L.total) return CC_EWORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int M = cells;
    if (n == 0) {
        if (moments_out && cudaMemsetAsync(moments_out, 0, sizeof(double) * CC_MOMENTS_LEN * M, st) != cudaSuccess)
            return CC_ECUDA;
        if (diag_out && cudaMemsetAsync(diag_out, 0, sizeof(double) * CC_DIAG_LEN, st) != cudaSuccess)
            return CC_ECUDA;
        return CC_OK;
    }
    if (!v_in || !cell_in || !v_out || !cell_out) return CC_EINVAL;
    if (!aligned(v_in, 16) || !aligned(v_out, 16) || !aligned(cell_in, 4) || !aligned(cell_out, 4))
        return CC_EINVAL;
    const size_t vbytes = sizeof(double) * static_cast<size_t>(2 * ldv + n);
    if (overlaps(v_in, vbytes, v_out, vbytes) || overlaps(cell_in, 4 * n, cell_out, 4 * n) ||
        overlaps(v_out, vbytes, cell_out, 4 * n) || (perm_out && overlaps(perm_out, 4 * n, v_out, vbytes)) ||
        (perm_out && overlaps(perm_out, 4 * n, cell_out, 4 * n)))
        return CC_EINVAL;
    // the workspace is written by every kernel: it may overlap no input or output
    if (overlaps(workspace, L.total, v_out, vbytes) || overlaps(workspace, L.total, v_in, vbytes) ||
        overlaps(workspace, L.total, cell_in, 4 * n) || overlaps(workspace, L.total, cell_out, 4 * n) ||
        (perm_out && overlaps(workspace, L.total, perm_out, 4 * n)) ||
        (moments_out && overlaps(workspace, L.total, moments_out, sizeof(double) * CC_MOMENTS_LEN * cells)) ||
        (diag_out && overlaps(workspace, L.total, diag_out, sizeof(double) * CC_DIAG_LEN)))
        return CC_EINVAL;

    const CellConst k = cell_const(p, dt);
    const int nn = static_cast<int>(n);
    void* const* ev = p.stage_events;
    const bool blocked = (p.flags & CC_CELL_UNIFORM) == 0;     // R1b (default) or R1
    int rc = run_binning(v_in, ldv, cell_in, nn, M, L, workspace, k, cell_base, static_cast<uint32_t>(step), seed,
                         st, ev, true, p.step_dev, blocked);
    if (rc) return rc;

    CollideArgs A;
    A.wsv = at<double>(workspace, L.o_wsv);
    A.cellref = at<double>(workspace, L.o_ref);
    A.cnt = at<int32_t>(workspace, L.o_cnt);
    A.off = at<int32_t>(workspace, L.o_off);
    A.chunk_off = at<int32_t>(workspace, L.o_chunk);
    A.chunk_cell = at<int4>(workspace, L.o_chunkcell);
    A.Cj = at<double>(workspace, L.o_C);
    A.keys = at<cc::U4>(workspace, L.o_keys);
    A.v_out = v_out;
    A.ldv = ldv;
    A.cell_out = cell_out;
    const bool preserve = (p.flags & CC_PRESERVE_ORDER) != 0;
    // CC_PRESERVE_ORDER: the kernels below produce the default (pair-ordered) output, which
    // k_unpermute / k_unpack then put back in input order; perm is needed for that even
    // when the caller does not ask for it
    int32_t* perm_pair = perm_out ? perm_out : (preserve ? at<int32_t>(workspace, L.o_perm) : nullptr);
    A.perm_out = perm_pair;
    A.recs = at<double>(workspace, L.o_recs);
    A.small_recs = at<double>(workspace, L.o_small);
    A.M = M;
    A.cell_base = cell_base;
    A.step = static_cast<uint32_t>(step);
    A.step_dev = p.step_dev;
    A.chunk = blocked ? cc::kBlock / 2 : L.chunk;
    A.blocked = blocked ? 1 : 0;
    A.index_modes = blocked ? 1 : 0;
    A.flags = at<int32_t>(workspace, L.o_err);
    A.n = nn;
    A.v_in = v_in;
    A.ldvi = ldv;
    A.vec16 = aligned(v_in, 16) && (ldv % 2 == 0);
    A.seg = at<int32_t>(workspace, L.o_seg);
    A.push = 0;
    A.E = nullptr; A.x_in = nullptr; A.x_out = nullptr;
    A.ldE = A.ldxi = A.ldxo = 0;
    A.kick = A.dt = 0.0;
    if (p.push) {
        const cc_push_params& q = *p.push;
        A.push = 1;
        A.pg.dims = q.grid->dims;
        A.pg.periodic = q.grid->periodic;
        for (int a = 0; a < 3; ++a) {
            A.pg.n[a] = a < q.grid->dims ? q.grid->n[a] : 1;
            A.pg.d[a] = a < q.grid->dims ? q.grid->d[a] : 1.0;
            A.pg.L[a] = static_cast<double>(A.pg.n[a]) * A.pg.d[a];
        }
        A.E = q.E; A.ldE = q.ldE;
        A.kick = dt * q.q_over_m;            // = __dmul_rn(dt, qm) of k_push (host IEEE double product)
        A.dt = dt;
        A.x_in = q.x_in; A.ldxi = q.ldx_in;
        A.x_out = q.x_out; A.ldxo = q.ldx_out;
    }
    A.s0 = static_cast<uint32_t>(seed);
    A.s1 = static_cast<uint32_t>(seed >> 32);
    A.model = p.flags & (CC_ODD_TRIPLET | CC_NANBU);
    A.trec = at<double>(workspace, L.o_trec);
    A.pair_vec = aligned(v_out, 16) && (ldv % 2 == 0) && aligned(cell_out, 8) && (!perm_out || aligned(perm_out, 8));

    mark(ev, 3, st);
    k_collide_small<<<(M + 7) / 8, 256, 0, st>>>(A);
    {
        const unsigned grid = static_cast<unsigned>(L.max_chunks);
        const bool nb = (A.model & CC_NANBU) != 0;
        if (blocked) rc = launch_collide_large<true>(A, grid, nb, A.push != 0, st);
        else rc = launch_collide_large<false>(A, grid, nb, A.push != 0, st);
        if (rc) return rc;
    }
    if (A.model & CC_ODD_TRIPLET) k_triplets<<<(M + 255) / 256, 256, 0, st>>>(A);
    k_copy_dead<<<148 * 4, 256, 0, st>>>(A, nn);
    if (preserve) {
        const unsigned g = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
        k_unpermute<<<g, 256, 0, st>>>(v_out, ldv, cell_out, perm_pair, n, at<double>(workspace, L.o_wsv));
        k_unpack<<<g, 256, 0, st>>>(A.wsv, n, v_out, ldv, cell_out, perm_out);
    }

    MomConst mc{p.weight, p.cell_volume, p.cell_volume_arr, p.mass / p.charge};
    double* cellsum = at<double>(workspace, L.o_cellsum);
    mark(ev, 4, st);
    k_finalize_cells<<<(M + 7) / 8, 256, 0, st>>>(A.cnt, A.chunk_off, A.recs, A.small_recs, A.cellref,
                                                      (A.model & CC_ODD_TRIPLET) ? A.trec : nullptr, M, mc,
                                                      moments_out, cellsum);
    if (diag_out)
        k_finalize_diag<<<1, 1024, 0, st>>>(A.cnt, cellsum, M, diag_out);
    mark(ev, 5, st);
    return launch_ok();
}

// ---------------------------------------------------------------- host-buffer entry (end-to-end path)
namespace {
struct HostLayout {
    int64_t ldd = 0;   // device row stride (even, so the pair-vectorised stores apply)
    size_t o_vin = 0, o_cin = 0, o_vout = 0, o_cout = 0, o_perm = 0, o_mom = 0, o_diag = 0, o_ws = 0, total = 0;
};

HostLayout host_layout(int64_t n, int32_t cells)
{
    HostLayout H;
    H.ldd = std::max<int64_t>(2, n + (n & 1));
    size_t o = 0;
    H.o_vin = o;  o = align256(o + sizeof(double) * 3 * static_cast<size_t>(H.ldd));
    H.o_vout = o; o = align256(o + sizeof(double) * 3 * static_cast<size_t>(H.ldd));
    H.o_cin = o;  o = align256(o + sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(n, 1)));
    H.o_cout = o; o = align256(o + sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(n, 1)));
    H.o_perm = o; o = align256(o + sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(n, 1)));
    H.o_mom = o;  o = align256(o + sizeof(double) * CC_MOMENTS_LEN * static_cast<size_t>(cells));
    H.o_diag = o; o = align256(o + sizeof(double) * CC_DIAG_LEN);
    H.o_ws = o;   o = align256(o + cc_workspace_bytes(n, cells));
    H.total = o;
    return H;
}
}  // namespace

size_t cc_host_buffer_bytes(int64_t n, int32_t cells)
{
    if (n < 0 || cells < 1) return 0;
    return host_layout(n, cells).total;
}

int coulomb_collide_host(const double* h_v_in, int64_t ldv, const int32_t* h_cell_in, double* h_v_out,
                         int32_t* h_cell_out, int32_t* h_perm_out, int64_t n, int32_t cells, uint32_t cell_base,
                         double dt, const cc_params* params, uint64_t seed, uint64_t step, double* h_moments_out,
                         double* h_diag_out, void* dev_buffer, size_t dev_bytes, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    {
        // every host-side argument error is reported before anything is enqueued (header contract)
        cc_params p;
        if (params) p = *params; else cc_default_params(&p);
        if (p.push) return CC_EINVAL;      // the host entry has no device positions to push
        if (const int rc = check_call(p, n, cells, ldv, dt, step)) return rc;
    }
    if (n > 0 && (!h_v_in || !h_cell_in || !h_v_out)) return CC_EINVAL;
    const HostLayout H = host_layout(n, cells);
    if (!dev_buffer || !aligned(dev_buffer, 256) || dev_bytes < H.total) return CC_EWORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* b = static_cast<char*>(dev_buffer);
    double* d_vin = reinterpret_cast<double*>(b + H.o_vin);
    double* d_vout = reinterpret_cast<double*>(b + H.o_vout);
    int32_t* d_cin = reinterpret_cast<int32_t*>(b + H.o_cin);
    int32_t* d_cout = reinterpret_cast<int32_t*>(b + H.o_cout);
    int32_t* d_perm = reinterpret_cast<int32_t*>(b + H.o_perm);
    double* d_mom = reinterpret_cast<double*>(b + H.o_mom);
    double* d_diag = reinterpret_cast<double*>(b + H.o_diag);
    const size_t row = sizeof(double) * static_cast<size_t>(n);
    if (n > 0) {
        // H2D: cell ids first (the count pass needs only them), then the three velocity rows
        // (contiguous rows on both sides: one linear copy of 3n doubles)
        const bool lin = (ldv == n && H.ldd == n);
        if (cudaMemcpyAsync(d_cin, h_cell_in, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            (lin ? cudaMemcpyAsync(d_vin, h_v_in, 3 * row, cudaMemcpyHostToDevice, st)
                 : cudaMemcpy2DAsync(d_vin, sizeof(double) * H.ldd, h_v_in, sizeof(double) * ldv, row, 3,
                                     cudaMemcpyHostToDevice, st)) != cudaSuccess) {
            cudaGetLastError();
            return CC_ECUDA;
        }
    }
    int rc = coulomb_collide(d_vin, H.ldd, d_cin, d_vout, d_cout, h_perm_out ? d_perm : nullptr, n, cells, cell_base,
                             dt, params, seed, step, h_moments_out ? d_mom : nullptr, h_diag_out ? d_diag : nullptr,
                             b + H.o_ws, H.total - H.o_ws, stream);
    if (rc) return rc;
    bool ok = true;
    if (n > 0) {
        ok = ok && ((ldv == n && H.ldd == n)
                        ? cudaMemcpyAsync(h_v_out, d_vout, 3 * row, cudaMemcpyDeviceToHost, st)
                        : cudaMemcpy2DAsync(h_v_out, sizeof(double) * ldv, d_vout, sizeof(double) * H.ldd, row, 3,
                                            cudaMemcpyDeviceToHost, st)) == cudaSuccess;
        if (h_cell_out)
            ok = ok && cudaMemcpyAsync(h_cell_out, d_cout, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st) == cudaSuccess;
        if (h_perm_out)
            ok = ok && cudaMemcpyAsync(h_perm_out, d_perm, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st) == cudaSuccess;
    }
    if (h_moments_out)
        ok = ok && cudaMemcpyAsync(h_moments_out, d_mom, sizeof(double) * CC_MOMENTS_LEN * cells,
                                   cudaMemcpyDeviceToHost, st) == cudaSuccess;
    if (h_diag_out)
        ok = ok && cudaMemcpyAsync(h_diag_out, d_diag, sizeof(double) * CC_DIAG_LEN, cudaMemcpyDeviceToHost, st) ==
                       cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        return CC_ECUDA;
    }
    return CC_OK;
}

int cc_device_status(void* workspace, void* stream)
{
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaStreamSynchronize(st) != cudaSuccess) return CC_ECUDA;
    if (!workspace) return CC_EWORKSPACE;
    int32_t err = 0;
    if (cudaMemcpy(&err, workspace, sizeof(err), cudaMemcpyDeviceToHost) != cudaSuccess) return CC_ECUDA;
    if (err) {
        if (cudaMemset(workspace, 0, sizeof(err)) != cudaSuccess) return CC_ECUDA;
        return CC_ECELL;
    }
    return CC_OK;
}

int cc_bin(const int32_t* cell_in, int64_t n, int32_t cells, int32_t* perm_out, int32_t* off_out,
           void* workspace, size_t workspace_bytes, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (n < 0 || cells < 1) return CC_EINVAL;
    if (n >= (1ll << 31) || cells > CC_MAX_CELLS) return CC_ECOUNT;
    if (!workspace || !aligned(workspace, 256)) return CC_EWORKSPACE;
    const Layout L = make_layout(n, cells);
    if (workspace_bytes < L.total) return CC_EWORKSPACE;
    if (!off_out || (n > 0 && (!cell_in || !perm_out))) return CC_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cc_params p;
    cc_default_params(&p);
    const CellConst k = cell_const(p, 1.0);
    if (n == 0) {
        return cudaMemsetAsync(off_out, 0, sizeof(int32_t) * (cells + 1), st) == cudaSuccess ? CC_OK : CC_ECUDA;
    }
    // the velocity payload is irrelevant for the order: bin without one
    const int nn = static_cast<int>(n);
    int rc = run_binning(nullptr, 0, cell_in, nn, cells, L, workspace, k, 0, 0, 0, st, nullptr, false);
    if (rc) return rc;
    k_extract_perm<<<(nn + 255) / 256, 256, 0, st>>>(at<double>(workspace, L.o_wsv), nn, perm_out);
    if (cudaMemcpyAsync(off_out, at<int32_t>(workspace, L.o_off), sizeof(int32_t) * (cells + 1),
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return CC_ECUDA;
    return launch_ok();
}

int cc_pairs(const int32_t* off, int32_t cells, uint32_t cell_base, uint64_t seed, uint64_t step,
             uint32_t flags, int32_t* pair_slots_out, int64_t max_pairs, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (!off || cells < 1 || step >= (1ull << 32) || max_pairs < 0 || (flags & ~CC_CELL_UNIFORM)) return CC_EINVAL;
    if (max_pairs > 0 && !pair_slots_out) return CC_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_pairs<<<cells, 256, 0, st>>>(off, cells, cell_base, static_cast<uint32_t>(step), static_cast<uint32_t>(seed),
                                   static_cast<uint32_t>(seed >> 32), pair_slots_out, max_pairs,
                                   (flags & CC_CELL_UNIFORM) ? 0 : 1);
    return launch_ok();
}

int cc_philox(const uint32_t* ctr4, uint64_t seed, uint32_t* out4, int64_t m, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (m < 0 || (m > 0 && (!ctr4 || !out4))) return CC_EINVAL;
    if (m == 0) return CC_OK;
    k_philox<<<static_cast<unsigned>((m + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        ctr4, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), out4, m);
    return launch_ok();
}

int cc_ppnd16(const double* u, double* z, int64_t m, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (m < 0 || (m > 0 && (!u || !z))) return CC_EINVAL;
    if (m == 0) return CC_OK;
    k_ppnd16<<<static_cast<unsigned>((m + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(u, z, m);
    return launch_ok();
}

int cc_ta_pairs(double* va, double* vb, const double* C, const double* u1, const double* u2, int64_t m,
                void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (m < 0 || (m > 0 && (!va || !vb || !C || !u1 || !u2))) return CC_EINVAL;
    if (m == 0) return CC_OK;
    k_ta_pairs<<<static_cast<unsigned>((m + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(va, vb, C, u1,
                                                                                                       u2, m);
    return launch_ok();
}

int cc_moments(const double* v, int64_t ldv, const int32_t* off, int32_t cells, const cc_params* params,
               double* out, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (!v || !off || !out || cells < 1 || ldv < 0) return CC_EINVAL;
    cc_params p;
    if (params) p = *params; else cc_default_params(&p);
    MomConst mc{p.weight, p.cell_volume, p.cell_volume_arr, p.mass / p.charge};
    k_moments<<<cells, 256, 0, static_cast<cudaStream_t>(stream)>>>(v, ldv, off, cells, mc, out);
    return launch_ok();
}

int cc_gather(const double* v, int64_t ldv, const int32_t* cell, const int32_t* idx, int64_t m, int32_t cell_shift,
              double* v_out, int64_t ldo, int32_t* cell_out, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (m < 0 || ldo < m) return CC_EINVAL;
    if (m == 0) return CC_OK;
    if (!v || !cell || !idx || !v_out || !cell_out) return CC_EINVAL;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((m + 255) / 256, 148 * 16));
    k_gather<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(v, ldv, cell, idx, m, cell_shift, v_out, ldo,
                                                                   cell_out);
    return launch_ok();
}

int cc_owner(const int32_t* cell, int64_t n, const int32_t* bounds, int32_t nranks, int32_t* owner_out, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (n < 0 || nranks < 1) return CC_EINVAL;
    if (n == 0) return CC_OK;
    if (!cell || !bounds || !owner_out) return CC_EINVAL;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_owner<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(cell, n, bounds, nranks, owner_out);
    return launch_ok();
}

int cc_coulomb_log(const double* moments, int32_t cells, double* out, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (!moments || !out || cells < 1) return CC_EINVAL;
    k_coulomb_log<<<(cells + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(moments, cells, out);
    return launch_ok();
}

int cc_push(const double* x_in, int64_t ldx_in, const int32_t* perm, double* x_out, int64_t ldx_out, double* v,
            int64_t ldv, int32_t* cell, int64_t n, int32_t cells, uint32_t cell_base, const cc_grid* grid,
            const double* E, int64_t ldE, double q_over_m, double dt, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    (void)cell_base;      // E is indexed by the local cell; the output ids are global by construction
    if (!grid || n < 0 || cells < 1 || !std::isfinite(q_over_m) || !std::isfinite(dt)) return CC_EINVAL;
    if (grid->dims < 1 || grid->dims > 3) return CC_EINVAL;
    PushGrid g;
    g.dims = grid->dims;
    g.periodic = grid->periodic;
    int64_t total = 1;
    for (int a = 0; a < 3; ++a) {
        if (a < grid->dims) {
            if (grid->n[a] < 1 || !finite_pos(grid->d[a])) return CC_EINVAL;
            g.n[a] = grid->n[a];
            g.d[a] = grid->d[a];
        } else {
            g.n[a] = 1;
            g.d[a] = 1.0;
        }
        g.L[a] = static_cast<double>(g.n[a]) * g.d[a];
        total *= g.n[a];
    }
    if (total >= (1ll << 31)) return CC_EINVAL;
    if (n == 0) return CC_OK;
    if (!x_in || !x_out || !v || !cell || ldx_in < n || ldx_out < n || ldv < n || (E && ldE < cells))
        return CC_EINVAL;
    if (perm && overlaps(x_in, sizeof(double) * static_cast<size_t>(2 * ldx_in + n), x_out,
                         sizeof(double) * static_cast<size_t>(2 * ldx_out + n)))
        return CC_EINVAL;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (E) launch_push<true>(blocks, st, x_in, ldx_in, perm, x_out, ldx_out, v, ldv, cell, n, g, E, ldE, q_over_m, dt);
    else launch_push<false>(blocks, st, x_in, ldx_in, perm, x_out, ldx_out, v, ldv, cell, n, g, E, ldE, q_over_m, dt);
    return launch_ok();
}

size_t cc_p2c_scratch_bytes(int32_t cells, int32_t sub)
{
    if (cells < 1 || sub < 1) return 0;
    return sizeof(double) * kRaw * static_cast<size_t>(cells) * static_cast<size_t>(sub);
}

int cc_p2c(const double* v, int64_t ldv, const int32_t* cell, int64_t n, int32_t cells, int32_t sub, double* raw_out,
           void* scratch, size_t scratch_bytes, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (n < 0 || cells < 1 || sub < 1 || sub > 1024 || !raw_out || ldv < n) return CC_EINVAL;
    if (n > 0 && (!v || !cell)) return CC_EINVAL;
    if (!scratch || scratch_bytes < cc_p2c_scratch_bytes(cells, sub)) return CC_EWORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double* acc = static_cast<double*>(scratch);
    if (cudaMemsetAsync(acc, 0, cc_p2c_scratch_bytes(cells, sub), st) != cudaSuccess) return CC_ECUDA;
    if (n > 0) {
        const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
        k_p2c_atomic<<<blocks, 256, 0, st>>>(v, ldv, cell, n, cells, sub, acc);
    }
    k_p2c_reduce<<<(cells + 255) / 256, 256, 0, st>>>(acc, cells, sub, raw_out);
    return launch_ok();
}

int cc_p2c_moments(const double* raw, int32_t cells, const cc_params* params, double* moments_out, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (!raw || !moments_out || cells < 1) return CC_EINVAL;
    cc_params p;
    if (params) p = *params; else cc_default_params(&p);
    MomConst mc{p.weight, p.cell_volume, p.cell_volume_arr, p.mass / p.charge};
    k_p2c_moments<<<(cells + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(raw, cells, mc, moments_out);
    return launch_ok();
}

int cc_recombine(double* v, int64_t ldv, int32_t* cell, int64_t n, int32_t cells, uint32_t cell_base,
                 const double* prob, double eps_bind, double mass, uint64_t seed, uint64_t step,
                 unsigned long long* stats_out, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (n < 0 || cells < 1 || ldv < n || !prob || !stats_out || !finite_pos(mass) || !std::isfinite(eps_bind) ||
        eps_bind < 0.0 || step >= (1ull << 32))
        return CC_EINVAL;
    if (n >= (1ll << 31) || cells > CC_MAX_CELLS) return CC_ECOUNT;
    if (n > 0 && (!v || !cell)) return CC_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(stats_out, 0, 3 * sizeof(unsigned long long), st) != cudaSuccess) return CC_ECUDA;
    if (n == 0) return CC_OK;
    k_recombine<<<cells, 256, 0, st>>>(v, ldv, cell, n, cells, cell_base, prob, 2.0 * eps_bind / mass,
                                       static_cast<uint32_t>(step), static_cast<uint32_t>(seed),
                                       static_cast<uint32_t>(seed >> 32), stats_out);
    k_recombine_finish<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(cell, n);
    return launch_ok();
}

int cc_step_advance(uint32_t* step_dev, uint32_t inc, void* stream)
{
    cudaGetLastError();
    if (!step_dev) return CC_EINVAL;
    k_step_advance<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(step_dev, inc);
    return launch_ok();
}

int cc_diag_sum_ranks(const double* gathered, int32_t nranks, double* out, void* stream)
{
    cudaGetLastError();   // launch errors below are ours, not a stale earlier one
    if (!gathered || !out || nranks < 1) return CC_EINVAL;
    k_diag_sum_ranks<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(gathered, nranks, out);
    return launch_ok();
}

}  // extern "C"
