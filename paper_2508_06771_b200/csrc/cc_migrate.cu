// cc_migrate.cu — device-side particle migration between cell-range shards
// (SURVEY §8(e)), with no host synchronisation.
//
// Every rank keeps its particles in n fixed slots, dead-padded (cell -1).
// coulomb_collide leaves the live particles in slots [0, L) and the dead in
// [L, n) (L = diag_out[0]); a push (cc_push) rewrites the cell ids as GLOBAL ids
// in place.  Migration then moves every live particle to the rank that owns its
// cell (the paper's ranks never exchange particles: each owns N/P electrons and
// replicates the grid; the cell-range shards here do, so that cells
// are never split and pairing stays global):
//   k_mig_count   per (tile, warp): leavers per destination rank
//   k_mig_scan    per destination: exclusive scan over (tile, warp) rows, totals,
//                 send-slot headers, receive headers zeroed
//   k_mig_pack    leavers copied, in input order, into their destination's slot
//                 (SoA rows of a fixed capacity) and marked dead here; stayers
//                 get their LOCAL cell id; ids outside every range are dropped
//   (cc_dist_mig_exchange: fixed-size slots over NCCL, csrc/cc_dist.cu)
//   k_mig_unpack  arrivals, in (source rank, source order), into [L, L + A)
// Counts never leave the device: message sizes are the fixed slot size.  The
// order is deterministic for a given world size (stable packing, arrivals in
// source-rank order), so a sharded run is reproducible.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/coulomb.h"

namespace {

constexpr int kMigThreads = 256;
constexpr int kMigWarps = kMigThreads / 32;
constexpr int kMigSub = 512;                       // ids per warp sub-range
constexpr int kMigTile = kMigWarps * kMigSub;      // ids per CTA
constexpr int kMigHdr = 64;                        // header bytes of a slot (int64 count + padding)

size_t align256(size_t x) { return (x + 255u) & ~static_cast<size_t>(255u); }

// owner rank of a GLOBAL cell id under bounds[0..P] (smem), -1 if outside every range
__device__ __forceinline__ int mig_owner(int32_t c, const int32_t* b, int P)
{
    if (c < b[0] || c >= b[P]) return -1;
    int lo = 0, hi = P;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (b[mid] <= c) lo = mid; else hi = mid;
    }
    return lo;
}

struct SlotView {
    char* base;
    size_t slot;
    int64_t cap;
    int32_t xrows;
    __device__ char* s(int p) const { return base + static_cast<size_t>(p) * slot; }
    __device__ int64_t* count(int p) const { return reinterpret_cast<int64_t*>(s(p)); }
    __device__ double* row(int p, int r) const   // rows 0-2 v, 3.. payload
    {
        return reinterpret_cast<double*>(s(p) + kMigHdr) + static_cast<int64_t>(r) * cap;
    }
    __device__ int32_t* cell(int p) const
    {
        return reinterpret_cast<int32_t*>(row(p, 3 + xrows));
    }
};

__global__ void __launch_bounds__(kMigThreads)
k_mig_count(const int32_t* __restrict__ cell, int64_t n, const int32_t* __restrict__ bounds, int P, int rank,
            int32_t* __restrict__ rows)
{
    __shared__ int32_t b[CC_MIG_MAX_RANKS + 1];
    for (int i = threadIdx.x; i <= P; i += blockDim.x) b[i] = bounds[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kMigWarps + w;          // (tile, warp) row
    const int64_t s0 = r * kMigSub, s1 = min(s0 + kMigSub, n);
    int32_t mine = 0;                 // lane p counts leavers to rank p (P <= 64: two words per lane)
    int32_t mine2 = 0;
    for (int64_t i0 = s0; i0 < s1; i0 += 32) {
        const int64_t i = i0 + lane;
        int o = -1;
        if (i < s1) {
            const int32_t c = __ldg(cell + i);
            if (c >= 0) o = mig_owner(c, b, P);
        }
        const bool leaver = o >= 0 && o != rank;
        unsigned m = __ballot_sync(0xFFFFFFFFu, leaver);
        while (m) {
            const int p0 = __shfl_sync(0xFFFFFFFFu, o, __ffs(m) - 1);
            const unsigned mp = __ballot_sync(0xFFFFFFFFu, leaver && o == p0);
            if (lane == (p0 & 31)) { if (p0 < 32) mine += __popc(mp); else mine2 += __popc(mp); }
            m &= ~mp;
        }
    }
    if (lane < P) rows[r * P + lane] = mine;
    if (lane + 32 < P) rows[r * P + lane + 32] = mine2;
}

// one CTA per destination rank p: exclusive scan of column p over the R rows, total -> header
__global__ void __launch_bounds__(1024)
k_mig_scan(int32_t* __restrict__ rows, int64_t R, int P, SlotView send, SlotView recv)
{
    __shared__ int64_t wsum[32];
    const int p = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t per = (R + blockDim.x - 1) / blockDim.x;
    const int64_t r0 = min(static_cast<int64_t>(tid) * per, R), r1 = min(r0 + per, R);
    int64_t a = 0;
    for (int64_t r = r0; r < r1; ++r) a += rows[r * P + p];
    int64_t ia = a;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t x = __shfl_up_sync(0xFFFFFFFFu, ia, d);
        if (lane >= d) ia += x;
    }
    if (lane == 31) wsum[wid] = ia;
    __syncthreads();
    if (wid == 0) {
        int64_t v = (lane < static_cast<int>(blockDim.x / 32)) ? wsum[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t x = __shfl_up_sync(0xFFFFFFFFu, v, d);
            if (lane >= d) v += x;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    int64_t run = ia - a + (wid > 0 ? wsum[wid - 1] : 0);
    for (int64_t r = r0; r < r1; ++r) {
        const int32_t x = rows[r * P + p];
        rows[r * P + p] = static_cast<int32_t>(run);
        run += x;
    }
    if (tid == blockDim.x - 1) {
        *send.count(p) = min(run, send.cap);     // what the slot holds (the rest is dropped, status[0])
        *recv.count(p) = 0;                      // slots of non-peers read as empty
    }
}

__global__ void __launch_bounds__(kMigThreads)
k_mig_pack(double* __restrict__ v, int64_t ldv, double* __restrict__ x, int64_t ldx, int32_t* __restrict__ cell,
           int64_t n, const int32_t* __restrict__ bounds, int P, int rank, const int32_t* __restrict__ rows,
           SlotView send, int32_t* __restrict__ status)
{
    __shared__ int32_t b[CC_MIG_MAX_RANKS + 1];
    __shared__ int32_t run[kMigWarps][CC_MIG_MAX_RANKS];
    for (int i = threadIdx.x; i <= P; i += blockDim.x) b[i] = bounds[i];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kMigWarps + w;
    for (int p = lane; p < P; p += 32) run[w][p] = rows[r * P + p];
    __syncthreads();
    const int32_t base = b[rank];
    const int64_t s0 = r * kMigSub, s1 = min(s0 + kMigSub, n);
    const unsigned lt = (1u << lane) - 1u;
    int dropped = 0, outside = 0;
    for (int64_t i0 = s0; i0 < s1; i0 += 32) {
        const int64_t i = i0 + lane;
        int32_t c = -1;
        int o = -1;
        if (i < s1) {
            c = cell[i];
            if (c >= 0) o = mig_owner(c, b, P);
        }
        const bool leaver = o >= 0 && o != rank;
        if (c >= 0 && o == rank) cell[i] = c - base;                  // stays: LOCAL id
        if (c >= 0 && o < 0) { cell[i] = -1; ++outside; }               // outside every range
        unsigned m = __ballot_sync(0xFFFFFFFFu, leaver);
        int64_t pos = -1;
        while (m) {
            const int p0 = __shfl_sync(0xFFFFFFFFu, o, __ffs(m) - 1);
            const unsigned mp = __ballot_sync(0xFFFFFFFFu, leaver && o == p0);
            const int32_t at = run[w][p0];
            if (leaver && o == p0) pos = at + __popc(mp & lt);
            __syncwarp();
            if (lane == __ffs(mp) - 1) run[w][p0] = at + __popc(mp);
            __syncwarp();
            m &= ~mp;
        }
        if (leaver) {
            if (pos < send.cap) {
#pragma unroll
                for (int q = 0; q < 3; ++q) send.row(o, q)[pos] = v[q * ldv + i];
                for (int q = 0; q < send.xrows; ++q) send.row(o, 3 + q)[pos] = x[q * ldx + i];
                send.cell(o)[pos] = c;                                  // GLOBAL id: the receiver converts
            } else {
                ++dropped;
            }
            cell[i] = -1;                                               // gone from this rank
        }
    }
    if (dropped) atomicAdd(status + 0, dropped);
    if (outside) atomicAdd(status + 1, outside);
}

// grid: (chunks, P); arrivals of source p at L + (arrivals of sources < p) + t
__global__ void __launch_bounds__(kMigThreads)
k_mig_unpack(double* __restrict__ v, int64_t ldv, double* __restrict__ x, int64_t ldx, int32_t* __restrict__ cell,
             int64_t n, const double* __restrict__ diag, SlotView recv, const int32_t* __restrict__ bounds, int P,
             int rank, int32_t* __restrict__ status)
{
    const int p = blockIdx.y;
    if (p == rank) return;
    int64_t pre = 0;
    for (int q = 0; q < p; ++q) pre += (q == rank) ? 0 : *recv.count(q);
    const int64_t cnt = *recv.count(p);
    const int64_t L = static_cast<int64_t>(diag[0]);
    const int32_t base = bounds[rank];
    int lost = 0;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < cnt;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t d = L + pre + t;
        if (d >= n) { ++lost; continue; }
#pragma unroll
        for (int q = 0; q < 3; ++q) v[q * ldv + d] = recv.row(p, q)[t];
        for (int q = 0; q < recv.xrows; ++q) x[q * ldx + d] = recv.row(p, 3 + q)[t];
        cell[d] = recv.cell(p)[t] - base;
    }
    if (lost) atomicAdd(status + 2, lost);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(status + 3, static_cast<int32_t>(cnt));
}

int64_t mig_rows(int64_t n) { return (n + kMigSub - 1) / kMigSub; }

bool ok_ptr(const void* p, size_t a) { return p && (reinterpret_cast<uintptr_t>(p) % a) == 0; }

}  // namespace

extern "C" {

size_t cc_mig_slot_bytes(int64_t cap, int32_t xrows)
{
    if (cap < 0 || xrows < 0) return 0;
    return align256(kMigHdr + static_cast<size_t>(cap) * (8u * (3u + static_cast<size_t>(xrows)) + 4u));
}

size_t cc_mig_workspace_bytes(int64_t n, int32_t nranks)
{
    if (n < 0 || nranks < 1) return 0;
    return align256(static_cast<size_t>(mig_rows(n) > 0 ? mig_rows(n) : 1) * nranks * sizeof(int32_t));
}

int cc_mig_pack(double* v, int64_t ldv, double* x, int64_t ldx, int32_t xrows, int32_t* cell, int64_t n,
                const int32_t* bounds, int32_t nranks, int32_t rank, int64_t cap, void* send, void* recv,
                int32_t* status, void* workspace, size_t workspace_bytes, void* stream)
{
    cudaGetLastError();
    if (n < 0 || nranks < 1 || nranks > CC_MIG_MAX_RANKS || rank < 0 || rank >= nranks || cap < 0 || xrows < 0 ||
        xrows > 3 || ldv < n || (xrows > 0 && ldx < n))
        return CC_EINVAL;
    if (n >= (1ll << 31)) return CC_ECOUNT;
    if (!bounds || !status || !ok_ptr(send, 256) || !ok_ptr(recv, 256) || (n > 0 && (!v || !cell)) ||
        (xrows > 0 && n > 0 && !x))
        return CC_EINVAL;
    if (!ok_ptr(workspace, 256) || workspace_bytes < cc_mig_workspace_bytes(n, nranks)) return CC_EWORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t slot = cc_mig_slot_bytes(cap, xrows);
    SlotView S{static_cast<char*>(send), slot, cap, xrows};
    SlotView Rv{static_cast<char*>(recv), slot, cap, xrows};
    int32_t* rows = static_cast<int32_t*>(workspace);
    const int64_t R = mig_rows(n);
    const unsigned blocks = static_cast<unsigned>((R + kMigWarps - 1) / kMigWarps);
    if (R > 0) k_mig_count<<<blocks, kMigThreads, 0, st>>>(cell, n, bounds, nranks, rank, rows);
    k_mig_scan<<<nranks, 1024, 0, st>>>(rows, R, nranks, S, Rv);
    if (R > 0) k_mig_pack<<<blocks, kMigThreads, 0, st>>>(v, ldv, x, ldx, cell, n, bounds, nranks, rank, rows, S, status);
    return cudaGetLastError() == cudaSuccess ? CC_OK : CC_ECUDA;
}

int cc_mig_unpack(double* v, int64_t ldv, double* x, int64_t ldx, int32_t xrows, int32_t* cell, int64_t n,
                  const double* diag, const void* recv, const int32_t* bounds, int32_t nranks, int32_t rank,
                  int64_t cap, int32_t* status, void* stream)
{
    cudaGetLastError();
    if (n < 0 || nranks < 1 || nranks > CC_MIG_MAX_RANKS || rank < 0 || rank >= nranks || cap < 0 || xrows < 0 ||
        xrows > 3 || ldv < n || (xrows > 0 && ldx < n))
        return CC_EINVAL;
    if (!diag || !bounds || !status || !ok_ptr(recv, 256) || (n > 0 && (!v || !cell)) || (xrows > 0 && n > 0 && !x))
        return CC_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SlotView Rv{static_cast<char*>(const_cast<void*>(recv)), cc_mig_slot_bytes(cap, xrows), cap, xrows};
    const unsigned chunks = static_cast<unsigned>(cap > 0 ? (cap + kMigThreads * 4 - 1) / (kMigThreads * 4) : 1);
    k_mig_unpack<<<dim3(chunks > 0 ? chunks : 1, nranks), kMigThreads, 0, st>>>(v, ldv, x, ldx, cell, n, diag, Rv,
                                                                              bounds, nranks, rank, status);
    return cudaGetLastError() == cudaSuccess ? CC_OK : CC_ECUDA;
}

}  // extern "C"
