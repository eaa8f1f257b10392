// ------------------------------------------------------------------ R1b collide (persistent)
// k_collide_blocks: the R1b collide as a persistent kernel.  Each CTA walks the blocks
// c = blockIdx.x, + gridDim.x, ... with a two-buffer stage: while block c is paired and
// collided out of one buffer, block c + gridDim.x is being copied into the other (cp.async
// groups), so the copy latency and the per-block metadata chain (block table -> segment
// starts -> input indices -> copies) overlap the previous block's arithmetic instead of
// stalling a short-lived CTA (the round-2 one-CTA-per-block form spent ~1 ms of a 1.6-1.9 ms
// call on that chain, CC_ABLATE study in DESIGN.md §11).  Stage layouts: kModeRec interleaved
// 32-byte records; index modes planar x, y, z, input index.  Per block the results are
// identical to the one-CTA-per-block form (same pi, randoms, arithmetic and record order).
#ifndef CC_BLK_CTAS
#define CC_BLK_CTAS 7
#endif
constexpr int kBlkCTAs = CC_BLK_CTAS;
constexpr int kBlkThreads = 64;
constexpr int kBlkItems = cc::kBlock / 2 / kBlkThreads;        // pair items per thread (3)
constexpr int kBlkWarpItems = 32 * kBlkItems;
constexpr int kBlkBuf = 4 * cc::kBlock + 4;                    // doubles per buffer: stage + ref
constexpr size_t kBlkSmem = 2ull * kBlkBuf * sizeof(double);
static_assert(cc::kBlock % (2 * kBlkThreads) == 0 && kBlkThreads == 2 * cc::kSeg, "block shape");

struct BlkMeta {
    int32_t j, o, N, i0;
};

// Issue the copies of block c into buf (one cp.async group per call, committed by the caller).
__device__ __forceinline__ void blk_issue(const CollideArgs& A, int mode, int c, double* buf, BlkMeta& md)
{
    const int4 cm = __ldg(A.chunk_cell + c);
    md.j = cm.x; md.o = cm.y; md.N = cm.z; md.i0 = cm.w;
    const int32_t b = md.i0 / (cc::kBlock / 2);
    const int32_t nb = min(md.N - b * cc::kBlock, cc::kBlock);
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    int32_t sg[cc::kBlockSegs];
    if (md.N > cc::kBlock) {
        const int4* sp = reinterpret_cast<const int4*>(A.seg + static_cast<int64_t>(c) * cc::kBlockSegs);
#pragma unroll
        for (int g4 = 0; g4 < cc::kBlockSegs / 4; ++g4) {
            const int4 q = __ldg(sp + g4);
            sg[4 * g4] = q.x; sg[4 * g4 + 1] = q.y; sg[4 * g4 + 2] = q.z; sg[4 * g4 + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int g = 0; g < cc::kBlockSegs; ++g) sg[g] = g * cc::kSeg;
    }
    double* ref = buf + 4 * cc::kBlock;
    if (mode == kModeRec) {
        // record r = t / 2 of every segment, 16-byte half t % 2: a warp copies 512 contiguous bytes
        const int r = t >> 1, h = t & 1;
#pragma unroll
        for (int g = 0; g < cc::kBlockSegs; ++g)
            if (g * cc::kSeg + r < nb)
                cp_async16(buf + 4 * (g * cc::kSeg + r) + 2 * h, A.wsv + 4 * (md.o + static_cast<int64_t>(sg[g]) + r) + 2 * h);
        if (t < 2) cp_async16(ref + 2 * t, A.wsv + 4 * static_cast<int64_t>(md.o) + 2 * t);
    } else {
        // block slot u = t + 64 q lies in segment 2 q + w; slot o + sg + lane is input index
        // itself (kModeSorted) or the one k_scatter wrote (kModePerm)
        const int32_t* sperm = reinterpret_cast<const int32_t*>(A.wsv);
        int32_t idx[cc::kBlockSegs / 2];
#pragma unroll
        for (int q = 0; q < cc::kBlockSegs / 2; ++q) {
            const int u = t + q * kBlkThreads;
            const int32_t st0 = w ? sg[2 * q + 1] : sg[2 * q];
            const int64_t sl = md.o + static_cast<int64_t>(st0) + lane;
            idx[q] = (u < nb) ? (mode == kModeSorted ? static_cast<int32_t>(sl) : __ldg(sperm + sl)) : -1;
        }
        int32_t* pw = reinterpret_cast<int32_t*>(buf + 3 * cc::kBlock);
#pragma unroll
        for (int q = 0; q < cc::kBlockSegs / 2; ++q) {
            const int u = t + q * kBlkThreads;
            if (idx[q] >= 0) {
                const double* src = A.v_in + idx[q];
                cp_async8(buf + u, src);
                cp_async8(buf + cc::kBlock + u, src + A.ldvi);
                cp_async8(buf + 2 * cc::kBlock + u, src + 2 * A.ldvi);
                pw[u] = idx[q];
            }
        }
        if (t < 3) {
            const int64_t i0 = (mode == kModeSorted) ? md.o : __ldg(sperm + md.o);
            cp_async8(ref + t, A.v_in + i0 + t * A.ldvi);
        }
    }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <bool NANBU, bool PUSH>
__global__ void __launch_bounds__(kBlkThreads, kBlkCTAs)
k_collide_blocks(CollideArgs A)
{
    extern __shared__ __align__(16) double sbuf[];             // [2][kBlkBuf]
    __shared__ int32_t pi_small[cc::kSmallCell];
    __shared__ double zq[2][kBlkWarpItems];                     // normal variate / Nanbu u1 per item
    __shared__ double u2q[2][kBlkWarpItems];
    __shared__ int16_t tq[2][kBlkWarpItems];
    __shared__ double aq[NANBU ? 2 : 1][NANBU ? kBlkWarpItems : 1];
    __shared__ double red[2][10];
    const int nchunks = __ldg(A.chunk_off + A.M);
    const int mode = call_mode(A);
    const bool planar = mode != kModeRec;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t step = eff_step(A);
    int c = blockIdx.x;
    BlkMeta md{0, 0, 0, 0}, mdn{0, 0, 0, 0};
    if (c < nchunks) blk_issue(A, mode, c, sbuf, md);
    cp_async_commit();
    for (int it = 0; c < nchunks; c += gridDim.x, ++it) {
        double* buf = sbuf + (it & 1) * kBlkBuf;
        const int cn = c + gridDim.x;
        if (cn < nchunks) blk_issue(A, mode, cn, sbuf + ((it + 1) & 1) * kBlkBuf, mdn);
        cp_async_commit();

        const int j = md.j;
        const int32_t N = md.N, o = md.o;
        const uint32_t i0 = static_cast<uint32_t>(md.i0);
        const uint32_t items = static_cast<uint32_t>(N + 1) / 2;
        const uint32_t i1 = min(i0 + static_cast<uint32_t>(cc::kBlock / 2), items);
        const bool triplet = (A.model & cc::kOddTriplet) && (N & 1);
        const uint32_t b = i0 / static_cast<uint32_t>(cc::kBlock / 2);
        const int32_t nb = min(N - static_cast<int32_t>(b) * cc::kBlock, cc::kBlock);
        const uint32_t G = A.cell_base + static_cast<uint32_t>(j);
        // tau_b of each item's two block slots
        uint32_t xs[kBlkItems][2];
        if (nb > cc::kSmallCell) {
            const cc::Feistel f = cc::make_feistel(static_cast<uint32_t>(nb), cc::philox4x32_10(cc::U4{b, G, step, 1u}, A.s0, A.s1));
#pragma unroll
            for (int q = 0; q < kBlkItems; ++q) {
                const uint32_t e = threadIdx.x + q * kBlkThreads;
                uint32_t x[2] = {2 * e, 2 * e + 1};
                if (i0 + e < i1) {
                    cc::feistel_E_multi(f, x);
                    while (x[0] >= f.N) x[0] = cc::feistel_E(f, x[0]);
                    if (2 * e + 1 < static_cast<uint32_t>(nb))
                        while (x[1] >= f.N) x[1] = cc::feistel_E(f, x[1]);
                }
                xs[q][0] = x[0];
                xs[q][1] = x[1];
            }
        } else {
            if (w == 0) cc::small_cell_perm(static_cast<uint32_t>(nb), G, step, A.s0, A.s1, lane, pi_small,
                                           b * static_cast<uint32_t>(cc::kBlock / 4), 2u);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < kBlkItems; ++q) {
                const uint32_t e = threadIdx.x + q * kBlkThreads;
                xs[q][0] = (2 * e < static_cast<uint32_t>(nb)) ? pi_small[2 * e] : 0u;
                xs[q][1] = (2 * e + 1 < static_cast<uint32_t>(nb)) ? pi_small[2 * e + 1] : 0u;
            }
        }
        // CCS4: Philox per pair and AS241 (central branch in place, tails compacted per warp)
        {
            const uint32_t lt = (1u << lane) - 1u;
            int qn = 0;
            double u1[kBlkItems], u2[kBlkItems];
#pragma unroll
            for (int t = 0; t < kBlkItems; ++t) pair_uniforms(A, j, i0 + threadIdx.x + t * kBlkThreads, step, u1[t], u2[t]);
#pragma unroll
            for (int t = 0; t < kBlkItems; ++t) {
                const uint32_t k = i0 + threadIdx.x + t * kBlkThreads;
                const bool pair = (k < i1) && (2 * k + 1 < static_cast<uint32_t>(N));
                const bool tail = pair && !NANBU && !cc::ppnd16_is_central(u1[t]);
                const int slot = t * 32 + lane;
                zq[w][slot] = NANBU ? u1[t] : tail ? cc::ppnd16_tail_arg(u1[t]) : cc::ppnd16_central(u1[t]);
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
        const double C = A.Cj[j];
        cp_async_wait_prev();                      // block c's copies (block c + gridDim.x may still fly)
        __syncthreads();
        const double* ref = buf + 4 * cc::kBlock;
        const double rx = ref[0], ry = ref[1], rz = ref[2];
        if (i0 == 0 && threadIdx.x == 0) {
            double* cr = A.cellref + 4 * static_cast<int64_t>(j);
            cr[0] = rx; cr[1] = ry; cr[2] = rz; cr[3] = 0.0;
        }
        if (NANBU) {
            const uint32_t lt = (1u << lane) - 1u;
            int qn = 0;
#pragma unroll 1
            for (int t = 0; t < kBlkItems; ++t) {
                const uint32_t k = i0 + threadIdx.x + t * kBlkThreads;
                const int slot = t * 32 + lane;
                bool newton = false;
                if (k < i1 && !(triplet && k + 2 >= items) && 2 * k + 1 < static_cast<uint32_t>(N)) {
                    const Rec a = stage_rec(buf, planar, xs[t][0]), bb = stage_rec(buf, planar, xs[t][1]);
                    double Av, x;
                    newton = !cc::nanbu_A_direct(cc::nanbu_s(a.x, a.y, a.z, bb.x, bb.y, bb.z, C), Av, x);
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
        double pre[4] = {0.0, 0.0, 0.0, 0.0};
        constexpr int kUnroll2b = NANBU ? 1 : kBlkItems;
#pragma unroll kUnroll2b
        for (int t = 0; t < kBlkItems; ++t) {
            const uint32_t k = i0 + threadIdx.x + t * kBlkThreads;
            if (k < i1 && !(triplet && k + 2 >= items)) {     // the triplet's two items: k_triplets
                const int32_t pa = o + 2 * static_cast<int32_t>(k);
                Rec a = stage_rec(buf, planar, xs[t][0]);
                pre_add(pre, a.x, a.y, a.z);
                if (2 * k + 1 < static_cast<uint32_t>(N)) {
                    Rec bb = stage_rec(buf, planar, xs[t][1]);
                    pre_add(pre, bb.x, bb.y, bb.z);
                    if (PUSH) {
                        prefetch_x(A, unpack_perm(a.w));
                        prefetch_x(A, unpack_perm(bb.w));
                    }
                    const int slot = t * 32 + lane;
                    if (NANBU)
                        cc::nanbu_apply(a.x, a.y, a.z, bb.x, bb.y, bb.z, aq[w][slot], zq[w][slot], u2q[w][slot]);
                    else
                        cc::ta_update_z(a.x, a.y, a.z, bb.x, bb.y, bb.z, C, zq[w][slot], u2q[w][slot]);
                    write_pair_out<PUSH>(A, pa, j, a, bb);
                    acc.post(bb.x, bb.y, bb.z, rx, ry, rz);
                } else {
                    write_out<PUSH>(A, pa, j, a);
                }
                acc.post(a.x, a.y, a.z, rx, ry, rz);
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
        __syncthreads();                           // red complete; buf, zq, u2q free for reuse
        if (threadIdx.x < kRec)
            A.recs[static_cast<int64_t>(c) * kRec + threadIdx.x] = (threadIdx.x < 10) ? red[0][threadIdx.x] + red[1][threadIdx.x] : 0.0;
        md = mdn;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

