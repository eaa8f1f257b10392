// Third-party cross-checks of the product path (SURVEY §8(c) "What pins each part"), test
// infrastructure only: library routines the product does NOT use, called on the same inputs.
//   tp_sort_pairs  cub::DeviceRadixSort::SortPairs (stable LSD radix sort) of (cell key, input
//                  index): the values it returns are the stable counting sort cc_bin must produce;
//   tp_philox      cuRAND's device Philox4x32-10 (curand_Philox4x32_10 of curand_philox4x32_x.h)
//                  on given counters and key: what cc_philox must return word for word.
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include <cstdint>
#include <cub/cub.cuh>

namespace {

__global__ void k_tp_philox(const uint32_t* __restrict__ ctr, uint32_t k0, uint32_t k1, uint32_t* __restrict__ out,
                            int64_t m)
{
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= m) return;
    const uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
    const uint4 r = curand_Philox4x32_10(c, make_uint2(k0, k1));
    out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
}

}  // namespace

extern "C" {

size_t tp_sort_temp_bytes(int n)
{
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), n);
    return bytes;
}

int tp_sort_pairs(const int32_t* keys_in, int32_t* keys_out, const int32_t* vals_in, int32_t* vals_out, int n,
                  int end_bit, void* temp, size_t temp_bytes, void* stream)
{
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, n, 0, end_bit,
                                           static_cast<cudaStream_t>(stream)) == cudaSuccess ? 0 : -3;
}

int tp_philox(const uint32_t* ctr4, uint64_t key, uint32_t* out4, int64_t m, void* stream)
{
    if (m <= 0) return 0;
    k_tp_philox<<<static_cast<unsigned>((m + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        ctr4, static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32), out4, m);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // extern "C"
