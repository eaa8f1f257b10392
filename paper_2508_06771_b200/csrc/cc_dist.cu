// cc_dist.cu — multi-GPU entry points of the C ABI: NCCL over
// NVLink 5 / NVSwitch, one process per GPU.  Cells never interact ("we only
// consider collisions between two particles in the same grid cell"), so
// the data path of coulomb_collide has no collective; NCCL carries only
//   * the 16-double diagnostics vector — all-gather, then the rank-ascending
//     device sum cc_diag_sum_ranks (deterministic for a given world size,
//     SPEC S:568-576), instead of the paper's O(M) MPI_AllReduce;
//   * particle migration after a push that crosses shard boundaries — grouped
//     ncclSend / ncclRecv of per-destination counts, then of the packed rows.
// Bootstrap: cc_nccl_get_unique_id on rank 0, broadcast by the caller (e.g.
// torch.distributed), cc_nccl_comm_init on every rank.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>

#include "../../include/coulomb.h"

namespace {

int nccl_ok(ncclResult_t r) { return r == ncclSuccess ? CC_OK : CC_ENCCL; }

}  // namespace

extern "C" {

int cc_nccl_get_unique_id(void* id_out)
{
    if (!id_out) return CC_EINVAL;
    static_assert(sizeof(ncclUniqueId) == CC_NCCL_ID_BYTES, "ncclUniqueId size");
    return nccl_ok(ncclGetUniqueId(static_cast<ncclUniqueId*>(id_out)));
}

int cc_nccl_comm_init(void** comm_out, int32_t nranks, int32_t rank, const void* id)
{
    if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks) return CC_EINVAL;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    const int rc = nccl_ok(ncclCommInitRank(&c, nranks, uid, rank));
    *comm_out = c;
    return rc;
}

int cc_nccl_comm_destroy(void* comm)
{
    if (!comm) return CC_EINVAL;
    return nccl_ok(ncclCommDestroy(static_cast<ncclComm_t>(comm)));
}

int cc_dist_diag_reduce(double* diag, double* scratch, void* comm, void* stream)
{
    if (!diag || !scratch || !comm) return CC_EINVAL;
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int nranks = 0;
    if (ncclCommCount(c, &nranks) != ncclSuccess) return CC_ENCCL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int rc = nccl_ok(ncclAllGather(diag, scratch, CC_DIAG_LEN, ncclFloat64, c, st));
    if (rc) return rc;
    return cc_diag_sum_ranks(scratch, nranks, diag, stream);
}

int cc_dist_alltoall_counts(const int64_t* send_counts, int64_t* recv_counts, void* comm, void* stream)
{
    if (!send_counts || !recv_counts || !comm) return CC_EINVAL;
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int nranks = 0;
    if (ncclCommCount(c, &nranks) != ncclSuccess) return CC_ENCCL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (ncclGroupStart() != ncclSuccess) return CC_ENCCL;
    ncclResult_t r = ncclSuccess;
    for (int p = 0; p < nranks && r == ncclSuccess; ++p) {
        r = ncclSend(send_counts + p, 1, ncclInt64, p, c, st);
        if (r == ncclSuccess) r = ncclRecv(recv_counts + p, 1, ncclInt64, p, c, st);
    }
    // the group is always closed; a failed post aborts it (no half-posted peer set)
    const ncclResult_t e = ncclGroupEnd();
    return (r == ncclSuccess && e == ncclSuccess) ? CC_OK : CC_ENCCL;
}

int cc_dist_exchange(const void* send, int64_t lds, void* recv, int64_t ldr, int32_t nrows, int32_t elem_bytes,
                     const int64_t* send_off, const int64_t* recv_off, void* comm, void* stream)
{
    if (!comm || !send_off || !recv_off || nrows < 1 || (elem_bytes != 4 && elem_bytes != 8)) return CC_EINVAL;
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int nranks = 0;
    if (ncclCommCount(c, &nranks) != ncclSuccess) return CC_ENCCL;
    if (send_off[0] != 0 || recv_off[0] != 0 || lds < send_off[nranks] || ldr < recv_off[nranks]) return CC_EINVAL;
    if ((send_off[nranks] > 0 && !send) || (recv_off[nranks] > 0 && !recv)) return CC_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const char* s = static_cast<const char*>(send);
    char* r = static_cast<char*>(recv);
    const size_t eb = static_cast<size_t>(elem_bytes);
    if (ncclGroupStart() != ncclSuccess) return CC_ENCCL;
    ncclResult_t res = ncclSuccess;
    for (int32_t row = 0; row < nrows && res == ncclSuccess; ++row)
        for (int p = 0; p < nranks && res == ncclSuccess; ++p) {
            const size_t ns = static_cast<size_t>(send_off[p + 1] - send_off[p]);
            const size_t nr = static_cast<size_t>(recv_off[p + 1] - recv_off[p]);
            if (ns) res = ncclSend(s + (row * lds + send_off[p]) * eb, ns * eb, ncclUint8, p, c, st);
            if (nr && res == ncclSuccess) res = ncclRecv(r + (row * ldr + recv_off[p]) * eb, nr * eb, ncclUint8, p, c, st);
        }
    const ncclResult_t e = ncclGroupEnd();
    return (res == ncclSuccess && e == ncclSuccess) ? CC_OK : CC_ENCCL;
}

int cc_dist_mig_exchange(const void* send, void* recv, size_t slot_bytes, const int32_t* peers, int32_t npeers,
                         void* comm, void* stream)
{
    if (!comm || npeers < 0 || (npeers > 0 && (!peers || !send || !recv)) || slot_bytes == 0) return CC_EINVAL;
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int nranks = 0, me = 0;
    if (ncclCommCount(c, &nranks) != ncclSuccess || ncclCommUserRank(c, &me) != ncclSuccess) return CC_ENCCL;
    for (int32_t i = 0; i < npeers; ++i)
        if (peers[i] < 0 || peers[i] >= nranks || peers[i] == me) return CC_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const char* s = static_cast<const char*>(send);
    char* r = static_cast<char*>(recv);
    if (ncclGroupStart() != ncclSuccess) return CC_ENCCL;
    ncclResult_t res = ncclSuccess;
    for (int32_t i = 0; i < npeers && res == ncclSuccess; ++i) {
        const size_t p = static_cast<size_t>(peers[i]);
        res = ncclSend(s + p * slot_bytes, slot_bytes, ncclUint8, peers[i], c, st);   // my slot for p
        if (res == ncclSuccess) res = ncclRecv(r + p * slot_bytes, slot_bytes, ncclUint8, peers[i], c, st);
    }
    const ncclResult_t e = ncclGroupEnd();
    return (res == ncclSuccess && e == ncclSuccess) ? CC_OK : CC_ENCCL;
}

}  // extern "C"
