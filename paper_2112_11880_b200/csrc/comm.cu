// comm.cu — NCCL communicator for row-partitioned runs: one process per GPU,
// the 128-byte ncclUniqueId broadcast by the caller (torch.distributed), libzk owns the comm.
#include <nccl.h>

#include <cstring>
#include <string>

#include "zk_host.h"

struct zk_comm_s {
    ncclComm_t nccl = nullptr;
    int nranks = 1, rank = 0, device = 0;
};

namespace zk {
static zk_status nccl_fail(ncclResult_t r, const char* what) {
    return fail(ZK_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
#define ZK_NCCL(call)                                   \
    do {                                                \
        ncclResult_t _r = (call);                       \
        if (_r != ncclSuccess) return nccl_fail(_r, #call); \
    } while (0)

zk_status comm_allreduce_sum(zk_comm_s* c, double* buf, int count, cudaStream_t s) {
    ZK_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, c->nccl, s));
    return ZK_OK;
}
zk_status comm_group_start() { ZK_NCCL(ncclGroupStart()); return ZK_OK; }
zk_status comm_group_end() { ZK_NCCL(ncclGroupEnd()); return ZK_OK; }
zk_status comm_send(zk_comm_s* c, const void* buf, size_t bytes, int peer, cudaStream_t s) {
    ZK_NCCL(ncclSend(buf, bytes, ncclUint8, peer, c->nccl, s));
    return ZK_OK;
}
zk_status comm_recv(zk_comm_s* c, void* buf, size_t bytes, int peer, cudaStream_t s) {
    ZK_NCCL(ncclRecv(buf, bytes, ncclUint8, peer, c->nccl, s));
    return ZK_OK;
}
zk_status comm_allgather(zk_comm_s* c, const void* send, void* recv, size_t bytes, cudaStream_t s) {
    ZK_NCCL(ncclAllGather(send, recv, bytes, ncclUint8, c->nccl, s));
    return ZK_OK;
}
int comm_rank(const zk_comm_s* c) { return c->rank; }
int comm_size(const zk_comm_s* c) { return c->nranks; }
}  // namespace zk

using namespace zk;

extern "C" zk_status zk_comm_get_unique_id(void* id128) {
    if (!id128) return fail(ZK_ERR_INVALID_VALUE, "NULL id");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    ZK_NCCL(ncclGetUniqueId(&id));
    memcpy(id128, &id, sizeof id);
    return ZK_OK;
}

extern "C" zk_status zk_comm_create(zk_comm* out, const void* id128, int32_t nranks, int32_t rank, int32_t device) {
    if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return fail(ZK_ERR_INVALID_VALUE, "bad argument");
    *out = nullptr;
    ZK_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    zk_comm_s* c = new zk_comm_s();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *out = c;
    return ZK_OK;
}

extern "C" zk_status zk_comm_destroy(zk_comm c) {
    if (!c) return ZK_OK;
    if (c->nccl) ncclCommDestroy(c->nccl);
    delete c;
    return ZK_OK;
}
