// comm.cu — communicators of the row-partitioned path (north star "rows are split
// into contiguous blocks ... halo exchange ... NCCL allreduce").  Two transports behind one set of
// internal calls (allreduce of a few doubles, allgather, grouped send/recv), all stream-ordered:
//
//  * NCCL — one process per GPU, the 128-byte ncclUniqueId broadcast by the caller
//    (torch.distributed); the product path for 2-8 B200s over NVLink 5 / NVSwitch.
//  * LOCAL — the ranks are host threads of ONE process (zk_local_group_create +
//    zk_comm_create_local), one CUDA stream each, on one or several GPUs.  A collective is a
//    rendezvous of the ranks' host threads: each rank records an event on its stream when its
//    operand is ready, the threads meet, every rank makes its stream wait for the peers' events and
//    moves the data with device copies (or a rank-order sum kernel), then a second rendezvous and
//    event wait keeps a rank from overwriting a buffer a peer is still reading.  Nothing spins on
//    the device, so several ranks can share one GPU: this is how the halo exchange and the
//    distributed reductions run with real multi-rank halos on the single B200 the tests lease
//    (NCCL refuses two ranks on one device).  Sums are taken in rank order: deterministic, and
//    bitwise identical on every rank, as the solvers' identical-branch rule needs.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "zk_host.h"

namespace zk {
constexpr int kLocalMaxRanks = 16;
constexpr int kLocalMaxRed = 128;  // doubles per local allreduce (BiCGStab(8)'s Gram totals: 81)

struct LocalOp {
    bool send;
    int peer;
    void* buf;
    size_t bytes;
};

struct LocalGroup {
    int n = 0;
    int refs = 0;  // live comms of this group
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;  // a rank timed out: every later rendezvous fails fast
    std::vector<const void*> ptr;
    std::vector<cudaEvent_t> ev_ready, ev_done;
    std::vector<std::vector<LocalOp>> sends;
    std::vector<int> joined;
    std::vector<int> dev;  // CUDA device of each rank

    // generation barrier with a timeout (a rank that errored out of a collective must not hang
    // its peers forever: they fail with ZK_ERR_NCCL after ZK_LOCAL_TIMEOUT_S, default 120 s)
    bool barrier() {
        static const double tmo = getenv("ZK_LOCAL_TIMEOUT_S") ? atof(getenv("ZK_LOCAL_TIMEOUT_S")) : 120.0;
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return false;
        const uint64_t g = gen;
        if (++arrived == n) {
            arrived = 0;
            gen++;
            cv.notify_all();
            return true;
        }
        const bool ok = cv.wait_for(lk, std::chrono::duration<double>(tmo), [&] { return gen != g || broken; });
        if (!ok || broken) {
            broken = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
};
}  // namespace zk

struct zk_local_group_s {
    zk::LocalGroup g;
    // the ranks' events belong to the group, not to the comms: a rank that leaves (zk_comm_destroy)
    // right after a collective must not invalidate an event a peer is about to wait on
    ~zk_local_group_s() {
        for (auto e : g.ev_ready)
            if (e) cudaEventDestroy(e);
        for (auto e : g.ev_done)
            if (e) cudaEventDestroy(e);
    }
};

struct zk_comm_s {
    ncclComm_t nccl = nullptr;
    int nranks = 1, rank = 0, device = 0;
    // LOCAL transport
    zk::LocalGroup* local = nullptr;
    zk_local_group_s* lg = nullptr;
    double* tmp = nullptr;  // device: this rank's allreduce result before it is copied back
    bool in_group = false;
    std::vector<zk::LocalOp> pending;
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

static zk_status local_rendezvous(zk_comm_s* c) {
    if (!c->local->barrier()) return fail(ZK_ERR_NCCL, "local group rendezvous failed (a peer rank timed out or errored)");
    return ZK_OK;
}

struct PeerPtrs {
    const double* p[kLocalMaxRanks];
};
// out[k] = Σ_q in[q][k], q = 0..n−1 in rank order (the same bits on every rank)
__global__ void local_sum_kernel(PeerPtrs in, int n, int count, double* out) {
    const int k = threadIdx.x;
    if (k >= count) return;
    double s = 0.0;
    for (int q = 0; q < n; q++) s += in.p[q][k];
    out[k] = s;
}

// phase 1 of every LOCAL collective: operand ready on this rank's stream, published, rendezvous
static zk_status local_publish(zk_comm_s* c, const void* p, cudaStream_t s) {
    LocalGroup* g = c->local;
    ZK_CUDA(cudaEventRecord(g->ev_ready[c->rank], s));
    g->ptr[c->rank] = p;
    return local_rendezvous(c);
}
// phase 3: this rank's consumers are done with what it published
static zk_status local_retire(zk_comm_s* c, cudaStream_t s) {
    LocalGroup* g = c->local;
    ZK_CUDA(cudaEventRecord(g->ev_done[c->rank], s));
    ZK_TRY(local_rendezvous(c));
    for (int q = 0; q < g->n; q++)
        if (q != c->rank) ZK_CUDA(cudaStreamWaitEvent(s, g->ev_done[q], 0));
    return ZK_OK;
}

zk_status comm_allreduce_sum(zk_comm_s* c, double* buf, int count, cudaStream_t s) {
    if (!c->local) {
        ZK_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, c->nccl, s));
        return ZK_OK;
    }
    if (count > kLocalMaxRed) return fail(ZK_ERR_INVALID_VALUE, "local allreduce count too large");
    LocalGroup* g = c->local;
    ZK_TRY(local_publish(c, buf, s));
    PeerPtrs pp{};
    for (int q = 0; q < g->n; q++) {
        pp.p[q] = (const double*)g->ptr[q];
        if (q != c->rank) ZK_CUDA(cudaStreamWaitEvent(s, g->ev_ready[q], 0));
    }
    local_sum_kernel<<<1, kLocalMaxRed, 0, s>>>(pp, g->n, count, c->tmp);
    ZK_CUDA(cudaGetLastError());
    ZK_TRY(local_retire(c, s));
    ZK_CUDA(cudaMemcpyAsync(buf, c->tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
    return ZK_OK;
}

zk_status comm_allgather(zk_comm_s* c, const void* send, void* recv, size_t bytes, cudaStream_t s) {
    if (!c->local) {
        ZK_NCCL(ncclAllGather(send, recv, bytes, ncclUint8, c->nccl, s));
        return ZK_OK;
    }
    LocalGroup* g = c->local;
    ZK_TRY(local_publish(c, send, s));
    for (int q = 0; q < g->n; q++) {
        if (q != c->rank) ZK_CUDA(cudaStreamWaitEvent(s, g->ev_ready[q], 0));
        if (bytes) ZK_CUDA(cudaMemcpyAsync((char*)recv + q * bytes, g->ptr[q], bytes, cudaMemcpyDefault, s));
    }
    return local_retire(c, s);
}

zk_status comm_group_start(zk_comm_s* c) {
    if (!c->local) {
        ZK_NCCL(ncclGroupStart());
        return ZK_OK;
    }
    c->in_group = true;
    c->pending.clear();
    return ZK_OK;
}

zk_status comm_send(zk_comm_s* c, const void* buf, size_t bytes, int peer, cudaStream_t s) {
    if (!c->local) {
        ZK_NCCL(ncclSend(buf, bytes, ncclUint8, peer, c->nccl, s));
        return ZK_OK;
    }
    if (!c->in_group) return fail(ZK_ERR_INVALID_VALUE, "local send outside a group");
    c->pending.push_back(LocalOp{true, peer, const_cast<void*>(buf), bytes});
    return ZK_OK;
}

zk_status comm_recv(zk_comm_s* c, void* buf, size_t bytes, int peer, cudaStream_t s) {
    if (!c->local) {
        ZK_NCCL(ncclRecv(buf, bytes, ncclUint8, peer, c->nccl, s));
        return ZK_OK;
    }
    if (!c->in_group) return fail(ZK_ERR_INVALID_VALUE, "local recv outside a group");
    c->pending.push_back(LocalOp{false, peer, buf, bytes});
    return ZK_OK;
}

// A group of sends/recvs is one collective of the whole group in the LOCAL transport (every rank
// calls it, possibly with no ops): the k-th recv from q takes the k-th send of q to this rank.
zk_status comm_group_end(zk_comm_s* c, cudaStream_t s) {
    if (!c->local) {
        ZK_NCCL(ncclGroupEnd());
        return ZK_OK;
    }
    LocalGroup* g = c->local;
    c->in_group = false;
    std::vector<LocalOp> ops;
    ops.swap(c->pending);
    g->sends[c->rank].clear();
    for (const LocalOp& o : ops)
        if (o.send) g->sends[c->rank].push_back(o);
    ZK_TRY(local_publish(c, nullptr, s));
    std::vector<int> taken(g->n, 0);
    zk_status st = ZK_OK;
    for (const LocalOp& o : ops) {
        if (o.send) continue;
        const int q = o.peer;
        const LocalOp* src = nullptr;
        int k = 0;
        for (const LocalOp& so : g->sends[q])
            if (so.peer == c->rank && k++ == taken[q]) {
                src = &so;
                break;
            }
        taken[q]++;
        if (!src || src->bytes != o.bytes) {
            st = fail(ZK_ERR_INVALID_VALUE, "local recv has no matching send of the same size");
            break;
        }
        ZK_CUDA(cudaStreamWaitEvent(s, g->ev_ready[q], 0));
        if (o.bytes) ZK_CUDA(cudaMemcpyAsync(o.buf, src->buf, o.bytes, cudaMemcpyDefault, s));
    }
    // the second rendezvous happens even on a mismatch, so the peers do not wait out the timeout
    zk_status st2 = local_retire(c, s);
    return st != ZK_OK ? st : st2;
}

int comm_rank(const zk_comm_s* c) { return c->rank; }
bool comm_is_local(const zk_comm_s* c) { return c && c->local; }
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

static std::mutex g_local_mu;  // guards LocalGroup::refs / joined across create and destroy

extern "C" zk_status zk_local_group_create(zk_local_group* out, int32_t nranks) {
    if (!out || nranks < 1 || nranks > kLocalMaxRanks) return fail(ZK_ERR_INVALID_VALUE, "nranks must be in [1, 16]");
    zk_local_group_s* lg = new zk_local_group_s();
    LocalGroup& g = lg->g;
    g.n = nranks;
    g.ptr.assign(nranks, nullptr);
    g.ev_ready.assign(nranks, nullptr);
    g.ev_done.assign(nranks, nullptr);
    g.sends.assign(nranks, {});
    g.joined.assign(nranks, 0);
    g.dev.assign(nranks, -1);
    g.refs = 1;  // the caller's reference
    *out = lg;
    return ZK_OK;
}

static void local_unref(zk_local_group_s* lg) {
    bool last;
    {
        std::lock_guard<std::mutex> lk(g_local_mu);
        last = --lg->g.refs == 0;
    }
    if (last) delete lg;
}

extern "C" zk_status zk_local_group_destroy(zk_local_group g) {
    if (!g) return ZK_OK;
    local_unref(g);
    return ZK_OK;
}

extern "C" zk_status zk_comm_create_local(zk_comm* out, zk_local_group lg, int32_t rank, int32_t device) {
    if (!out || !lg || rank < 0 || rank >= lg->g.n) return fail(ZK_ERR_INVALID_VALUE, "bad argument");
    *out = nullptr;
    ZK_CUDA(cudaSetDevice(device));
    zk_comm_s* c = new zk_comm_s();
    c->nranks = lg->g.n;
    c->rank = rank;
    c->device = device;
    c->local = &lg->g;
    c->lg = lg;
    cudaError_t e = cudaMalloc(&c->tmp, sizeof(double) * kLocalMaxRed);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "zk_comm_create_local", __FILE__, __LINE__);
    }
    {
        std::lock_guard<std::mutex> lk(g_local_mu);
        LocalGroup& g = lg->g;
        if (g.joined[rank]) {
            cudaFree(c->tmp);
            delete c;
            return fail(ZK_ERR_INVALID_VALUE, "rank already joined this local group");
        }
        if (g.dev[rank] != device) {  // first join of this rank (or on another device): its events
            if (g.ev_ready[rank]) cudaEventDestroy(g.ev_ready[rank]);
            if (g.ev_done[rank]) cudaEventDestroy(g.ev_done[rank]);
            g.ev_ready[rank] = g.ev_done[rank] = nullptr;
            e = cudaEventCreateWithFlags(&g.ev_ready[rank], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g.ev_done[rank], cudaEventDisableTiming);
            if (e != cudaSuccess) {
                cudaFree(c->tmp);
                delete c;
                return cuda_fail(e, "zk_comm_create_local(events)", __FILE__, __LINE__);
            }
        }
        g.joined[rank] = 1;
        g.dev[rank] = device;
        g.refs++;
    }
    // every rank of the group exists before the first collective (events published)
    zk_status st = local_rendezvous(c);
    if (st != ZK_OK) {
        zk_comm_destroy(c);
        return st;
    }
    // ranks on different GPUs read each other's buffers (sum kernel): peer access where needed
    for (int q = 0; q < lg->g.n; q++) {
        const int d = lg->g.dev[q];
        if (d == device) continue;
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, device, d) == cudaSuccess && can) {
            const cudaError_t pe = cudaDeviceEnablePeerAccess(d, 0);
            if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        }
    }
    *out = c;
    return ZK_OK;
}

extern "C" zk_status zk_comm_destroy(zk_comm c) {
    if (!c) return ZK_OK;
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->local) {
        {
            std::lock_guard<std::mutex> lk(g_local_mu);
            c->local->joined[c->rank] = 0;  // its events stay with the group (peers may still wait on them)
        }
        cudaFree(c->tmp);
        local_unref(c->lg);
    }
    delete c;
    return ZK_OK;
}
