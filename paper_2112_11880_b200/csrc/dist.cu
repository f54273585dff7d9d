// dist.cu — row-partitioned matrices over NCCL: each rank owns a contiguous row
// block with global column ids; setup builds the halo plan (which off-rank x entries each rank
// references, grouped by owner), renumbers columns to [local rows | halo slots], and exchanges the
// send lists.  Each SpMV first fills the halo slots with grouped ncclSend/ncclRecv to the owning
// peers (NVLink through NVSwitch); each reduction point ends with an ncclAllReduce of the
// block partials' sums (≤ 4 doubles), identical on every rank, so all ranks take the same branch.
#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/zk_dist.h"
#include "spmv.cuh"
#include "zk_host.h"

namespace zk {
zk_status comm_allreduce_sum(zk_comm_s* c, double* buf, int count, cudaStream_t s);
zk_status comm_group_start();
zk_status comm_group_end();
zk_status comm_send(zk_comm_s* c, const void* buf, size_t bytes, int peer, cudaStream_t s);
zk_status comm_recv(zk_comm_s* c, void* buf, size_t bytes, int peer, cudaStream_t s);
zk_status comm_allgather(zk_comm_s* c, const void* send, void* recv, size_t bytes, cudaStream_t s);
int comm_rank(const zk_comm_s* c);
int comm_size(const zk_comm_s* c);
zk_status zcsrmv_local(const zk_csr_s* A, double2 alpha, const double2* x, double2 beta, double2* y,
                       cudaStream_t s);

struct DistPlan {
    int nranks = 1, rank = 0;
    std::vector<int64_t> offsets;              // [nranks+1] global row ranges
    int64_t n_ext = 0;                         // halo slots
    std::vector<int64_t> recv_cnt, recv_off;   // per peer, into the halo slots
    std::vector<int64_t> send_cnt, send_off;   // per peer, into the send list
    int64_t n_send = 0;
    int* d_send_idx = nullptr;                 // local rows to pack, concatenated per peer
    double2* d_sendbuf = nullptr;
    double2* d_xg = nullptr;                   // gather scratch of zk_zcsrmv: [x | halo]
};

static DistPlan* plan(const zk_csr_s* A) { return (DistPlan*)A->dist; }

__global__ void pack_kernel(const double2* __restrict__ x, const int* __restrict__ idx, int64_t n,
                            double2* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = x[idx[i]];
}

void dist_destroy(zk_csr_s* A) {
    DistPlan* P = plan(A);
    if (!P) return;
    cudaFree(P->d_send_idx);
    cudaFree(P->d_sendbuf);
    cudaFree(P->d_xg);
    delete P;
    A->dist = nullptr;
}

int64_t dist_gather_len(const zk_csr_s* A) { return A->n_rows + (plan(A) ? plan(A)->n_ext : 0); }

zk_status dist_setup(zk_csr_s* A, const int64_t*, const int*, cudaStream_t s) {
    zk_comm_s* c = A->comm;
    const int np = comm_size(c), me = comm_rank(c);
    DistPlan* P = new DistPlan();
    A->dist = P;
    P->nranks = np;
    P->rank = me;
    // ---- 1. row ranges of all ranks
    int64_t* d_rng = nullptr;
    ZK_CUDA(cudaMalloc(&d_rng, sizeof(int64_t) * 2 * (np + np * (size_t)np + 1)));
    int64_t mine[2] = {A->row_begin, A->n_rows};
    ZK_CUDA(cudaMemcpyAsync(d_rng, mine, sizeof mine, cudaMemcpyHostToDevice, s));
    ZK_TRY(comm_allgather(c, d_rng, d_rng + 2, sizeof mine, s));
    std::vector<int64_t> rng(2 * np);
    ZK_CUDA(cudaMemcpyAsync(rng.data(), d_rng + 2, sizeof(int64_t) * 2 * np, cudaMemcpyDeviceToHost, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    P->offsets.assign(np + 1, 0);
    for (int r = 0; r < np; r++) {
        if (rng[2 * r] != P->offsets[r]) {
            cudaFree(d_rng);
            return fail(ZK_ERR_INVALID_VALUE, "rank row blocks must be contiguous and in rank order");
        }
        P->offsets[r + 1] = rng[2 * r] + rng[2 * r + 1];
    }
    A->n_global = P->offsets[np];
    // ---- 2. halo plan from this rank's global column ids
    std::vector<int> col(A->nnz);
    if (A->nnz) ZK_CUDA(cudaMemcpyAsync(col.data(), A->col, sizeof(int) * A->nnz, cudaMemcpyDeviceToHost, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    int64_t n_ext = 0;
    std::vector<int64_t> cnt(np, 0);
    zk_status st = zk_halo_plan(A->nnz, col.data(), np, me, P->offsets.data(), &n_ext, nullptr, nullptr);
    if (st != ZK_OK) { cudaFree(d_rng); return st; }
    std::vector<int> ext(n_ext > 0 ? n_ext : 1);
    ZK_TRY(zk_halo_plan(A->nnz, col.data(), np, me, P->offsets.data(), &n_ext, ext.data(), cnt.data()));
    P->n_ext = n_ext;
    P->recv_cnt = cnt;
    P->recv_off.assign(np + 1, 0);
    for (int r = 0; r < np; r++) P->recv_off[r + 1] = P->recv_off[r] + cnt[r];
    // ---- 3. who needs what from whom: allgather the count rows → counts[i][j]
    int64_t* d_cnt = d_rng + 2 + 2 * np;
    ZK_CUDA(cudaMemcpyAsync(d_cnt, cnt.data(), sizeof(int64_t) * np, cudaMemcpyHostToDevice, s));
    ZK_TRY(comm_allgather(c, d_cnt, d_cnt + np, sizeof(int64_t) * np, s));
    std::vector<int64_t> all(np * (size_t)np);
    ZK_CUDA(cudaMemcpyAsync(all.data(), d_cnt + np, sizeof(int64_t) * np * np, cudaMemcpyDeviceToHost, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_rng);
    P->send_cnt.assign(np, 0);
    P->send_off.assign(np + 1, 0);
    for (int q = 0; q < np; q++) P->send_cnt[q] = all[(size_t)q * np + me];
    for (int q = 0; q < np; q++) P->send_off[q + 1] = P->send_off[q] + P->send_cnt[q];
    P->n_send = P->send_off[np];
    // ---- 4. exchange the requested global ids (grouped p2p), turn them into local rows
    int *d_req_out = nullptr, *d_req_in = nullptr;
    ZK_CUDA(cudaMalloc(&d_req_out, sizeof(int) * (n_ext > 0 ? n_ext : 1)));
    ZK_CUDA(cudaMalloc(&d_req_in, sizeof(int) * (P->n_send > 0 ? P->n_send : 1)));
    if (n_ext) ZK_CUDA(cudaMemcpyAsync(d_req_out, ext.data(), sizeof(int) * n_ext, cudaMemcpyHostToDevice, s));
    ZK_TRY(comm_group_start());
    for (int q = 0; q < np; q++) {
        if (q == me) continue;
        if (P->recv_cnt[q]) ZK_TRY(comm_send(c, d_req_out + P->recv_off[q], sizeof(int) * P->recv_cnt[q], q, s));
        if (P->send_cnt[q]) ZK_TRY(comm_recv(c, d_req_in + P->send_off[q], sizeof(int) * P->send_cnt[q], q, s));
    }
    ZK_TRY(comm_group_end());
    std::vector<int> req(P->n_send > 0 ? P->n_send : 1);
    if (P->n_send) ZK_CUDA(cudaMemcpyAsync(req.data(), d_req_in, sizeof(int) * P->n_send, cudaMemcpyDeviceToHost, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_req_out);
    for (int64_t k = 0; k < P->n_send; k++) {
        const int64_t loc = (int64_t)req[k] - A->row_begin;
        if (loc < 0 || loc >= A->n_rows) {
            cudaFree(d_req_in);
            return fail(ZK_ERR_INVALID_VALUE, "halo request outside this rank's rows");
        }
        req[k] = (int)loc;
    }
    if (P->n_send) ZK_CUDA(cudaMemcpyAsync(d_req_in, req.data(), sizeof(int) * P->n_send, cudaMemcpyHostToDevice, s));
    P->d_send_idx = d_req_in;
    ZK_CUDA(cudaMalloc(&P->d_sendbuf, sizeof(double2) * (P->n_send > 0 ? P->n_send : 1)));
    ZK_CUDA(cudaMalloc(&P->d_xg, sizeof(double2) * (A->n_rows + n_ext > 0 ? A->n_rows + n_ext : 1)));
    // ---- 5. renumber columns to [local | halo] in the library's own copy
    ZK_TRY(zk_halo_renumber(A->nnz, col.data(), A->row_begin, A->n_rows, n_ext, ext.data(), col.data()));
    if (A->nnz) ZK_CUDA(cudaMemcpyAsync(A->col, col.data(), sizeof(int) * A->nnz, cudaMemcpyHostToDevice, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    return ZK_OK;
}

zk_status dist_halo(const zk_csr_s* A, double2* xg, cudaStream_t s) {
    const DistPlan* P = plan(A);
    if (P->n_send) {
        const int G = grid_for(P->n_send, kBlock, A->dev.num_sms * 4);
        pack_kernel<<<G, kBlock, 0, s>>>(xg, P->d_send_idx, P->n_send, P->d_sendbuf);
        ZK_CUDA(cudaGetLastError());
    }
    ZK_TRY(comm_group_start());
    for (int q = 0; q < P->nranks; q++) {
        if (q == P->rank) continue;
        if (P->send_cnt[q])
            ZK_TRY(comm_send(A->comm, P->d_sendbuf + P->send_off[q], sizeof(double2) * P->send_cnt[q], q, s));
        if (P->recv_cnt[q])
            ZK_TRY(comm_recv(A->comm, xg + A->n_rows + P->recv_off[q], sizeof(double2) * P->recv_cnt[q], q, s));
    }
    return comm_group_end();
}

zk_status dist_allreduce_ctx(const zk_csr_s* A, double* red, int count, cudaStream_t s) {
    return comm_allreduce_sum(A->comm, red, count, s);
}

zk_status dist_zcsrmv(const zk_csr_s* A, double2 alpha, const double2* x, double2 beta, double2* y,
                      cudaStream_t s) {
    const DistPlan* P = plan(A);
    ZK_CUDA(cudaMemcpyAsync(P->d_xg, x, sizeof(double2) * A->n_rows, cudaMemcpyDeviceToDevice, s));
    ZK_TRY(dist_halo(A, P->d_xg, s));
    return zcsrmv_local(A, alpha, P->d_xg, beta, y, s);
}

int64_t dist_n_halo(const zk_csr_s* A) { return plan(A) ? plan(A)->n_ext : 0; }
int dist_nranks(const zk_csr_s* A) { return plan(A) ? plan(A)->nranks : 1; }

}  // namespace zk

using namespace zk;

extern "C" zk_status zk_partition_rows(int64_t n, const int64_t* row_ptr, int32_t nranks, int64_t* offsets) {
    if (n < 0 || !row_ptr || nranks < 1 || !offsets) return fail(ZK_ERR_INVALID_VALUE, "bad argument");
    const int64_t nnz = row_ptr[n];
    offsets[0] = 0;
    for (int r = 1; r < nranks; r++) {
        const int64_t target = (int64_t)((__int128)nnz * r / nranks);
        int64_t i = std::lower_bound(row_ptr, row_ptr + n + 1, target) - row_ptr;
        if (i < offsets[r - 1]) i = offsets[r - 1];
        if (i > n) i = n;
        offsets[r] = i;
    }
    offsets[nranks] = n;
    return ZK_OK;
}

extern "C" zk_status zk_halo_plan(int64_t nnz, const int32_t* col, int32_t nranks, int32_t rank, const int64_t* offsets,
                                  int64_t* n_ext, int32_t* ext_cols, int64_t* count_per_rank) {
    if (nnz < 0 || (nnz > 0 && !col) || nranks < 1 || rank < 0 || rank >= nranks || !offsets || !n_ext)
        return fail(ZK_ERR_INVALID_VALUE, "bad argument");
    const int64_t lo = offsets[rank], hi = offsets[rank + 1], n = offsets[nranks];
    std::vector<int32_t> ext;
    for (int64_t p = 0; p < nnz; p++) {
        const int64_t c = col[p];
        if (c < 0 || c >= n) return fail(ZK_ERR_INVALID_CSR, "column outside the global range");
        if (c < lo || c >= hi) ext.push_back((int32_t)c);
    }
    std::sort(ext.begin(), ext.end());
    ext.erase(std::unique(ext.begin(), ext.end()), ext.end());
    *n_ext = (int64_t)ext.size();
    if (ext_cols) std::copy(ext.begin(), ext.end(), ext_cols);
    if (count_per_rank) {
        for (int r = 0; r < nranks; r++) count_per_rank[r] = 0;
        int r = 0;
        for (int32_t c : ext) {
            while (c >= offsets[r + 1]) r++;
            count_per_rank[r]++;
        }
    }
    return ZK_OK;
}

extern "C" zk_status zk_halo_renumber(int64_t nnz, const int32_t* col, int64_t row_begin, int64_t n_rows, int64_t n_ext,
                                      const int32_t* ext_cols, int32_t* col_local) {
    if (nnz < 0 || (nnz > 0 && (!col || !col_local)) || (n_ext > 0 && !ext_cols))
        return fail(ZK_ERR_INVALID_VALUE, "bad argument");
    for (int64_t p = 0; p < nnz; p++) {
        const int64_t c = col[p];
        if (c >= row_begin && c < row_begin + n_rows) {
            col_local[p] = (int32_t)(c - row_begin);
        } else {
            const int32_t* it = std::lower_bound(ext_cols, ext_cols + n_ext, (int32_t)c);
            if (it == ext_cols + n_ext || *it != c) return fail(ZK_ERR_INVALID_VALUE, "column missing from the halo plan");
            col_local[p] = (int32_t)(n_rows + (it - ext_cols));
        }
    }
    return ZK_OK;
}
