// dist.cu — row-partitioned matrices over NCCL: each rank owns a contiguous row
// block with global column ids; setup builds the halo plan (which off-rank x entries each rank
// references, grouped by owner), renumbers columns to [local rows | halo slots], and exchanges the
// send lists.  Each SpMV first fills the halo slots with grouped ncclSend/ncclRecv to the owning
// peers (NVLink through NVSwitch); each reduction point ends with an ncclAllReduce of the
// block partials' sums (≤ 4 doubles), identical on every rank, so all ranks take the same branch.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/zk_dist.h"
#include "spmv.cuh"
#include "zk_host.h"

namespace zk {
zk_status comm_allreduce_sum(zk_comm_s* c, double* buf, int count, cudaStream_t s);
zk_status comm_group_start(zk_comm_s* c);
zk_status comm_group_end(zk_comm_s* c, cudaStream_t s);
zk_status comm_send(zk_comm_s* c, const void* buf, size_t bytes, int peer, cudaStream_t s);
zk_status comm_recv(zk_comm_s* c, void* buf, size_t bytes, int peer, cudaStream_t s);
zk_status comm_allgather(zk_comm_s* c, const void* send, void* recv, size_t bytes, cudaStream_t s);
int comm_rank(const zk_comm_s* c);
int comm_size(const zk_comm_s* c);
zk_status zcsrmv_local(const zk_csr_s* A, double2 alpha, const double2* x, double2 beta, double2* y,
                       cudaStream_t s);
zk_status zcsrmv_part(const zk_csr_s* A, double2 alpha, const double2* x, double2 beta, double2* y,
                      cudaStream_t s, const CsrDev& part);

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
    // interior / boundary split (SURVEY.md §8(e) "Halo" row): the longest run of 32-row slices
    // whose rows reference no halo column, [ov_lo, ov_hi); their SpMV overlaps the exchange
    int ov_lo = 0, ov_hi = 0, n_slices = 0;
    cudaStream_t cs = nullptr;                 // exchange stream
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
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
    dev_free(P->d_send_idx, true);  // (zk_csr_destroy synchronised the device)
    dev_free(P->d_sendbuf, true);
    dev_free(P->d_xg, true);
    if (P->cs) cudaStreamDestroy(P->cs);
    if (P->ev_pack) cudaEventDestroy(P->ev_pack);
    if (P->ev_halo) cudaEventDestroy(P->ev_halo);
    delete P;
    A->dist = nullptr;
}

// *any_failed = 1 if `failed` on any rank (one allreduce of a double; every rank calls it)
zk_status dist_agree_failed(zk_comm_s* c, bool failed, cudaStream_t s, int* any_failed) {
    double* d = nullptr;
    double h = failed ? 1.0 : 0.0;
    ZK_CUDA(scratch_alloc(&d, sizeof(double), s));
    cudaError_t e = cudaMemcpyAsync(d, &h, sizeof h, cudaMemcpyHostToDevice, s);
    zk_status st = e == cudaSuccess ? comm_allreduce_sum(c, d, 1, s) : cuda_fail(e, "agree", __FILE__, __LINE__);
    if (st == ZK_OK) {
        e = cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = cuda_fail(e, "agree", __FILE__, __LINE__);
    }
    scratch_free(d, s);
    *any_failed = h > 0.0 ? 1 : 0;
    return st;
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
    ZK_CUDA(scratch_alloc(&d_rng, sizeof(int64_t) * 2 * (np + np * (size_t)np + 1), s));
    int64_t mine[2] = {A->row_begin, A->n_rows};
    ZK_CUDA(cudaMemcpyAsync(d_rng, mine, sizeof mine, cudaMemcpyHostToDevice, s));
    ZK_TRY(comm_allgather(c, d_rng, d_rng + 2, sizeof mine, s));
    std::vector<int64_t> rng(2 * np);
    ZK_CUDA(cudaMemcpyAsync(rng.data(), d_rng + 2, sizeof(int64_t) * 2 * np, cudaMemcpyDeviceToHost, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    P->offsets.assign(np + 1, 0);
    for (int r = 0; r < np; r++) {
        if (rng[2 * r] != P->offsets[r]) {
            scratch_free(d_rng, s);
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
    if (st != ZK_OK) { scratch_free(d_rng, s); return st; }
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
    scratch_free(d_rng, s);
    P->send_cnt.assign(np, 0);
    P->send_off.assign(np + 1, 0);
    for (int q = 0; q < np; q++) P->send_cnt[q] = all[(size_t)q * np + me];
    for (int q = 0; q < np; q++) P->send_off[q + 1] = P->send_off[q] + P->send_cnt[q];
    P->n_send = P->send_off[np];
    // ---- 4. exchange the requested global ids (grouped p2p), turn them into local rows
    int *d_req_out = nullptr, *d_req_in = nullptr;
    ZK_CUDA(scratch_alloc(&d_req_out, sizeof(int) * (n_ext > 0 ? n_ext : 1), s));
    ZK_CUDA(dev_alloc(&d_req_in, sizeof(int) * (P->n_send > 0 ? P->n_send : 1), s));
    if (n_ext) ZK_CUDA(cudaMemcpyAsync(d_req_out, ext.data(), sizeof(int) * n_ext, cudaMemcpyHostToDevice, s));
    ZK_TRY(comm_group_start(c));
    for (int q = 0; q < np; q++) {
        if (q == me) continue;
        if (P->recv_cnt[q]) ZK_TRY(comm_send(c, d_req_out + P->recv_off[q], sizeof(int) * P->recv_cnt[q], q, s));
        if (P->send_cnt[q]) ZK_TRY(comm_recv(c, d_req_in + P->send_off[q], sizeof(int) * P->send_cnt[q], q, s));
    }
    ZK_TRY(comm_group_end(c, s));
    std::vector<int> req(P->n_send > 0 ? P->n_send : 1);
    if (P->n_send) ZK_CUDA(cudaMemcpyAsync(req.data(), d_req_in, sizeof(int) * P->n_send, cudaMemcpyDeviceToHost, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    scratch_free(d_req_out, s);
    for (int64_t k = 0; k < P->n_send; k++) {
        const int64_t loc = (int64_t)req[k] - A->row_begin;
        if (loc < 0 || loc >= A->n_rows) {
            scratch_free(d_req_in, s);
            return fail(ZK_ERR_INVALID_VALUE, "halo request outside this rank's rows");
        }
        req[k] = (int)loc;
    }
    if (P->n_send) ZK_CUDA(cudaMemcpyAsync(d_req_in, req.data(), sizeof(int) * P->n_send, cudaMemcpyHostToDevice, s));
    P->d_send_idx = d_req_in;
    ZK_CUDA(dev_alloc(&P->d_sendbuf, sizeof(double2) * (P->n_send > 0 ? P->n_send : 1), s));
    ZK_CUDA(dev_alloc(&P->d_xg, sizeof(double2) * (A->n_rows + n_ext > 0 ? A->n_rows + n_ext : 1), s));
    // ---- 5. renumber columns to [local | halo] in the library's own copy
    ZK_TRY(zk_halo_renumber(A->nnz, col.data(), A->row_begin, A->n_rows, n_ext, ext.data(), col.data()));
    if (A->nnz) ZK_CUDA(cudaMemcpyAsync(A->col, col.data(), sizeof(int) * A->nnz, cudaMemcpyHostToDevice, s));
    // ---- 6. interior slices: the longest run of 32-row slices with no halo column
    std::vector<int64_t> rp(A->n_rows + 1);
    ZK_CUDA(cudaMemcpyAsync(rp.data(), A->row_ptr, sizeof(int64_t) * (A->n_rows + 1), cudaMemcpyDeviceToHost, s));
    ZK_CUDA(cudaStreamSynchronize(s));
    const int64_t ns = (A->n_rows + 31) / 32;
    P->n_slices = (int)ns;
    int64_t best_lo = 0, best_len = 0, run_lo = 0;
    for (int64_t sl = 0; sl <= ns; sl++) {
        bool interior = sl < ns;
        if (interior) {
            const int64_t r0 = sl * 32, r1 = std::min<int64_t>(r0 + 32, A->n_rows);
            for (int64_t p = rp[r0]; p < rp[r1] && interior; p++) interior = col[p] < A->n_rows;
        }
        if (!interior) {
            if (sl - run_lo > best_len) {
                best_len = sl - run_lo;
                best_lo = run_lo;
            }
            run_lo = sl + 1;
        }
    }
    P->ov_lo = (int)best_lo;
    P->ov_hi = (int)(best_lo + best_len);
    ZK_CUDA(cudaStreamCreateWithFlags(&P->cs, cudaStreamNonBlocking));
    ZK_CUDA(cudaEventCreateWithFlags(&P->ev_pack, cudaEventDisableTiming));
    ZK_CUDA(cudaEventCreateWithFlags(&P->ev_halo, cudaEventDisableTiming));
    return ZK_OK;
}

// halo exchange with the interior slices overlapped: is it available for this matrix?
// (SELL mapping, a non-empty interior run; ZK_DIST_OVERLAP=0 turns it off)
bool dist_overlap(const zk_csr_s* A) {
    const int on = getenv("ZK_DIST_OVERLAP") ? atoi(getenv("ZK_DIST_OVERLAP")) : 1;
    const DistPlan* P = plan(A);
    return on && P && A->spmv_mode == 3 && P->ov_hi > P->ov_lo && P->n_slices == (int)A->n_slices;
}
// the interior run and the boundary rest (prefix + suffix) of the slice set of `a`
void dist_split(const zk_csr_s* A, const CsrDev& a, CsrDev* in, CsrDev* bd) {
    const DistPlan* P = plan(A);
    *in = a;
    in->sl_lo = P->ov_lo;
    in->sl_cnt = P->ov_hi - P->ov_lo;
    in->sl_gap_at = in->sl_cnt;
    in->sl_gap = 0;
    in->main_part = 1;
    *bd = a;
    bd->sl_lo = 0;
    bd->sl_cnt = P->ov_lo + (P->n_slices - P->ov_hi);
    bd->sl_gap_at = P->ov_lo;
    bd->sl_gap = P->ov_hi - P->ov_lo;
    bd->main_part = 0;
}

static zk_status halo_pack(const zk_csr_s* A, const double2* xg, cudaStream_t s) {
    const DistPlan* P = plan(A);
    if (P->n_send) {
        const int G = grid_for(P->n_send, kBlock, A->dev.num_sms * 4);
        pack_kernel<<<G, kBlock, 0, s>>>(xg, P->d_send_idx, P->n_send, P->d_sendbuf);
        ZK_CUDA(cudaGetLastError());
    }
    return ZK_OK;
}
// grouped send/recv of the packed entries into xg's halo slots, on stream s
static zk_status halo_exchange(const zk_csr_s* A, double2* xg, cudaStream_t s) {
    const DistPlan* P = plan(A);
    ZK_TRY(comm_group_start(A->comm));
    for (int q = 0; q < P->nranks; q++) {
        if (q == P->rank) continue;
        if (P->send_cnt[q])
            ZK_TRY(comm_send(A->comm, P->d_sendbuf + P->send_off[q], sizeof(double2) * P->send_cnt[q], q, s));
        if (P->recv_cnt[q])
            ZK_TRY(comm_recv(A->comm, xg + A->n_rows + P->recv_off[q], sizeof(double2) * P->recv_cnt[q], q, s));
    }
    return comm_group_end(A->comm, s);
}

// blocking halo: xg's halo slots are filled in stream order on s
zk_status dist_halo(const zk_csr_s* A, double2* xg, cudaStream_t s) {
    ZK_TRY(halo_pack(A, xg, s));
    return halo_exchange(A, xg, s);
}

// overlapped halo: pack on s, exchange on the plan's own stream; dist_halo_end makes s wait for it
zk_status dist_halo_begin(const zk_csr_s* A, double2* xg, cudaStream_t s) {
    const DistPlan* P = plan(A);
    ZK_TRY(halo_pack(A, xg, s));
    ZK_CUDA(cudaEventRecord(P->ev_pack, s));
    ZK_CUDA(cudaStreamWaitEvent(P->cs, P->ev_pack, 0));
    ZK_TRY(halo_exchange(A, xg, P->cs));
    ZK_CUDA(cudaEventRecord(P->ev_halo, P->cs));
    return ZK_OK;
}
zk_status dist_halo_end(const zk_csr_s* A, cudaStream_t s) {
    ZK_CUDA(cudaStreamWaitEvent(s, plan(A)->ev_halo, 0));
    return ZK_OK;
}

zk_status dist_allreduce_ctx(const zk_csr_s* A, double* red, int count, cudaStream_t s) {
    return comm_allreduce_sum(A->comm, red, count, s);
}

zk_status dist_zcsrmv(const zk_csr_s* A, double2 alpha, const double2* x, double2 beta, double2* y,
                      cudaStream_t s) {
    const DistPlan* P = plan(A);
    ZK_CUDA(cudaMemcpyAsync(P->d_xg, x, sizeof(double2) * A->n_rows, cudaMemcpyDeviceToDevice, s));
    if (!dist_overlap(A)) {
        ZK_TRY(dist_halo(A, P->d_xg, s));
        return zcsrmv_local(A, alpha, P->d_xg, beta, y, s);
    }
    CsrDev in, bd;
    dist_split(A, csr_dev(A), &in, &bd);
    ZK_TRY(dist_halo_begin(A, P->d_xg, s));
    ZK_TRY(zcsrmv_part(A, alpha, P->d_xg, beta, y, s, in));  // interior rows: local x only
    ZK_TRY(dist_halo_end(A, s));
    return bd.sl_cnt > 0 ? zcsrmv_part(A, alpha, P->d_xg, beta, y, s, bd) : ZK_OK;
}

bool comm_is_local(const zk_comm_s* c);
// libzk kernels a distributed SpMV / allreduce launches beyond the SpMV / finish kernel itself
void dist_launch_extra(const zk_csr_s* A, int* per_spmv, int* per_allreduce) {
    const DistPlan* P = plan(A);
    *per_spmv = (P && P->n_send ? 1 : 0) + (dist_overlap(A) ? 1 : 0);
    *per_allreduce = comm_is_local(A->comm) ? 1 : 0;
}
int64_t dist_n_send(const zk_csr_s* A) { return plan(A) ? plan(A)->n_send : 0; }
// rows of the interior slice run whose SpMV overlaps the halo exchange (0 without an overlap)
int64_t dist_interior_rows(const zk_csr_s* A) {
    if (!dist_overlap(A)) return 0;
    const DistPlan* P = plan(A);
    return std::min<int64_t>((int64_t)P->ov_hi * 32, A->n_rows) - (int64_t)P->ov_lo * 32;
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
