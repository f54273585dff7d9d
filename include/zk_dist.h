/*
 * zk_dist.h — host-only helpers of libzk's row-partitioned (multi-GPU) path, SURVEY.md §8(e).
 * They need no GPU and no NCCL: zk_csr_create uses them to build the halo plan of a rank's row
 * block, and the CPU tests use them (with a gloo process group standing in for NCCL) to check
 * the partition logic.  Citations: the paper partitions nothing on this path (its multi-GPU
 * Schwarz DDM, is out of scope); the plan follows the north star's "rows are split
 * into contiguous blocks ... each SpMV first runs a halo exchange of the x entries the local
 * block references".
 */
#ifndef ZK_DIST_H
#define ZK_DIST_H
#include "zk.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Contiguous row blocks balanced by nonzeros: offsets[0..nranks] with offsets[0] = 0,
 * offsets[nranks] = n, rank r owning rows [offsets[r], offsets[r+1]) and about nnz/nranks
 * nonzeros each (row_ptr is the GLOBAL int64[n+1] row pointer).  Host memory. */
zk_status zk_partition_rows(int64_t n, const int64_t* row_ptr, int32_t nranks, int64_t* offsets);

/* Halo plan of rank `rank` whose block is rows [offsets[rank], offsets[rank+1]):
 * the distinct off-rank GLOBAL column ids its nnz entries reference, sorted ascending (so grouped
 * by owner), and how many of them each rank owns.
 *   col            int32[nnz] global column ids of this rank's rows (host).
 *   offsets        int64[nranks+1] row ranges of all ranks (host).
 *   n_ext          out: number of distinct off-rank columns.
 *   ext_cols       out (may be NULL to query n_ext): int32[n_ext] sorted.
 *   count_per_rank out (may be NULL): int64[nranks], count_per_rank[rank] = 0.
 * Errors: ZK_ERR_INVALID_VALUE (NULL, bad rank), ZK_ERR_INVALID_CSR (column outside [0, offsets[nranks])). */
zk_status zk_halo_plan(int64_t nnz, const int32_t* col, int32_t nranks, int32_t rank, const int64_t* offsets,
                       int64_t* n_ext, int32_t* ext_cols, int64_t* count_per_rank);

/* Local renumbering: col_local[p] = col[p] − row_begin for owned columns, n_rows + k for the
 * k-th entry of ext_cols (the halo slot the exchange fills).  Host memory; col_local may alias col. */
zk_status zk_halo_renumber(int64_t nnz, const int32_t* col, int64_t row_begin, int64_t n_rows, int64_t n_ext,
                           const int32_t* ext_cols, int32_t* col_local);

#ifdef __cplusplus
}
#endif
#endif /* ZK_DIST_H */
