"""Multi-process CPU tests (gloo, world_size 2) of the row-partitioned path's host logic
(SURVEY.md §8(e)): libzk's partition and halo-plan functions (include/zk_dist.h, no GPU needed),
the request/send-list exchange and the halo exchange protocol zk_csr_create / dist_halo run over
NCCL — here over gloo — and the reduction combine.  The distributed SpMV assembled from
per-rank local products equals the single-rank product bitwise; distributed dot products
match the global one within the L5 bound."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_2112_11880_b200 import zk


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange(send_lists, recv_counts, rank, world, dtype):
    """Grouped point-to-point exchange (the ncclSend/ncclRecv group of dist.cu) over gloo."""
    out = {}
    reqs = []
    for q in range(world):
        if q == rank:
            continue
        if len(send_lists[q]):
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(send_lists[q])), q))
        if recv_counts[q]:
            buf = torch.empty(int(recv_counts[q]), dtype=dtype)
            out[q] = buf
            reqs.append(dist.irecv(buf, q))
    for r in reqs:
        r.wait()
    return {q: b.numpy() for q, b in out.items()}


def _worker(rank, world, port, spec_name, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        spec = gen.CONFIGS[spec_name] if spec_name in gen.CONFIGS else gen.cube(int(spec_name))
        full = gen.make_matrix(spec)
        n = full["n"]
        offsets = zk.partition_rows(full["row_ptr"], world)
        lo, hi = int(offsets[rank]), int(offsets[rank + 1])
        loc = gen.make_matrix(spec, row_range=(lo, hi))                       # this rank's slab only
        ext, cnt = zk.halo_plan(loc["col_idx"], world, rank, offsets)
        # counts[i][j] = how many entries rank i needs from rank j (allgather of count rows)
        rows = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(rows, torch.from_numpy(cnt))
        counts = torch.stack(rows).numpy()
        send_cnt = counts[:, rank]
        recv_off = np.concatenate([[0], np.cumsum(cnt)])
        need = {qq: ext[recv_off[qq]:recv_off[qq + 1]] for qq in range(world)}
        req = _exchange(need, send_cnt, rank, world, torch.int32)              # requested global ids
        send_idx = {qq: (req[qq].astype(np.int64) - lo) for qq in req}
        for qq, s in send_idx.items():
            assert np.all((s >= 0) & (s < hi - lo))
        col_local = zk.halo_renumber(loc["col_idx"], lo, hi - lo, ext)
        # halo exchange of x (complex128 as 2 float64)
        x = gen.rand_vector(n, 77)
        x_loc = x[lo:hi]
        payload = {qq: np.ascontiguousarray(x_loc[send_idx[qq]]).view(np.float64) for qq in send_idx}
        halo_in = _exchange({qq: payload.get(qq, np.zeros(0)) for qq in range(world)}, 2 * cnt, rank, world,
                            torch.float64)
        xg = np.zeros(hi - lo + len(ext), np.complex128)
        xg[: hi - lo] = x_loc
        for qq, v in halo_in.items():
            xg[hi - lo + recv_off[qq]: hi - lo + recv_off[qq + 1]] = v.view(np.complex128)
        A_loc = dict(row_ptr=loc["row_ptr"], col_idx=col_local, values=loc["values"], n=len(xg))
        y_loc = oracle.zcsrmv(A_loc, xg)
        y_ref = oracle.zcsrmv(full, x)[lo:hi]
        assert np.array_equal(y_loc, y_ref)                                   # same terms, same order
        # reduction point: sum of per-rank partials (the ncclAllReduce of dist.cu)
        yv = gen.rand_vector(n, 78)
        part = oracle.zdotc(x_loc, yv[lo:hi])
        t = torch.tensor([part.real, part.imag], dtype=torch.float64)
        dist.all_reduce(t)
        glob = oracle.zdotc(x, yv)
        assert abs(complex(t[0].item(), t[1].item()) - glob) <= 1e-12 * oracle.dznrm2(x) * oracle.dznrm2(yv)
        q.put((rank, "ok", len(ext), int(loc["nnz"])))
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc(), 0, 0))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("spec_name", ["C2", "24"])
def test_two_rank_halo_spmv_and_reduction(spec_name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, spec_name, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, status, n_ext, nnz in res:
        assert status == "ok", status
        assert n_ext > 0


def test_partition_balanced():
    m = gen.make_matrix("C3")
    for P in (2, 3, 4, 8):
        off = zk.partition_rows(m["row_ptr"], P)
        assert off[0] == 0 and off[-1] == m["n"] and np.all(np.diff(off) > 0)
        per = np.diff(m["row_ptr"][off])
        assert per.max() - per.min() <= 2 * 27


def test_halo_plan_cube_slabs():
    """z-slab blocks of an N³ cube: each rank references exactly the neighbouring planes."""
    N = 10
    spec = gen.cube(N)
    full = gen.make_matrix(spec)
    offsets = np.array([0, 5 * N * N, N ** 3])
    for r in range(2):
        lo, hi = offsets[r], offsets[r + 1]
        loc = gen.make_matrix(spec, row_range=(lo, hi))
        ext, cnt = zk.halo_plan(loc["col_idx"], 2, r, offsets)
        assert len(ext) == N * N and cnt[1 - r] == N * N and cnt[r] == 0
        plane = np.arange(N * N) + (5 * N * N if r == 0 else 4 * N * N)
        assert np.array_equal(ext, plane)
    with pytest.raises(zk.ZkError):
        zk.halo_plan(np.array([0, N ** 3], np.int32), 2, 0, offsets)
