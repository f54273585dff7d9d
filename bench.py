#!/usr/bin/env python
"""bench.py — the hot path of arXiv 2112.11880 on B200: one step = one device-resident BiCGStab
solve to 1e-8 (x0 = 0) of the C4 synthetic 27-point Q1-hex complex Helmholtz system
(unit-cube interior 200³: n = 8,000,000, nnz = 213,847,192; BASELINE.json configs[3]) through
libzk's C-ABI: every step runs ZSpMV (fused K1/K3), the fused BLAS-1 updates with zdotc/dznrm2
reductions (K2/K4/K5) and the device-resident driver, plus the final true-residual SpMV.

value  = counted (algorithmic) bytes of the step ÷ device time  [GB/s], whole job over N GPUs.
         Per step: iters·(2·Mat + 304n) + 80n (init) + Mat + 32n (true residual),
         Mat = 20·nnz + 8·(n+1)   (paper_2112_11880_b200/metrics.py).
Also printed: BiCGStab ms/iteration and time-to-1e-8, ZSpMV GB/s and GFLOP/s (8 flops/nnz,
PAPER.md T8 convention), roofline of the dominant kernel (the in-loop ZSpMV), the CPU oracle
baseline on a bounded sample, the end-to-end number with host buffers, and SM clocks.

--impl reference runs the CPU oracle (the reference arm of this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "ZSpMV GB/s & GFLOP/s vs HBM roofline; BiCGStab ms/iteration & time-to-1e-8"
FALLBACK_HBM_GBS = 6650.0


def args_():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="zk", choices=["zk", "reference"])
    p.add_argument("--config", default="C4")
    p.add_argument("--method", default="bicgstab", choices=["bicgstab"])
    p.add_argument("--tol", type=float, default=1e-8)
    p.add_argument("--maxit", type=int, default=2000)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--spmv-reps", type=int, default=100)
    p.add_argument("--no-shapes", action="store_true", help="skip the PAPER.md T1-shape latency runs")
    p.add_argument("--no-methods", action="store_true",
                   help="skip the per-method C4 solves (CG, Jacobi-BiCGStab, COCG, TFQMR, BiCGStab(2), BiCGStab(8))")
    p.add_argument("--no-blas1", action="store_true", help="skip the BLAS-1 GB/s sweep")
    p.add_argument("--local-ranks", type=int, default=0,
                   help="run the row-partitioned path on ONE GPU with N in-process ranks (LOCAL transport, "
                        "threads): the C5 z-slab split of the strong-scaling run, timed as max over ranks")
    p.add_argument("--local-config", default=None,
                   help="--local-ranks: the system to split (default C5, the strong-scaling system)")
    p.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                   help="N > 1: strong = the fixed C5 system (400^3, 64M rows; BASELINE.json configs[4]) "
                        "split into z-slabs; weak = a 200x200x(200N) box, 8M rows per GPU")
    return p.parse_args()


# ---------------------------------------------------------------- BLAS-1 sweep (north star: dot-product GB/s)
BLAS1_SIZES = (648_849, 2_000_000, 9_000_000, 14_000_000, 1 << 26, 1 << 28)  # PAPER.md T2-T7 h + B200 sizes


def blas1_sweep(zk, torch, dev, stream, peak, read_gbs, reps=10):
    """zdotc, dznrm2, zaxpy, zscal, zassign, zaxmy GB/s (algorithmic bytes, metrics.blas1_bytes) at
    the paper's vector lengths (T2-T7: 648,849 / 2M / 9M / 14M) and at 64M / 256M elements.  Each
    rep: a 512 MB L2 flush by READING a buffer (outside the timed pair: L2 is left full of clean
    lines, so the timed call pays no write-back of the flush's own data), then CUDA events around
    the one call on its stream; the median rep is reported."""
    from paper_2112_11880_b200 import metrics as M
    flush = torch.ones(1 << 27, dtype=torch.float32, device=dev)
    out = {}
    res_c = torch.empty(1, dtype=torch.complex128, device=dev)
    res_d = torch.empty(1, dtype=torch.float64, device=dev)
    for n in BLAS1_SIZES:
        x = torch.full((n,), 0.5 - 0.25j, dtype=torch.complex128, device=dev)
        y = torch.full((n,), 0.125 + 1j, dtype=torch.complex128, device=dev)
        ops = {"zdotc": lambda: zk.zdotc(x, y, res_c, stream=stream),
               "dznrm2": lambda: zk.dznrm2(x, res_d, stream=stream),
               "zaxpy": lambda: zk.zaxpy(1e-3, x, y, stream=stream),
               "zscal": lambda: zk.zscal(1.0 + 0j, y, stream=stream),
               "zassign": lambda: zk.zassign(0.5 - 0.25j, y, stream=stream),
               "zaxmy": lambda: zk.zaxmy(x, y, stream=stream)}
        row = {}
        for name, f in ops.items():
            f()
            ts = []
            for _ in range(reps):
                with torch.cuda.stream(stream):
                    flush.sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                f()
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            gbs = M.blas1_bytes(name, n) / (ms * 1e-3) / 1e9
            row[name] = {"us": round(1e3 * ms, 2), "gbs": round(gbs, 1), "frac_of_copy_peak": round(gbs / peak, 3),
                         "frac_of_read_stream": round(gbs / read_gbs, 3), "frac_of_8tbs_spec": round(gbs / 8000.0, 3),
                         "gflops": round(M.FLOPS_PER_ELEM[name] * n / (ms * 1e-3) / 1e9, 1)}
        out[str(n)] = row
        del x, y
    del flush
    return {"sizes": out, "l2": "512 MB read (clean-line L2 flush) before every timed call", "reps": reps, "stat": "median",
            "headline_zdotc_gbs_256M": out[str(1 << 28)]["zdotc"]["gbs"]}


def workload_name(cfg: str, spec) -> str:
    if cfg in ("C4", "C5"):
        return f"{cfg}: scaled 27-point Q1-hex complex Helmholtz, unit-cube interior {spec.nx}^3 (n={spec.n:,})"
    return f"{cfg}: PAPER.md T1-shaped synthetic complex Helmholtz {spec.nx}x{spec.ny}x{spec.nz} + {spec.pad} pad"


def step_bytes(n: int, nnz: int, iters: int) -> int:
    from paper_2112_11880_b200 import metrics as M
    return iters * M.bicgstab_iter_bytes(n, nnz) + 5 * 16 * n + M.csr_bytes(n, nnz) + 32 * n


# ---------------------------------------------------------------- clocks (during the timed region)
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        time.sleep(0.3)

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.count(",") >= 6]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].strip() == "Active"})
        busy = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg: str):
    """profiles/ncu_traffic.json[cfg]: DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and
    duration per in-loop SpMV launch from the ncu launch list of this bench command (cold-cache,
    serialised), or None for a config without a capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(cfg)
        if d:
            return d
    return None


# ---------------------------------------------------------------- CPU oracle (reference arm / baseline)
def oracle_sample(mat, b, maxit: int):
    """The oracle as it stands, single-threaded: BiCGStab capped at `maxit` iterations."""
    import oracle
    t = time.perf_counter()
    r = oracle.bicgstab(mat, b, tol=1e-8, maxit=maxit)
    dt = time.perf_counter() - t
    return r, dt


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import gen
    world = int(os.environ.get("WORLD_SIZE", "1"))
    scaling = "weak"
    if world > 1 and a.scaling == "strong" and a.config == "C4":
        a.config = "C5"  # the N-GPU zk arm's workload: the fixed C5 system (BASELINE.json configs[4])
        scaling = "strong"  # (C5 on rank 0: ~16 s per 1-iteration step, ~45 GB of host memory)
    spec = gen.CONFIGS[a.config]
    mat = gen.make_matrix(spec)
    b = gen.make_rhs(mat)
    n, nnz = mat["n"], mat["nnz"]
    for _ in range(a.warmup):
        oracle_sample(mat, b, 1)
    times, its = [], []
    for _ in range(a.steps):
        r, dt = oracle_sample(mat, b, 1)
        times.append(dt)
        its.append(r["iters"])
    tot = sum(times)
    byts = sum(step_bytes(n, nnz, i) for i in its)
    v = byts / tot / 1e9
    sample = (f"each step: oracle BiCGStab on {a.config} capped at 1 iteration "
              f"(init + 2 SpMV + fused-vector work + true-residual SpMV), single thread")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "complex128 (f64)", "data": "synthetic",
            "config": {"workload": workload_name(a.config, spec), "n": n, "nnz": nnz, "method": "bicgstab",
                       "tol": 1e-8, "parallelism": "cpu oracle, 1 thread"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- the zk arm
def run_local_ranks(a):
    """The strong-scaling partition (C5 split into N z-slabs) on ONE GPU through the LOCAL transport:
    N host threads, one stream and one rank each, halo exchange overlapped with the interior rows,
    rank-order allreduces.  Not a scaling number (the ranks share one GPU's HBM): it measures the
    row-partitioned loop at full size against the same system on one rank."""
    import threading

    import torch

    import gen
    from paper_2112_11880_b200 import metrics as M
    from paper_2112_11880_b200 import zk
    N = a.local_ranks
    cfg = a.local_config or ("C5" if a.config == "C4" else a.config)
    spec = gen.CONFIGS[cfg]
    plane = spec.nx * spec.ny
    group = zk.LocalGroup(N)
    out, errs = [None] * N, [None] * N
    ready = threading.Barrier(N)

    def rank(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                comm = zk.Comm.local(group, r, 0)
                z0, z1 = r * spec.nz // N, (r + 1) * spec.nz // N
                mat = gen.make_matrix(spec, row_range=(z0 * plane, z1 * plane))
                b = torch.from_numpy(gen.make_rhs(mat)).cuda()
                A = zk.csr_create(mat["row_ptr"], mat["col_idx"], mat["values"], spec.n, comm=comm,
                                  row_begin=mat["row_begin"], stream=st)
                n, nnz = len(mat["row_ptr"]) - 1, mat["nnz"]
                del mat
                ws = zk.alloc_workspace(A, "bicgstab", a.maxit)
                x = torch.empty_like(b)
                for _ in range(max(a.warmup, 1)):
                    zk.solve(A, b, None, a.tol, a.maxit, "bicgstab", x=x, workspace=ws, stream=st)
                st.synchronize()
                ready.wait()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                res = [zk.solve(A, b, None, a.tol, a.maxit, "bicgstab", x=x, workspace=ws, stream=st)
                       for _ in range(a.steps)]
                e1.record(st)
                st.synchronize()
                out[r] = dict(ms=e0.elapsed_time(e1), iters=res[-1]["iters"], n=n, nnz=nnz,
                              n_halo=A.info["n_halo"], interior=A.info["interior_rows"],
                              status=res[-1]["status"], true_relres=res[-1]["true_relres"])
                A.close()
            comm.close()
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=rank, args=(r,)) for r in range(N)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    group.close()
    for e in errs:
        if e is not None:
            raise e
    ms = max(q["ms"] for q in out)
    iters = out[0]["iters"]
    byts = sum(step_bytes(q["n"], q["nnz"], q["iters"]) for q in out) * a.steps
    line = {"metric": METRIC, "value": byts / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": 1, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "none (one GPU)",
            "dtype": "complex128 (f64)", "data": "synthetic",
            "config": {"workload": f"{cfg}: {spec.nx}x{spec.ny}x{spec.nz} (n={spec.n:,}) split into {N} z-slabs",
                       "parallelism": f"LOCAL transport: {N} in-process ranks (threads) on one GPU, halo overlapped"},
            "bicgstab": {"iters": iters, "status": out[0]["status"], "ms_per_iteration": ms / a.steps / iters,
                         "true_relres": out[0]["true_relres"]},
            "ranks": [{k: q[k] for k in ("n", "nnz", "n_halo", "interior", "ms", "iters")} for q in out]}
    print(json.dumps(line), flush=True)


def main():
    a = args_()
    if a.impl == "reference":
        return run_reference(a)
    if a.local_ranks > 1:
        return run_local_ranks(a)

    import torch
    import torch.distributed as dist

    import gen
    from paper_2112_11880_b200 import metrics as M
    from paper_2112_11880_b200 import zk

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    zk.lib()

    comm = None
    scaling = "weak"
    if world > 1:
        uid = [zk.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = zk.Comm(uid[0], world, rank, local)
        if a.scaling == "strong":
            # BASELINE.json configs[4]: the fixed C5 system (unit-cube interior 400^3, 64M rows) split
            # into N contiguous z-slabs (rank r: planes [r*400/N, (r+1)*400/N)); NCCL halo + allreduce
            a.config = "C5" if a.config == "C4" else a.config
            spec = gen.CONFIGS[a.config]
            plane = spec.nx * spec.ny
            z0, z1 = rank * spec.nz // world, (rank + 1) * spec.nz // world
            row_range = (z0 * plane, z1 * plane)
            scaling = "strong"
        else:
            # weak scaling: a 200 x 200 x (200*N) box at the C4 spacing, rank r owns the z-slab of
            # rows [r*8M, (r+1)*8M) (exactly C4 at N = 1)
            base = gen.CONFIGS[a.config]
            spec = gen.BoxSpec(base.nx, base.ny, base.nz * world, base.h, base.lam, base.shell, 0)
            plane = spec.nx * spec.ny
            row_range = (rank * base.nz * plane, (rank + 1) * base.nz * plane)
    else:
        spec = gen.CONFIGS[a.config]
        row_range = None
    if a.config == "C5" and world == 1:
        # 64M rows on one GPU: CSR 34.9 GB + its SELL copy + workspace ≈ 78 GB; a second handle
        # (e2e upload, the CG matrix of methods_c4) would not fit beside it
        a.no_e2e = a.no_methods = True
    t_gen = time.perf_counter()
    mat = gen.make_matrix(spec, row_range=row_range)
    b_h = gen.make_rhs(mat)
    t_gen = time.perf_counter() - t_gen
    n_glob = mat["n"]
    n, nnz = len(mat["row_ptr"]) - 1, mat["nnz"]   # this rank's rows / nonzeros

    # inputs resident in HBM; validation + stats (+ halo plan on N > 1) at create (setup)
    b = torch.from_numpy(b_h).to(dev)
    if comm is None:
        rp = torch.from_numpy(mat["row_ptr"]).to(dev)
        ci = torch.from_numpy(mat["col_idx"]).to(dev)
        va = torch.from_numpy(mat["values"]).to(dev)
        A = zk.csr_create(rp, ci, va, n, borrow=True)
    else:
        A = zk.csr_create(mat["row_ptr"], mat["col_idx"], mat["values"], n_glob, comm=comm,
                          row_begin=mat["row_begin"])
    ws = zk.alloc_workspace(A, "bicgstab", a.maxit, dev)
    x = torch.empty_like(b)
    stream = torch.cuda.current_stream()

    def step():
        return zk.solve(A, b, None, a.tol, a.maxit, "bicgstab", x=x, workspace=ws, stream=stream)

    for _ in range(max(a.warmup, 3)):
        r = step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local) if rank == 0 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results = []
    e0.record(stream)
    for _ in range(a.steps):
        results.append(step())
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ck = clocks.stop() if clocks else None
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    iters = results[-1]["iters"]
    assert all(r["iters"] == iters for r in results), "non-deterministic iteration count"
    bytes_step = step_bytes(n, nnz, iters)           # this rank's HBM bytes per step
    if world > 1:
        t = torch.tensor([float(bytes_step)], device=dev, dtype=torch.float64)
        dist.all_reduce(t)                            # units all ranks processed
        bytes_step_all = float(t.item())
    else:
        bytes_step_all = float(bytes_step)
    total_bytes = bytes_step_all * a.steps
    value = total_bytes / (ms * 1e-3) / 1e9
    ms_step = ms / a.steps

    # dominant kernel: the in-loop ZSpMV (K1: Mat+48n, K3: Mat+32n algorithmic bytes), timed by
    # the device global timer inside the timed solves (first block start → last block end)
    k_ms = sum(r["kernel_ms"][0] for r in results)
    k_n = sum(r["kernel_launches"][0] for r in results)
    mat_b = M.csr_bytes(n, nnz)
    spmv_alg = sum(r["kernel_launches"][0] // 2 * (2 * mat_b + 80 * n) for r in results)
    spmv_gbs = spmv_alg / (k_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    roofline = {"bound": "hbm", "achieved": spmv_gbs, "peak": peak, "unit": "GB/s", "frac": spmv_gbs / peak,
                "traffic": (ncu_traffic(a.config) or {}).get("spmv_dram_bytes_per_launch"),
                "kernel": ("in-loop ZSpMV (BiCGStab K1/K3: SELL-32 SpMV with its dot products fused by per-slice "
                           "warp reductions)" if n >= (1 << 20) and comm is None else
                           "in-loop ZSpMV (BiCGStab K1/K3: SELL-32 SpMV, its dot products in the same kernel's tail)"
                           if n >= (1 << 18) and comm is None else
                           "in-loop ZSpMV (BiCGStab K1/K3: interior + boundary SELL launches around the halo "
                           "exchange, then the reduction pass)" if comm is not None else
                           "in-loop ZSpMV (BiCGStab K1/K3, fused epilogues)"),
                "launch_us": 1e3 * k_ms / max(k_n, 1), "bytes_per_launch": spmv_alg / max(k_n, 1),
                "peak_source": peak_src,
                "share_of_step": k_ms / ms}
    vec_ms = sum(r["kernel_ms"][1] for r in results)

    # standalone zk_zcsrmv (β = 0) with CUDA events on the launching stream: GB/s and GFLOP/s
    # (on N > 1 it includes the halo copy + exchange of zk_zcsrmv's distributed path)
    y = torch.empty_like(b)
    for _ in range(3):
        zk.zcsrmv(A, 1.0, b, 0.0, y, stream)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.spmv_reps + 1)]
    evs[0].record(stream)
    for i in range(a.spmv_reps):                     # back to back; per-launch events
        zk.zcsrmv(A, 1.0, b, 0.0, y, stream)
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    per = sorted(1e3 * evs[i].elapsed_time(evs[i + 1]) for i in range(a.spmv_reps))
    spmv_us = 1e3 * evs[0].elapsed_time(evs[-1]) / a.spmv_reps
    # measured read-only stream peak (SURVEY.md §8(d) "Reporting"): zk_dznrm2 over a 4 GiB vector
    big = torch.ones(1 << 28, dtype=torch.complex128, device=dev)
    for _ in range(2):
        zk.dznrm2(big, stream=stream)
    q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    q0.record(stream)
    for _ in range(10):
        zk.dznrm2(big, stream=stream)
    q1.record(stream)
    torch.cuda.synchronize()
    read_gbs = 16.0 * (1 << 28) * 10 / (q0.elapsed_time(q1) * 1e-3) / 1e9
    del big
    roofline["read_stream_gbs"] = read_gbs
    roofline["frac_of_8tbs_spec"] = spmv_gbs / 8000.0  # also against the 8.0 TB/s spec
    nt = ncu_traffic(a.config)
    if nt and nt.get("duration_us_per_launch"):
        # ncu-measured DRAM GB/s of the same kernel (cold-cache, serialised launches)
        roofline["ncu_dram_gbs"] = nt["spmv_dram_bytes_per_launch"] / (nt["duration_us_per_launch"] * 1e-6) / 1e9
        roofline["ncu_dram_frac"] = roofline["ncu_dram_gbs"] / peak
        roofline["ncu_dram_frac_of_8tbs_spec"] = roofline["ncu_dram_gbs"] / 8000.0
        roofline["ncu_source"] = nt.get("source")
    roofline["frac_of_read_stream"] = spmv_gbs / read_gbs
    spmv = {"us": spmv_us, "us_median": per[len(per) // 2], "us_min": per[0], "reps": a.spmv_reps,
            "gbs": M.spmv_bytes(n, nnz) / (spmv_us * 1e-6) / 1e9,
            "frac_of_read_stream": M.spmv_bytes(n, nnz) / (spmv_us * 1e-6) / 1e9 / read_gbs,
            "gflops": M.spmv_flops(nnz) / (spmv_us * 1e-6) / 1e9,
            "frac_of_peak": M.spmv_bytes(n, nnz) / (spmv_us * 1e-6) / 1e9 / peak,
            "frac_of_8tbs_spec": M.spmv_bytes(n, nnz) / (spmv_us * 1e-6) / 1e9 / 8000.0,
            "lanes_per_row": A.info["lanes_per_row"],
            "mapping": {0: "CSR sub-warp",
                        3: "sliced ELL (SELL-32 device copy)"}[A.info["spmv_mode"]],
            "stored_entries": A.info["sell_entries"] or nnz}

    blas1 = None
    if world == 1 and not a.no_blas1:
        blas1 = blas1_sweep(zk, torch, dev, stream, peak, read_gbs)

    # the paper's own matrix shapes (PAPER.md T1; latency-bound on B200): BiCGStab per iteration
    shapes = None
    if world == 1 and not a.no_shapes:
        shapes = {}
        for cfg in ("C1", "C2", "C3", "C3T"):
            ms_ = gen.make_matrix(cfg)
            As = zk.csr_create(ms_["row_ptr"], ms_["col_idx"], ms_["values"], ms_["n"])
            bs = torch.from_numpy(gen.make_rhs(ms_)).to(dev)
            wss = zk.alloc_workspace(As, "bicgstab", a.maxit, dev)
            for _ in range(2):
                rs_ = zk.solve(As, bs, None, a.tol, a.maxit, "bicgstab", workspace=wss, stream=stream)
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(5):
                rs_ = zk.solve(As, bs, None, a.tol, a.maxit, "bicgstab", workspace=wss, stream=stream)
            g1.record(stream)
            torch.cuda.synchronize()
            t_ms = g0.elapsed_time(g1) / 5
            shapes[cfg] = {"n": ms_["n"], "nnz": ms_["nnz"], "iters": rs_["iters"], "time_to_tol_ms": t_ms,
                           "us_per_iteration": 1e3 * t_ms / max(rs_["iters"], 1),
                           "gbs": step_bytes(ms_["n"], ms_["nnz"], rs_["iters"]) / (t_ms * 1e-3) / 1e9}
            As.close()

    # PAPER.md T9/T10 context: the paper's three solvers (P-BiCGSTAB → Jacobi-BiCGStab, P-TFQMR →
    # TFQMR, P-BiCGSTAB(8) → BiCGStab(8)) at the paper's tol 1e-9, x0 = 0 (reading L10) on
    # the T1 shapes; iteration counts are not comparable (synthetic matrices, L8), per-iteration times
    # are shown beside the paper's derived K20c ms/iteration
    table9 = None
    if world == 1 and not a.no_shapes:
        table9 = {}
        k20c = {"C1": 1.43, "C2": 2.00, "T0": 1.79, "C3": 50.3, "C3T": 37.7}  # P-BiCGSTAB ms/iter (T9/T10, derived)
        for cfg in ("C1", "T0", "C2", "C3", "C3T"):
            ms_ = gen.make_matrix(cfg)
            As = zk.csr_create(ms_["row_ptr"], ms_["col_idx"], ms_["values"], ms_["n"])
            bs = torch.from_numpy(gen.make_rhs(ms_)).to(dev)
            row = {"n": ms_["n"], "nnz": ms_["nnz"], "k20c_p_bicgstab_ms_per_iter": k20c[cfg]}
            for meth, ell, key in (("bicgstab_jacobi", 8, "p_bicgstab"), ("tfqmr", 8, "tfqmr"),
                                   ("bicgstab_l", 8, "bicgstab8")):
                wss = zk.alloc_workspace(As, meth, 1000, dev, ell)
                rs_ = zk.solve(As, bs, None, 1e-9, 1000, meth, workspace=wss, stream=stream, ell=ell)
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                for _ in range(3):
                    rs_ = zk.solve(As, bs, None, 1e-9, 1000, meth, workspace=wss, stream=stream, ell=ell)
                g1.record(stream)
                torch.cuda.synchronize()
                t_ms = g0.elapsed_time(g1) / 3
                row[key] = {"iters": rs_["iters"], "status": rs_["status"], "time_to_tol_ms": t_ms,
                            "ms_per_iteration": t_ms / max(rs_["iters"], 1), "loop_mode": rs_["loop_mode"]}
                del wss
            table9[cfg] = row
            As.close()

    # the other solvers of the path on the same C4 system, after the timed
    # region: per-iteration time and counted GB/s of their fused kernels (one warm-up + 2 timed solves)
    methods = None
    if world == 1 and not a.no_methods:
        methods = {}
        # CG (A7) needs Hermitian positive definite A: the gauge-twisted eta = 0 version of the same
        # box (reading L9), same n / nnz / pattern
        mg = gen.make_matrix(spec, eta=0.0, twist_seed=gen.SEED_TWIST)
        bg = torch.from_numpy(np.exp(1j * mg["phase"]) * gen.make_rhs(mg)).to(dev)
        Ag = zk.csr_create(torch.from_numpy(mg["row_ptr"]).to(dev), torch.from_numpy(mg["col_idx"]).to(dev),
                           torch.from_numpy(mg["values"]).to(dev), n, stream=stream)
        del mg
        wsg = zk.alloc_workspace(Ag, "cg", a.maxit, dev)
        rm = zk.solve(Ag, bg, None, a.tol, a.maxit, "cg", workspace=wsg, stream=stream)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(2):
            rm = zk.solve(Ag, bg, None, a.tol, a.maxit, "cg", workspace=wsg, stream=stream)
        h1.record(stream)
        torch.cuda.synchronize()
        t_ms = h0.elapsed_time(h1) / 2
        its = max(rm["iters"], 1)
        gbs = M.cg_iter_bytes(n, nnz) * its / (t_ms * 1e-3) / 1e9
        methods["cg_twisted_hpd"] = {"status": rm["status"], "iters": rm["iters"], "time_to_tol_ms": t_ms,
                                     "ms_per_iteration": t_ms / its, "bytes_per_iteration": M.cg_iter_bytes(n, nnz),
                                     "iter_gbs": gbs, "frac_of_peak": gbs / peak, "true_relres": rm["true_relres"],
                                     "spmv_launch_us": 1e3 * rm["kernel_ms"][0] / max(rm["kernel_launches"][0], 1)}
        Ag.close()
        del wsg, bg
        runs = [("bicgstab_jacobi", 0, M.bicgstab_iter_bytes(n, nnz)), ("cocg", 0, M.cocg_iter_bytes(n, nnz)),
                ("tfqmr", 0, M.tfqmr_iter_bytes(n, nnz)),
                ("bicgstab_l", 2, M.bicgstab_l_cycle_bytes(n, nnz, 2)),
                ("bicgstab_l", 8, M.bicgstab_l_cycle_bytes(n, nnz, 8))]
        for meth, ell, it_bytes in runs:
            wsm = zk.alloc_workspace(A, meth, a.maxit, dev, ell=ell or 8)
            rm = zk.solve(A, b, None, a.tol, a.maxit, meth, workspace=wsm, stream=stream, ell=ell or 8)
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            for _ in range(2):
                rm = zk.solve(A, b, None, a.tol, a.maxit, meth, workspace=wsm, stream=stream, ell=ell or 8)
            h1.record(stream)
            torch.cuda.synchronize()
            t_ms = h0.elapsed_time(h1) / 2
            its = max(rm["iters"], 1)
            gbs = it_bytes * its / (t_ms * 1e-3) / 1e9
            key = f"bicgstab({ell})" if meth == "bicgstab_l" else meth
            methods[key] = {"status": rm["status"], "iters": rm["iters"], "time_to_tol_ms": t_ms,
                            "ms_per_iteration": t_ms / its, "bytes_per_iteration": it_bytes, "iter_gbs": gbs,
                            "frac_of_peak": gbs / peak, "true_relres": rm["true_relres"],
                            "spmv_launch_us": 1e3 * rm["kernel_ms"][0] / max(rm["kernel_launches"][0], 1)}
            del wsm

    # end to end through the public API with HOST buffers (pinned): CSR upload + b H2D + solve + x D2H
    e2e = None
    if not a.no_e2e:
        rp_h = torch.from_numpy(mat["row_ptr"]).pin_memory()
        ci_h = torch.from_numpy(mat["col_idx"]).pin_memory()
        va_h = torch.from_numpy(mat["values"]).pin_memory()
        b_pin = torch.from_numpy(b_h).pin_memory()
        x_h = torch.empty(n, dtype=torch.complex128).pin_memory()
        ws2 = zk.alloc_workspace(A, "bicgstab", a.maxit, dev)

        def e2e_step():
            if comm is None:
                Ah = zk.csr_create(rp_h, ci_h, va_h, n, stream=stream)
            else:
                Ah = zk.csr_create(rp_h, ci_h, va_h, n_glob, comm=comm, row_begin=mat["row_begin"], stream=stream)
            bd = b_pin.to(dev, non_blocking=True)
            re = zk.solve(Ah, bd, None, a.tol, a.maxit, "bicgstab", workspace=ws2, stream=stream)
            x_h.copy_(re["x"], non_blocking=True)
            Ah.close()

        e2e_step()  # untimed warm-up: first-use costs (device memory pool growth, CUDA-graph build)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(a.e2e_steps):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        e_ms = f0.elapsed_time(f1) / a.e2e_steps
        h2d = 8 * (n + 1) + 4 * nnz + 16 * nnz + 16 * n
        d2h = 16 * n + 8 * (a.maxit + 1)
        e2e = {"value": bytes_step_all / (e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world}
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["ms_per_step"] = float(t.item())
            e2e["value"] = bytes_step_all / (e2e["ms_per_step"] * 1e-3) / 1e9

    cpu = cpu_all = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        rr, dt = oracle_sample(mat, b_h, 3)
        cb = step_bytes(n, nnz, rr["iters"])
        cpu = {"value": cb / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"oracle BiCGStab on {a.config} capped at 3 iterations (+ init and true-residual SpMV), "
                         f"single thread, {dt:.1f} s", "ms_per_iteration": 1e3 * dt / max(rr["iters"], 1)}
        # all host cores (SURVEY.md §8(d) "CPU oracle timing" (ii)): the same oracle source built with
        # -fopenmp, its per-row / per-element loops split over the affinity set (same bits)
        import oracle
        cores = len(os.sched_getaffinity(0))
        os.environ["OMP_NUM_THREADS"] = str(cores)
        oracle.use_all_cores(True)
        try:
            rr, dt = oracle_sample(mat, b_h, 10)
        finally:
            oracle.use_all_cores(False)
        cb = step_bytes(n, nnz, rr["iters"])
        cpu_all = {"value": cb / dt / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle (OpenMP build)",
                   "sample": f"oracle BiCGStab on {a.config} capped at 10 iterations, liboracle_omp.so "
                             f"(SpMV rows and vector updates over {cores} threads, dots sequential), {dt:.1f} s",
                   "ms_per_iteration": 1e3 * dt / max(rr["iters"], 1)}

    if rank == 0:
        r = results[-1]
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "complex128 (f64)", "data": "synthetic",
            "config": {"workload": workload_name(a.config, spec) if world == 1 else
                       f"{a.config}: 27-point Q1-hex complex Helmholtz box {spec.nx}x{spec.ny}x{spec.nz} "
                       f"(n={n_glob:,}), {scaling} scaling, z-slab row blocks of {n:,} rows on rank 0",
                       "n": n_glob, "nnz_rank0": nnz, "method": "bicgstab",
                       "tol": a.tol, "x0": "zero",
                       "l2": f"inputs larger than L2 (matrix {M.csr_bytes(n, nnz) / 1e9:.1f} GB per GPU)",
                       "parallelism": "1 GPU" if world == 1 else
                       f"row-partitioned x{world}: NCCL halo exchange per SpMV + allreduce per reduction point"},
            "bicgstab": {"iters": iters, "status": r["status"], "ms_per_iteration": ms_step / iters,
                         "time_to_tol_ms": ms_step, "true_relres": r["true_relres"], "loop_mode": r["loop_mode"],
                         "bytes_per_iteration": M.bicgstab_iter_bytes(n, nnz),
                         "iter_gbs": M.bicgstab_iter_bytes(n, nnz) * iters / (ms_step * 1e-3) / 1e9,
                         "spmv_share_of_solve": k_ms / sum(q["solve_ms"] for q in results),
                         "vector_kernels_ms_per_iter": vec_ms / a.steps / iters},
            "spmv": spmv,
            "paper_shapes_bicgstab": shapes,
            "paper_table9_solvers_tol1e-9": table9,
            "methods_c4": methods,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "cpu_baseline_all_cores": cpu_all,
            "blas1": blas1,
            "e2e": e2e,
            "clocks": ck,
            "gpu_launches": sum(q["gpu_launches"] for q in results) + 0,
            "paper_context": "PAPER.md P:7: up to 28x dot, 9.8x SpMV/solvers (i7-920 vs Tesla K20c / GTX 570); "
                             "K20c ZSpMV 6.74 GFLOP/s on Audi3D-4 (T8 P:297)",
            "setup_s": {"generate": t_gen},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
