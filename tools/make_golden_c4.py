"""Write tests/golden/c4_oracle.json: the CPU oracle's solves of the full-size C4 system
(BASELINE.json configs[3], the bench workload), so the GPU test can check the iteration-count
envelope, a residual-history prefix and a seeded sample of x at full size (VERDICT r1 "Next" 2).

Calls only oracle/ (the plain C oracle) and gen/ (seeded inputs).  Runs the solves in threads
(ctypes releases the GIL); about 10-15 min on 8 cores.

  BiCGStab (O6) on C4, tol 1e-8, orders seq / rev / block-256   (L11 envelope)
  CG (O7) on the gauge-twisted HPD C4 (eta = 0, L9), orders seq / rev / block-256
  TFQMR and COCG on C4 (seq order; NEXT-2 / NEXT-4)

With --bl: tests/golden/c4_oracle_bicgstab_l.json, BiCGStab(2) and BiCGStab(8) (NEXT-3) under the three
orders (cycles, history, x sample).

With --tight: tests/golden/c4_oracle_tol1e-10.json, BiCGStab at tol 1e-10 (orders seq / rev), the
L12 optional mode "run both sides at tol 1e-10 and require 1e-6 agreement there" (at tol 1e-8 the
oracle's own orders disagree by 1e-5 on x at C4, κ = 6.1e3).
"""
from __future__ import annotations

import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c4_oracle.json")
ORDERS = {"seq": oracle.ORD_SEQ, "rev": oracle.ORD_REV, "block256": oracle.ORD_BLOCK256}


def sample_idx(n: int) -> np.ndarray:
    rng = np.random.default_rng(7)
    idx = set(rng.choice(n, size=64, replace=False).tolist()) | {0, n // 2, n - 1}
    return np.array(sorted(idx), dtype=np.int64)


def summarise(r: dict, idx: np.ndarray, t: float) -> dict:
    x = r["x"]
    return dict(status=r["status"], iters=int(r["iters"]), hist=[float(h) for h in r["hist"]],
                true_relres=float(r["true_relres"]), xnorm=float(np.linalg.norm(x)),
                x_sample_re=[float(v) for v in x[idx].real], x_sample_im=[float(v) for v in x[idx].imag],
                seconds=round(t, 1))


def main(tight=False, extra=False, bl=False):
    m = gen.make_matrix("C4")
    b = gen.make_rhs(m)
    mg = gen.make_matrix("C4", eta=0.0, twist_seed=gen.SEED_TWIST)
    bg = np.exp(1j * mg["phase"]) * gen.make_rhs(mg)
    idx = sample_idx(m["n"])
    jobs = []
    if tight:
        mg = bg = None
        for name in ("seq", "rev"):
            jobs.append((f"bicgstab/{name}", lambda o=ORDERS[name]: oracle.bicgstab(m, b, tol=1e-10, maxit=1000, order=o)))
    for name, o in ([] if tight else ORDERS.items()):
        jobs.append((f"bicgstab/{name}", lambda o=o: oracle.bicgstab(m, b, tol=1e-8, maxit=1000, order=o)))
        jobs.append((f"cg_twisted_hpd/{name}", lambda o=o: oracle.cg(mg, bg, tol=1e-8, maxit=3000, order=o)))
    if bl:
        jobs = [(f"bicgstab_l{ell}/{name}", lambda o=o, ell=ell: oracle.bicgstab_l(m, b, tol=1e-8, maxit=300, ell=ell, order=o))
                for ell in (2, 8) for name, o in ORDERS.items()]
    elif extra:  # the other two orders of TFQMR and COCG, merged into the existing file
        jobs = []
        for name in ("rev", "block256"):
            jobs.append((f"tfqmr/{name}", lambda o=ORDERS[name]: oracle.tfqmr(m, b, tol=1e-8, maxit=1000, order=o)))
            jobs.append((f"cocg/{name}", lambda o=ORDERS[name]: oracle.cocg(m, b, tol=1e-8, maxit=2000, order=o)))
    elif not tight:
        jobs.append(("tfqmr/seq", lambda: oracle.tfqmr(m, b, tol=1e-8, maxit=1000)))
        jobs.append(("cocg/seq", lambda: oracle.cocg(m, b, tol=1e-8, maxit=2000)))
    res = {}

    def run(key, fn):
        t = time.time()
        r = fn()
        res[key] = summarise(r, idx, time.time() - t)
        print(key, r["status"], r["iters"], f"{time.time() - t:.0f}s", flush=True)

    th = [threading.Thread(target=run, args=j) for j in jobs]
    for t in th:
        t.start()
    for t in th:
        t.join()
    out = dict(config="C4", n=int(m["n"]), nnz=int(m["nnz"]), tol=1e-10 if tight else 1e-8, sample_idx=idx.tolist(),
               generator="gen.make_matrix('C4') / make_rhs seed 42; CG: eta=0, twist seed 43, b = e^{i phase} b",
               written_by="tools/make_golden_c4.py (oracle/ only)", results=res)
    path = OUT.replace(".json", "_tol1e-10.json") if tight else OUT.replace(".json", "_bicgstab_l.json") if bl else OUT
    if extra:
        with open(OUT) as f:
            old = json.load(f)
        old["results"].update(res)
        out = old
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main(tight="--tight" in sys.argv, extra="--extra" in sys.argv, bl="--bl" in sys.argv)
