"""Mutation check of the BiCGStab(l) oracle pins: applies one plausible mistake to a copy of
oracle/zk_oracle.c, rebuilds it under /tmp and runs the bicgstab_l pins against it (they must fail).
Usage: PYTHONPATH=. python tools/mutate_oracle.py {x_uses_rj,g_conj,beta_sign,rho0_nosign,u_update,chol_conj,rr_index}"""
import sys, subprocess, re
import oracle, pytest
src = open("oracle/zk_oracle.c").read()  # run from the repo root: PYTHONPATH=. python tools/mutate_oracle.py NAME
i = src.index("int oracle_bicgstab_l(")
muts = {
 "x_uses_rj": ("cplx a = cmul(gm[j], rp)", "cplx a = cmul(gm[j], rj)"),
 "g_conj": ("cplx s = G[i + 1][0];", "cplx s = G[0][i + 1];"),
 "beta_sign": ("cplx beta = cdiv(cmul(alpha, rho1), rho0);", "cplx beta = cdiv(cmul(alpha, rho1), rho0); beta.re = -beta.re; beta.im = -beta.im;"),
 "rho0_nosign": ("cplx mw = {-omega.re, -omega.im};", "cplx mw = {omega.re, omega.im};"),
 "u_update": ("u0r -= d.re; u0i -= d.im;", "u0r += d.re; u0i += d.im;"),
 "chol_conj": ("cplx cj = {L[j][q].re, -L[j][q].im};", "cplx cj = {L[j][q].re, L[j][q].im};"),
 "rr_index": ("spmv(&A, rr[j], rr[j + 1]);", "spmv(&A, rr[0], rr[j + 1]);"),
}
name = sys.argv[1]
a, b = muts[name]
t = src[i:]
assert a in t, name
m = src[:i] + t.replace(a, b, 1)
open("/tmp/mut.c", "w").write(m)
subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared", "-o", "/tmp/mut.so", "/tmp/mut.c", "-lm"])
oracle._SRC = "/tmp/mut.c"; oracle._SO = "/tmp/mut.so"
rc = pytest.main(["-q", "-x", "tests/test_oracle_solvers.py", "-k", "bicgstab_l", "-p", "no:cacheprovider"])
print("MUTANT", name, "caught" if rc != 0 else "SURVIVED")
