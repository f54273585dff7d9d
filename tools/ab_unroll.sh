# A/B: iterations per WHILE-graph body (ZK_WHILE_UNROLL; the default is solve.cu kWhileUnroll)
export AB_METHODS=${AB_METHODS:-bicgstab,cg,tfqmr}
for r in 1 2; do
for u in ${AB_UNROLLS:-1 2 4}; do echo "UNROLL=$u"; ZK_WHILE_UNROLL=$u python tools/ab_lib.py ${AB_CFGS:-C3 C3T}; done
done
