# A/B of the opposite-sweep directions: the in-tree build vs -DZK_SWEEP=0.
# Build the variant first (here, then it travels with gpurun):
#   python -m paper_2112_11880_b200.build --out paper_2112_11880_b200/variants/nosweep.so -D ZK_SWEEP=0
export AB_METHODS=${AB_METHODS:-bicgstab,cg,cocg,tfqmr}
for r in 1 2; do
for lib in paper_2112_11880_b200/variants/nosweep.so paper_2112_11880_b200/libzk.so; do
ZK_LIB=$lib python tools/ab_lib.py ${AB_CFGS:-C3 C3T C4}
done
done
