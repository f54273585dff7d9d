# A/B: the in-tree libzk vs a variant build (VARIANT=path/to/variant.so), tools/ab_lib.py on
# ${AB_CFGS:-C3 C3T C4} with ${AB_METHODS:-bicgstab,cg,tfqmr}, alternating, twice
# Variants: python -m paper_2112_11880_b200.build --out paper_2112_11880_b200/variants/X.so -D MACRO=VALUE
export AB_METHODS=${AB_METHODS:-bicgstab,cg,tfqmr}
for r in 1 2; do
ZK_LIB=${VARIANT:?set VARIANT=path/to/variant.so} python tools/ab_lib.py ${AB_CFGS:-C3 C3T C4}
python tools/ab_lib.py ${AB_CFGS:-C3 C3T C4}
done
