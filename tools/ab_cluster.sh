# cluster-solver A/B: the in-tree libzk vs a variant build (VARIANT=path/to/variant.so) on the
# paper's small shapes (METHOD: bicgstab by default)
# Variants: python -m paper_2112_11880_b200.build --out paper_2112_11880_b200/variants/X.so -D MACRO=VALUE
for r in 1 2; do
python tools/latency_probe.py --cfgs C1,T0,C2 --modes 5 --method ${METHOD:-bicgstab}
ZK_LIB=${VARIANT:?set VARIANT=path/to/variant.so} python tools/latency_probe.py --cfgs C1,T0,C2 --modes 5 --method ${METHOD:-bicgstab}
done
