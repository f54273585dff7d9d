# cluster-solver A/B: the in-tree libzk vs a variant build (VARIANT=path/to/variant.so) on the
# paper's small shapes (METHOD: bicgstab by default)
for r in 1 2; do
python tools/latency_probe.py --cfgs C1,T0,C2 --modes 5 --method ${METHOD:-bicgstab}
ZK_LIB=${VARIANT:?set VARIANT=path/to/variant.so} python tools/latency_probe.py --cfgs C1,T0,C2 --modes 5 --method ${METHOD:-bicgstab}
done
