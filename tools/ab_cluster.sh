# cluster-solver A/B: the in-tree libzk vs a variant build (ZK_LIB=...) on the paper's small shapes
for r in 1 2; do
python tools/latency_probe.py --cfgs C1,T0,C2 --modes 5
ZK_LIB=${VARIANT:?set VARIANT=path/to/variant.so} python tools/latency_probe.py --cfgs C1,T0,C2 --modes 5
done
