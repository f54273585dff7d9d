set -x
for w in 2 4 8; do ZK_CLUSTER_W=$w timeout 600 python tools/latency_probe.py --cfgs C1,T0,C2 --modes 5 2>&1 | tail -3; done
for vs in 0 1; do ZK_CLUSTER_VS=$vs timeout 600 python tools/latency_probe.py --cfgs C1,T0 --modes 5 2>&1 | tail -2; done
