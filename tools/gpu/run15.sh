set -x
python __graft_entry__.py build
timeout 1200 python -m pytest tests/test_gpu_solve.py -q -k "cluster" 2>&1 | tail -5
for mg in 0 1; do ZK_CLUSTER_MERGE=$mg timeout 600 python tools/latency_probe.py --cfgs C1,T0,C2 --modes 5 2>&1 | tail -3; done
