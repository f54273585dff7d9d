# A/B of the zero-copy readback of cluster solves (ZK_ZERO_COPY=0 keeps the D2H copy)
for r in 1 2; do
ZK_ZERO_COPY=0 python tools/host_overhead.py; python tools/host_overhead.py
ZK_ZERO_COPY=0 python tools/latency_probe.py --cfgs C1,C2 --modes 5; python tools/latency_probe.py --cfgs C1,C2 --modes 5
done
