set -x
python __graft_entry__.py build
timeout 900 python -m pytest tests/test_gpu_dist_local.py -q -k "c4_zslabs" 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1
timeout 900 python tools/latency_probe.py 2>&1 | tail -30
