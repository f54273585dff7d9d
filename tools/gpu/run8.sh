set -x
python __graft_entry__.py build
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
ZK_TRACE=1 timeout 600 python tools/e2e_probe.py 2>&1 | tee gpurun_out/e2e_probe2.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench rc=$?; tail -3 gpurun_out/bench_r2b.err
