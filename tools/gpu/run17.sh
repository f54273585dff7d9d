set -x
python __graft_entry__.py build
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -8
timeout 1200 python bench.py > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; echo bench rc=$?; tail -2 gpurun_out/bench_r2d.err
