set -x
python __graft_entry__.py build
timeout 900 python -m pytest tests/test_gpu_dist_local.py -q 2>&1 | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/solve_target.py C3 bicgstab 10 2 > gpurun_out/c3_launches.log 2>&1; echo ncu rc=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-shapes > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo bench rc=$?; tail -3 gpurun_out/bench_r2a.err
