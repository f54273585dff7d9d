set -x
mkdir -p gpurun_out/san
python __graft_entry__.py build
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -8
ZK_LOOP_MODE=3 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/solve_target.py C4 bicgstab 20 1 > gpurun_out/c4_launches.log 2>&1; echo ncu1 rc=$?
ZK_LOOP_MODE=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_bicg -s 4 -c 1 -o gpurun_out/k1_bicg_c4_full -f python tools/solve_target.py C4 bicgstab 10 1 > gpurun_out/k1_full.log 2>&1; echo ncu2 rc=$?
timeout 1200 python bench.py > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err; echo bench rc=$?; tail -2 gpurun_out/bench_r2c.err
