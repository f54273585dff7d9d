set -x
python __graft_entry__.py build
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_tfqmr.py -q -k "split" 2>&1 | tail -5
timeout 900 python tools/ab_split.py C3 C3T C4 2>&1 | tee gpurun_out/ab_split.txt
for t in 0 1; do ZK_SPLIT_TAIL=$t ZK_LOOP_MODE=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_launches_tail$t.csv python tools/solve_target.py C3 bicgstab 10 2 > /dev/null 2>&1; echo ncu rc=$?; done
