set -x
python __graft_entry__.py build
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -8
ZK_LOOP_MODE=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_launches_r2.csv python tools/solve_target.py C3 bicgstab 10 2 > /dev/null 2>&1; echo ncu rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
