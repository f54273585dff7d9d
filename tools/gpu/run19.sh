set -x
mkdir -p gpurun_out/san
python __graft_entry__.py build
for tail in 1 2; do
  ZK_SPLIT_RED=1 ZK_SPLIT_TAIL=$tail SAN_MODES=3 SAN_SPLIT=1 SAN_MAXIT=12 timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/racecheck_tail$tail.txt 2>&1; echo rc=$?; tail -2 gpurun_out/san/racecheck_tail$tail.txt
  ZK_SPLIT_RED=1 ZK_SPLIT_TAIL=$tail SAN_MODES=3 SAN_SPLIT=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/memcheck_tail$tail.txt 2>&1; echo rc=$?; tail -2 gpurun_out/san/memcheck_tail$tail.txt
  ZK_SPLIT_RED=1 ZK_SPLIT_TAIL=$tail SAN_MODES=3 SAN_SPLIT=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/synccheck_tail$tail.txt 2>&1; echo rc=$?; tail -2 gpurun_out/san/synccheck_tail$tail.txt
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_dist_local.py -q -x -k "C1 and not c4" > gpurun_out/san/memcheck_dist_local.txt 2>&1; echo rc=$?; tail -3 gpurun_out/san/memcheck_dist_local.txt
ZK_LOOP_MODE=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_bicg -s 4 -c 1 -o gpurun_out/k1_bicg_c3_full -f python tools/solve_target.py C3 bicgstab 10 1 > /dev/null 2>&1; echo ncu rc=$?
