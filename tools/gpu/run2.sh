set -x
mkdir -p gpurun_out/san
python __graft_entry__.py build
timeout 900 python -m pytest tests/test_gpu_dist_local.py -x -q 2>&1 | tail -30
SAN_MODES=3,5 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/memcheck_m35.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/memcheck_m35.txt
ZK_PDL=0 SAN_MODES=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/memcheck_m1_nopdl.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/memcheck_m1_nopdl.txt
SAN_MODES=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/memcheck_m1.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/memcheck_m1.txt
SAN_MODES=3,5 timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/synccheck_m35.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/synccheck_m35.txt
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
