set -x
mkdir -p gpurun_out/san
python __graft_entry__.py build
timeout 900 python -m pytest tests/test_gpu_dist_local.py -q 2>&1 | tail -30
SAN_MODES=2 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/memcheck_m2.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/memcheck_m2.txt
ZK_PDL=0 SAN_MODES=1 SAN_SPLIT=0 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 --show-backtrace device python tools/sanitize_target.py C1 > gpurun_out/san/memcheck_m1_b.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/memcheck_m1_b.txt
ZK_PDL=0 SAN_MODES=1 SAN_SPLIT=0 timeout 600 python tools/sanitize_target.py C1 > gpurun_out/san/nosan_m1.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/nosan_m1.txt
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -15
