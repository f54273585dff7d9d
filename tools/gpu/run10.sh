set -x
mkdir -p gpurun_out/san
python __graft_entry__.py build
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_tfqmr.py -q -k "single_rank or c5 or update_values" 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_blas.py -q -k "update_values" 2>&1 | tail -3
SAN_MODES=3,5 ZK_PDL=0 SAN_MAXIT=12 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/racecheck_m35.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/racecheck_m35.txt
SAN_MODES=1,2 SAN_MAXIT=12 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/racecheck_m12.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/racecheck_m12.txt
timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 --no-shapes > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench rc=$?; tail -3 gpurun_out/bench_c5.err
