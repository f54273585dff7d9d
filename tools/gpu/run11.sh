set -x
mkdir -p gpurun_out/san
python __graft_entry__.py build
AB_TAILS=1,2 timeout 900 python tools/ab_split.py C3 C3T C4 2>&1 | tee gpurun_out/ab_wacc.txt
ZK_PDL=0 SAN_MODES=1,2 SAN_MAXIT=12 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/racecheck_m12_nopdl.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/racecheck_m12_nopdl.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-shapes --no-methods --no-e2e --no-cpu-baseline > gpurun_out/bench_blas1.json 2> gpurun_out/bench_blas1.err; echo bench rc=$?
