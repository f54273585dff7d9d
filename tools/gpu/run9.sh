set -x
python __graft_entry__.py build
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -15
SAN_MODES=3,5 ZK_PDL=0 SAN_MAXIT=12 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/racecheck_m35.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/racecheck_m35.txt
SAN_MODES=1,2 SAN_MAXIT=12 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_target.py C1 > gpurun_out/san/racecheck_m12.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san/racecheck_m12.txt
