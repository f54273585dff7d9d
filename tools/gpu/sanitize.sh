set -x
mkdir -p gpurun_out/san
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py build
for t in memcheck synccheck initcheck; do timeout 900 compute-sanitizer --tool $t --print-limit 40 python tools/sanitize_target.py C1 > gpurun_out/san/$t.txt 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/san/$t.txt; done
SAN_MAXIT=12 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 40 python tools/sanitize_target.py C1 > gpurun_out/san/racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san/racecheck.txt
