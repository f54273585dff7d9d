set -x
python __graft_entry__.py build
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?; tail -2 gpurun_out/bench_final.err
timeout 900 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/bench_reference.json; echo ref rc=$?
