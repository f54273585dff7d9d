set -x
timeout 1500 python bench.py --local-ranks 2 --steps 2 --warmup 1 > gpurun_out/bench_local2_c5.json 2> gpurun_out/bench_local2_c5.err; echo rc=$?; tail -3 gpurun_out/bench_local2_c5.err; cat gpurun_out/bench_local2_c5.json
timeout 1500 python bench.py --local-ranks 4 --config C4 --steps 2 --warmup 1 > gpurun_out/bench_local4.json 2> gpurun_out/bench_local4.err; echo rc=$?; cat gpurun_out/bench_local4.json
