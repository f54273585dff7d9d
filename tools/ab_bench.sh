#!/bin/bash
# A/B: bench configurations "lib|ENV=V ENV2=V" (default: in-tree lib + each variant), one line each
CONFIGS=${CONFIGS:-"paper_2112_11880_b200/libzk.so|"}
IFS=';' read -ra CS <<< "$CONFIGS"
for cfg in "${CS[@]}"; do
  lib=${cfg%%|*}; envs=${cfg#*|}
  env ZK_LIB=$lib $envs python bench.py --steps ${STEPS:-5} --no-e2e --no-cpu-baseline --no-shapes 2>/dev/null | python3 -c "
import sys, json
d = json.loads(sys.stdin.read())
print('$(basename $lib) [$envs]', round(d['value']), 'ms/it', round(d['bicgstab']['ms_per_iteration'], 4), 'spmv_us', round(d['spmv']['us'], 1),
      'inloop_us', round(d['roofline']['launch_us'], 1), 'vec_ms/it', round(d['bicgstab']['vector_kernels_ms_per_iter'], 4), 'clk', d['clocks']['sm_mhz'])"
done
