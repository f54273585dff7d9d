#!/bin/bash
# A/B: bench the in-tree libzk and each variant in paper_2112_11880_b200/variants/ (one line each)
for lib in paper_2112_11880_b200/libzk.so paper_2112_11880_b200/variants/*.so; do
  ZK_LIB=$lib python bench.py --steps ${STEPS:-5} --no-e2e --no-cpu-baseline 2>/dev/null | python3 -c "
import sys, json
d = json.loads(sys.stdin.read())
print('$lib', round(d['value']), 'ms/it', round(d['bicgstab']['ms_per_iteration'], 4), 'spmv_us', round(d['spmv']['us'], 1),
      'inloop_us', round(d['roofline']['launch_us'], 1), 'vec_ms/it', round(d['bicgstab']['vector_kernels_ms_per_iter'], 4))"
done
