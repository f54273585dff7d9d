#!/bin/bash
# microbench.py spmv for each lib in $LIBS with maps $MAPS, printing lib, map, µs, GB/s only
for L in $LIBS; do
  ZK_LIB=$L python tools/microbench.py spmv --config ${CFG:-C4} --maps ${MAPS:-0:4,3:32} --reps ${REPS:-30} --beta ${BETA:-0} 2>/dev/null |
  python3 -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$(basename $L)', d['map'], round(d['us'], 1), round(d['gbs']))"
done
