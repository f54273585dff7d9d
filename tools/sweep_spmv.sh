#!/bin/bash
# ZSpMV sweep over libzk variants (paper_2112_11880_b200/variants) and mappings; compact output
MAPS=${MAPS:-"0:8,0:8:::2,0:8:::4,0:8:::8,1:8:2:756,1:8:3:756,1:8:4:756,1:4:3:1512"}
for lib in paper_2112_11880_b200/libzk.so ${VARIANTS:-paper_2112_11880_b200/variants/*.so}; do
  ZK_LIB=$lib python tools/microbench.py spmv --reps ${REPS:-60} --maps "$MAPS" 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$(basename $lib)', d['map'], round(d['us'], 1), round(d['gbs']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:300])"
done
