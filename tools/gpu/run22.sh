set -x
python __graft_entry__.py build
timeout 900 python tools/ab_bl.py C4 2>&1 | tee gpurun_out/ab_bl.txt
timeout 900 python -m pytest tests/test_gpu_bicgstab_l.py tests/test_gpu_dist_local.py -q -k "c4 or single_rank or local_bicgstab_l or split" 2>&1 | tail -4
