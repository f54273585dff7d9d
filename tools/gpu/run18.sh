set -x
python __graft_entry__.py build
timeout 1200 python -m pytest tests/test_gpu_dist_local.py tests/test_gpu_bicgstab_l.py -q -x 2>&1 | tail -25
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -5
