set -x
python __graft_entry__.py build
timeout 900 python -m pytest tests/test_gpu_dist_local.py -q -x -k "validation or cg_cocg" 2>&1 | tail -60
timeout 900 python -m pytest tests/test_gpu_dist_local.py tests/test_gpu_solve.py tests/test_gpu_tfqmr.py tests/test_gpu_bicgstab_l.py -q 2>&1 | tail -30
