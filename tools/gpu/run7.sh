set -x
python __graft_entry__.py build
for lib in paper_2112_11880_b200/libzk.so paper_2112_11880_b200/variants/libzk_lp4.so; do ZK_LIB=$PWD/$lib timeout 600 python tools/ab_lib.py C3 C3T C4 2>&1 | tee -a gpurun_out/ab_lp.txt; done
ZK_LIB=$PWD/paper_2112_11880_b200/libzk.so timeout 600 python tools/ab_lib.py C3 C3T C4 2>&1 | tee -a gpurun_out/ab_lp.txt
timeout 900 python tools/e2e_probe.py 2>&1 | tee gpurun_out/e2e_probe.txt
