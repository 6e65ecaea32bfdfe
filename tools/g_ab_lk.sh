#!/bin/bash
# usage (GPU box): bash tools/g_ab_lk.sh TAG -- 3D parity tests, then A/B of the K=2 layouts (lk0 vs lk1)
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_paths.py tests/test_gpu_rom.py tests/test_gpu_fom.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
V=paper_2104_11404_b200/_build/var
timeout 1500 python tools/ab_lib.py 2 c2,tg,c4 $V/lk0.so $V/lk1.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
