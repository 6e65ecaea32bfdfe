#!/bin/bash
# usage (GPU box): bash tools/g_lane2.sh TAG -- 2D tests, C1/C0 A/B of the 2D kernels, ncu of the lane kernel on C1
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for r in 1 2; do timeout 300 python tools/ab.py c1 K2D=element K2D=lane >> $O/ab_c1.txt 2>&1; done
timeout 300 python tools/ab.py c0 K2D=lane K2D=point >> $O/ab_c0.txt 2>&1
bash tools/g_ncu1.sh $TAG c1 force2d --k2d lane
