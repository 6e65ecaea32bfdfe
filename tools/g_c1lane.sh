#!/bin/bash
# usage (GPU box): bash tools/g_c1lane.sh TAG -- 2D kernel-path tests, C1 A/B of the 2D kernels, ncu of the lane kernel
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for r in 1 2; do timeout 300 python tools/ab.py c1 K2D=element K2D=lane K2D=point >> $O/ab_c1.txt 2>&1; done
timeout 300 python tools/ab.py c0 K2D=element K2D=lane K2D=point >> $O/ab_c0.txt 2>&1
echo "ab rc=$?" >> $O/rc.txt
cat > /tmp/pl.py <<'PY'
import sys; sys.argv=[sys.argv[0],'c1','--iters','2']
from paper_2104_11404_b200 import hydro; hydro.set_kernel_2d('lane')
sys.path.insert(0,'tools'); import runpy; runpy.run_path('tools/prof_case.py', run_name='__main__')
PY
timeout 300 python /tmp/pl.py > $O/p_c1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:force2d -s 1 -c 1 -o $O/c1_lane_full python /tmp/pl.py > $O/ncu_c1.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
