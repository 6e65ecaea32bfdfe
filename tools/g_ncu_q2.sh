#!/bin/bash
# usage (GPU box): bash tools/g_ncu_q2.sh TAG -- ncu --set full of the C4 and C2 force kernels
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
for w in c4 c2; do
  timeout 600 python tools/prof_case.py $w --iters 2 > $O/p_$w.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 2 -c 1 \
     -o $O/${w}_full python tools/prof_case.py $w --iters 2 > $O/ncu_$w.log 2>&1
  echo "ncu $w rc=$?" >> $O/rc.txt
done
