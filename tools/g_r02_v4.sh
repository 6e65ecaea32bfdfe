#!/bin/bash
# usage (GPU box): bash tools/g_r02_v4.sh TAG -- smoke + pytest -m gpu + bench + ncu full of c3 / c1 force kernels
TAG=$1
cd $GRAFT_REPO_ROOT
bash tools/g_tests.sh $TAG
O=gpurun_out/$TAG
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
for w in c3 c1; do
  timeout 600 python tools/prof_case.py $w --iters 2 > $O/p_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:force -s 2 -c 1 \
     -o $O/${w}_full python tools/prof_case.py $w --iters 2 > $O/ncu_$w.log 2>&1
  echo "ncu $w rc=$?" >> $O/rc.txt
done
