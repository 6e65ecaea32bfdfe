#!/bin/bash
# usage (GPU box): bash tools/g_prof_c3.sh TAG [cfg ...] -- ncu --set full of the force kernel per config
TAG=$1; shift
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
for c in "$@"; do
timeout 600 python tools/prof_case.py $c --iters 2 > $O/p_$c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 2 -c 1 -o $O/${c}_full python tools/prof_case.py $c --iters 2 > $O/ncu_$c.log 2>&1; echo "ncu $c rc=$?" >> $O/rc.txt
done
