#!/bin/bash
# usage (GPU box): bash tools/g_ncu1.sh TAG WORKLOAD KREGEX [prof_case args...] -- one ncu --set full capture
TAG=$1; W=$2; KR=$3; shift 3
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 300 python tools/prof_case.py $W --iters 2 "$@" > $O/p_$W.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KR -s 1 -c 1 -o $O/${W}_full python tools/prof_case.py $W --iters 2 "$@" > $O/ncu_$W.log 2>&1; echo "ncu $W rc=$?" >> $O/rc.txt
