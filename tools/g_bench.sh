#!/bin/bash
# usage (on the GPU box via gpurun): bash tools/g_bench.sh TAG [ncu workloads...]
# full default bench line, then (optional) ncu --set full of the force kernel per workload
TAG=$1; shift
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
for w in "$@"; do
  timeout 600 python tools/prof_case.py $w --iters 2 > $O/p_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 2 -c 1 \
     -o $O/${w}_full python tools/prof_case.py $w --iters 2 > $O/ncu_$w.log 2>&1
  echo "ncu $w rc=$?" >> $O/rc.txt
done
