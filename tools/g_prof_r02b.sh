#!/bin/bash
# usage (GPU box): bash tools/g_prof_r02b.sh TAG -- launch list of the bench command (C4 headline),
# ncu --set full of the C4 and C3 force kernels and of the C4-sized projection kernels
# (each after a plain run of the same command)
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 600 python bench.py --only --no-cpu --steps 2 --warmup 3 > $O/b_only.json 2> $O/b_only.err; echo "bench-only rc=$?" >> $O/rc.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --only --no-cpu --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
for w in c4 c3; do
  timeout 600 python tools/prof_case.py $w --iters 2 > $O/p_$w.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 2 -c 1 \
     -o $O/${w}_full python tools/prof_case.py $w --iters 2 > $O/ncu_$w.log 2>&1
  echo "ncu $w rc=$?" >> $O/rc.txt
done
timeout 600 python tools/gemm_bench.py > $O/gemm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:project_mma -c 4 \
  -o $O/proj_full python tools/gemm_bench.py > $O/ncu_proj.log 2>&1; echo "ncu proj rc=$?" >> $O/rc.txt
