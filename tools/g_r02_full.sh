#!/bin/bash
# usage (GPU box): bash tools/g_r02_full.sh TAG -- smoke + pytest -m gpu + bench + ncu (tg force, c4 lift/project)
TAG=$1
cd $GRAFT_REPO_ROOT
bash tools/g_tests.sh $TAG
O=gpurun_out/$TAG
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python tools/prof_case.py tg --iters 2 > $O/p_tg.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 2 -c 1 -o $O/tg_full python tools/prof_case.py tg --iters 2 > $O/ncu_tg.log 2>&1; echo "ncu tg rc=$?" >> $O/rc.txt
timeout 600 python tools/prof_case.py c4 --iters 2 > $O/p_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lift_mma|project_mma" -s 8 -c 8 -o $O/c4_liftproj python tools/prof_case.py c4 --iters 2 > $O/ncu_lp.log 2>&1; echo "ncu lp rc=$?" >> $O/rc.txt
