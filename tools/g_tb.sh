#!/bin/bash
# usage (GPU box): bash tools/g_tb.sh TAG -- smoke + pytest -m gpu + the default bench line
TAG=$1
cd $GRAFT_REPO_ROOT
bash tools/g_tests.sh $TAG
O=gpurun_out/$TAG
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
