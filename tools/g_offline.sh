#!/bin/bash
# usage (GPU box): bash tools/g_offline.sh TAG -- offline GPU tests + offline bench (+ launch list)
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_offline.py tests/test_gpu_window_ops.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python tools/offline_bench.py > $O/offline.json 2> $O/offline.err; echo "offline rc=$?" >> $O/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/offline_bench.py > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
