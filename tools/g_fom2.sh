#!/bin/bash
# usage (GPU box): bash tools/g_fom2.sh TAG -- FOM tests (incl. the random FOM sweep), the FOM bench rows, the
# launch list of one C2 step
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fom.py tests/test_gpu_random_sweep.py tests/test_gpu_indicator.py tests/test_gpu_window_ops.py tests/test_gpu_offline.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
tail -3 $O/pytest.log
timeout 900 python tools/fom_bench.py c2 tg c1 > $O/fom.json 2> $O/fom.err; echo "fom rc=$?" >> $O/rc.txt
cut -c1-400 $O/fom.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/fom_step_once.py c2 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
