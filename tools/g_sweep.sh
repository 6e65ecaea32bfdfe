#!/bin/bash
# usage (GPU box): bash tools/g_sweep.sh TAG START COUNT [KINDS] -- the seeded random parity sweep
# (tests/test_gpu_random_sweep.py): its pytest cases, then COUNT more seeds from START
TAG=$1; START=$2; COUNT=$3
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_random_sweep.py -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
tail -15 $O/pytest.log
PYTHONPATH=$PWD timeout 2400 python tests/test_gpu_random_sweep.py sweep $START $COUNT $4 > $O/sweep.txt 2>&1; echo "sweep rc=$?" >> $O/rc.txt
grep -c . $O/sweep.txt; grep FAILED $O/sweep.txt | head -20; tail -1 $O/sweep.txt
