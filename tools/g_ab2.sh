#!/bin/bash
# usage (GPU box): bash tools/g_ab2.sh TAG CFGS LIB_A LIB_B [ROUNDS] [pytest files...] -- optional tests, then an A/B of two library builds
TAG=$1; CFGS=$2; A=$3; Bv=$4; R=${5:-2}; shift 5
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
if [ $# -gt 0 ]; then timeout 1200 python -m pytest "$@" -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt; fi
timeout 1500 python tools/ab_lib.py $R $CFGS $A $Bv > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
