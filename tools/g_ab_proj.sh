#!/bin/bash
# usage (GPU box): bash tools/g_ab_proj.sh TAG LIB...  -- C4-sized projection/lift timing per library build
TAG=$1; shift
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
for r in 0 1; do for L in "$@"; do
  echo -n "$(basename $L) round $r: " >> $O/ab.txt
  HYDRO_LIB_PATH=$PWD/$L timeout 300 python tools/gemm_bench.py >> $O/ab.txt 2>&1
done; done
echo "ab rc=$?" >> $O/rc.txt
