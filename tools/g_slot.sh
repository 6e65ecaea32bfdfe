#!/bin/bash
# usage (GPU box): bash tools/g_slot.sh TAG -- A/B of the lane kernel with the assembly slots loaded in the
# gather (slot.so) against the base build, C0 and C1 with K2D=lane (and element for reference)
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
V=paper_2104_11404_b200/_build/var
for r in 0 1 2; do for L in base slot; do for c in c0 c1; do
  echo -n "round $r $L $c: " >> $O/ab.txt
  HYDRO_LIB_PATH=$PWD/$V/$L.so timeout 300 python tools/ab.py $c K2D=lane K2D=element 2>&1 | grep median | tr '\n' '|' >> $O/ab.txt; echo >> $O/ab.txt
done; done; done
cat $O/ab.txt
