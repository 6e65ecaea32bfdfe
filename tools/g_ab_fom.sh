#!/bin/bash
# usage (GPU box): bash tools/g_ab_fom.sh TAG LIB_A LIB_B -- FOM tests (in-tree lib) + FOM step A/B (fom_step_once.py)
TAG=$1; A=$2; Bv=$3
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fom.py tests/test_gpu_rom_step.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for r in 1 2; do for L in $A $Bv; do
  echo "== $L" >> $O/ab.txt
  HYDRO_LIB_PATH=$PWD/$L timeout 600 python tools/fom_step_once.py c2 >> $O/ab.txt 2>&1
done; done
timeout 900 env HYDRO_LIB_PATH=$PWD/$Bv ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"assemble_dot|mass_apply3|cg_" --csv --log-file $O/launches.csv python tools/fom_step_once.py c2 > $O/ncu.log 2>&1
