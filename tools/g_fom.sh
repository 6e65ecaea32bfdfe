#!/bin/bash
# usage (GPU box): bash tools/g_fom.sh TAG -- FOM step bench + launch list + ncu full of the mass kernel
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 600 python tools/fom_step_once.py c2 > $O/fom.json 2> $O/fom.err; echo "fom rc=$?" >> $O/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/fom_step_once.py c2 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mass_apply3|assemble_dot|cg_xr" -s 30 -c 3 -o $O/fom_full python tools/fom_step_once.py c2 > $O/ncu2.log 2>&1; echo "ncu2 rc=$?" >> $O/rc.txt
