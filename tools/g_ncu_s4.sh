#!/bin/bash
# usage (GPU box): bash tools/g_ncu_s4.sh TAG -- ncu --set full of the kernels changed in session 4: the fused PCG
# passes (one FOM step on the C2 mesh) and the 2D lane kernel on C0 (each after a plain run of the same command)
TAG=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
timeout 600 python tools/fom_step_once.py c2 > $O/fom.json 2> $O/fom.err; echo "fom rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_xr_dot_fused|cg_p_fused|assemble_dot|mass_apply3" -s 40 -c 4 -o $O/fom_full python tools/fom_step_once.py c2 > $O/ncu_fom.log 2>&1; echo "ncu fom rc=$?" >> $O/rc.txt
timeout 300 python tools/prof_case.py c0 --iters 2 > $O/p_c0.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:force2d -s 1 -c 1 -o $O/c0_full python tools/prof_case.py c0 --iters 2 > $O/ncu_c0.log 2>&1; echo "ncu c0 rc=$?" >> $O/rc.txt
ls -la $O
