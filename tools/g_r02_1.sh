cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_g1; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 600 python tools/prof_case.py c4 --iters 2 > $O/plain_c4.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_launches.csv python tools/prof_case.py c4 --iters 2 > $O/ncu_l.log 2>&1; echo "launches rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 2 -c 1 -o $O/c4_force python tools/prof_case.py c4 --iters 2 > $O/ncu_f.log 2>&1; echo "ncu force rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lift_kernel|project" -s 8 -c 8 -o $O/c4_liftproj python tools/prof_case.py c4 --iters 2 > $O/ncu_lp.log 2>&1; echo "ncu liftproj rc=$?" >> $O/rc.txt
