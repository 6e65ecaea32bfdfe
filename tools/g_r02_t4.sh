cd $GRAFT_REPO_ROOT
bash tools/g_tests.sh r02_t4
O=gpurun_out/r02_t4
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
bash tools/fp64_sustained.sh r02_t4/fp64 6; echo "fp64 rc=$?" >> $O/rc.txt
timeout 600 python tools/prof_case.py c4 --iters 2 > $O/p_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lift_mma|project_mma" -s 8 -c 8 -o $O/c4_liftproj python tools/prof_case.py c4 --iters 2 > $O/ncu_lp.log 2>&1; echo "ncu lp rc=$?" >> $O/rc.txt
