cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/v4l
python tools/prof_case.py c1 --iters 5 > gpurun_out/v4l/p.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v4l/c1_launches.csv python tools/prof_case.py c1 --iters 5 > gpurun_out/v4l/ncu.log 2>&1
python tools/prof_case.py c2 --iters 3 > gpurun_out/v4l/p2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v4l/c2_launches.csv python tools/prof_case.py c2 --iters 3 > gpurun_out/v4l/ncu2.log 2>&1
