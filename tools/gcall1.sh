cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/rc.txt
timeout 300 python tools/prof_case.py c2 --iters 3 > gpurun_out/p2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 2 -c 1 -o gpurun_out/r01_c2_full python tools/prof_case.py c2 --iters 3 > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?" >> gpurun_out/rc.txt
timeout 300 python tools/prof_case.py c1 --iters 3 > gpurun_out/p1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 2 -c 1 -o gpurun_out/r01_c1_full python tools/prof_case.py c1 --iters 3 > gpurun_out/ncu_c1.log 2>&1; echo "ncu c1 rc=$?" >> gpurun_out/rc.txt
timeout 300 python tools/prof_case.py c3 --iters 3 > gpurun_out/p3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 2 -c 1 -o gpurun_out/r01_c3_full python tools/prof_case.py c3 --iters 3 > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_short.json 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/rc.txt
