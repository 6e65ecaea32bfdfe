#!/bin/bash
# usage (on the GPU box via gpurun): bash tools/gcall.sh TAG [ncu-workloads...]
# runs: build check, smoke, pytest -m gpu, bench (all configs), then ncu --set full of
# force_kernel for each listed workload (after a plain run of the same command).
TAG=$1; shift
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
for w in "$@"; do
  timeout 300 python tools/prof_case.py $w --iters 3 > $O/p_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:force -s 2 -c 1 \
     -o $O/${w}_full python tools/prof_case.py $w --iters 3 > $O/ncu_$w.log 2>&1
  echo "ncu $w rc=$?" >> $O/rc.txt
done
# launch list of the bench command itself (ncu's per-launch durations; first 400 launches)
if [ -n "$LAUNCHES" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --only --no-cpu > $O/ncu_launch.log 2>&1
  echo "ncu launches rc=$?" >> $O/rc.txt
fi
