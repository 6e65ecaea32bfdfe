cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_t2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for w in c2 c4 c3 tg c1; do timeout 900 python bench.py --workload $w --only --no-cpu --steps 10 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?" >> $O/rc.txt; done
