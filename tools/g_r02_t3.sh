cd $GRAFT_REPO_ROOT
bash tools/g_tests.sh r02_t3
O=gpurun_out/r02_t3
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
