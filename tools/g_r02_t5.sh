cd $GRAFT_REPO_ROOT
bash tools/g_tests.sh r02_t5
O=gpurun_out/r02_t5
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
