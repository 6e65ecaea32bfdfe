cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab21; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_paths.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 2400 python tools/ab_lib.py 2 c3,c2,tg,c4 $V/base.so $V/tc0.so $V/q1n4.so $V/q2n4.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
