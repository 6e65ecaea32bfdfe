cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab23; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_paths.py tests/test_gpu_fom.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_lib.py 2 c3 $V/base.so $V/pad0.so $V/pad14.so $V/seps.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
