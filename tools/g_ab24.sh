cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab24; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_paths.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 1800 python tools/ab_lib.py 2 c3 $V/base.so $V/s1p0.so $V/f1s2.so $V/b2s2.so $V/b3s2.so $V/b3s4.so $V/b1s3.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
