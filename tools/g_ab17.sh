cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab17; mkdir -p $O
V=paper_2104_11404_b200/_build/var
HYDRO_LIB_PATH=$V/pf4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_paths.py tests/test_gpu_rom.py -q -x > $O/pytest_pf4.log 2>&1; echo "pytest pf4 rc=$?" >> $O/rc.txt
timeout 2400 python tools/ab_lib.py 2 c3,c2,tg,c4 $V/base.so $V/pf2.so $V/pf4.so $V/pf8.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
