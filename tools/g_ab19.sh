cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab19; mkdir -p $O
V=paper_2104_11404_b200/_build/var
HYDRO_LIB_PATH=$V/r1.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c3 or 3d or Q3 or q3" > $O/pytest_r1.log 2>&1; echo "pytest r1 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_lib.py 2 c3 $V/base.so $V/r1.so $V/r2.so $V/r3.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
