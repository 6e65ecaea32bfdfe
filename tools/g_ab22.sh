cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab22; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 1500 python tools/ab_lib.py 2 c3 $V/base.so $V/b1r1.so $V/b1r2.so $V/dl1.so $V/dl1b1r2.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
