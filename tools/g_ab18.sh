cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab18; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 900 python tools/ab_lib.py 3 c1 $V/base.so $V/u2.so $V/u2q1.so $V/u4q1.so $V/mx168.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
