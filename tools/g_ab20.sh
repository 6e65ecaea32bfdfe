cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab20; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 2000 python tools/ab_lib.py 2 c3 $V/base.so $V/r3.so $V/q3n2.so $V/q3n4.so $V/q2n2.so $V/q6n2.so $V/q3n1.so $V/q2n4.so $V/q3n3.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
