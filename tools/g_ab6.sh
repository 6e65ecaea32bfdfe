cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab6; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 2400 python tools/ab_lib.py 2 c3,c2 $V/cur.so $V/m3.so $V/m5.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
