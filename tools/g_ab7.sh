cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab7; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 2400 python tools/ab_lib.py 2 c1 $V/cur.so $V/tpe1.so $V/tpe2_128.so $V/tpe2_80.so $V/tpe2_64.so $V/tpe4_64.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
