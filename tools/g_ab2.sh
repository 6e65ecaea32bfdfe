cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab2; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 2400 python tools/ab_lib.py 2 c4,c2 $V/base.so $V/upc2.so $V/upc4.so $V/upc16.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
