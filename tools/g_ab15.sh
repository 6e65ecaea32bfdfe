cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab15; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 2400 python tools/ab_lib.py 2 c3 $V/base.so $V/seps.so > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
