cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab13; mkdir -p $O
V=paper_2104_11404_b200/_build/var
for r in 0 1; do for lib in wm2 wm1m3 wm1m4; do echo "$lib: $(HYDRO_LIB_PATH=$V/$lib.so timeout 600 python tools/gemm_bench.py 2>&1 | tail -1)" >> $O/ab.txt; done; done
