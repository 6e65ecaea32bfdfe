cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab12; mkdir -p $O
V=paper_2104_11404_b200/_build/var
for r in 0 1; do for lib in cur p8; do echo "$lib: $(HYDRO_LIB_PATH=$V/$lib.so timeout 600 python tools/gemm_bench.py 2>&1 | tail -1)" >> $O/ab.txt; done; done
timeout 900 python -m pytest tests/test_gpu_rom.py tests/test_gpu_rom_step.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
