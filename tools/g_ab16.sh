cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ab16; mkdir -p $O
V=paper_2104_11404_b200/_build/var
timeout 900 python -m pytest tests/test_gpu_fom.py tests/test_gpu_indicator.py tests/test_gpu_window_ops.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for r in 0 1; do for lib in nocolor color; do echo "$lib: $(HYDRO_LIB_PATH=$V/$lib.so timeout 900 python tools/fom_bench.py c2 tg 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['workload'], round(d['ms_per_step'], 2), 'ms', d['cg_iterations_per_step'], 'it', d.get('indicator_ms'), d.get('window_ops_oblique_v_ms'), end='; ')
")" >> $O/ab.txt; done; done
