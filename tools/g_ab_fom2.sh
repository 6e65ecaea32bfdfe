#!/bin/bash
# usage (GPU box): bash tools/g_ab_fom2.sh TAG LIB... -- FOM step timing (tools/fom_bench.py c2 tg) per library build
TAG=$1; shift
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
for r in 0 1; do for L in "$@"; do
  echo "$(basename $L) round $r:" >> $O/ab.txt
  HYDRO_LIB_PATH=$PWD/$L timeout 600 python tools/fom_bench.py c2 tg 2>&1 | python -c "
import sys, json
for line in sys.stdin:
    try: d = json.loads(line)
    except Exception: continue
    print('  ', d['workload'], 'ms_per_step', round(d['ms_per_step'], 3), 'cg_it', d.get('cg_iterations_per_step'), 'drift', d.get('rel_energy_drift'), 'status', d.get('status'))
" >> $O/ab.txt
done; done
cat $O/ab.txt
