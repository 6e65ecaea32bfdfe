#!/bin/bash
# usage (on the GPU box via gpurun): bash tools/g_tests.sh TAG [pytest args...]
# build check, smoke, pytest -m gpu (logs under gpurun_out/TAG)
TAG=$1; shift
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 2400 python -m pytest tests -m gpu -q -x "$@" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
tail -5 $O/pytest.log
