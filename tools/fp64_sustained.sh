#!/bin/bash
# on the GPU box: sustained FP64 DFMA / DMMA rates with the SM clock sampled beside them
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-fp64_sustained}; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/fp64_sustained.cu -o /tmp/fp64_sustained || exit 1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $O/clocks.csv &
SMI=$!
/tmp/fp64_sustained ${2:-6} > $O/rates.txt 2>&1
kill $SMI
