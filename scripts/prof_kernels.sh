#!/bin/bash
# One `ncu --set full` capture of each select kernel (bench configuration,
# chunk of 32 streams per launch), plus the SASS/source pages needed to read
# it here.  usage: bash scripts/prof_kernels.sh <tag>
TAG=${1:-x}
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $CMD > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"k448_rows_fwd|k448_cols|k448_rows_inv|k_select" -s 40 -c 4 \
    -o gpurun_out/kprof_$TAG $CMD > gpurun_out/kprof_$TAG.log 2>&1
echo ncu_rc=$?
