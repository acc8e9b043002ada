#!/bin/bash
# Launch list + full ncu capture of the select/splice kernels (run under gpurun, 1 GPU).
# usage: bash scripts/ncu_profile.sh <tag>
TAG=${1:-v0}
mkdir -p gpurun_out
CMD="python bench.py --streams 64 --steps 2 --warmup 1 --ring 2 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_$TAG.json 2> gpurun_out/ncu_plain_$TAG.err || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k448_rows_fwd|k448_cols|k448_rows_inv|k_splice16|k_select" -s 5 -c 5 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full_rc=$?
ls -la gpurun_out | tail -8
