#!/bin/bash
# Round evidence: default bench line, ncu launch list of the same command,
# and one `--set full` capture per kernel at the bench configuration.
mkdir -p gpurun_out
TAG=${1:-r01}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err || { echo "bench failed"; tail gpurun_out/bench_$TAG.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k448|k_select|k_splice" --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --no-cpu-baseline > /dev/null 2>&1
echo launches_rc=$?
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on \
    -k regex:"k448_rows_fwd|k448_cols|k448_rows_inv|k_select|k_splice16" -s 5 -c 5 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full_rc=$?
