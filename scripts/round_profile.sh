#!/bin/bash
# Full default bench + ncu launch list of the same command + one full capture per kernel.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err || { echo "bench failed"; tail gpurun_out/bench_full.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k448|k_select|k_splice" --csv \
    --log-file gpurun_out/launches_full.csv python bench.py --no-cpu-baseline > /dev/null 2>&1
echo launches_rc=$?
CMD="python bench.py --streams 64 --steps 2 --warmup 1 --ring 2 --e2e-steps 1 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on \
    -k regex:"k448_rows_fwd|k448_cols|k448_rows_inv|k_select|k_splice16" -s 5 -c 5 \
    -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
