#!/bin/bash
# Round evidence: default bench line, ncu launch list of the same command,
# and one `--set full` capture per kernel at the bench configuration.
# usage: bash scripts/round_profile.sh <tag> [skip_tests]
mkdir -p gpurun_out
TAG=${1:-r01}
if [ -z "$2" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1
  echo smoke_rc=$?; tail -2 gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err || { echo "bench failed"; tail gpurun_out/bench_$TAG.err; exit 1; }
cat gpurun_out/bench_$TAG.json
KRE="k448|k_select|k_rank|k_splice"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$KRE" --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --no-cpu-baseline --sustained-s 0 > /dev/null 2>&1
echo launches_rc=$?
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --sustained-s 0"
timeout 600 $CMD > /dev/null 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"k448_rows_fwd|k448_cols|k448_rows_inv|k_select|k_rank|k_splice_ip|k_splice_plan" -s 14 -c 7 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full_rc=$?
