#!/bin/bash
# Stream-priority knobs of the pipelined bench step (front / back / splice branches).
S=${1:-64}
run() {  # label, env...
  local lab=$1; shift
  env "$@" timeout 300 python bench.py --streams $S --no-cpu-baseline --e2e-steps 1 --sustained-s 0 $EXTRA > gpurun_out/pr_$lab.json 2> gpurun_out/pr_$lab.err
  python -c "import json; d=json.loads(open('gpurun_out/pr_$lab.json').read()); print('$S $lab', round(d['value']), round(d['ms_per_step'],4))" || tail -2 gpurun_out/pr_$lab.err
}
EXTRA="--no-pipeline" run nopipe
run base
run back_hi FC_BENCH_BACK_PRIO=-2
run back_hi_side_lo FC_BENCH_BACK_PRIO=-2 FC_BENCH_SIDE_PRIO=-1
run back_hi_side_0 FC_BENCH_BACK_PRIO=-1 FC_BENCH_SIDE_PRIO=0
run nolanes FC_LANES=1 FC_CHUNK=512
run nolanes_backhi FC_LANES=1 FC_CHUNK=512 FC_BENCH_BACK_PRIO=-2
