#!/bin/bash
# Chunk / lane knobs at a small per-GPU batch (default 64 streams).
S=${1:-64}
for cfg in "64 1" "32 2" "16 4" "22 3" "11 6"; do
  set -- $cfg
  FC_CHUNK=$1 FC_LANES=$2 timeout 300 python bench.py --streams $S --no-cpu-baseline --e2e-steps 1 --sustained-s 0 > gpurun_out/kn_$1_$2.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/kn_$1_$2.json').read().splitlines()[-1]); print('streams $S chunk $1 lanes $2', round(d['value']), round(d['ms_per_step'],4))"
done
