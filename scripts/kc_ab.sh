#!/bin/bash
# K_C pairs-per-warp A/B (bench + K_C alone in the serial pass).
run() {
  local lab=$1; shift
  env "$@" timeout 300 python bench.py --steps 128 --no-cpu-baseline --e2e-steps 1 --sustained-s 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lab', round(d['value']), round(d['ms_per_step'],4), 'K_C', round(d['kernels']['rows_inv']['ms'],4))"
}
for r in 1 2; do
  run ppw1
  run ppw2c7 FC_KC_PPW=2
  run ppw2c6 FC_KC_PPW=2 FC_OCC_C=6
done
