#!/bin/bash
# K_B / K_C occupancy variants inside the pipelined step (default 512 streams).
S=${S:-512}
run() {
  local lab=$1; shift
  env "$@" timeout 300 python bench.py --streams $S --steps 128 --no-cpu-baseline --e2e-steps 1 --sustained-s 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$S $lab', round(d['value']), round(d['ms_per_step'],4))"
}
for r in 1 2; do
  for ob in 4 5 6; do for oc in 6 7 8 10; do run b${ob}c${oc} FC_OCC_B=$ob FC_OCC_C=$oc; done; done
done
