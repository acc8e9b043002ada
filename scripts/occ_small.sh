#!/bin/bash
# K_B / K_C occupancy variants (wave quantisation) at a small per-GPU batch.
S=${1:-64}
for lanes in 1 2; do
  for ob in 4 5 6; do
    for oc in 6 7 8 10; do
      for pipe in "" "--no-pipeline"; do
        if [ $lanes = 1 ]; then CH=512; else CH=$(( (S + 1) / 2 )); fi
        FC_OCC_B=$ob FC_OCC_C=$oc FC_LANES=$lanes FC_CHUNK=$CH timeout 120 python bench.py --streams $S --no-cpu-baseline \
          --e2e-steps 1 --sustained-s 0 $pipe > gpurun_out/oc.json 2>/dev/null
        python -c "import json; d=json.loads(open('gpurun_out/oc.json').read()); print('S $S lanes $lanes occB $ob occC $oc ${pipe:-pipe}', round(d['value']), round(d['ms_per_step'],4))" 2>/dev/null || echo "S $S lanes $lanes $ob $oc failed"
      done
    done
  done
done
