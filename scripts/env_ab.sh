#!/bin/bash
# Same-box A/B of environment knobs on the pipelined bench step.
# usage: bash scripts/env_ab.sh "<streams list>" rounds "LABEL_A:VAR=v VAR=v" "LABEL_B:VAR=v" ...
SL=$1; R=$2; shift 2
for r in $(seq "$R"); do
  for s in $SL; do
    for spec in "$@"; do
      label=${spec%%:*}; envs=${spec#*:}
      env $envs timeout 300 python bench.py --streams "$s" --steps 256 --sustained-s 0 --no-cpu-baseline --e2e-steps 2 \
        2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$label S=$s', round(d['value']), 'ms/step %.4f' % d['ms_per_step'], 'mhz', d['clocks']['sm_mhz'])"
    done
  done
done
