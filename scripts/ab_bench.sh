#!/bin/bash
# Pipelined bench (select + splice) under env variants; prints value, ms/step,
# step roofline fraction and the serial per-kernel times.
for v in "$@"; do
  echo -n "[$v] "
  env $v timeout 300 python bench.py --steps 64 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline_step']['frac'],3), {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
done
