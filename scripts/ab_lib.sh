#!/bin/bash
# Same-box A/B of two library builds through the pipelined bench.
# usage: bash scripts/ab_lib.sh A.so B.so [rounds]
L=paper_2604_24391_b200/_lib/libfreqcache_b200.so
for r in $(seq ${3:-2}); do
  for lib in "$1" "$2"; do
    cp "$lib" "$L"
    echo -n "[$lib] "; timeout 300 python bench.py --steps 64 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
  done
done
