#!/bin/bash
# Same-box A/B over library builds x env settings through the pipelined bench.
# usage: bash scripts/ab_libs_env.sh "lib1.so lib2.so" "ENV=a" "ENV=b" ...
L=paper_2604_24391_b200/_lib/libfreqcache_b200.so
libs=$1; shift
for lib in $libs; do
  cp "$lib" "$L"
  for v in "$@"; do
    echo -n "[$lib $v] "; env $v timeout 300 python bench.py --steps 64 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
  done
done
