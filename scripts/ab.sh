#!/bin/bash
# A/B timing of kernel variants selected by environment variables (one GPU).
# usage: bash scripts/ab.sh "ENV1=a ENV2=b" "ENV1=c" ...   (each arg = one variant)
mkdir -p gpurun_out
for v in "$@"; do
  echo -n "[$v] "; env $v timeout 300 python scripts/time_parts.py 2>&1 | tail -1
done
