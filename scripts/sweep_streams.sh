#!/bin/bash
# Per-GPU throughput against streams per GPU (the literal config-5 split puts
# 512 / N streams on each GPU), graph and eager launch.
# usage: bash scripts/sweep_streams.sh <tag> [streams...]
mkdir -p gpurun_out
TAG=${1:-sweep}; shift
LIST=${@:-64 128 256 512}
for s in $LIST; do
  for g in "" "--no-graph"; do
    timeout 300 python bench.py --streams $s --no-cpu-baseline --e2e-steps 1 --sustained-s 0 $g \
      > gpurun_out/sw_${TAG}_${s}${g}.json 2> gpurun_out/sw_${TAG}_${s}${g}.err
    python - "$s" "$g" gpurun_out/sw_${TAG}_${s}${g}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read())
    k = d["kernels"]
    print(f"streams {sys.argv[1]:>4} {sys.argv[2] or 'graph':>10}: {d['value']:9.0f} frames/s "
          f"{d['ms_per_step']:.4f} ms/step | " + " ".join(f"{n} {v['ms']:.4f}" for n, v in k.items()))
except Exception as e:
    print("failed", sys.argv[1:], e)
PY
  done
done
