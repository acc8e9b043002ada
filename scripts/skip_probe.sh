#!/bin/bash
# Critical-path sensitivity of the pipelined step's select branches: the
# graph-captured front + back (no splice, so the decision's data cannot change
# the work) with one kernel kind not launched (FC_PROBE_SKIP; timing only).
OUT=${1:-gpurun_out/skip_probe.txt}
mkdir -p "$(dirname "$OUT")"; : > "$OUT"
for s in 64 512; do
  for sk in 0 1 2 4 8 16; do
    echo "== S=$s skip=$sk" >> "$OUT"
    S=$s FC_PROBE_SKIP=$sk PROBE_ONLY="front + back" timeout 300 python scripts/overlap_probe.py 2>/dev/null | grep "us/step" >> "$OUT"
  done
done
cat "$OUT"
