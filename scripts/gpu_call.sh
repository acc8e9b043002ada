#!/bin/bash
# gpurun with retries on transient infrastructure failures.
# usage: bash scripts/gpu_call.sh <log> <timeout_s> '<command>'
LOG=$1; TO=$2; CMD=$3
for i in $(seq 1 12); do
  /usr/local/graft/bin/gpurun --timeout "$TO" -- "$CMD" > "$LOG" 2>&1
  if grep -q "status=transient\|backing off\|status=noslot\|no box" "$LOG"; then sleep 45; continue; fi
  break
done
tail -25 "$LOG"
