#!/bin/bash
# Same-box A/B of the K_B + K_C flow kernel (FC_BC_FLOW) against the split
# kernels on the pipelined bench step, two rounds, 512 and 64 streams.
# usage: bash scripts/flow_ab.sh [out]
OUT=${1:-gpurun_out/flow_ab.txt}
mkdir -p "$(dirname "$OUT")"; : > "$OUT"
run() {  # label, streams, env...
  local label=$1 s=$2; shift 2
  env "$@" timeout 300 python bench.py --streams "$s" --steps 256 --sustained-s 0 --no-cpu-baseline --e2e-steps 2 \
    2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$label S=$s', round(d['value']), 'ms/step %.4f' % d['ms_per_step'], 'mhz', d['clocks']['sm_mhz'])" >> "$OUT"
}
for r in 1 2; do
  for s in 512 64; do
    run split "$s" FC_BC_FLOW=0
    run flow_l4 "$s" FC_BC_FLOW=1 FC_BC_LAG=4
    run flow_l8 "$s" FC_BC_FLOW=1 FC_BC_LAG=8
    run flow_l16 "$s" FC_BC_FLOW=1 FC_BC_LAG=16
    run flow_l8_nodiscard "$s" FC_BC_FLOW=1 FC_BC_LAG=8 FC_BC_DISCARD=0
  done
done
cat "$OUT"
