#!/bin/bash
# A/B: K_B + K_C flow kernel variants and K_C's L2 discard vs the split kernels
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stages.py -m gpu -x -q -k "flow" > gpurun_out/flow_test.log 2>&1; tail -3 gpurun_out/flow_test.log
OUT=gpurun_out/flow_ab2.txt; : > $OUT
run() { local label=$1 s=$2; shift 2
  env "$@" timeout 300 python bench.py --streams "$s" --steps 256 --sustained-s 0 --no-cpu-baseline --e2e-steps 2 \
    2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$label S=$s', round(d['value']), 'ms/step %.4f' % d['ms_per_step'], {n: round(v['ms'],4) for n,v in k.items()})" >> $OUT; }
for r in 1 2; do
run split 512 FC_BC_FLOW=0
run kc_discard 512 FC_KC_DISCARD=1
run pflow_l8 512 FC_BC_FLOW=1 FC_BC_LAG=8
run pflow_l32 512 FC_BC_FLOW=1 FC_BC_LAG=32
run pflow5_l16 512 FC_BC_FLOW=1 FC_BC_LAG=16 FC_BC_FLOW_OCC=5
done
cat $OUT
