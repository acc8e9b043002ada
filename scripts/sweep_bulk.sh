#!/bin/bash
# In-place splice copier sweep inside the pipelined bench (run under gpurun).
# args per config: bulk NL ctas side-priority
for cfg in "1 8 1 -1" "1 8 1 0" "1 4 2 -1" "1 4 1 -1" "1 16 1 -1" "1 2 4 -1" "1 4 2 0" "1 8 2 0"; do
  set -- $cfg
  tag="$1_$2_$3_$4"
  FC_SPLICE_BULK=$1 FC_SPLICE_BULK_NL=$2 FC_SPLICE_BULK_CTAS=$3 FC_BENCH_SIDE_PRIO=$4 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
    > gpurun_out/sb_$tag.json 2>gpurun_out/sb_$tag.err
  python - "$tag" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/sb_{sys.argv[1]}.json"))
print(f"{sys.argv[1]} value={d['value']:.0f} ms/step={d['ms_per_step']:.3f} frac={d['roofline_step']['frac']:.3f} "
      + " ".join(f"{n}={v['ms']:.3f}" for n,v in d["kernels"].items()))
PY
done
