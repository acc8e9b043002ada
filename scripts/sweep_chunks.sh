#!/bin/bash
# Chunk / lane sweep of the fast select path (run under gpurun).
for cfg in "32 2" "64 2" "32 3"; do
  set -- $cfg
  FC_CHUNK=$1 FC_LANES=$2 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/sw_$1_$2.json 2>/dev/null
  python - "$1" "$2" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/sw_{sys.argv[1]}_{sys.argv[2]}.json"))
k=d["kernels"]
print(f"chunk={sys.argv[1]:>3} lanes={sys.argv[2]} value={d['value']:.0f} ms/step={d['ms_per_step']:.3f} frac={d['roofline_step']['frac']:.3f} "
      + " ".join(f"{n}={v['ms']:.3f}" for n,v in k.items()))
PY
done
