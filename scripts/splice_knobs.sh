#!/bin/bash
# Splice-copier sizing inside the pipelined 3-branch step (default 512 streams).
S=${S:-512}
run() {
  local lab=$1; shift
  env "$@" timeout 300 python bench.py --streams $S --steps 128 --no-cpu-baseline --e2e-steps 1 --sustained-s 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$S $lab', round(d['value']), round(d['ms_per_step'],4))"
}
for r in 1 2; do
  run base
  run c1n8 FC_SPLICE_BULK_CTAS=1
  run c1n4 FC_SPLICE_BULK_CTAS=1 FC_SPLICE_BULK_NL=4
  run c1n2 FC_SPLICE_BULK_CTAS=1 FC_SPLICE_BULK_NL=2
  run g111n8 FC_SPLICE_BULK_GRID=111
  run g74n8 FC_SPLICE_BULK_GRID=74
  run g74n16 FC_SPLICE_BULK_GRID=74 FC_SPLICE_BULK_NL=16
  run g148n16 FC_SPLICE_BULK_GRID=148 FC_SPLICE_BULK_NL=16
  run c1n8s3 FC_SPLICE_BULK_CTAS=1 FC_SPLICE_BULK_SLOTS=3
done
