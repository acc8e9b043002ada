S=${S:-512}
run() {
  local lab=$1; shift
  env "$@" timeout 300 python bench.py --streams $S --steps 128 --no-cpu-baseline --e2e-steps 1 --sustained-s 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$S $lab', round(d['value']), round(d['ms_per_step'],4))"
}
for r in 1 2; do
  run c1n8 FC_SPLICE_BULK_CTAS=1
  run g185n8 FC_SPLICE_BULK_GRID=185
  run g222n8 FC_SPLICE_BULK_GRID=222
  run g130n8 FC_SPLICE_BULK_GRID=130
done
