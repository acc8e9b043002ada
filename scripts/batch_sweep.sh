for s in 64 128 256 512 1024; do
  echo -n "streams=$s "; timeout 300 python bench.py --streams $s --steps 64 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline_step']['frac'],3))"
done
