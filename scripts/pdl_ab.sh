# A/B: programmatic dependent launch on / off (NC_PDL) for the small configs and C4
for c in 0 1 2; do for m in 1 0 1 0; do
  NC_PDL=$m python bench.py --config $c --steps 30 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c pdl=$m', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
done; done
