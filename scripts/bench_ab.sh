# same-box A/B: the current tree vs an older checkout in ./oldtree (its own bench.py and library)
for rep in 1 2; do
  for tree in . oldtree; do
    (cd $tree && python bench.py --no-cpu --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tree', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), '%.3g' % d['e2e']['value'])")
  done
done
