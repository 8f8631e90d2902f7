for lib in varlib/*.so; do for v in do ds; do
  NC_LIB=$lib python bench.py --config 0 --variant $v --steps 30 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $v', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
done; done
