# full GPU suite + per-workload bench lines (auto build) + scaling shares (dev)
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2c_tests.log
for w in cfg1 cfg2 cfg3 cfg4 cfg4idl cfg5; do
  python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_$w.json 2>/dev/null
  tail -1 gpurun_out/r2c_$w.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"
done
