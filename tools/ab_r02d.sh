timeout 900 python -m pytest tests/test_gpu.py -q -x -m gpu -k "golden_parity or config_parity or frame_independence or smaller" -p no:cacheprovider 2>&1 | tail -2
for w in cfg5 cfg4 cfg3; do for v in r2 base r2 base; do
  if [ "$v" = base ]; then unset BM_NATIVE_VARIANT; else export BM_NATIVE_VARIANT=$v; fi
  python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $v', round(d['value']), round(d['ms_per_step'],2))"
done; done
