# ab.sh <workload> <steps> <variant>... : cfg bench line per build variant (dev A/B tool)
w=$1; k=$2; shift 2
for v in "$@"; do
  if [ "$v" = "base" ]; then unset BM_NATIVE_VARIANT; else export BM_NATIVE_VARIANT=$v; fi
  python bench.py --workload $w --steps $k --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'], round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"
done
