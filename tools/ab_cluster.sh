# cluster build: parity first, then narrow-DAG timings 512 vs cluster (dev A/B)
timeout 900 python -m pytest tests/test_gpu.py -q -x -m gpu -k "cluster" -p no:cacheprovider > gpurun_out/cl_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/cl_tests.log
for w in cfg1 cfg3 cfg2; do for b in 512 cluster; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --kernel-build $b 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $b', round(d['value']), round(d['ms_per_step'],2))"
done; done
