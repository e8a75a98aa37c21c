# FP32 IDL-estimate experiment: the build variant
# _blockmend_b200.idl32.so (-DBM_IDL_FP32=1) through the parity suites that
# exercise the IDL estimate, then cfg4idl throughput against the product build.
export BM_NATIVE_VARIANT=idl32
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullframe.py -q -s -m gpu -p no:cacheprovider \
  -k "golden_parity or config_parity or idl or vs_reference" > gpurun_out/fp32_idl_parity.log 2>&1
echo parity rc=$?
grep -E "passed|failed|FAILED|forced IDL|vs reference:|idl " gpurun_out/fp32_idl_parity.log | tail -40
for v in idl32 base; do
  if [ "$v" = base ]; then unset BM_NATIVE_VARIANT; else export BM_NATIVE_VARIANT=$v; fi
  python bench.py --workload cfg4idl --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg4idl', round(d['value']), round(d['ms_per_step'],2))"
done
