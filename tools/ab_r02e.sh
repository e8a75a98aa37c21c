# round 2: LOO/exp FP64 trimming (product), one-pass covariance, LOO single-row SIMT (dev A/B)
python tools/cli_case_debug.py > gpurun_out/e_cli.log 2>&1; echo cli rc=$?
for v in base nofast cov1p row1 all3; do
  if [ "$v" = base ]; then unset BM_NATIVE_VARIANT; else export BM_NATIVE_VARIANT=$v; fi
  timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fullframe.py -q -m gpu -p no:cacheprovider -x > gpurun_out/e_tests_$v.log 2>&1; echo "$v tests rc=$?"; tail -1 gpurun_out/e_tests_$v.log
done
unset BM_NATIVE_VARIANT
bash tools/ab.sh cfg5 3 base nofast cov1p row1 all3 base
bash tools/ab.sh cfg4 3 base nofast cov1p row1 all3
