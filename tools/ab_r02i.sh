# round 2: register-resident beta epilogue + paired nearest-set distances (bit-identical), alpha sums on two lanes (dev A/B)
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/i_bit.log 2>&1
python tools/bitcmp.py base prev 1 1 >> gpurun_out/i_bit.log 2>&1
python tools/bitcmp.py base prev 4 1 256 >> gpurun_out/i_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/i_bit.log 2>&1
grep cfg gpurun_out/i_bit.log
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_fullframe.py tests/test_cli_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/i_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/i_tests.log
bash tools/ab.sh cfg5 3 base prev near2 base
bash tools/ab.sh cfg4 3 base prev
bash tools/ab.sh cfg1 10 base prev
bash tools/ab.sh cfg3 3 base prev
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/i_ph_cfg5.log 2>&1
