# round 2: right-looking Cholesky + paired nearest-set distances (both meant bit-identical) (dev A/B)
python tools/bitcmp.py base prev 5 8 > gpurun_out/h_bit.log 2>&1
python tools/bitcmp.py base prev 1 1 >> gpurun_out/h_bit.log 2>&1
python tools/bitcmp.py base prev 4 1 >> gpurun_out/h_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 512 >> gpurun_out/h_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/h_bit.log 2>&1
cat gpurun_out/h_bit.log | grep cfg
bash tools/ab.sh cfg5 3 base prev chol base
bash tools/ab.sh cfg4 3 base prev
bash tools/ab.sh cfg1 10 base prev chol
bash tools/ab.sh cfg3 3 base prev
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/h_ph_cfg5.log 2>&1
BM_NATIVE_VARIANT=diag python tools/phases.py 1 1 sentinel cluster > gpurun_out/h_ph_cfg1.log 2>&1
