# round 2: L^-1 substitution to row n + paired nearest distances (bit-identical) (dev A/B)
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/k_bit.log 2>&1
python tools/bitcmp.py base prev 1 1 >> gpurun_out/k_bit.log 2>&1
grep cfg gpurun_out/k_bit.log
bash tools/ab.sh cfg5 3 base prev base prev
bash tools/ab.sh cfg4 3 base prev
bash tools/ab.sh cfg1 10 base prev
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/k_ph_cfg5.log 2>&1
BM_NATIVE_VARIANT=diagprev python tools/phases.py 5 256 efficient > gpurun_out/k_ph_cfg5_prev.log 2>&1
BM_NATIVE_VARIANT=diag python tools/phases.py 1 1 sentinel cluster > gpurun_out/k_ph_cfg1.log 2>&1
