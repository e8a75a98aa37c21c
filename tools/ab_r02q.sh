# round 2: single-barrier tree-order reductions in the 512-thread / cluster builds (bit-identical) (dev A/B)
python tools/bitcmp.py base prev 1 1 > gpurun_out/q_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/q_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 512 >> gpurun_out/q_bit.log 2>&1
python tools/bitcmp.py base prev 4 1 cluster >> gpurun_out/q_bit.log 2>&1
grep cfg gpurun_out/q_bit.log
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_fullframe.py -q -m gpu -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/q_tests.log
bash tools/ab.sh cfg1 10 base prev base prev
bash tools/ab.sh cfg3 3 base prev
bash tools/ab.sh cfg2 10 base prev
python tools/scale_sim.py 32 > gpurun_out/q_scale.log 2>&1; cat gpurun_out/q_scale.log
