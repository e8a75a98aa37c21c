# round 2: gate nu scan four rings per step (BM_SCAN4) (bit-identical) (dev A/B): scan4 = working tree, base = prev = c3b24a0;
# then the phase breakdown of the working tree (diag) and the cfg5 per-rank share at N = 8
python tools/bitcmp.py scan4 base 5 8 256 > gpurun_out/w_bit.log 2>&1
python tools/bitcmp.py scan4 base 2 1 >> gpurun_out/w_bit.log 2>&1
python tools/bitcmp.py scan4 base 3 2 cluster >> gpurun_out/w_bit.log 2>&1
python tools/bitcmp.py scan4 base 5 8 512 >> gpurun_out/w_bit.log 2>&1
grep cfg gpurun_out/w_bit.log
bash tools/ab.sh cfg5 3 scan4 base scan4 base
bash tools/ab.sh cfg2 10 scan4 base
bash tools/ab.sh cfg3 3 scan4 base
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/w_phases_cfg5.txt 2>&1; grep "gate2\|sidl_scan\|per-patch" gpurun_out/w_phases_cfg5.txt
python tools/scale_sim.py 32 > gpurun_out/w_scale.log 2>&1; cat gpurun_out/w_scale.log
