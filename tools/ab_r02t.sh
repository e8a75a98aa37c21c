# round 2: the gate's sequential nu loop on warp 0 with the ring sums on its lanes (BM_WARP_SCAN) (bit-identical)
# (dev A/B); prev = the commit before
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 2 1 >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 512 >> gpurun_out/t_bit.log 2>&1
grep cfg gpurun_out/t_bit.log
bash tools/ab.sh cfg5 3 base prev base prev
bash tools/ab.sh cfg2 10 base prev
bash tools/ab.sh cfg3 3 base prev
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/t_phases_cfg5.txt 2>&1; grep "gate2\|sidl\|^gate\|per-patch" gpurun_out/t_phases_cfg5.txt
