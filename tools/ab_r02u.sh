# round 2: loop-invariant DMMA A fragments held in registers: quadforms L^-1 (BM_QF_HOIST), LOO U / nearest / d_i
# (BM_LOO_HOIST) (bit-identical) (dev A/B); prev = the commit before; noqh / nolh = base without one of them
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/u_bit.log 2>&1
python tools/bitcmp.py base prev 1 1 >> gpurun_out/u_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/u_bit.log 2>&1
python tools/bitcmp.py base prev 4 1 >> gpurun_out/u_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 512 >> gpurun_out/u_bit.log 2>&1
grep cfg gpurun_out/u_bit.log
bash tools/ab.sh cfg5 3 base prev noqh nolh base prev
bash tools/ab.sh cfg4 3 base prev noqh nolh
bash tools/ab.sh cfg1 10 base prev
bash tools/ab.sh cfg3 3 base prev
