# round 2: tree reductions with named barriers over the warps a level involves (BM_TREE_NB) (bit-identical) (dev A/B):
# new = working tree, base = HEAD
python tools/bitcmp.py new base 5 8 256 > gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 1 1 >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 3 2 cluster >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 4 1 >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 5 8 512 >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 2 1 >> gpurun_out/x_bit.log 2>&1
grep cfg gpurun_out/x_bit.log
bash tools/ab.sh cfg5 3 new base new base
bash tools/ab.sh cfg4 3 new base
bash tools/ab.sh cfg1 10 new base
bash tools/ab.sh cfg3 3 new base
