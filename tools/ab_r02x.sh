# round 2: Cholesky column dot product unrolled (BM_CHOL_UNR), L^-1 substitution two rows per step (BM_LINV_PAIR)
# (bit-identical) (dev A/B): new = working tree, nolp = new without BM_LINV_PAIR, base = HEAD
python tools/bitcmp.py new base 5 8 256 > gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 1 1 >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 3 2 cluster >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 4 1 >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 5 8 512 >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 2 1 >> gpurun_out/x_bit.log 2>&1
grep cfg gpurun_out/x_bit.log
bash tools/ab.sh cfg5 3 new nolp base new nolp base
bash tools/ab.sh cfg4 3 new nolp base
bash tools/ab.sh cfg1 10 new nolp base
bash tools/ab.sh cfg3 3 new nolp base
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/x_phases_cfg5.txt 2>&1; grep "^cholesky\|^nearest \|chol_only\|per-patch" gpurun_out/x_phases_cfg5.txt
