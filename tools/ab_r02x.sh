# round 2: nearest-set distances with 16-byte offset / y0 loads (BM_NEAR_VEC), IDL tail dims' squares before their
# ordered additions (BM_IDL_TAIL) (bit-identical) (dev A/B): new = working tree, base = 008f7b0, nonv / noit = new without one
python tools/bitcmp.py new base 5 8 256 > gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 1 1 >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 3 2 cluster >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 4 1 >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 5 8 512 >> gpurun_out/x_bit.log 2>&1
python tools/bitcmp.py new base 2 1 >> gpurun_out/x_bit.log 2>&1
grep cfg gpurun_out/x_bit.log
bash tools/ab.sh cfg5 3 new base nonv noit new base
bash tools/ab.sh cfg4 3 new base nonv
bash tools/ab.sh cfg4idl 3 new base noit
bash tools/ab.sh cfg3 3 new base
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/x_phases_cfg5.txt 2>&1; grep "^cholesky\|^nearest\|chol_only\|per-patch\|sidl_dist" gpurun_out/x_phases_cfg5.txt
