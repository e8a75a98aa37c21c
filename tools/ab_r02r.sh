# round 2: first-window nu accounting in every warp (BM_WARP_NU), warp-0 IDL for m <= 32 (BM_IDL_SMALL),
# 16-byte offset / y0 loads in the IDL and nearest-set distances (bit-identical) (dev A/B)
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/r_bit.log 2>&1
python tools/bitcmp.py base prev 1 1 >> gpurun_out/r_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/r_bit.log 2>&1
python tools/bitcmp.py base prev 4 1 >> gpurun_out/r_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 512 >> gpurun_out/r_bit.log 2>&1
python tools/bitcmp.py base prev 2 1 >> gpurun_out/r_bit.log 2>&1
grep cfg gpurun_out/r_bit.log
bash tools/ab.sh cfg5 3 base prev nowarpnu nosmall base prev
bash tools/ab.sh cfg4 3 base prev
bash tools/ab.sh cfg4idl 3 base prev
bash tools/ab.sh cfg2 10 base prev
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/r_phases_cfg5.txt 2>&1; tail -22 gpurun_out/r_phases_cfg5.txt
