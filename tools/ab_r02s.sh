# round 2: Gram staging / alpha with the nearest rows on the lanes (BM_TSTAGE), 1024-entry gate chunks with
# prefetched expansion-map entries (BM_GH=4, BM_TABPF) (bit-identical) (dev A/B); prev = 0cf3435, nots = base without BM_TSTAGE
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/s_bit.log 2>&1
python tools/bitcmp.py base prev 1 1 >> gpurun_out/s_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/s_bit.log 2>&1
python tools/bitcmp.py base prev 4 1 >> gpurun_out/s_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 512 >> gpurun_out/s_bit.log 2>&1
python tools/bitcmp.py base prev 2 1 >> gpurun_out/s_bit.log 2>&1
grep cfg gpurun_out/s_bit.log
bash tools/ab.sh cfg5 3 base prev nots base prev
bash tools/ab.sh cfg4 3 base prev nots
bash tools/ab.sh cfg1 10 base prev
bash tools/ab.sh cfg3 3 base prev
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/s_phases_cfg5.txt 2>&1; head -16 gpurun_out/s_phases_cfg5.txt
